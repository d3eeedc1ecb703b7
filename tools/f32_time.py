"""C5 ACO step time with fp32 pheromone storage, steps 150..250 (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1412_4933_b200 as p  # noqa: E402

kernel = sys.argv[1] if len(sys.argv) > 1 else "fused_f32"
cfg, reps, desc = bench.scenario("c5_aco")
e = p.Ensemble(cfg, replicas=1, kernel=kernel)
e.run(150)
e.ctx.prepare_steps(100)
t, _ = e.time_steps(100)
print(kernel, os.environ.get("PEDFLOW_STRIP_SEGS", "default"), f"{t * 10:.1f} us/step")
