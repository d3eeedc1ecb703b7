import sys, os
sys.path.insert(0, os.getcwd())
import bench, paper_1412_4933_b200 as p
cfg, reps, desc = bench.scenario("c5_aco")
e = p.Ensemble(cfg, replicas=1, kernel="fused_f32"); e.run(150); e.ctx.prepare_steps(100); t, _ = e.time_steps(100)
print("c5_aco_f32", t * 10)
