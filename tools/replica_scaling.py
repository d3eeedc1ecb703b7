"""480^2 100K-agent throughput vs replica batch size (dev tool).

    python tools/replica_scaling.py 16 64 256
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_4933_b200 as p  # noqa: E402

for model in (p.Model.Aco, p.Model.Lem):
    for reps in [int(x) for x in sys.argv[1:]]:
        cfg = p.ScenarioConfig(width=480, height=480, agents_per_side=51_200, model=model, seed=42)
        e = p.Ensemble(cfg, replicas=reps)
        e.run(5)
        tot, _ = e.time_steps(1000)
        print(f"{model.name} x{reps}: {tot / 1000 * 1e3:8.1f} us/step  "
              f"{2 * 51_200 * reps * 1000 / (tot / 1e3) / 1e9:6.2f} G agent-upd/s (steps 5..1005)", flush=True)
        e.close()
