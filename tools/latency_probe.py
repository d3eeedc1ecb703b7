"""Per-step time of single 480^2 scenarios at several densities, including an
empty grid (the kernel's fixed per-step cost), one launch per step (dev tool).

    python tools/latency_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_4933_b200 as p  # noqa: E402

for model in (p.Model.Lem, p.Model.Aco):
    for n in (0, 1024, 51200):
        cfg = p.ScenarioConfig(width=480, height=480, agents_per_side=n, model=model, seed=42)
        e = p.Ensemble(cfg, replicas=1)
        e.run(5)
        tot, ker = e.time_steps(1000)
        _, ker = e.time_steps(100, kernel=True)
        print(f"{model.name} n={n:6d}: {tot:.3f} us/step in graphs, {ker * 1e3:.2f} us isolated launch", flush=True)
        e.close()
