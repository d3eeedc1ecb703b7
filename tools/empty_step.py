"""An empty 480^2 grid (no agents) stepped N times: the step kernel's fixed cost (dev tool for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_4933_b200 as p  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
aps = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = p.ScenarioConfig(width=480, height=480, agents_per_side=aps, model=p.Model.Lem, seed=42)
e = p.Ensemble(cfg, replicas=1)
e.run(n)
