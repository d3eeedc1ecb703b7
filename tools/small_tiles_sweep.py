"""Dev sweep: regular vs small-grid geometry (PEDFLOW_SMALL_TILES) for 480^2
batches of R replicas (steps 5..505).

    python tools/small_tiles_sweep.py 1 2 4 8 16
"""
import os
import subprocess
import sys

CODE = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import paper_1412_4933_b200 as p
reps = int(sys.argv[1])
for model, n in ((p.Model.Aco, 51200), (p.Model.Lem, 51200), (p.Model.Aco, 1024)):
    cfg = p.ScenarioConfig(width=480, height=480, agents_per_side=n, model=model, seed=42)
    e = p.Ensemble(cfg, replicas=reps); e.run(5)
    tot, _ = e.time_steps(500)
    print(f"  {model.name}{n} x{reps}: {tot/500*1e3:8.1f} us/step", flush=True); e.close()
'''
for reps in sys.argv[1:]:
    for st in ("0", "1"):
        print(f"PEDFLOW_SMALL_TILES={st}", flush=True)
        subprocess.run([sys.executable, "-c", CODE, reps], env=dict(os.environ, PEDFLOW_SMALL_TILES=st))
