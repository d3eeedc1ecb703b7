"""Single-scenario step time, cluster-resident kernel vs the bit-plane
kernel, against agent density (dev tool; picks pf_cluster.cu's density cut).

    python tools/cluster_sweep.py [--size 480] [--steps 1000] [--model lem|aco] N_PER_SIDE...
"""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import paper_1412_4933_b200 as p
size, steps, model = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
for n in sys.argv[4:]:
    cfg = p.ScenarioConfig(width=size, height=size, agents_per_side=int(n),
                           model=p.Model.Lem if model == "lem" else p.Model.Aco, seed=42)
    e = p.Ensemble(cfg, replicas=1); e.run(5)
    e.ctx.prepare_steps(steps)
    e.time_steps(steps)
    e.ctx.prepare_steps(steps)
    tot, _ = e.time_steps(steps)
    print(f"{n} {tot/steps*1e3:.2f} {e.ctx.launches}", flush=True); e.close()
'''

ap = argparse.ArgumentParser()
ap.add_argument("agents", nargs="+")
ap.add_argument("--size", type=int, default=480)
ap.add_argument("--steps", type=int, default=1000)
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--model", default="lem")
args = ap.parse_args()
res = {}
for r in range(args.rounds):
    for flag in ("0", "1"):
        env = dict(os.environ, PEDFLOW_CLUSTER=flag, PEDFLOW_CLUSTER_MAX_DENSITY="1")
        out = subprocess.run([sys.executable, "-c", CODE, str(args.size), str(args.steps), args.model] + args.agents, env=env,
                             cwd=ROOT, capture_output=True, text=True)
        for line in out.stdout.split("\n"):
            if line.strip():
                n, us, _ = line.split()
                res.setdefault((n, flag), []).append(float(us))
        if out.returncode:
            print(out.stderr[-2000:])
for n in args.agents:
    a, b = min(res.get((n, "0"), [0])), min(res.get((n, "1"), [0]))
    dens = 2 * int(n) / args.size ** 2
    print(f"{args.size}^2 {n:>7s}/side (density {dens:6.3f})  bit-plane {a:8.2f} us   cluster {b:8.2f} us   "
          f"ratio {b / a if a else 0:.3f}")
