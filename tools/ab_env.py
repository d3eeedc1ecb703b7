"""Same-box A/B of one library under two environments (dev tool).

    python tools/ab_env.py "PEDFLOW_MULTISTEP=0" "PEDFLOW_MULTISTEP=1" c4_aco_x64 ... [--steps N] [--skip S]
"""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import bench, paper_1412_4933_b200 as p
steps, skip = int(sys.argv[1]), int(sys.argv[2])
for name in sys.argv[3:]:
    cfg, reps, desc = bench.scenario(name)
    e = p.Ensemble(cfg, replicas=reps); e.run(5 + skip)
    e.ctx.prepare_steps(steps)  # graph capture outside the timed region (as bench.py)
    e.time_steps(steps)  # warm
    e.ctx.prepare_steps(steps)
    tot, _ = e.time_steps(steps)
    print(f"{name} {tot/steps*1e3:.2f}", flush=True); e.close()
'''

ap = argparse.ArgumentParser()
ap.add_argument("env_a")
ap.add_argument("env_b")
ap.add_argument("workloads", nargs="+")
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--skip", type=int, default=0)
args = ap.parse_args()
res = {}
for r in range(args.rounds):
    for tag in (args.env_a, args.env_b):
        env = dict(os.environ)
        for kv in tag.split(","):
            if kv:
                k, v = kv.split("=", 1)
                env[k] = v
        out = subprocess.run([sys.executable, "-c", CODE, str(args.steps), str(args.skip)] + args.workloads, env=env,
                             cwd=ROOT, capture_output=True, text=True).stdout
        for line in out.split("\n"):
            if line.strip():
                name, us = line.split()
                res.setdefault((name, tag), []).append(float(us))
for name in args.workloads:
    a, b = min(res.get((name, args.env_a), [0])), min(res.get((name, args.env_b), [0]))
    print(f"{name:12s} [{args.env_a}] {a:9.1f} us   [{args.env_b}] {b:9.1f} us   ratio {b / a if a else 0:.3f}")
