"""Same-box A/B step timing of tools/debug/lib_base.so vs lib_new.so (dev tool).

    python tools/ab_time.py c5_lem c4_aco_x64 [--rounds 3] [--steps 100] [--skip 0]

--skip runs that many extra steps before the timed window (the 480^2 crowds
jam after ~125 steps, so --skip 200 times the congested regime).
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
    tot, _ = e.time_steps(steps)
    print(f"{name} {tot/steps*1e3:.2f}", flush=True); e.close()
'''

ap = argparse.ArgumentParser()
ap.add_argument("workloads", nargs="+")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--skip", type=int, default=0)
ap.add_argument("--tags", default="base,new", help="tools/debug/lib_<tag>.so to compare (first = baseline)")
args = ap.parse_args()
res = {}
for r in range(args.rounds):
    for tag in args.tags.split(","):
        env = dict(os.environ, PEDFLOW_B200_LIB=os.path.join(ROOT, "tools", "debug", f"lib_{tag}.so"))
        out = subprocess.run([sys.executable, "-c", CODE, str(args.steps), str(args.skip)] + args.workloads, env=env, cwd=ROOT,
                             capture_output=True, text=True).stdout
        for line in out.split("\n"):
            if line.strip():
                name, us = line.split()
                res.setdefault((name, tag), []).append(float(us))
tags = args.tags.split(",")
for name in args.workloads:
    b = min(res.get((name, tags[0]), [0]))
    line = f"{name:12s} {tags[0]} {b:9.1f} us"
    for t in tags[1:]:
        n = min(res.get((name, t), [0]))
        line += f"   {t} {n:9.1f} us ({n / b if b else 0:.3f})"
    print(line)
