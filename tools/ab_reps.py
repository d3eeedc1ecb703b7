"""A/B of tools/debug/lib_{base,new}.so on 480^2 C3/C4 batches of several sizes (dev tool).

    python tools/ab_reps.py 64 128 256
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for tag in ("base", "new", "base", "new"):
    env = dict(os.environ, PEDFLOW_B200_LIB=os.path.join(ROOT, "tools", "debug", f"lib_{tag}.so"))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "replica_scaling.py")] + sys.argv[1:], env=env,
                         capture_output=True, text=True).stdout
    for line in out.splitlines():
        print(tag, line, flush=True)
