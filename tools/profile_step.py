"""Minimal driver for ncu: set up one workload, run a few steps (dev tool).

    ncu --set full -k regex:step_fused -s 2 -c 1 -o gpurun_out/prof python tools/profile_step.py c5_aco 3
    python tools/profile_step.py W STEPS fused THEN   # then THEN more steps in a second batch

Dense batched workloads run each graph batch as ONE multi-step launch: to
capture steps S..S+K of those, run `W S fused K` and capture launch 1.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_1412_4933_b200 as p  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5_aco"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kernel = sys.argv[3] if len(sys.argv) > 3 else "fused"
cfg, reps, desc = bench.scenario(name)
ens = p.Ensemble(cfg, replicas=reps, kernel=kernel)
ens.run(steps)
then = int(sys.argv[4]) if len(sys.argv) > 4 else 0
if then:
    ens.run(then)
print(desc, "steps", steps, "+", then, "launches", ens.ctx.launches)
