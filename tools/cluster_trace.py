"""Per-warp phase clocks of the cluster-resident LEM kernel (dev tool; needs a
library built with -DPF_CLUSTER_TRACE, e.g. tools/debug/lib_trace.so):

    PEDFLOW_B200_LIB=tools/debug/lib_trace.so python tools/cluster_trace.py AGENTS_PER_SIDE SKIP STEPS
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_4933_b200 as p  # noqa: E402

n, skip, steps = (int(x) for x in sys.argv[1:4])
cfg = p.ScenarioConfig(width=480, height=480, agents_per_side=n, model=p.Model.Lem, seed=42)
e = p.Ensemble(cfg, replicas=1)
e.run(skip)
e.ctx.synchronize()
print("---", flush=True)
e.run(steps)
e.ctx.synchronize()
