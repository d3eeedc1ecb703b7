"""Fused-halo overhead on ONE device (dev tool): a workload split into k
linked row shards (pf_peer_attach, same process), all stepped with
graph-batched pf_step_async, vs the unsharded context. The shards share the
GPU, so the ideal is equal total time; the difference is the per-step
handshake + boundary mirroring + the extra launches.

    python tools/shard_time.py c5_aco 2 4
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1412_4933_b200 as p  # noqa: E402
from paper_1412_4933_b200 import _lib  # noqa: E402
from paper_1412_4933_b200.engine import _pf_config  # noqa: E402
from paper_1412_4933_b200.sharding import row_partition  # noqa: E402

name = sys.argv[1]
cfg, reps, desc = bench.scenario(name)
steps = 100
for k in [1] + [int(x) for x in sys.argv[2:]]:
    ctxs = []
    for lo, hi in row_partition(cfg.height, k):
        c = _lib.Context(_pf_config(cfg, 42, replicas=reps, row_begin=0 if k == 1 else lo, row_end=0 if k == 1 else hi))
        c.init_environment()
        ctxs.append(c)
    if k > 1:
        _lib.link_shards(ctxs)
    for c in ctxs:
        c.step_async(5)
    for c in ctxs:
        c.synchronize()
    t0 = time.perf_counter()
    for c in ctxs:
        c.step_async(steps)
    for c in ctxs:
        c.synchronize()
    dt = (time.perf_counter() - t0) / steps * 1e3
    print(f"{name} shards={k}: {dt:.3f} ms/step (wall, {steps} steps, all shards on one GPU)", flush=True)
    for c in ctxs:
        c.close()
    torch.cuda.empty_cache()
