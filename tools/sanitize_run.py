"""Small workloads for compute-sanitizer (dev tool): every step kernel
variant on a few small grids, including 4 linked shards (fused halo).

    compute-sanitizer --tool memcheck  python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py
    SANITIZE_NO_LINK=1 compute-sanitizer --tool synccheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_4933_b200 as p  # noqa: E402
from paper_1412_4933_b200 import _lib  # noqa: E402
from paper_1412_4933_b200.engine import _pf_config  # noqa: E402
from paper_1412_4933_b200.sharding import row_partition  # noqa: E402

steps = int(os.environ.get("STEPS", "12"))
if os.environ.get("SANITIZE_NO_LINK"):  # kernels one at a time: no in-kernel waits between CTAs either
    os.environ["PEDFLOW_MULTISTEP"] = "0"
C = p.ScenarioConfig
for model in (p.Model.Lem, p.Model.Aco):
    # Small single grids take the small-grid geometry; the 64-replica 96^2
    # batch the regular 256-column one (several one-tile items per CTA); the
    # 20-replica 624-wide LEM batch the 320-column / 32-row one.
    # Dense bands (96^2 with 3000 per side: 32 rows) put agents in the ghost
    # rows of the 4-way shard split from step 0.
    # 192^2 x 64 (768 one-tile items per step) runs as multi-step launches.
    for w, h, n, reps in ((96, 96, 3000, 2), (624, 48, 6000, 1), (480, 64, 9000, 1), (96, 96, 3000, 64),
                          (624, 96, 9000, 20), (192, 192, 6000, 64)):
        cfg = C(width=w, height=h, agents_per_side=n, model=model, seed=5)
        for kernel in ("fused", "tile", "pipeline"):
            e = p.Ensemble(cfg, replicas=reps, kernel=kernel)
            e.run(steps)
            e.state(0)
            e.audit(0)
            e.close()
        if os.environ.get("SANITIZE_NO_LINK"):
            # synccheck runs kernels one at a time; linked shards on one GPU
            # wait inside their kernels for each other and need them concurrent.
            print(f"ok {model.name} {w}x{h} n={n} x{reps} (unlinked)", flush=True)
            continue
        shards = []
        for lo, hi in row_partition(h, 4):
            c = _lib.Context(_pf_config(cfg, 5, replicas=reps, row_begin=lo, row_end=hi))
            c.init_environment()
            shards.append(c)
        _lib.link_shards(shards)
        for c in shards:
            c.step_async(steps)
        for c in shards:
            c.synchronize()
            c.close()
        print(f"ok {model.name} {w}x{h} n={n} x{reps}", flush=True)
# The cluster-resident LEM kernel (pf_cluster.cu): sparse single grids take it
# by default; a dense one forced onto it; two replicas (two clusters); 16- and
# 8-CTA clusters (a 16-column grid needs 2-column slices: 8 CTAs).
for (w, h, n, reps, dens) in ((480, 480, 1024, 1, None), (96, 96, 200, 2, None), (96, 96, 3000, 1, "1"),
                              (16, 64, 16, 1, "1")):
    if dens:
        os.environ["PEDFLOW_CLUSTER_MAX_DENSITY"] = dens
    cfg = C(width=w, height=h, agents_per_side=n, model=p.Model.Lem, seed=5)
    e = p.Ensemble(cfg, replicas=reps)
    e.run(steps)
    e.state(0)
    e.audit(0)
    e.close()
    os.environ.pop("PEDFLOW_CLUSTER_MAX_DENSITY", None)
    print(f"ok cluster LEM {w}x{h} n={n} x{reps}", flush=True)
print("sanitize_run done")
