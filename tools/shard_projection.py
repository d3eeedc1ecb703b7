"""Per-GPU step time of one row shard of C5 at P = 1, 2, 4, 8 GPUs, measured on ONE
GPU (dev tool). Each shard context owns rows [H*r/P, H*(r+1)/P) plus 3 ghost rows
and is stepped alone (unlinked: its ghost rows are not refreshed, so this times
the shard's own work, not the exchange). Interior and edge shards are timed.
The exchange cost is measured separately by linked shards on one GPU
(bench secondary c5_aco_linked_shards_one_gpu). Projection, not a scaling run.

    python tools/shard_projection.py [c5_aco|c5_lem] [steps] [equal|balanced]

equal: row_partition (equal rows; an edge and an interior shard are timed);
balanced: balanced_row_partition (ShardedEngine's cost-weighted rows; every
shard is timed).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1412_4933_b200 import _lib  # noqa: E402
from paper_1412_4933_b200.engine import _pf_config  # noqa: E402
from paper_1412_4933_b200.sharding import balanced_row_partition, row_partition  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5_aco"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
mode = sys.argv[3] if len(sys.argv) > 3 else "equal"
cfg, reps, desc = bench.scenario(name)
out = {"workload": desc, "steps": steps, "window": f"steps 5..{5 + steps}", "partition": mode, "per_P": {}}
for P in (1, 2, 4, 8):
    parts = row_partition(cfg.height, P) if mode == "equal" else balanced_row_partition(cfg, P)
    times = {}
    ranks = sorted({0, P // 2}) if mode == "equal" else range(P)
    for r in ranks:  # equal: an edge shard (band rows) and an interior one
        lo, hi = parts[r]
        c = _lib.Context(_pf_config(cfg, 42, row_begin=0 if P == 1 else lo, row_end=0 if P == 1 else hi))
        c.init_environment()
        c.step(5)
        c.prepare_steps(steps)
        tot, _ = c.time_steps(steps)
        times[f"shard{r}_rows_{lo}_{hi}"] = tot / steps
        c.close()
    worst = max(times.values())
    out["per_P"][P] = {"ms_per_step_by_shard": times, "ms_per_step_max": worst}
base = out["per_P"][1]["ms_per_step_max"]
for P, v in out["per_P"].items():
    v["projected_speedup_compute_only"] = base / v["ms_per_step_max"]
print(json.dumps(out, indent=1))
