"""Generate tests/golden/anchors.json from the UNMODIFIED reference.

Runs oracle/_ref/libpedflow_ref.so (the reference library compiled from
/root/reference/proj/src by oracle/Makefile, Parallel executor, 8 threads — the
reference guarantees results independent of thread count) from
new_environment(cfg, seed) through StepEngine::step x N, and records:

* scalar anchors — step-0 moved, sum of moved, cumulative crossings;
* FNV-1a 64 hashes (offset 0xcbf29ce484222325, prime 0x100000001b3) over
  little-endian bytes of: ``index`` (u32 grid, row-major), ``occ`` (u8 grid),
  ``agents`` (per id: i32 row, i32 col, f64 tour_length, u8 crossed — 17 B),
  ``pher`` (top then bottom f64 grids, ACO only), ``series`` (per step the
  16-byte StepReport);
* the full per-step series as a list (for first-divergence reports).

The scalar anchors of SURVEY.md §8(c) are reproduced exactly (checked below);
its hex hashes use a byte layout the survey does not fully specify, so the
hashes here are regenerated with the definition above.

Usage (build container only; needs /root/reference):
    python tests/golden/make_golden.py [--big | --c5-long]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference, Scenario, series_hash  # noqa: E402

# name: (scenario kwargs, steps, survey scalar anchors (step0 moved, crossed T, crossed B, sum moved) or None)
CONFIGS = {
    "C1_lem_480_1024": (dict(width=480, height=480, agents_per_side=1024, model="lem"), 2000, (1338, 1024, 1024, 2394866)),
    "C2_aco_480_1024": (dict(width=480, height=480, agents_per_side=1024, model="aco"), 2000, (1329, 1024, 1024, 2261415)),
    "C3_lem_480_51200": (dict(width=480, height=480, agents_per_side=51200, model="lem"), 1000, (1274, 0, 0, 19889429)),
    "C4_aco_480_51200": (dict(width=480, height=480, agents_per_side=51200, model="aco"), 1000, (1274, 0, 0, 19354110)),
    "S96_aco_96_256": (dict(width=96, height=96, agents_per_side=256, model="aco"), 5000, (232, 256, 256, 987041)),
    # small grids in the spirit of SPEC acceptance #1 (32x32 / 96x96, both models, 200 steps)
    "s32_lem_64_s7": (dict(width=32, height=32, agents_per_side=64, model="lem", seed=7), 200, None),
    "s32_aco_64_s7": (dict(width=32, height=32, agents_per_side=64, model="aco", seed=7), 200, None),
    "s32_lem_200_s3": (dict(width=32, height=32, agents_per_side=200, model="lem", seed=3), 200, None),
    "s32_aco_200_s3": (dict(width=32, height=32, agents_per_side=200, model="aco", seed=3), 200, None),
    "s96_lem_900_s11": (dict(width=96, height=96, agents_per_side=900, model="lem", seed=11), 200, None),
    "s96_aco_900_s11": (dict(width=96, height=96, agents_per_side=900, model="aco", seed=11), 200, None),
    "s96_aco_2000_s5_alt": (dict(width=96, height=96, agents_per_side=2000, model="aco", seed=5, alpha=0.0,
                                 beta=1.0, rho=0.3, tau0=0.5, q=2.0), 200, None),
    "s96_lem_2000_s5_alt": (dict(width=96, height=96, agents_per_side=2000, model="lem", seed=5, d0=3.0,
                                 sel_mu=0.8, sel_sigma=1.5), 200, None),
    "r48x32_aco_300_s9": (dict(width=48, height=32, agents_per_side=300, model="aco", seed=9), 300, None),
    "r16x64_lem_16_s1": (dict(width=16, height=64, agents_per_side=16, model="lem", seed=1), 100, None),
    "empty_aco_32": (dict(width=32, height=32, agents_per_side=0, model="aco"), 20, None),
    "full_band_lem_16": (dict(width=16, height=16, agents_per_side=128, model="lem"), 50, None),
}

BIG = {
    # C5 is too large for per-step oracle runs: a short window anchors it.
    "C5_aco_16384_25M": (dict(width=16384, height=16384, agents_per_side=25_000_000, model="aco"), 3, None),
    "C5_lem_16384_25M": (dict(width=16384, height=16384, agents_per_side=25_000_000, model="lem"), 3, None),
}


def run_one(name, kw, steps, survey, threads):
    sc = Scenario(**kw)
    t0 = time.time()
    ref = Reference(sc, threads=threads)
    t_setup = time.time() - t0
    rep, secs = ref.run(steps)
    h = ref.hashes()
    moved = rep["moved"].astype("int64")
    entry = {
        "scenario": kw,
        "steps": steps,
        "step0_moved": int(moved[0]) if steps else 0,
        "sum_moved": int(moved.sum()),
        "crossed_top": int(rep["newly_crossed_top"].sum()),
        "crossed_bottom": int(rep["newly_crossed_bottom"].sum()),
        "hash": {k: f"{v:016x}" for k, v in h.items()},
        "series_hash": f"{series_hash(rep):016x}",
    }
    if steps <= 5000 and sc.width * sc.height <= 480 * 480:
        entry["series"] = rep.view("<u4").reshape(-1, 4)[:, 1:].tolist()  # moved, top, bottom
    if survey is not None:
        got = (entry["step0_moved"], entry["crossed_top"], entry["crossed_bottom"], entry["sum_moved"])
        entry["survey_scalar_anchors_match"] = got == survey
        assert got == survey, (name, got, survey)
    print(f"{name}: setup {t_setup:.1f}s, {steps} steps {secs:.1f}s, {entry['hash']}", flush=True)
    return entry


# Long C5 horizons with checkpoints: one reference run per model, hashed at each
# checkpoint (the bench window and the sharded tests sit inside them).
C5_LONG = {
    "C5_aco_long": dict(width=16384, height=16384, agents_per_side=25_000_000, model="aco"),
    "C5_lem_long": dict(width=16384, height=16384, agents_per_side=25_000_000, model="lem"),
}
C5_CHECKPOINTS = (10, 30, 100, 300)


def run_long(name, kw, checkpoints, threads):
    sc = Scenario(**kw)
    t0 = time.time()
    ref = Reference(sc, threads=threads)
    print(f"{name}: setup {time.time() - t0:.1f}s", flush=True)
    reps, cps, done = [], {}, 0
    for cp in checkpoints:
        rep, secs = ref.run(cp - done)
        reps.append(rep)
        done = cp
        h = ref.hashes()
        cps[str(cp)] = {k: f"{v:016x}" for k, v in h.items()}
        print(f"{name}: step {cp} ({secs:.1f}s) {cps[str(cp)]}", flush=True)
    import numpy as np

    rep = np.concatenate(reps)
    return {
        "scenario": kw,
        "steps": done,
        "checkpoints": cps,
        "series": rep.view("<u4").reshape(-1, 4)[:, 1:].tolist(),
        "series_hash": f"{series_hash(rep):016x}",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also anchor C5 (needs ~14 GB RAM, ~2 min)")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--c5-long", action="store_true",
                    help="only the C5 checkpointed anchors (steps %s; ~1 h on 8 cores)" % (C5_CHECKPOINTS,))
    args = ap.parse_args()
    path = os.path.join(HERE, "anchors.json")
    old = json.load(open(path)) if os.path.exists(path) else {}
    out = dict(old)
    if args.c5_long:
        for name, kw in C5_LONG.items():
            out[name] = run_long(name, kw, C5_CHECKPOINTS, args.threads)
            with open(path, "w") as f:
                json.dump(out, f, indent=1, sort_keys=True)
        print("wrote", path)
        return
    todo = dict(CONFIGS)
    if args.big:
        todo.update(BIG)
    for name, (kw, steps, survey) in todo.items():
        out[name] = run_one(name, kw, steps, survey, args.threads)
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
