"""`simulate` on the GPU engine with the reference CLI's CSV outputs.

    python -m paper_1412_4933_b200.cli simulate --model aco --agents-per-side 1280 --steps 2000 --repeats 2 --out runs/

The reference's `pedflow simulate` (tools/pedflow.cpp:132-146) runs `repeats`
seeds (seed, seed+1, ..., tools/pedflow.cpp:135) through run_scenario and
writes steps.csv / summary.csv with the headers of SPEC.md:519-522 and
doubles as %.10g (src/csv.cpp:8-44). This mirror runs all repeats in one
replica-batched launch per step. Runtime columns are the GPU job's wall time
(split evenly over the repeats), or blank with --zero-timings
(inc/csv.hpp:11-16). Exit codes: 2 config error, 1 other (tools/pedflow.cpp:253-258).
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

from .engine import ConfigError, Model, ScenarioConfig, validate
from .ensemble import Ensemble

STEPS_HEADER = "run_id,seed,model,executor,step,crossed_top,crossed_bottom,crossed_total,moved"
SUMMARY_HEADER = "run_id,seed,model,executor,agents_total,steps,throughput,runtime_seconds"


def format_double(v: float) -> str:
    return "%.10g" % v  # src/csv.cpp:8-12


def simulate(cfg: ScenarioConfig, out_dir: str, zero_timings: bool = False, device: int = 0) -> list[dict]:
    validate(cfg)
    os.makedirs(out_dir, exist_ok=True)
    model = "lem" if Model(cfg.model) == Model.Lem else "aco"
    t0 = time.perf_counter()
    ens = Ensemble(cfg, replicas=cfg.repeats, seed=cfg.seed, device=device)
    rep = ens.run(cfg.steps) if cfg.steps else np.zeros((cfg.repeats, 0))
    ens.close()
    wall = time.perf_counter() - t0
    runs = []
    with open(os.path.join(out_dir, "steps.csv"), "w") as f:
        f.write(STEPS_HEADER + "\n")
        for i in range(cfg.repeats):
            r = rep[i]
            top = np.cumsum(r["newly_crossed_top"].astype(np.int64)) if cfg.steps else np.zeros(0, np.int64)
            bot = np.cumsum(r["newly_crossed_bottom"].astype(np.int64)) if cfg.steps else np.zeros(0, np.int64)
            for s in range(cfg.steps):
                f.write(f"{i},{cfg.seed + i},{model},gpu,{int(r['step'][s])},{int(top[s])},{int(bot[s])},"
                        f"{int(top[s] + bot[s])},{int(r['moved'][s])}\n")
            runs.append(dict(run_id=i, seed=cfg.seed + i, throughput=int(top[-1] + bot[-1]) if cfg.steps else 0))
    with open(os.path.join(out_dir, "summary.csv"), "w") as f:
        f.write(SUMMARY_HEADER + "\n")
        for r in runs:
            rt = "" if zero_timings else format_double(wall / cfg.repeats)
            f.write(f"{r['run_id']},{r['seed']},{model},gpu,{2 * cfg.agents_per_side},{cfg.steps},{r['throughput']},{rt}\n")
    return runs


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="pedflow-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("simulate")
    d = ScenarioConfig()
    for name in ("width", "height", "agents_per_side", "steps", "seed", "repeats"):
        s.add_argument("--" + name.replace("_", "-"), type=int, default=getattr(d, name))
    for name in ("d0", "sel_mu", "sel_sigma", "alpha", "beta", "rho", "tau0", "q"):
        s.add_argument("--" + name.replace("_", "-"), type=float, default=getattr(d, name))
    s.add_argument("--model", choices=["lem", "aco"], default="aco")
    s.add_argument("--out", default=".")
    s.add_argument("--zero-timings", action="store_true")
    s.add_argument("--device", type=int, default=0)
    args = ap.parse_args(argv)
    try:
        cfg = ScenarioConfig(width=args.width, height=args.height, agents_per_side=args.agents_per_side,
                             model=Model.Lem if args.model == "lem" else Model.Aco, steps=args.steps, seed=args.seed,
                             repeats=args.repeats, d0=args.d0, sel_mu=args.sel_mu, sel_sigma=args.sel_sigma,
                             alpha=args.alpha, beta=args.beta, rho=args.rho, tau0=args.tau0, q=args.q,
                             out_dir=args.out)
        simulate(cfg, args.out, args.zero_timings, args.device)
        print(f"wrote {os.path.join(args.out, 'steps.csv')} and summary.csv")
        return 0
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 - CLI boundary, mirrors tools/pedflow.cpp:253-258
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
