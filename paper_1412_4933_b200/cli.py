"""The reference CLI's `simulate` and `sweep` on the GPU engine, with its CSV outputs.

    python -m paper_1412_4933_b200.cli simulate --model aco --agents-per-side 1280 --steps 2000 --repeats 2 --out runs/
    python -m paper_1412_4933_b200.cli sweep --model lem --steps 1000 --repeats 10 --densities 1280,2560 --out runs/

Flags, the `--config` scenario file and their precedence follow
tools/pedflow.cpp:40-97 (only flags the user passed override the file).
`simulate` (tools/pedflow.cpp:132-146) runs `repeats` seeds (seed, seed+1, ...)
and writes steps.csv / summary.csv; `sweep` (tools/pedflow.cpp:148-189) runs
every density x model x repeat and writes sweep.csv. Headers, row order,
%.10g doubles, the summary's `mean` row and --zero-timings (0 in the
wall-clock columns) follow src/csv.cpp:8-54. All runs of one model share each
step's launch (paper_1412_4933_b200/sweep.py). The executor column reads `gpu`.
Runtime columns are the batch's wall time split evenly over its runs. Exit
codes: 2 config error, 1 other (tools/pedflow.cpp:253-258). The reference's
`bench` (sequential vs parallel CPU executors) has no GPU counterpart; see
bench.py.
"""
from __future__ import annotations

import argparse
import os
import re
import sys

from .config import parse_config
from .engine import ConfigError, Model, RunReport
from .sweep import SweepRow, aggregate, run_batch, sweep

STEPS_HEADER = "run_id,seed,model,executor,step,crossed_top,crossed_bottom,crossed_total,moved"
SUMMARY_HEADER = "run_id,seed,model,executor,agents_total,steps,throughput,runtime_seconds"
SWEEP_HEADER = "agents_total,model,repeats,throughput_mean,throughput_sd,runtime_mean_seconds"
EXECUTOR = "gpu"
_STOI = re.compile(r"[ \t\n\v\f\r]*[+-]?[0-9]+\Z")


def format_double(v: float) -> str:
    return "%.10g" % v  # src/csv.cpp:8-12


def _model(m) -> str:
    return "lem" if Model(m) == Model.Lem else "aco"  # src/config.cpp:12


def write_steps_csv(runs: list[RunReport]) -> str:
    """src/csv.cpp:14-24."""
    out = [STEPS_HEADER + "\n"]
    for i, r in enumerate(runs):
        for row in r.series:
            out.append(f"{i},{r.seed},{_model(r.model)},{EXECUTOR},{row.step},{row.crossed_top},"
                       f"{row.crossed_bottom},{row.crossed_total},{row.moved}\n")
    return "".join(out)


def write_summary_csv(runs: list[RunReport], zero_timings: bool) -> str:
    """src/csv.cpp:26-44, including the trailing `mean` row for repeats > 1."""
    out = [SUMMARY_HEADER + "\n"]
    for i, r in enumerate(runs):
        rt = 0.0 if zero_timings else r.runtime_seconds
        out.append(f"{i},{r.seed},{_model(r.model)},{EXECUTOR},{r.agents_total},{r.config.steps},{r.throughput},"
                   f"{format_double(rt)}\n")
    if len(runs) > 1:
        agg = aggregate(runs)
        rt = 0.0 if zero_timings else agg.runtime_mean_seconds
        out.append(f"mean,{runs[0].seed},{_model(runs[0].model)},{EXECUTOR},{agg.agents_total},"
                   f"{runs[0].config.steps},{format_double(agg.throughput_mean)},{format_double(rt)}\n")
    return "".join(out)


def write_sweep_csv(rows: list[SweepRow], zero_timings: bool) -> str:
    """src/csv.cpp:46-54."""
    out = [SWEEP_HEADER + "\n"]
    for r in rows:
        rt = 0.0 if zero_timings else r.runtime_mean_seconds
        out.append(f"{r.agents_total},{_model(r.model)},{r.repeats},{format_double(r.throughput_mean)},"
                   f"{format_double(r.throughput_sd)},{format_double(rt)}\n")
    return "".join(out)


def _write(path: str, text: str):
    with open(path, "w", encoding="utf-8", newline="") as f:
        f.write(text)


def simulate(cfg, zero_timings: bool = False, device: int = 0) -> list[RunReport]:
    """cmd_simulate (tools/pedflow.cpp:132-146)."""
    runs = run_batch(cfg, [(cfg.agents_per_side, (cfg.seed + i) % 2**64) for i in range(cfg.repeats)], device=device)
    os.makedirs(cfg.out_dir, exist_ok=True)
    _write(os.path.join(cfg.out_dir, "steps.csv"), write_steps_csv(runs))
    _write(os.path.join(cfg.out_dir, "summary.csv"), write_summary_csv(runs, zero_timings))
    return runs


def run_sweep(cfg, densities: list[int] | None, zero_timings: bool = False, device: int = 0) -> list[SweepRow]:
    """cmd_sweep (tools/pedflow.cpp:159-189)."""
    rows = sweep(cfg, densities, device=device)
    os.makedirs(cfg.out_dir, exist_ok=True)
    _write(os.path.join(cfg.out_dir, "sweep.csv"), write_sweep_csv(rows, zero_timings))
    return rows


def parse_densities(text: str) -> list[int]:
    """tools/pedflow.cpp:91-111: comma-separated items, each a whole std::stoi
    parse (leading whitespace and sign allowed) of a non-negative int."""
    out = []
    pos = 0
    while pos < len(text):
        comma = text.find(",", pos)
        if comma < 0:
            comma = len(text)
        item = text[pos:comma]
        if not _STOI.match(item) or not 0 <= int(item) <= 2**31 - 1:
            raise ConfigError(f"malformed value for key 'densities': '{item}'")
        out.append(int(item))
        pos = comma + 1
    return out


_FLAGS = [  # (flag, config key, argparse type)
    ("--width", "width", int), ("--height", "height", int), ("--agents-per-side", "agents_per_side", int),
    ("--model", "model", str), ("--steps", "steps", int), ("--seed", "seed", int), ("--repeats", "repeats", int),
    ("--executor", "executor", str), ("--threads", "threads", int), ("--d0", "d0", float),
    ("--sel-mu", "sel_mu", float), ("--sel-sigma", "sel_sigma", float), ("--alpha", "alpha", float),
    ("--beta", "beta", float), ("--rho", "rho", float), ("--tau0", "tau0", float), ("--q", "q", float),
    ("--out", "out_dir", str),
]


def _fmt(v) -> str:
    return "%.17g" % v if isinstance(v, float) else str(v)  # fmt_full, tools/pedflow.cpp:35-39


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="pedflow-b200", description="bi-directional pedestrian flow simulator (GPU)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    cmds = {"simulate": sub.add_parser("simulate", help="run one scenario over repeated seeds"),
            "sweep": sub.add_parser("sweep", help="density sweep over one or both models")}
    for name, p in cmds.items():
        p.add_argument("--config", default="", help="flat key = value scenario file")
        for flag, key, typ in _FLAGS:
            p.add_argument(flag, dest=key, type=typ, default=None)
        p.add_argument("--zero-timings", action="store_true")
        p.add_argument("--device", type=int, default=0)
        if name == "sweep":
            p.add_argument("--densities", default="")
    args = ap.parse_args(argv)
    try:
        overrides = [(key, _fmt(getattr(args, key))) for _, key, _ in _FLAGS if getattr(args, key) is not None]
        cfg = parse_config(args.config, overrides)
        densities = parse_densities(args.densities) if getattr(args, "densities", "") else []
        if args.cmd == "simulate":
            simulate(cfg, args.zero_timings, args.device)
            print(f"wrote {os.path.join(cfg.out_dir, 'steps.csv')} and {os.path.join(cfg.out_dir, 'summary.csv')}")
        else:
            run_sweep(cfg, densities or None, args.zero_timings, args.device)
            print(f"wrote {os.path.join(cfg.out_dir, 'sweep.csv')}")
        return 0
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 - CLI boundary, mirrors tools/pedflow.cpp:253-258
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
