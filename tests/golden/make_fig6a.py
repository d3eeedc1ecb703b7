"""Generate tests/golden/fig6a.json: SPEC.md acceptance #5 (the desk-scale
Fig. 6a analog) as run by the UNMODIFIED reference library.

96x96 grid, 5000 steps, seeds 42..51, 230 / 507 / 1843 agents per side
(5% / 11% / 40% of the cells), both models, through oracle/_ref (the
reference's src/ compiled by oracle/Makefile) with its parallel executor. The
fixture holds every run's throughput (final cumulative crossings,
src/engine.cpp:223) and series hash, so the GPU sweep is checked run by run
and the acceptance properties are evaluated on the reference's own numbers.

Usage (build container only; needs /root/reference and oracle/_ref):
    python tests/golden/make_fig6a.py
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference, Scenario, series_hash  # noqa: E402

FILLS = {"5%": 230, "11%": 507, "40%": 1843}
SEEDS = list(range(42, 52))
STEPS = 5000


def main():
    out = {"grid": [96, 96], "steps": STEPS, "seeds": SEEDS, "fills": FILLS, "runs": {}}
    for model in ("lem", "aco"):
        for name, d in FILLS.items():
            rows = []
            for s in SEEDS:
                rep, _ = Reference(Scenario(width=96, height=96, agents_per_side=d, model=model, seed=s),
                                   threads=os.cpu_count() or 1).run(STEPS)
                thr = int(rep["newly_crossed_top"].sum() + rep["newly_crossed_bottom"].sum())
                rows.append({"seed": s, "throughput": thr, "series_hash": f"{series_hash(rep):016x}"})
            out["runs"][f"{model}/{name}"] = rows
            mean = sum(r["throughput"] for r in rows) / len(rows) / (2 * d)
            print(f"{model} {name}: mean throughput fraction {mean:.4f}")
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "fig6a.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
