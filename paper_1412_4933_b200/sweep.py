"""Density sweeps and repeat batches on the GPU engine.

The reference's `sweep` (tools/pedflow.cpp:148-189) runs, for every density
and model, `repeats` seeds (seed, seed+1, ...) through run_scenario and
aggregates each group with `aggregate` (src/metrics.cpp:34-59) into one
SweepRow (inc/metrics.hpp:50-57). At 480x480 one scenario is far too small to
fill a B200, so here every (density, repeat) run of one model shares each
step's launch: one context with per-replica densities and seeds
(pf_set_replicas). The results per run are bit-identical to running them one
by one (tests/test_sweep.py checks against the oracle).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, replace

import numpy as np

from .engine import ConfigError, Model, RunReport, ScenarioConfig, StepSeriesRow, validate
from .ensemble import Ensemble

# Device bytes per cell and replica for the step planes (2 cell words + 2 tau
# pairs + tour for ACO), used to split very large batches.
_BYTES_PER_CELL = {Model.Lem: 8, Model.Aco: 8 + 32 + 8}
DEFAULT_BATCH_BYTES = 48 << 30


@dataclass
class SweepRow:
    """inc/metrics.hpp:50-57."""

    agents_total: int = 0
    model: Model = Model.Lem
    repeats: int = 0
    throughput_mean: float = 0.0
    throughput_sd: float = 0.0
    runtime_mean_seconds: float = 0.0


def aggregate(reports: list[RunReport]) -> SweepRow:
    """aggregate (src/metrics.cpp:34-59): mean/sample-sd of throughput and mean
    runtime over the repeats of one configuration, accumulated in run order."""
    if not reports:
        raise ValueError("aggregate: empty report list")
    row = SweepRow(agents_total=reports[0].agents_total, model=reports[0].model, repeats=len(reports))
    sum_thr = 0.0
    sum_rt = 0.0
    for r in reports:
        sum_thr += float(r.throughput)
        sum_rt += r.runtime_seconds
    n = float(len(reports))
    row.throughput_mean = sum_thr / n
    row.runtime_mean_seconds = sum_rt / n
    if len(reports) > 1:
        ss = 0.0
        for r in reports:
            d = float(r.throughput) - row.throughput_mean
            ss += d * d
        row.throughput_sd = math.sqrt(ss / (n - 1.0))
    return row


@dataclass
class ProportionTest:
    """inc/metrics.hpp:40-43."""

    p_value: float = 1.0
    defined: bool = True  # False when both runs have zero agents


def proportion_test(a: RunReport, b: RunReport) -> ProportionTest:
    """proportion_test (src/metrics.cpp:18-32): two-sided two-proportion z-test
    on the crossing fractions of two runs with the same agents_total."""
    if a.agents_total != b.agents_total:
        raise ValueError("proportion_test: runs must share agents_total")
    if a.agents_total == 0:
        return ProportionTest(1.0, False)
    if a.throughput == b.throughput:
        return ProportionTest(1.0, True)
    n = float(a.agents_total)
    p1 = float(a.throughput) / n
    p2 = float(b.throughput) / n
    pooled = (float(a.throughput) + float(b.throughput)) / (2.0 * n)
    se = math.sqrt(pooled * (1.0 - pooled) * (2.0 / n))
    if se == 0.0:
        return ProportionTest(1.0, True)
    z = (p1 - p2) / se
    return ProportionTest(math.erfc(abs(z) / math.sqrt(2.0)), True)


def default_sweep_densities(cfg: ScenarioConfig) -> list[int]:
    """tools/pedflow.cpp:148-157: 1,280 .. 51,200 per side on 480x480."""
    if cfg.width == 480 and cfg.height == 480:
        return [1280 * k for k in range(1, 41)]
    raise ConfigError("no default densities for this grid size; pass --densities")


def models_to_run(cfg: ScenarioConfig) -> list[Model]:
    """tools/pedflow.cpp:113-116: both models unless the model was picked."""
    return [Model(cfg.model)] if cfg.model_explicit else [Model.Lem, Model.Aco]


def run_batch(cfg: ScenarioConfig, runs: list[tuple[int, int]], *, device: int = 0, kernel: str = "fused",
              batch_bytes: int = DEFAULT_BATCH_BYTES) -> list[RunReport]:
    """run_scenario (src/engine.cpp:195-231) for every (agents_per_side, seed)
    in `runs`, all of `cfg.model`, stepped together `cfg.steps` times.
    runtime_seconds is the batch's wall time (setup included, like the
    reference) split evenly over its runs."""
    model = Model(cfg.model)
    for aps, _ in runs:
        validate(replace(cfg, agents_per_side=aps))
    per_rep = (cfg.height + 6) * cfg.width * _BYTES_PER_CELL[model]
    chunk = max(1, min(65535, batch_bytes // per_rep))
    out: list[RunReport] = []
    for i0 in range(0, len(runs), chunk):
        part = runs[i0:i0 + chunk]
        t0 = time.perf_counter()
        ens = Ensemble(replace(cfg, agents_per_side=part[0][0]), replicas=len(part), device=device, kernel=kernel,
                       agents_per_side=[a for a, _ in part], seeds=[s for _, s in part])
        rep = ens.run(cfg.steps) if cfg.steps else None
        ens.close()
        share = (time.perf_counter() - t0) / len(part)
        for j, (aps, seed) in enumerate(part):
            series = []
            thr = 0
            if rep is not None:
                r = rep[j]
                top = np.cumsum(r["newly_crossed_top"].astype(np.int64))
                bot = np.cumsum(r["newly_crossed_bottom"].astype(np.int64))
                series = [StepSeriesRow(int(r["step"][s]), int(top[s]), int(bot[s]), int(top[s] + bot[s]),
                                        int(r["moved"][s])) for s in range(cfg.steps)]
                thr = int(top[-1] + bot[-1])
            c = replace(cfg, agents_per_side=aps)
            out.append(RunReport(config=c, seed=seed, model=model, executor=cfg.executor, threads=cfg.threads,
                                 agents_total=2 * aps, series=series, throughput=thr, runtime_seconds=share))
    return out


def sweep(cfg: ScenarioConfig, densities: list[int] | None = None, *, device: int = 0, kernel: str = "fused",
          batch_bytes: int = DEFAULT_BATCH_BYTES) -> list[SweepRow]:
    """cmd_sweep (tools/pedflow.cpp:159-189): one SweepRow per (density,
    model) in the reference's order, each over cfg.repeats seeds. Every
    density is validated before anything runs."""
    densities = list(densities) if densities else default_sweep_densities(cfg)
    for d in densities:
        validate(replace(cfg, agents_per_side=d))
    by_model = {}
    for m in models_to_run(cfg):
        mcfg = replace(cfg, model=m, model_explicit=True)
        runs = [(d, (cfg.seed + i) % 2**64) for d in densities for i in range(cfg.repeats)]  # uint64 wrap
        by_model[m] = run_batch(mcfg, runs, device=device, kernel=kernel, batch_bytes=batch_bytes)
    rows = []
    for k, _ in enumerate(densities):
        for m in models_to_run(cfg):
            rows.append(aggregate(by_model[m][k * cfg.repeats:(k + 1) * cfg.repeats]))
    return rows


__all__ = ["ProportionTest", "SweepRow", "aggregate", "proportion_test", "default_sweep_densities", "models_to_run", "run_batch", "sweep"]
