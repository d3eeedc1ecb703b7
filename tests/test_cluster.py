"""The cluster-resident LEM kernel (pf_cluster.cu): small LEM grids run all the
steps of a launch inside one thread-block cluster, state in distributed
shared memory. Bit-exact against the reference anchors (tests/golden, made
from oracle/_ref) and the oracle, with the bit-plane kernel as the other arm
(PEDFLOW_CLUSTER=0)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from tests.helpers import first_divergence, hashes_of, hex_hashes, to_config, to_scenario

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _any_density(monkeypatch):
    """The product takes the cluster path only for sparse grids
    (kMaxDensity); these tests force it at every density so the dense
    anchors (C3, the full bands) check it too."""
    monkeypatch.setenv("PEDFLOW_CLUSTER_MAX_DENSITY", "1")

LEM_ANCHORS = ["s32_lem_64_s7", "s32_lem_200_s3", "s96_lem_900_s11", "s96_lem_2000_s5_alt", "r16x64_lem_16_s1",
               "full_band_lem_16", "C1_lem_480_1024", "C3_lem_480_51200"]


def _with_env(env: dict, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _run(kw, steps, env):
    import paper_1412_4933_b200 as p

    def go():
        cfg = to_config(kw)
        seed = kw.get("seed", 42)
        state = p.new_environment(cfg, seed)
        eng = p.StepEngine(p.EngineOptions.from_config(cfg, seed))
        rep = eng.run_array(state, steps)
        return state, rep, eng.context.launches

    return _with_env(env, go)


@pytest.mark.parametrize("cluster", ["1", "0"])
@pytest.mark.parametrize("name", LEM_ANCHORS)
def test_lem_anchor_cluster_and_bitplane(anchors, name, cluster):
    a = anchors[name]
    state, rep, launches = _run(a["scenario"], a["steps"], {"PEDFLOW_CLUSTER": cluster})
    ser = np.stack([rep["moved"], rep["newly_crossed_top"], rep["newly_crossed_bottom"]], 1)
    bad = np.nonzero((ser != np.asarray(a["series"])).any(1))[0]
    assert len(bad) == 0, f"series first differs at step {bad[0]}"
    assert list(rep["step"]) == list(range(a["steps"]))
    assert hex_hashes(hashes_of(state)) == a["hash"]
    # The cluster path is one launch per batch of up to 256 steps; the
    # bit-plane kernel takes one launch per step on these single small grids.
    if cluster == "1":
        assert launches < a["steps"] // 2, f"{launches} launches: the cluster path did not run"
    else:
        assert launches >= a["steps"]


def test_cluster_replicas_match_single_runs():
    """Several replicas, one cluster each (seed + i), against the oracle."""
    import paper_1412_4933_b200 as p
    from oracle.oracle import OracleState

    kw = dict(width=96, height=96, agents_per_side=900, model="lem", seed=100)
    ens = p.Ensemble(to_config(kw), replicas=5, seed=100)
    l0 = ens.ctx.launches
    rep = ens.run(120)
    assert ens.ctx.launches - l0 < 10
    for i in range(5):
        ora = OracleState(to_scenario(dict(kw, seed=100 + i)))
        o = ora.run(120)
        assert (rep[i]["moved"] == o["moved"]).all()
        assert (rep[i]["newly_crossed_top"] == o["newly_crossed_top"]).all()
        assert first_divergence(ens.state(i), ora) == "identical"


@pytest.mark.parametrize("shape", [(48, 16, 40), (80, 48, 300), (480, 16, 60), (16, 128, 50)])
def test_cluster_odd_shapes_vs_oracle(shape):
    """Widths that are multiples of 16 but not of 32 (partial plane
    segments and claim words), few rows, and batches split at odd step
    counts (one launch per call: 1, 7, 13, ... steps; the 1- and 7-step
    calls run on the bit-plane kernel, so the two kernels alternate on one
    state)."""
    import paper_1412_4933_b200 as p
    from oracle.oracle import OracleState

    w, h, n = shape
    kw = dict(width=w, height=h, agents_per_side=n, model="lem", seed=3)
    cfg = to_config(kw)
    state = p.new_environment(cfg, 3)
    ora = OracleState(to_scenario(kw))
    eng = p.StepEngine(p.EngineOptions.from_config(cfg, 3))
    done = 0
    for k in (1, 7, 13, 29, 50):
        rep = eng.run_array(state, k)
        o = ora.run(k)
        assert (rep["moved"] == o["moved"]).all(), (done, k)
        assert list(rep["step"]) == list(range(done, done + k))
        done += k
        assert first_divergence(state, ora) == "identical", done


def test_cluster_one_launch_per_step_matches_batches():
    """PEDFLOW_MULTISTEP=0 (one launch per step: the bit-plane kernel, as
    every launch of fewer than 8 steps) against the default batched cluster
    launch, C3 over 150 steps."""
    kw = dict(width=480, height=480, agents_per_side=51200, model="lem")
    s1, r1, l1 = _run(kw, 150, {"PEDFLOW_MULTISTEP": "0"})
    s2, r2, l2 = _run(kw, 150, {"PEDFLOW_MULTISTEP": "1"})
    assert (r1 == r2).all()
    assert hashes_of(s1) == hashes_of(s2)
    assert l1 > l2


def test_default_density_cut(monkeypatch):
    """Without the override, sparse C1 takes the cluster path and dense C3
    the bit-plane kernel (one launch per step on a single 480^2 grid)."""
    monkeypatch.delenv("PEDFLOW_CLUSTER_MAX_DENSITY")
    for n, cluster in ((1024, True), (51200, False)):
        kw = dict(width=480, height=480, agents_per_side=n, model="lem")
        _, _, launches = _run(kw, 100, {})
        assert (launches < 50) == cluster, (n, launches)


def test_sparse_batch_in_waves_vs_oracle(monkeypatch):
    """A sparse 64-replica C1 batch runs one cluster per replica in waves
    (more replicas than resident clusters); replicas 0, 31 and 63 against the
    oracle over 300 steps."""
    import paper_1412_4933_b200 as p
    from oracle.oracle import OracleState

    monkeypatch.delenv("PEDFLOW_CLUSTER_MAX_DENSITY")
    kw = dict(width=480, height=480, agents_per_side=1024, model="lem", seed=7)
    ens = p.Ensemble(to_config(kw), replicas=64, seed=7)
    l0 = ens.ctx.launches  # (after the setup kernels)
    rep = ens.run(300)
    assert ens.ctx.launches - l0 < 10  # batches of <= 256 steps, one launch each
    for i in (0, 31, 63):
        ora = OracleState(to_scenario(dict(kw, seed=7 + i)))
        o = ora.run(300)
        assert (rep[i]["moved"] == o["moved"]).all()
        assert (rep[i]["newly_crossed_bottom"] == o["newly_crossed_bottom"]).all()
        assert first_divergence(ens.state(i), ora) == "identical"
