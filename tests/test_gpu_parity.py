"""GPU parity: the CUDA path (through the C-ABI) against the golden anchors
generated from the unmodified reference and against the C oracle, step by
step, bit-exact (integer planes, per-step counters AND the fp64 pheromone
fields: every double op is an IEEE round-to-nearest in reference order)."""
from __future__ import annotations

import numpy as np
import pytest

from tests.helpers import first_divergence, hashes_of, hex_hashes, to_config, to_scenario

pytestmark = pytest.mark.gpu

SMALL = ["s32_lem_64_s7", "s32_aco_64_s7", "s32_lem_200_s3", "s32_aco_200_s3", "s96_lem_900_s11",
         "s96_aco_900_s11", "s96_aco_2000_s5_alt", "s96_lem_2000_s5_alt", "r48x32_aco_300_s9",
         "r16x64_lem_16_s1", "empty_aco_32", "full_band_lem_16"]
BIG = ["C1_lem_480_1024", "C2_aco_480_1024", "C3_lem_480_51200", "C4_aco_480_51200", "S96_aco_96_256"]


def _run_gpu(kw, steps, kernel="fused"):
    import paper_1412_4933_b200 as p

    cfg = to_config(kw)
    seed = kw.get("seed", 42)
    state = p.new_environment(cfg, seed)
    eng = p.StepEngine(p.EngineOptions.from_config(cfg, seed, kernel=kernel))
    rep = eng.run_array(state, steps) if steps else np.zeros(0)
    return state, rep


@pytest.mark.parametrize("kernel", ["fused", "pipeline", "tile"])
@pytest.mark.parametrize("name", SMALL + BIG)
def test_golden_anchor(anchors, name, kernel):
    a = anchors[name]
    state, rep = _run_gpu(a["scenario"], a["steps"], kernel)
    got = hex_hashes(hashes_of(state))
    if a["steps"]:
        moved = rep["moved"].astype(np.int64)
        assert int(moved.sum()) == a["sum_moved"]
        assert int(rep["newly_crossed_top"].sum()) == a["crossed_top"]
        assert int(rep["newly_crossed_bottom"].sum()) == a["crossed_bottom"]
        if "series" in a:
            ser = np.stack([rep["moved"], rep["newly_crossed_top"], rep["newly_crossed_bottom"]], 1)
            bad = np.nonzero((ser != np.asarray(a["series"])).any(1))[0]
            assert len(bad) == 0, f"series first differs at step {bad[0]}"
        assert list(rep["step"]) == list(range(a["steps"]))
    assert got == a["hash"]
    assert state.step == a["steps"]


@pytest.mark.parametrize("name", ["s96_aco_900_s11", "s96_lem_2000_s5_alt", "s96_aco_2000_s5_alt", "r48x32_aco_300_s9"])
def test_step_by_step_vs_oracle(anchors, name):
    """Every step compared with the oracle; the first divergence is reported."""
    import paper_1412_4933_b200 as p
    from oracle.oracle import OracleState

    kw = anchors[name]["scenario"]
    ora = OracleState(to_scenario(kw))
    cfg = to_config(kw)
    seed = kw.get("seed", 42)
    state = p.new_environment(cfg, seed)
    eng = p.StepEngine(p.EngineOptions.from_config(cfg, seed))
    for t in range(60):
        r = eng.step(state)
        o = ora.run(1)[0]
        assert (r.step, r.moved, r.newly_crossed_top, r.newly_crossed_bottom) == tuple(int(x) for x in o), t
        msg = first_divergence(state, ora)
        assert msg == "identical", f"step {t}: {msg}"


def test_replicas_match_single_runs(anchors):
    """A replica-batched launch (seed+i per replica) equals independent runs."""
    import paper_1412_4933_b200 as p
    from oracle.oracle import OracleState

    kw = dict(width=96, height=96, agents_per_side=900, model="aco", seed=100)
    cfg = to_config(kw)
    ens = p.Ensemble(cfg, replicas=5, seed=100)
    rep = ens.run(40)
    for i in range(5):
        ora = OracleState(to_scenario(dict(kw, seed=100 + i)))
        o = ora.run(40)
        assert (rep[i]["moved"] == o["moved"]).all()
        s = ens.state(i)
        assert first_divergence(s, ora) == "identical"


@pytest.mark.parametrize("model", ["lem", "aco"])
def test_multistep_launch_matches_per_step_launches_and_oracle(model):
    """Dense batches run as multi-step launches with tile-level dependencies
    (pf_bitstep.cuh, launch()): 480^2 x 16 replicas at C3/C4 density (960
    one-tile items per step on ~600 resident CTAs) in graph batches of 256,
    100 and 1 steps must equal one launch per step (PEDFLOW_MULTISTEP=0) on
    every replica and every plane, through the crowds' meeting (~step 130),
    and the oracle on two replicas."""
    import os

    import paper_1412_4933_b200 as p
    from oracle.oracle import OracleState

    kw = dict(width=480, height=480, agents_per_side=51_200, model=model, seed=42)
    cfg = to_config(kw)
    R, steps = 16, 357
    ens = {}
    for flag in ("1", "0"):
        os.environ["PEDFLOW_MULTISTEP"] = flag
        try:
            e = p.Ensemble(cfg, replicas=R)
        finally:
            os.environ.pop("PEDFLOW_MULTISTEP", None)
        reps = [e.run(256), e.run(100), e.run(1)]
        ens[flag] = (e, np.concatenate(reps, axis=1))
    (em, rm), (es, rs) = ens["1"], ens["0"]
    assert (rm == rs).all()
    for i in range(R):
        assert hashes_of(em.state(i)) == hashes_of(es.state(i)), f"replica {i}"
    for i in (0, 11):
        ora = OracleState(to_scenario(dict(kw, seed=42 + i)))
        o = ora.run(steps)
        assert (rm[i]["moved"] == o["moved"]).all()
        assert first_divergence(em.state(i), ora) == "identical"
    em.close()
    es.close()


def test_multistep_launch_with_multi_tile_items():
    """Multi-step launches whose work items are chunks of several tiles
    (PEDFLOW_ITEMS_PER_CTA=1: 480^2 x 40 ACO, 4-tile items, 640 items per
    step): the dependency window spans the chunk's tiles +- 1. Equal to one
    launch per step on every replica over 200 steps."""
    import os

    import paper_1412_4933_b200 as p

    cfg = to_config(dict(width=480, height=480, agents_per_side=51_200, model="aco", seed=7))
    R = 40
    got = {}
    for flag in ("1", "0"):
        os.environ["PEDFLOW_MULTISTEP"] = flag
        os.environ["PEDFLOW_ITEMS_PER_CTA"] = "1"
        try:
            e = p.Ensemble(cfg, replicas=R, seed=7)
        finally:
            os.environ.pop("PEDFLOW_MULTISTEP", None)
            os.environ.pop("PEDFLOW_ITEMS_PER_CTA", None)
        rep = e.run(200)
        got[flag] = (rep, [hashes_of(e.state(i)) for i in range(R)])
        e.close()
    assert (got["1"][0] == got["0"][0]).all()
    assert got["1"][1] == got["0"][1]


def test_device_rng_matches_oracle():
    """Device Philox / uniform / AS241 normal vs the oracle (all three branches)."""
    from oracle.oracle import oracle
    from paper_1412_4933_b200 import _lib

    rng = np.random.default_rng(0)
    n = 20000
    seed = rng.integers(0, 2**63, n, dtype=np.uint64)
    step = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    phase = rng.integers(0, 5, n).astype(np.uint32)
    ent = rng.integers(0, 2**63, n, dtype=np.uint64)
    ctr = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    bits, uni, nrm = _lib.selftest_rng(seed, step, phase, ent, ctr, mu=0.7, sigma=0.35)
    lib = oracle()
    ob = np.array([lib.pfo_random_bits(int(a), int(b), int(c), int(d), int(e))
                   for a, b, c, d, e in zip(seed, step, phase, ent, ctr)], np.uint64)
    on = np.array([lib.pfo_normal(int(a), int(b), int(c), int(d), int(e), 0.7, 0.35)
                   for a, b, c, d, e in zip(seed, step, phase, ent, ctr)])
    assert (bits == ob).all()
    assert (uni == (ob >> np.uint64(11)).astype(np.float64) * 2.0**-53).all()
    # Every branch is exact: the tails' log is glibc's algorithm restated on the
    # device (pfdev::glibc_log).
    assert (nrm.view(np.uint64) == on.view(np.uint64)).all()


def test_as241_tails_bit_identical_1m():
    """About 10^6 AS241 tail draws (|p - 0.5| > 0.425, where the reference calls
    std::log, src/rng.cpp:93-96): the device normal equals the host oracle's
    (glibc log) bit for bit."""
    import ctypes

    from oracle.oracle import oracle
    from paper_1412_4933_b200 import _lib

    rng = np.random.default_rng(1)
    n = 7_000_000
    seed = rng.integers(0, 2**63, n, dtype=np.uint64)
    step = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    phase = np.full(n, 1, np.uint32)
    ent = rng.integers(0, 2**63, n, dtype=np.uint64)
    ctr = np.zeros(n, np.uint32)
    bits, uni, nrm = _lib.selftest_rng(seed, step, phase, ent, ctr, mu=1.0, sigma=0.5)
    on = np.zeros(n)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    oracle().pfo_normal_batch(n, vp(seed), vp(step), vp(phase), vp(ent), vp(ctr), 1.0, 0.5, vp(on))
    u = ((bits >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0**-53
    tail = np.abs(u - 0.5) > 0.425
    assert tail.sum() > 1_000_000
    bad = np.nonzero(nrm.view(np.uint64) != on.view(np.uint64))[0]
    assert len(bad) == 0, f"{len(bad)} differ, first key {bad[0]}: {nrm[bad[0]]!r} vs {on[bad[0]]!r}"


def test_store_load_roundtrip():
    import paper_1412_4933_b200 as p

    cfg = to_config(dict(width=96, height=96, agents_per_side=900, model="aco", seed=3))
    s = p.new_environment(cfg, 3)
    eng = p.StepEngine(p.EngineOptions.from_config(cfg, 3))
    eng.run(s, 25)
    snap = s.copy()
    eng2 = p.StepEngine(p.EngineOptions.from_config(cfg, 3, kernel="pipeline"))
    eng.run(s, 10)
    eng2.run(snap, 10)
    assert hashes_of(s) == hashes_of(snap)
    assert s.step == snap.step == 35


def test_pinned_host_planes_match_pageable():
    """SimState planes in page-locked memory (pf_host_alloc: direct DMA, no
    staging) give the same trajectory as pageable planes, on a grid large
    enough (> 4 MB planes) to take the staged path when pageable."""
    import paper_1412_4933_b200 as p

    cfg = to_config(dict(width=1024, height=1024, agents_per_side=60000, model="aco", seed=9))
    a = p.new_environment(cfg, 9)
    b = p.new_environment(cfg, 9, pinned=True)
    assert hashes_of(a) == hashes_of(b)
    for s in (a, b):
        eng = p.StepEngine(p.EngineOptions.from_config(cfg, 9))
        eng.run(s, 30)
    assert hashes_of(a) == hashes_of(b)
    assert a.step == b.step == 30


def test_corrupt_state_rejected():
    import paper_1412_4933_b200 as p

    cfg = to_config(dict(width=32, height=32, agents_per_side=64, model="lem", seed=7))
    s = p.new_environment(cfg, 7)
    s.index[0, 0], s.index[0, 1] = s.index[0, 1], s.index[0, 0]
    if s.index[0, 0] == s.index[0, 1]:
        s.occupancy[5, 5] = 1
    s.touch()
    eng = p.StepEngine(p.EngineOptions.from_config(cfg, 7))
    with pytest.raises(p.StateCorrupt):
        eng.step(s)


def _oracle_select(lib, kind, mask, num, seed, step, ent, d0=2.0, mu=1.0, sigma=0.5):
    """The oracle's lem_select / aco_select (goal-relative slot, -1 stay) or
    the movement-phase winner draw (src/engine.cpp:116-120) for one key."""
    import ctypes as C

    if kind == 2:
        k = bin(int(mask)).count("1")
        if k == 0:
            return -1
        u = lib.pfo_uniform(int(seed), int(step), 3, int(ent), 0)
        j = min(int(u * k), k - 1)
        return [b for b in range(8) if mask >> b & 1][j]
    op = (C.c_uint8 * 8)(*[(int(mask) >> b) & 1 for b in range(8)])
    if kind == 0:
        d = (C.c_double * 8)()
        lib.pfo_distance_table(d0, d)
        sc = (C.c_double * 8)()
        lib.pfo_lem_scores(op, d, sc)
        return lib.pfo_lem_select(sc, op, int(seed), int(step), int(ent), mu, sigma)
    return lib.pfo_aco_select((C.c_double * 8)(*num), op, int(seed), int(step), int(ent))


@pytest.mark.parametrize("kind", [0, 1, 2], ids=["lem_select", "aco_select", "resolve"])
def test_device_selection_matches_oracle(kind):
    """The selection functions the step kernels use, per key, against the
    oracle: all open masks (F open / blocked / boxed in), random keys, random
    ACO numerators including zeros (the degenerate uniform branch)."""
    from oracle.oracle import oracle
    from paper_1412_4933_b200 import _lib

    rng = np.random.default_rng(kind + 10)
    n = 6000
    mask = rng.integers(0, 256, n).astype(np.uint8)
    seed = rng.integers(0, 2**63, n, dtype=np.uint64)
    step = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    ent = rng.integers(1, 2**29, n, dtype=np.uint64) if kind < 2 else rng.integers(0, 2**32, n, dtype=np.uint64)
    num = None
    if kind == 1:
        num = rng.random((n, 8)) * (rng.random((n, 8)) < 0.8)
        num[rng.random(n) < 0.05] = 0.0
    got = _lib.selftest_select(kind, mask, seed, step, ent, num=num)
    lib = oracle()
    exp = np.array([_oracle_select(lib, kind, mask[i], None if num is None else list(num[i]), seed[i], step[i], ent[i])
                    for i in range(n)])
    assert (got == exp).all(), f"{int((got != exp).sum())} of {n} selections differ"


def test_aco_selection_frequencies_chi_square():
    """SPEC acceptance #2 on the device: Eq. 2 frequencies (ACO, F blocked,
    uniform tau = 0.1, beta = 2: P = num_i / sum, e.g. P(FL) = 0.29221) over
    200,000 keyed draws, chi-square against the expected probabilities."""
    from scipy.stats import chisquare

    from paper_1412_4933_b200 import _lib

    d = np.array([1, 2**0.5, 2**0.5, 5**0.5, 5**0.5, 3, 10**0.5, 10**0.5])
    num = 0.1 * (1.0 / d) ** 2
    num[0] = 0.0
    p = num / num.sum()
    assert abs(p[1] - 0.29221) < 1e-5
    n = 200_000
    rng = np.random.default_rng(5)
    got = _lib.selftest_select(1, np.full(n, 0xFE, np.uint8), 42, rng.integers(0, 2**32, n, dtype=np.uint64),
                               np.arange(1, n + 1, dtype=np.uint64), num=num)
    counts = np.bincount(got, minlength=8)
    assert counts[0] == 0
    stat = chisquare(counts[1:], p[1:] * n)
    assert stat.pvalue > 1e-3, stat


def test_winner_draw_uniform_among_five_contenders():
    """SPEC acceptance #3 on the device: a destination with 5 contenders picks
    each with probability 1/5 (keyed by the global cell index)."""
    from scipy.stats import chisquare

    from paper_1412_4933_b200 import _lib

    mask = 0b10110101  # contenders at row-major codes 0, 2, 4, 5, 7
    n = 200_000
    got = _lib.selftest_select(2, np.full(n, mask, np.uint8), 7, 123, np.arange(n, dtype=np.uint64))
    assert set(np.unique(got)) == {0, 2, 4, 5, 7}
    counts = np.bincount(got, minlength=8)[[0, 2, 4, 5, 7]]
    assert chisquare(counts).pvalue > 1e-3


_TOP_OFFSETS = [(1, 0), (1, -1), (1, 1), (0, -1), (0, 1), (-1, 0), (-1, -1), (-1, 1)]  # inc/grid.hpp:19-43


def _neighbourhood(s, a):
    """Goal-relative slots of agent record a: (row, col) and open flag (in
    bounds and empty at the step-start snapshot, inc/grid.hpp:109-125)."""
    sign = 1 if a["group"] == 1 else -1
    out = []
    for dr, dc in _TOP_OFFSETS:
        r, c = int(a["row"]) + sign * dr, int(a["col"]) + sign * dc
        ok = 0 <= r < s.height and 0 <= c < s.width and s.occupancy[r, c] == 0
        out.append((r, c, 1 if ok else 0))
    return out


@pytest.mark.parametrize("model", ["lem", "aco"])
def test_phase_level_api_matches_reference_phases(model):
    """score_phase / intention_phase / movement_phase / reset_phase
    (src/engine.cpp:64-193) one at a time on a PF_KERNEL_PIPELINE engine:
    the scores after score_phase and the futures after intention_phase equal
    the oracle's lem_scores / aco_numerators and lem_select / aco_select per
    agent; movement_phase moves agents as a fused step does and leaves denied
    agents' futures at their targets; reset_phase completes a step identical
    to StepEngine::step; repeated phase steps equal pf_step."""
    import ctypes as C

    import paper_1412_4933_b200 as p
    from oracle.oracle import oracle

    kw = dict(width=96, height=96, agents_per_side=1500, model=model, seed=3)
    cfg = to_config(kw)
    state = p.new_environment(cfg, 3)
    eng = p.StepEngine(p.EngineOptions.from_config(cfg, 3, kernel="pipeline"))
    eng.run(state, 40)
    s0 = state.copy()
    ref = s0.copy()
    fused = p.StepEngine(p.EngineOptions.from_config(cfg, 3))
    ref_report = fused.step(ref)
    lib = oracle()
    o = p.EngineOptions.from_config(cfg, 3)
    d = (C.c_double * 8)()
    lib.pfo_distance_table(o.d0, d)
    eta = (C.c_double * 8)(*[(1.0 / x) ** o.beta for x in d])

    eng.score_phase(state)
    exp_scores = np.zeros((len(s0.agents), 8))
    exp_future = np.zeros((len(s0.agents), 2), np.int64)
    for i, a in enumerate(s0.agents):
        nb = _neighbourhood(s0, a)
        op = (C.c_uint8 * 8)(*[x[2] for x in nb])
        sc = (C.c_double * 8)()
        if model == "lem":
            lib.pfo_lem_scores(op, d, sc)
            slot = lib.pfo_lem_select(sc, op, 3, s0.step, int(a["index"]), o.sel_mu, o.sel_sigma)
        else:
            tau = s0.pheromone_top if a["group"] == 1 else s0.pheromone_bottom
            t8 = (C.c_double * 8)(*[tau[r, c] if ok else 0.0 for r, c, ok in nb])
            lib.pfo_aco_numerators(op, t8, o.alpha, eta, sc)
            slot = lib.pfo_aco_select(sc, op, 3, s0.step, int(a["index"]))
        exp_scores[i] = list(sc)
        exp_future[i] = (nb[slot][0], nb[slot][1]) if slot >= 0 else (a["row"], a["col"])
    assert (state.scores == exp_scores).all()
    assert (state.score_owners == s0.agents["index"]).all()
    assert (state.agents["future_row"] == s0.agents["row"]).all()  # no intentions yet

    eng.intention_phase(state)
    assert (state.agents["future_row"] == exp_future[:, 0]).all()
    assert (state.agents["future_col"] == exp_future[:, 1]).all()
    assert (state.agents["row"] == s0.agents["row"]).all()  # nobody moved yet
    assert state.step == s0.step

    report = eng.movement_phase(state)
    assert (report.moved, report.newly_crossed_top, report.newly_crossed_bottom) == (
        ref_report.moved, ref_report.newly_crossed_top, ref_report.newly_crossed_bottom)
    assert (state.index == ref.index).all() and (state.occupancy == ref.occupancy).all()
    ag = state.agents
    assert (ag["row"] == ref.agents["row"]).all() and (ag["col"] == ref.agents["col"]).all()
    moved = (ag["row"] != s0.agents["row"]) | (ag["col"] != s0.agents["col"])
    assert moved.sum() == report.moved
    # movers' futures are their new cells; denied agents keep their targets
    assert (ag["future_row"] == exp_future[:, 0]).all() and (ag["future_col"] == exp_future[:, 1]).all()
    assert state.step == s0.step

    eng.reset_phase(state)
    assert state.step == s0.step + 1
    assert hashes_of(state) == hashes_of(ref)
    assert (state.agents["future_row"] == state.agents["row"]).all()
    assert not state.scores.any()

    # phase-level steps == full steps
    for _ in range(5):
        eng.score_phase(state)
        eng.intention_phase(state)
        eng.movement_phase(state)
        eng.reset_phase(state)
    fused.run(ref, 5)
    assert hashes_of(state) == hashes_of(ref)

    with pytest.raises(ValueError):  # out of order (PF_ERR_ARG)
        eng.movement_phase(state)
    with pytest.raises(p.ConfigError):  # the fused kernel has no separate phases
        fused.score_phase(ref)
