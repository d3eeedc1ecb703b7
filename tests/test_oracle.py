"""Pinning the C oracle (CPU): Random123 Philox known-answer vectors, the SPEC
per-operation examples, the golden anchors generated from the unmodified
reference, and (when oracle/_ref is built) direct differential runs."""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import pytest

from oracle.oracle import OracleState, Reference, Scenario, oracle, series_hash

SMALL = ["s32_lem_64_s7", "s32_aco_64_s7", "s32_lem_200_s3", "s32_aco_200_s3", "s96_lem_900_s11",
         "s96_aco_900_s11", "s96_aco_2000_s5_alt", "s96_lem_2000_s5_alt", "r48x32_aco_300_s9",
         "r16x64_lem_16_s1", "empty_aco_32", "full_band_lem_16", "S96_aco_96_256"]


def arr(vals, t=C.c_double):
    return (t * len(vals))(*vals)


# ---------------------------------------------------------------- det-rng

@pytest.mark.parametrize("seed,step,phase,entity,counter,expect", [
    # Random123 philox4x32-10 KATs mapped through the packing of src/rng.cpp:47-52
    (0, 0, 0, 0, 0, 0x6627E8D5E169C58D),
    (0xFFFFFFFFFFFFFFFF, 0xFFFFFFFF, 0xF, 0xFFFFFFFFFFFFFFFF, 0x0FFFFFFF, 0x408F276D41C83B0E),
    (0x299F31D0A4093822, 0x13198A2E, 0x0, 0x85A308D3243F6A88, 0x03707344, 0xD16CFE0994FDCCEB),
])
def test_philox_known_answers(seed, step, phase, entity, counter, expect):
    assert oracle().pfo_random_bits(seed, step, phase, entity, counter) == expect


def test_uniform_and_normal_properties():
    lib = oracle()
    u = np.array([lib.pfo_uniform(42, 1, 3, i, 0) for i in range(20000)])
    assert 0.0 <= u.min() and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 0.01
    z = np.array([lib.pfo_normal(7, 3, 1, i, 0, 0.0, 1.0) for i in range(20000)])
    assert abs(z.mean()) < 0.03 and abs(z.std() - 1.0) < 0.03
    assert lib.pfo_normal(1, 2, 1, 3, 0, 0.25, 0.0) == 0.25  # sigma = 0 -> exactly mu


def test_inverse_normal_cdf_values():
    lib = oracle()
    assert lib.pfo_inverse_normal_cdf(0.5) == 0.0
    for p, z in [(0.975, 1.959963984540054), (0.025, -1.959963984540054), (1e-10, -6.361340902404056)]:
        assert abs(lib.pfo_inverse_normal_cdf(p) - z) < 1e-12


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")
def test_rng_matches_reference_library():
    lib, ref = oracle(), Reference.lib()
    rng = np.random.default_rng(1)
    for _ in range(3000):
        k = (int(rng.integers(0, 2**63)), int(rng.integers(0, 2**32)), int(rng.integers(0, 5)),
             int(rng.integers(0, 2**63)), int(rng.integers(0, 2**32)))
        assert lib.pfo_random_bits(*k) == ref.ref_random_bits(*k)
        assert lib.pfo_normal(*k, 0.3, 1.7) == ref.ref_normal(*k, 0.3, 1.7)


# ---------------------------------------------------------- SPEC examples

def test_distance_table_examples():
    lib = oracle()
    out = (C.c_double * 8)()
    assert lib.pfo_distance_table(2.0, out) == 0
    assert list(out) == [1.0, math.sqrt(2), math.sqrt(2), math.sqrt(5), math.sqrt(5), 3.0, math.sqrt(10), math.sqrt(10)]
    lib.pfo_distance_table(3.0, out)
    assert out[0] == 2.0 and out[5] == 4.0 and out[6] == math.sqrt(17)
    assert lib.pfo_distance_table(1.0, out) == 2  # d0 <= 1 -> config error


def test_lem_scores_examples():
    lib = oracle()
    d = (C.c_double * 8)()
    lib.pfo_distance_table(2.0, d)
    out = (C.c_double * 8)()
    lib.pfo_lem_scores(arr([1] * 8, C.c_uint8), d, out)
    assert np.allclose(list(out), [1, .70711, .70711, .44721, .44721, .33333, .31623, .31623], atol=5e-6)
    lib.pfo_lem_scores(arr([0] * 8, C.c_uint8), d, out)
    assert list(out) == [0.0] * 8
    lib.pfo_lem_scores(arr([0] + [1] * 7, C.c_uint8), d, out)
    assert out[0] == 0.0 and abs(out[1] - 0.70711) < 5e-6


def test_lem_select_examples():
    lib = oracle()
    d = (C.c_double * 8)()
    lib.pfo_distance_table(2.0, d)
    sc = (C.c_double * 8)()
    allopen = arr([1] * 8, C.c_uint8)
    lib.pfo_lem_scores(allopen, d, sc)
    assert lib.pfo_lem_select_u(sc, allopen, 0.1, 0.9) == 0  # F empty -> F
    fblk = arr([0] + [1] * 7, C.c_uint8)
    lib.pfo_lem_scores(fblk, d, sc)
    # r clamps to C_max = 0.70711, tie-break u = 0.3 -> FL (SPEC lem_select example)
    assert lib.pfo_lem_select_u(sc, fblk, 5.0, 0.3) == 1
    assert lib.pfo_lem_select_u(sc, fblk, 5.0, 0.7) == 2
    none = arr([0] * 8, C.c_uint8)
    lib.pfo_lem_scores(none, d, sc)
    assert lib.pfo_lem_select_u(sc, none, 0.5, 0.5) == -1  # boxed in -> stay


def test_aco_numerators_and_select_examples():
    lib = oracle()
    d = (C.c_double * 8)()
    lib.pfo_distance_table(2.0, d)
    eta = arr([(1.0 / x) ** 2.0 for x in d])
    fblk = arr([0] + [1] * 7, C.c_uint8)
    num = (C.c_double * 8)()
    lib.pfo_aco_numerators(fblk, arr([0.1] * 8), 1.0, eta, num)
    assert np.allclose(list(num), [0, .05, .05, .02, .02, .011111, .01, .01], atol=1e-6)
    total = sum(num)
    assert abs(total - 0.171111) < 1e-6
    assert abs(num[1] / total - 0.29221) < 1e-5  # P(FL)
    assert lib.pfo_aco_select_u(num, fblk, 0.0) == 1
    assert lib.pfo_aco_select_u(num, fblk, 0.2922) == 1
    assert lib.pfo_aco_select_u(num, fblk, 0.2923) == 2
    assert lib.pfo_aco_select_u(num, fblk, 0.9999999) == 7
    zero = (C.c_double * 8)()
    assert lib.pfo_aco_select_u(zero, fblk, 0.5) == 4  # degenerate total -> uniform over open


def test_band_height_examples():
    lib = oracle()
    assert lib.pfo_band_height(1280, 480) == 3
    assert lib.pfo_band_height(6720, 480) == 14
    assert lib.pfo_band_height(0, 480) == 0


@pytest.mark.parametrize("H", [16, 32, 64])
def test_single_agent_closed_form(H):
    """SPEC acceptance #8: one Top agent, band 1 -> crosses at step H-2."""
    o = OracleState(Scenario(width=16, height=H, agents_per_side=1, model="lem"))
    rep = o.run(H)
    assert int(np.nonzero(rep["newly_crossed_top"])[0][0]) == H - 2


def test_pheromone_mass_accounting():
    """SPEC acceptance #4: mass(t+1) = (1-rho) mass(t) + sum q/L over movers."""
    sc = Scenario(width=48, height=48, agents_per_side=400, model="aco", seed=4)
    o = OracleState(sc)
    for _ in range(30):
        m0 = o.tau_top.sum() + o.tau_bot.sum()
        before = o.agents["tour_length"].copy()
        o.run(1)
        moved = o.agents["tour_length"] != before
        dep = (sc.q / o.agents["tour_length"][moved]).sum()
        m1 = o.tau_top.sum() + o.tau_bot.sum()
        assert abs(m1 - ((1 - sc.rho) * m0 + dep)) <= 1e-9 * m1


# ------------------------------------------------------------ golden anchors

@pytest.mark.parametrize("name", SMALL)
def test_oracle_matches_golden(anchors, name):
    a = anchors[name]
    o = OracleState(Scenario(**a["scenario"]))
    rep = o.run(a["steps"])
    assert {k: f"{v:016x}" for k, v in o.hashes().items()} == a["hash"]
    assert f"{series_hash(rep):016x}" == a["series_hash"]


@pytest.mark.parametrize("name", ["C1_lem_480_1024", "C2_aco_480_1024"])
def test_oracle_matches_golden_c1_c2_prefix(anchors, name):
    """First 300 steps of C1/C2 against the per-step series of the anchor."""
    a = anchors[name]
    o = OracleState(Scenario(**a["scenario"]))
    rep = o.run(300)
    ser = np.stack([rep["moved"], rep["newly_crossed_top"], rep["newly_crossed_bottom"]], 1)
    assert (ser == np.asarray(a["series"][:300])).all()
    assert int(rep["moved"][0]) == a["step0_moved"]


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("kw", [dict(width=64, height=64, agents_per_side=700, model="aco", seed=13),
                                dict(width=64, height=48, agents_per_side=500, model="lem", seed=17),
                                dict(width=32, height=32, agents_per_side=256, model="aco", seed=2, alpha=0.5)])
def test_oracle_matches_reference_library(kw):
    sc = Scenario(**kw)
    o = OracleState(sc)
    r = Reference(sc, threads=3)
    ro = o.run(150)
    rr, _ = r.run(150)
    assert (ro == rr).all()
    assert o.hashes() == r.hashes()


def test_oracle_aco_selection_chi_square():
    """SPEC acceptance #2 (CPU, the oracle's aco_select): Eq. 2 frequencies
    over 100,000 keyed draws match P_i = num_i / sum (chi-square)."""
    from scipy.stats import chisquare

    lib = oracle()
    d = (C.c_double * 8)()
    lib.pfo_distance_table(2.0, d)
    eta = arr([(1.0 / x) ** 2.0 for x in d])
    op = arr([0] + [1] * 7, C.c_uint8)
    num = (C.c_double * 8)()
    lib.pfo_aco_numerators(op, arr([0.1] * 8), 1.0, eta, num)
    n = 100_000
    got = np.array([lib.pfo_aco_select(num, op, 42, s % 977, s + 1) for s in range(n)])
    counts = np.bincount(got, minlength=8)
    p = np.array(list(num)) / sum(num)
    assert counts[0] == 0
    assert chisquare(counts[1:], p[1:] * n).pvalue > 1e-3


def test_oracle_winner_draw_uniform():
    """SPEC acceptance #3 (CPU): the keyed winner draw min(int(u*k), k-1)
    (src/engine.cpp:118-120) picks each of 5 contenders with probability 1/5."""
    from scipy.stats import chisquare

    lib = oracle()
    k = 5
    idx = [min(int(lib.pfo_uniform(7, 123, 3, cell, 0) * k), k - 1) for cell in range(100_000)]
    assert chisquare(np.bincount(idx, minlength=k)).pvalue > 1e-3


def test_log_restatement_matches_host_glibc():
    """The restatement of glibc's log that the device uses (oracle's
    pfo_log_restated, constants from tools/gen_log_table.py) equals this host's
    log bit for bit over 2M AS241 tail arguments, and at hand-picked points."""
    import math

    from oracle.oracle import oracle

    lib = oracle()
    assert lib.pfo_log_restated_matches_host(2_000_000, 7) == 1
    for x in (2.0**-54, 1e-300 * 1e290, 1e-5, 0.01, 0.0499, 0.075, 0.5, 0.9, 2.0, 1e300):
        assert lib.pfo_log_restated(x).hex() == math.log(x).hex(), x
