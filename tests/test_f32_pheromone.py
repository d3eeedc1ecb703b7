"""PF_KERNEL_FUSED_F32: the fused kernel with the ACO pheromone stored as fp32.

The north star asks for "a float pheromone field" whose values "agree within a
stated float tolerance"; the reference's fields are fp64
(/root/reference/proj/include/pedflow/aco.hpp:21-37), so the product default
stays fp64 and bit-exact, and fp32 storage is an option.
Arithmetic stays fp64 in the reference's order; each store rounds once. So per
step the relative error grows by at most 2^-24 (evaporation is a contraction,
deposits are positive): after t steps |tau32 - tau64| <= t * 2^-24 * |tau64|
while the values are normal floats. Decisions use the fields only through
u * total against cumulative sums, so a trajectory differs only when a draw
lands within ~1e-7 relative of a boundary; for the seeded cases below the
trajectories are identical to the oracle's, and the fields agree within the
bound. (Past ~900 steps of pure evaporation a never-visited cell drops below
the fp32 subnormal range and reads 0 where fp64 still holds ~1e-40: from then
on fp32 runs may take the reference's "total <= 0" branch elsewhere, so fp32
mode is a short-horizon / throughput option, not a parity mode.)
"""
from __future__ import annotations

import numpy as np
import pytest

from tests.helpers import to_config, to_scenario

pytestmark = pytest.mark.gpu

CASES = [
    (dict(width=96, height=96, agents_per_side=900, model="aco", seed=11), 200),
    (dict(width=480, height=480, agents_per_side=1024, model="aco", seed=42), 300),
    (dict(width=96, height=96, agents_per_side=2000, model="aco", seed=5, alpha=0.0, beta=1.0, rho=0.3, tau0=0.5,
          q=2.0), 100),
    # wide enough for the 320-column strips fp32 storage takes on large grids (C5's geometry)
    (dict(width=2560, height=512, agents_per_side=20_000, model="aco", seed=13), 80),
]


def _rel_bound(steps):
    return steps * 2.0**-24 * 1.01


@pytest.mark.parametrize("kw,steps", CASES)
def test_f32_pheromone_within_tolerance_and_same_trajectory(kw, steps):
    import paper_1412_4933_b200 as p
    from oracle.oracle import OracleState

    cfg = to_config(kw)
    seed = kw["seed"]
    state = p.new_environment(cfg, seed)
    eng = p.StepEngine(p.EngineOptions.from_config(cfg, seed, kernel="fused_f32"))
    rep = eng.run_array(state, steps)
    ora = OracleState(to_scenario(kw))
    orep = ora.run(steps)
    assert (rep == orep).all(), "per-step reports differ from the oracle"
    assert (state.index == ora.index).all() and (state.occupancy == ora.occ).all()
    for f in ("row", "col", "tour_length", "crossed"):
        assert (state.agents[f] == ora.agents[f]).all(), f
    for g, o in ((state.pheromone_top, ora.tau_top), (state.pheromone_bottom, ora.tau_bot)):
        rel = np.abs(g - o) / np.abs(o)
        assert rel.max() <= _rel_bound(steps), rel.max()
        assert (g != o).any()  # fp32 storage really is in use
    eng.close()


def test_f32_storage_halves_the_pheromone_planes_on_load_and_store():
    """A state loaded into an fp32 context and stored back equals the input
    rounded to fp32 (exactly), for every cell."""
    import paper_1412_4933_b200 as p
    from paper_1412_4933_b200 import _lib
    from paper_1412_4933_b200.engine import _pf_config

    kw = dict(width=64, height=48, agents_per_side=300, model="aco", seed=3)
    cfg = to_config(kw)
    s = p.new_environment(cfg, 3)
    rng = np.random.default_rng(0)
    s.pheromone_top[:] = rng.random(s.pheromone_top.shape) * 10.0 ** rng.integers(-30, 3, s.pheromone_top.shape)
    s.pheromone_bottom[:] = rng.random(s.pheromone_bottom.shape)
    c = _lib.Context(_pf_config(cfg, 3, kernel="fused_f32"))
    c.load(0, s.occupancy, s.index, s.agents, s.pheromone_top, s.pheromone_bottom, 7)
    occ, idx = np.zeros_like(s.occupancy), np.zeros_like(s.index)
    ag = np.zeros_like(s.agents)
    tt, tb = np.zeros_like(s.pheromone_top), np.zeros_like(s.pheromone_bottom)
    assert c.store(0, occ, idx, ag, tt, tb) == 7
    assert (tt == s.pheromone_top.astype(np.float32).astype(np.float64)).all()
    assert (tb == s.pheromone_bottom.astype(np.float32).astype(np.float64)).all()
    assert (idx == s.index).all() and (ag == s.agents).all()
    c.close()


def test_f32_linked_shards_equal_unsharded_f32():
    """fp32 storage through the fused halo exchange: 3 linked row shards
    (mirror stores of float2 pheromone rows) equal the unsharded fp32 run
    bit for bit (both round the same fp64 results)."""
    import paper_1412_4933_b200 as p
    from paper_1412_4933_b200 import _lib
    from paper_1412_4933_b200.engine import _pf_config
    from paper_1412_4933_b200.sharding import row_partition

    kw = dict(width=96, height=112, agents_per_side=1500, model="aco", seed=4)
    cfg = to_config(kw)
    steps = 150
    whole = p.Ensemble(cfg, replicas=1, seed=4, kernel="fused_f32")
    whole_rep = whole.run(steps)
    ref = whole.state(0)
    shards = []
    for lo, hi in row_partition(cfg.height, 3):
        c = _lib.Context(_pf_config(cfg, 4, row_begin=lo, row_end=hi, kernel="fused_f32"))
        c.init_environment()
        shards.append(c)
    _lib.link_shards(shards)
    for c in shards:
        c.step_async(steps)
    for c in shards:
        c.synchronize()
    tot = sum(c.read_reports(steps)["moved"].astype(np.int64) for c in shards)
    assert (tot == whole_rep["moved"]).all()
    H, W = cfg.height, cfg.width
    occ, idx = np.zeros((H, W), np.uint8), np.zeros((H, W), np.uint32)
    ag = np.zeros(2 * cfg.agents_per_side, _lib.AGENT_DTYPE)
    tt, tb = np.zeros((H, W)), np.zeros((H, W))
    for c in shards:
        assert c.store(0, occ, idx, ag, tt, tb) == steps
    assert (idx == ref.index).all() and (occ == ref.occupancy).all()
    assert (tt == ref.pheromone_top).all() and (tb == ref.pheromone_bottom).all()
    for c in shards:
        c.close()
    whole.close()
