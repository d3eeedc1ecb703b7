"""Lazy host/device sync of the Python StepEngine mirror (engine.py).

The reference's StepEngine::step(SimState&) (inc/pedflow/engine.hpp:53,
src/engine.cpp:53-62) works on any caller-owned SimState, so an engine that
keeps a device copy must (1) pull the state it holds before loading another
one and (2) never trust a device copy after another engine advanced the same
state. The CPU tests drive engine.py against a stand-in Context that "steps"
by incrementing every index word; the GPU tests repeat the same call
sequences on the real library against oracle runs.
"""
from __future__ import annotations

import gc

import numpy as np
import pytest

from tests.helpers import hashes_of, to_config


class FakeContext:
    """Records planes like pf_load_state / pf_store_state; a step adds 1 to
    every index word and to the step counter."""

    loads = 0

    def __init__(self, cfg):
        self.cfg = cfg
        self.state = None
        self.cur = 0

    def load(self, replica, occ, index, agents, tau_top, tau_bot, step):
        FakeContext.loads += 1
        self.state = (occ.copy(), index.copy(), agents.copy())
        self.cur = step

    def store(self, replica, occ, index, agents, tau_top, tau_bot):
        o, i, a = self.state
        occ[...] = o
        index[...] = i
        agents[...] = a
        return self.cur

    def store_scores(self, replica, scores):
        scores[...] = 0

    def step(self, n, want_reports=True):
        o, i, a = self.state
        self.state = (o, i + np.uint32(n), a)
        from paper_1412_4933_b200._lib import REPORT_DTYPE

        out = np.zeros((1, n), REPORT_DTYPE)
        out[0]["step"] = np.arange(self.cur, self.cur + n)
        self.cur += n
        return out

    @property
    def current_step(self):
        return self.cur

    def close(self):
        self.state = None


@pytest.fixture
def fake(monkeypatch):
    from paper_1412_4933_b200 import _lib

    monkeypatch.setattr(_lib, "Context", FakeContext)
    FakeContext.loads = 0
    return FakeContext


def _state(seed=7):
    import paper_1412_4933_b200 as p

    cfg = to_config(dict(width=32, height=32, agents_per_side=8, model="lem", seed=seed))
    s = p.SimState(cfg.width, cfg.height, cfg.model, 16)
    s._index[...] = seed  # distinguishable planes without the native new_environment
    return cfg, s


def _engine(cfg, seed=7):
    import paper_1412_4933_b200 as p

    return p.StepEngine(p.EngineOptions(model=p.Model(cfg.model), seed=seed))


def test_two_states_on_one_engine(fake):
    """eng.run(a, 1); eng.run(b, 5) must leave a at step 1 with its own planes."""
    cfg, a = _state(1)
    _, b = _state(2)
    eng = _engine(cfg)
    eng.run(a, 1)
    eng.run(b, 5)
    assert a.step == 1 and (a.index == 2).all()
    assert b.step == 5 and (b.index == 7).all()
    eng.run(a, 2)  # a comes back: re-uploaded from its (now current) host planes
    assert a.step == 3 and (a.index == 4).all()
    assert b.step == 5 and (b.index == 7).all()


def test_one_state_on_two_engines(fake):
    """e1.run(s); e2.run(s); e1.run(s) must not drop e2's step."""
    cfg, s = _state(3)
    e1, e2 = _engine(cfg), _engine(cfg)
    e1.run(s, 1)
    e2.run(s, 1)
    e1.run(s, 1)
    assert s.step == 3 and (s.index == 6).all()


def test_no_reupload_when_unchanged(fake):
    """The fast path stays: repeated steps on one state load once; reading a
    plane in between does not force a reload; touch() does."""
    cfg, s = _state(4)
    eng = _engine(cfg)
    for _ in range(5):
        eng.step(s)
    assert fake.loads == 1
    assert (s.index == 9).all()
    eng.step(s)
    assert fake.loads == 1 and (s.index == 10).all()
    s.touch()
    eng.step(s)
    assert fake.loads == 2 and (s.index == 11).all()


def test_tokens_not_reused_after_gc(fake):
    """A fresh state that happens to reuse a collected state's id() must still
    be uploaded."""
    cfg, a = _state(5)
    eng = _engine(cfg)
    eng.run(a, 1)
    _ = a.index  # pull: the engine's copy equals a's host planes
    del a
    gc.collect()
    for _ in range(20):
        _, b = _state(9)
        eng.run(b, 1)
        assert (b.index == 10).all()
        del b
        gc.collect()


def test_close_pulls_resident_state(fake):
    cfg, s = _state(6)
    eng = _engine(cfg)
    eng.run(s, 2)
    eng.close()
    assert s.step == 2 and (s.index == 8).all()


# --- the same sequences on the B200 -------------------------------------------


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["lem", "aco"])
def test_gpu_two_states_one_engine_and_two_engines(model):
    import paper_1412_4933_b200 as p
    from oracle.oracle import OracleState
    from tests.helpers import to_scenario

    kw_a = dict(width=64, height=64, agents_per_side=300, model=model, seed=11)
    kw_b = dict(kw_a, seed=12)
    cfg = to_config(kw_a)
    a = p.new_environment(cfg, 11)
    b = p.new_environment(cfg, 12)
    # one engine keyed with seed 11 steps both states (the engine's seed keys
    # the draws, as in the reference where options() carry the seed)
    eng = p.StepEngine(p.EngineOptions.from_config(cfg, 11))
    eng.run(a, 7)
    eng.run(b, 13)
    eng.run(a, 5)
    oa = OracleState(to_scenario(kw_a), seed=11)
    oa.run(12)
    ob = OracleState(to_scenario(kw_b), seed=12)  # placement of seed 12 ...
    ob.seed = 11  # ... stepped with the engine's seed 11
    ob.run(13)
    assert hashes_of(a) == oa.hashes() and a.step == 12
    assert hashes_of(b) == ob.hashes() and b.step == 13

    # one state, two engines, interleaved
    s = p.new_environment(cfg, 11)
    e1 = p.StepEngine(p.EngineOptions.from_config(cfg, 11))
    e2 = p.StepEngine(p.EngineOptions.from_config(cfg, 11))
    for i in range(6):
        (e1 if i % 2 == 0 else e2).run(s, 2)
    o = OracleState(to_scenario(kw_a), seed=11)
    o.run(12)
    assert s.step == 12 and hashes_of(s) == o.hashes()
    for e in (eng, e1, e2):
        e.close()
