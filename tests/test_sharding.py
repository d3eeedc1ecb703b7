"""Row sharding (the N>1 path).

CPU (gloo, world_size 2 and 3): the product's HaloExchanger drives shards of
the C oracle (pfo_step_cells: one reference step over a row window of the
cell-resident layout); gathering the owned rows must reproduce the
single-domain oracle bit-for-bit. This pins the decomposition, the ghost depth
of 3, the plane set and the global RNG keys.

GPU: several shard contexts on one device, exchanging through the same halo
ranges via pf_exchange_pair, must equal the unsharded GPU run and the oracle.
"""
from __future__ import annotations

import ctypes as C
import os
import socket

import numpy as np
import pytest

from oracle.oracle import OracleState, Scenario, _oracle_lib

GHOST = 3


def _cells_from_oracle(o: OracleState):
    """Cell-resident planes (the product's device layout) from an oracle SimState."""
    H, W = o.index.shape
    cell = np.zeros((H, W), np.uint32)
    tour = np.zeros((H, W), np.float64)
    occ = o.index != 0
    ids = o.index[occ]
    a = o.agents[ids - 1]
    cell[occ] = ids | (a["crossed"].astype(np.uint32) << 29) | (a["group"].astype(np.uint32) << 30)
    tour[occ] = a["tour_length"]
    return cell, tour


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, kw, steps, out_q):
    import torch
    import torch.distributed as dist

    from paper_1412_4933_b200.sharding import HaloExchanger, row_partition

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = Scenario(**kw)
        H, W = sc.height, sc.width
        o = OracleState(sc)
        gcell, gtour = _cells_from_oracle(o)
        aco = sc.model == "aco"
        lo, hi = row_partition(H, world)[rank]
        row0 = lo - GHOST
        nrows = hi - lo + 2 * GHOST
        cell = np.zeros((nrows, W), np.uint32)
        tour = np.zeros((nrows, W), np.float64)
        tt = np.zeros((nrows, W), np.float64)
        tb = np.zeros((nrows, W), np.float64)
        for b in range(nrows):
            g = row0 + b
            if 0 <= g < H:
                cell[b], tour[b] = gcell[g], gtour[g]
                if aco:
                    tt[b], tb[b] = o.tau_top[g], o.tau_bot[g]
        own = hi - lo

        def planes(side, recv):
            if side == 0:
                rows = slice(0, GHOST) if recv else slice(GHOST, 2 * GHOST)
                trow = GHOST - 1 if recv else GHOST
            else:
                rows = slice(GHOST + own, 2 * GHOST + own) if recv else slice(own, own + GHOST)
                trow = GHOST + own if recv else GHOST + own - 1
            out = [torch.from_numpy(cell[rows])]
            if aco:
                out += [torch.from_numpy(tt[rows]), torch.from_numpy(tb[rows]), torch.from_numpy(tour[trow])]
            return out

        ex = HaloExchanger(rank, world)
        lib = _oracle_lib()
        cfg = sc.cstruct()
        rep = np.zeros(4, np.uint32)
        reps = []
        for t in range(steps):
            rc = lib.pfo_step_cells(C.byref(cfg), sc.seed, t, row0, nrows, cell.ctypes.data, tour.ctypes.data,
                                    tt.ctypes.data if aco else None, tb.ctypes.data if aco else None,
                                    GHOST, GHOST + own, rep.ctypes.data)
            assert rc == 0
            reps.append(rep.copy())
            ex.exchange(planes)
        out_q.put((rank, lo, hi, cell[GHOST:GHOST + own].copy(), tour[GHOST:GHOST + own].copy(),
                   tt[GHOST:GHOST + own].copy() if aco else None, tb[GHOST:GHOST + own].copy() if aco else None,
                   np.array(reps)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kw", [
    dict(width=48, height=48, agents_per_side=400, model="aco", seed=5),
    dict(width=32, height=48, agents_per_side=300, model="lem", seed=9),
])
def test_gloo_sharded_oracle_matches_single_domain(kw, world):
    import torch.multiprocessing as mp

    steps = 40
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, kw, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort(key=lambda r: r[0])

    sc = Scenario(**kw)
    o = OracleState(sc)
    ref_rep = o.run(steps)
    cell, tour = _cells_from_oracle(o)
    for rank, lo, hi, c, t, tt, tb, reps in results:
        assert (c == cell[lo:hi]).all(), f"rank {rank} cell words differ"
        occ = c != 0
        assert (t[occ] == tour[lo:hi][occ]).all(), f"rank {rank} tour lengths differ"
        if tt is not None:
            assert (tt == o.tau_top[lo:hi]).all() and (tb == o.tau_bot[lo:hi]).all()
    tot = sum(r[7] for r in results)
    assert (tot[:, 1] == ref_rep["moved"]).all()
    assert (tot[:, 2] == ref_rep["newly_crossed_top"]).all()
    assert (tot[:, 3] == ref_rep["newly_crossed_bottom"]).all()


def test_row_partition():
    from paper_1412_4933_b200 import ConfigError
    from paper_1412_4933_b200.sharding import row_partition

    assert row_partition(16384, 8) == [(2048 * i, 2048 * (i + 1)) for i in range(8)]
    parts = row_partition(100, 3)
    assert parts[0][0] == 0 and parts[-1][1] == 100
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    with pytest.raises(ConfigError):
        row_partition(16, 8)


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["lem", "aco"])
@pytest.mark.parametrize("nshards", [2, 4])
def test_gpu_multishard_one_device(model, nshards):
    """k shard contexts on one GPU exchanging via pf_exchange_pair == unsharded run."""
    import paper_1412_4933_b200 as p
    from paper_1412_4933_b200 import _lib
    from paper_1412_4933_b200.engine import _pf_config
    from paper_1412_4933_b200.sharding import row_partition

    cfg = p.ScenarioConfig(width=96, height=96, agents_per_side=1500, model=p.Model.Lem if model == "lem" else p.Model.Aco,
                           seed=21)
    steps = 60
    whole = p.Ensemble(cfg, replicas=2, seed=21)
    whole_rep = whole.run(steps)
    shards = []
    for lo, hi in row_partition(cfg.height, nshards):
        c = _lib.Context(_pf_config(cfg, 21, replicas=2, row_begin=lo, row_end=hi))
        c.init_environment()
        shards.append(c)
    for _ in range(steps):
        for c in shards:
            c.step_async(1)
        for up, dn in zip(shards, shards[1:]):
            _lib.exchange_pair(up, dn)
    tot = sum(c.read_reports(steps)["moved"].astype(np.int64) for c in shards)
    assert (tot == whole_rep["moved"]).all()
    for r in range(2):
        ref = whole.state(r)
        H, W = cfg.height, cfg.width
        occ = np.zeros((H, W), np.uint8)
        idx = np.zeros((H, W), np.uint32)
        ag = np.zeros(2 * cfg.agents_per_side, _lib.AGENT_DTYPE)
        tt = np.zeros((H, W)) if model == "aco" else None
        tb = np.zeros((H, W)) if model == "aco" else None
        for c in shards:
            assert c.store(r, occ, idx, ag, tt, tb) == steps
        assert (idx == ref.index).all() and (occ == ref.occupancy).all()
        assert (ag["tour_length"] == ref.agents["tour_length"]).all()
        assert (ag["crossed"] == ref.agents["crossed"]).all()
        if tt is not None:
            assert (tt == ref.pheromone_top).all() and (tb == ref.pheromone_bottom).all()


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["lem", "aco"])
@pytest.mark.parametrize("nshards", [2, 3])
def test_gpu_fused_halo_one_device(model, nshards):
    """Fused halo exchange (the step kernel stores its boundary rows into the
    neighbours' ghost rows; device flag handshake per step): k linked shard
    contexts on one GPU, stepped by graph-batched pf_step_async only (no host
    exchange), equal the unsharded run in every plane. 300 steps = two graph
    batches; shards of unequal height (112 rows over 3)."""
    import paper_1412_4933_b200 as p
    from paper_1412_4933_b200 import _lib
    from paper_1412_4933_b200.engine import _pf_config
    from paper_1412_4933_b200.sharding import row_partition

    cfg = p.ScenarioConfig(width=96, height=112 if nshards == 3 else 96, agents_per_side=1500,
                           model=p.Model.Lem if model == "lem" else p.Model.Aco, seed=21)
    steps = 300
    whole = p.Ensemble(cfg, replicas=2, seed=21)
    whole_rep = whole.run(steps)
    shards = []
    for lo, hi in row_partition(cfg.height, nshards):
        c = _lib.Context(_pf_config(cfg, 21, replicas=2, row_begin=lo, row_end=hi))
        c.init_environment()
        shards.append(c)
    _lib.link_shards(shards)
    for c in shards:
        c.step_async(steps)
    for c in shards:
        c.synchronize()
    tot = sum(c.read_reports(steps)["moved"].astype(np.int64) for c in shards)
    assert (tot == whole_rep["moved"]).all()
    for r in range(2):
        ref = whole.state(r)
        H, W = cfg.height, cfg.width
        occ = np.zeros((H, W), np.uint8)
        idx = np.zeros((H, W), np.uint32)
        ag = np.zeros(2 * cfg.agents_per_side, _lib.AGENT_DTYPE)
        tt = np.zeros((H, W)) if model == "aco" else None
        tb = np.zeros((H, W)) if model == "aco" else None
        for c in shards:
            assert c.store(r, occ, idx, ag, tt, tb) == steps
        assert (idx == ref.index).all() and (occ == ref.occupancy).all()
        assert (ag["tour_length"] == ref.agents["tour_length"]).all()
        assert (ag["crossed"] == ref.agents["crossed"]).all()
        if tt is not None:
            assert (tt == ref.pheromone_top).all() and (tb == ref.pheromone_bottom).all()
        for c in shards:
            c.audit(r)
    for c in shards:
        c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["lem", "aco"])
def test_gpu_fused_halo_minimum_shards(model):
    """Shards of the minimum height (3 rows: every row is a ghost row of both
    neighbours, every work item touches both sides): 16 rows over 5 linked
    shards (3/3/3/3/4), 200 steps, equal to the unsharded run."""
    import paper_1412_4933_b200 as p
    from paper_1412_4933_b200 import _lib
    from paper_1412_4933_b200.engine import _pf_config
    from paper_1412_4933_b200.sharding import row_partition

    cfg = p.ScenarioConfig(width=96, height=16, agents_per_side=300, model=p.Model.Lem if model == "lem" else p.Model.Aco,
                           seed=4)
    steps = 200
    whole = p.Ensemble(cfg, replicas=3, seed=4)
    whole_rep = whole.run(steps)
    parts = row_partition(cfg.height, 5)
    assert [hi - lo for lo, hi in parts] == [3, 3, 3, 3, 4]
    shards = []
    for lo, hi in parts:
        c = _lib.Context(_pf_config(cfg, 4, replicas=3, row_begin=lo, row_end=hi))
        c.init_environment()
        shards.append(c)
    _lib.link_shards(shards)
    for c in shards:
        c.step_async(steps)
    for c in shards:
        c.synchronize()
    tot = sum(c.read_reports(steps)["moved"].astype(np.int64) for c in shards)
    assert (tot == whole_rep["moved"]).all()
    for r in range(3):
        ref = whole.state(r)
        H, W = cfg.height, cfg.width
        idx = np.zeros((H, W), np.uint32)
        occ = np.zeros((H, W), np.uint8)
        ag = np.zeros(2 * cfg.agents_per_side, _lib.AGENT_DTYPE)
        tt = np.zeros((H, W)) if model == "aco" else None
        tb = np.zeros((H, W)) if model == "aco" else None
        for c in shards:
            c.store(r, occ, idx, ag, tt, tb)
        assert (idx == ref.index).all() and (occ == ref.occupancy).all()
        if tt is not None:
            assert (tt == ref.pheromone_top).all() and (tb == ref.pheromone_bottom).all()
    for c in shards:
        c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["lem", "aco"])
def test_gpu_fused_halo_regular_geometry(model):
    """Linked shards large enough for the regular geometry (the C5-style
    path: 16-row tiles, boundary items claimed first, multi-tile items):
    96 x 160 over 2 shards x 64 replicas, equal to the unsharded batch."""
    import paper_1412_4933_b200 as p
    from paper_1412_4933_b200 import _lib
    from paper_1412_4933_b200.engine import _pf_config
    from paper_1412_4933_b200.sharding import row_partition

    cfg = p.ScenarioConfig(width=96, height=160, agents_per_side=3000, model=p.Model.Lem if model == "lem" else p.Model.Aco,
                           seed=8)
    steps, reps = 120, 64
    whole = p.Ensemble(cfg, replicas=reps, seed=8)
    whole_rep = whole.run(steps)
    shards = []
    for lo, hi in row_partition(cfg.height, 2):
        c = _lib.Context(_pf_config(cfg, 8, replicas=reps, row_begin=lo, row_end=hi))
        c.init_environment()
        shards.append(c)
    _lib.link_shards(shards)
    for c in shards:
        c.step_async(steps)
    for c in shards:
        c.synchronize()
    tot = sum(c.read_reports(steps)["moved"].astype(np.int64) for c in shards)
    assert (tot == whole_rep["moved"]).all()
    for r in (0, 37, 63):
        ref = whole.state(r)
        H, W = cfg.height, cfg.width
        idx = np.zeros((H, W), np.uint32)
        occ = np.zeros((H, W), np.uint8)
        ag = np.zeros(2 * cfg.agents_per_side, _lib.AGENT_DTYPE)
        tt = np.zeros((H, W)) if model == "aco" else None
        tb = np.zeros((H, W)) if model == "aco" else None
        for c in shards:
            c.store(r, occ, idx, ag, tt, tb)
        assert (idx == ref.index).all() and (occ == ref.occupancy).all()
        if tt is not None:
            assert (tt == ref.pheromone_top).all() and (tb == ref.pheromone_bottom).all()
    for c in shards:
        c.close()


@pytest.mark.gpu
def test_gpu_fused_halo_rejects_mismatched_peers():
    import paper_1412_4933_b200 as p
    from paper_1412_4933_b200 import _lib
    from paper_1412_4933_b200.engine import _pf_config

    cfg = p.ScenarioConfig(width=96, height=96, agents_per_side=500, model=p.Model.Aco)
    a = _lib.Context(_pf_config(cfg, 1, row_begin=0, row_end=48))
    b = _lib.Context(_pf_config(cfg, 1, row_begin=48, row_end=96))
    c = _lib.Context(_pf_config(cfg, 1, row_begin=0, row_end=40))
    t = _lib.Context(_pf_config(cfg, 1, row_begin=48, row_end=96, kernel="tile"))
    for x in (a, b, c):
        x.init_environment()
    with pytest.raises(_lib.CommError):
        b.attach_peer(0, c.peer_desc(), ipc=False)  # not adjacent
    with pytest.raises(_lib.CommError):
        a.attach_peer(0, b.peer_desc(), ipc=False)  # wrong side
    with pytest.raises(p.ConfigError):
        t.peer_desc()  # the tile kernel has no fused exchange
    a.step(1)
    with pytest.raises(_lib.CommError):
        b.attach_peer(0, a.peer_desc(), ipc=False)  # different step
    for x in (a, b, c, t):
        x.close()


def _gpu_rank_main(rank, world, port, kw, steps, out_q, exchange=None):
    import torch
    import torch.distributed as dist

    import paper_1412_4933_b200 as p
    from paper_1412_4933_b200 import _lib
    from paper_1412_4933_b200.sharding import ShardedEngine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        model = kw.pop("model")
        cfg = p.ScenarioConfig(model=p.Model.Lem if model == "lem" else p.Model.Aco, **kw)
        eng = ShardedEngine(cfg, rank, world, device=0, replicas=2, exchange=exchange)
        eng.step(steps)
        eng.synchronize()
        rep = eng.reports(steps)
        H, W = cfg.height, cfg.width
        res = []
        for r in range(2):
            occ = np.zeros((H, W), np.uint8)
            idx = np.zeros((H, W), np.uint32)
            ag = np.zeros(2 * cfg.agents_per_side, _lib.AGENT_DTYPE)
            tt = np.zeros((H, W)) if model == "aco" else None
            tb = np.zeros((H, W)) if model == "aco" else None
            eng.store(r, occ, idx, ag, tt, tb)
            res.append((occ, idx, ag, tt, tb))
        out_q.put((rank, eng.lo, eng.hi, rep, res))
        eng.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", ["collective", "p2p"])
@pytest.mark.parametrize("model", ["lem", "aco"])
def test_gpu_sharded_engine_two_ranks_one_device(model, exchange):
    """The N>1 product path with 2 ranks (processes) sharing cuda:0 over gloo,
    against the unsharded run. collective: ShardedEngine's per-step halo swap
    through the exchanger (host-staged for gloo), halo ranges from pf_halo.
    p2p: the fused halo exchange across processes — CUDA IPC handles of each
    rank's planes all-gathered over gloo, the step kernels storing into each
    other's ghost rows, the device flag handshake between processes."""
    import torch.multiprocessing as mp

    import paper_1412_4933_b200 as p

    kw = dict(width=96, height=96, agents_per_side=1500, model=model, seed=21)
    steps, world = 60, 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_rank_main, args=(r, world, port, dict(kw), steps, q, exchange))
             for r in range(world)]
    for pr in procs:
        pr.start()
    results = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    cfg = p.ScenarioConfig(width=96, height=96, agents_per_side=1500,
                           model=p.Model.Lem if model == "lem" else p.Model.Aco, seed=21)
    whole = p.Ensemble(cfg, replicas=2, seed=21)
    whole_rep = whole.run(steps)
    tot = sum(r[3]["moved"].astype(np.int64) for r in results)
    assert (tot == whole_rep["moved"]).all()
    for rep_i in range(2):
        ref = whole.state(rep_i)
        for rank, lo, hi, _, res in results:
            occ, idx, ag, tt, tb = res[rep_i]
            assert (idx[lo:hi] == ref.index[lo:hi]).all(), f"rank {rank} index differs"
            assert (occ[lo:hi] == ref.occupancy[lo:hi]).all()
            if tt is not None:
                assert (tt[lo:hi] == ref.pheromone_top[lo:hi]).all()
                assert (tb[lo:hi] == ref.pheromone_bottom[lo:hi]).all()


def test_balanced_row_partition():
    """ShardedEngine's cost-weighted rows: contiguous, covering, >= 3 rows
    each, equal rows without agents, fewer rows for the band shards."""
    import paper_1412_4933_b200 as p
    from paper_1412_4933_b200.sharding import balanced_row_partition, row_partition

    for model in (p.Model.Lem, p.Model.Aco):
        cfg = p.ScenarioConfig(width=16384, height=16384, agents_per_side=25_000_000, model=model)
        for P in (1, 2, 3, 4, 8):
            parts = balanced_row_partition(cfg, P)
            assert parts[0][0] == 0 and parts[-1][1] == 16384
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert all(hi - lo >= 3 for lo, hi in parts)
        eight = balanced_row_partition(cfg, 8)
        assert eight[0][1] - eight[0][0] < 2048 and eight[-1][1] - eight[-1][0] < 2048
    empty = p.ScenarioConfig(width=96, height=96, agents_per_side=0, model=p.Model.Aco)
    assert balanced_row_partition(empty, 3) == row_partition(96, 3)
    tiny = p.ScenarioConfig(width=16, height=16, agents_per_side=120, model=p.Model.Lem)
    assert all(hi - lo >= 3 for lo, hi in balanced_row_partition(tiny, 5))
