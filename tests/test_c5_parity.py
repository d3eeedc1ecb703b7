"""BASELINE config 5 (ACO/LEM, 16384 x 16384, 25M agents per side, seed 42)
checked bit-exact against the unmodified reference over a long horizon, whole
and row-sharded.

The anchors `C5_aco_long` / `C5_lem_long` in tests/golden/anchors.json come
from one run of oracle/_ref (the reference library compiled from
/root/reference/proj/src, tests/golden/make_golden.py --c5-long), hashed at
the checkpoints 10, 30, 100 and 300 (every plane: index, occupancy, agents,
pheromone) plus the full 300-step StepReport series. The bench window and the
builder's 300-step timing window lie inside them.

Row shards: the contiguous row blocks of SURVEY.md §8(e), linked by the fused
halo exchange (the step kernel stores its boundary rows into the neighbours'
ghost rows, pf_peer_attach), either as contexts of one process (ipc=0) or as
ranks in separate processes through CUDA IPC handles (ipc=1). All share the one
B200 here. Keys by agent id and global cell index
(/root/reference/proj/src/engine.cpp:82, 118-119) make every shard count
bit-identical to the reference.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from tests.helpers import hashes_of, hex_hashes, to_config

pytestmark = pytest.mark.gpu

C5 = ["C5_aco_long", "C5_lem_long"]


def _anchor(anchors, name):
    if name not in anchors:
        pytest.skip(f"{name} not generated (tests/golden/make_golden.py --c5-long)")
    return anchors[name]


def _checkpoints(a):
    return sorted(int(k) for k in a["checkpoints"])


def _series(rep):
    return np.stack([rep["moved"], rep["newly_crossed_top"], rep["newly_crossed_bottom"]], 1)


def _check_series(got, a):
    want = np.asarray(a["series"])[: len(got)]
    bad = np.nonzero((got != want).any(1))[0]
    assert len(bad) == 0, f"series first differs at step {bad[0]}: {got[bad[0]]} vs {want[bad[0]]}"


@pytest.mark.parametrize("name", C5)
def test_c5_long_horizon(anchors, name):
    """The product API (new_environment -> StepEngine.run_array) on the whole
    grid, hashed at every checkpoint."""
    import paper_1412_4933_b200 as p

    a = _anchor(anchors, name)
    cfg = to_config(a["scenario"])
    state = p.new_environment(cfg, 42)
    eng = p.StepEngine(p.EngineOptions.from_config(cfg, 42))
    done, reps = 0, []
    for cp in _checkpoints(a):
        reps.append(eng.run_array(state, cp - done))
        done = cp
        assert state.step == cp
        assert hex_hashes(hashes_of(state)) == a["checkpoints"][str(cp)], f"step {cp}"
    rep = np.concatenate(reps)
    assert list(rep["step"]) == list(range(done))
    _check_series(_series(rep), a)
    eng.close()


def _full_planes(cfg, aco):
    H, W = cfg.height, cfg.width
    from paper_1412_4933_b200 import _lib

    return dict(occ=np.zeros((H, W), np.uint8), idx=np.zeros((H, W), np.uint32),
                ag=np.zeros(2 * cfg.agents_per_side, _lib.AGENT_DTYPE),
                tt=np.zeros((H, W)) if aco else None, tb=np.zeros((H, W)) if aco else None)


@pytest.mark.parametrize("nshards", [2, 4])
@pytest.mark.parametrize("name", C5)
def test_c5_linked_shards_one_process(anchors, name, nshards):
    """nshards linked row-shard contexts (ipc=0) stepped only by graph-batched
    pf_step_async, stored into the global planes at every checkpoint."""
    from oracle.oracle import state_hashes
    from paper_1412_4933_b200 import _lib
    from paper_1412_4933_b200.engine import _pf_config
    from paper_1412_4933_b200.sharding import row_partition

    a = _anchor(anchors, name)
    cfg = to_config(a["scenario"])
    aco = a["scenario"]["model"] == "aco"
    shards = []
    for lo, hi in row_partition(cfg.height, nshards):
        c = _lib.Context(_pf_config(cfg, 42, row_begin=lo, row_end=hi))
        c.init_environment()
        shards.append(c)
    _lib.link_shards(shards)
    pl = _full_planes(cfg, aco)
    done, ser = 0, []
    for cp in _checkpoints(a):
        for c in shards:
            c.step_async(cp - done)
        for c in shards:
            c.synchronize()
        ser.append(sum(_series(c.read_reports(cp - done)[0]).astype(np.int64) for c in shards))
        done = cp
        for c in shards:
            assert c.store(0, pl["occ"], pl["idx"], pl["ag"], pl["tt"], pl["tb"]) == cp
        got = hex_hashes(state_hashes(pl["occ"], pl["idx"], pl["ag"], pl["tt"], pl["tb"]))
        assert got == a["checkpoints"][str(cp)], f"{nshards} shards, step {cp}"
    _check_series(np.concatenate(ser), a)
    for c in shards:
        c.audit(0)
    for c in shards:
        c.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ring_fnv(dist, rank, world, chunk: bytes, start: int) -> int:
    """FNV-1a 64 of the concatenation of every rank's chunk in rank order:
    the running hash travels rank 0 -> 1 -> ... and the last rank broadcasts
    the result."""
    import torch

    from oracle.oracle import fnv1a

    t = torch.zeros(1, dtype=torch.int64)
    if rank == 0:
        h = start
    else:
        dist.recv(t, src=rank - 1)
        h = int(t.item()) & (2**64 - 1)
    h = fnv1a(chunk, h)
    if rank + 1 < world:
        t[0] = np.uint64(h).astype(np.int64)
        dist.send(t, dst=rank + 1)
    t[0] = np.uint64(h).astype(np.int64)
    dist.broadcast(t, src=world - 1)
    return int(t.item()) & (2**64 - 1)


def _c5_rank_main(rank, world, port, kw, checkpoints, out_q):
    import torch
    import torch.distributed as dist

    from oracle.oracle import FNV_OFFSET
    from paper_1412_4933_b200.sharding import ShardedEngine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = to_config(kw)
        aco = kw["model"] == "aco"
        eng = ShardedEngine(cfg, rank, world, device=0, exchange="p2p")
        lo, hi = eng.lo, eng.hi
        pl = _full_planes(cfg, aco)
        done = 0
        for cp in checkpoints:
            eng.step(cp - done)
            eng.synchronize()
            rep = eng.reports(cp - done)[0]
            done = cp
            assert eng.store(0, pl["occ"], pl["idx"], pl["ag"], pl["tt"], pl["tb"]) == cp
            h = {"index": _ring_fnv(dist, rank, world, pl["idx"][lo:hi].tobytes(), FNV_OFFSET),
                 "occ": _ring_fnv(dist, rank, world, pl["occ"][lo:hi].tobytes(), FNV_OFFSET)}
            if aco:
                top = _ring_fnv(dist, rank, world, pl["tt"][lo:hi].tobytes(), FNV_OFFSET)
                h["pher"] = _ring_fnv(dist, rank, world, pl["tb"][lo:hi].tobytes(), top)
            ids = pl["idx"][lo:hi][pl["occ"][lo:hi] != 0].astype(np.int64) - 1  # agents living in my rows
            ag = pl["ag"][ids]
            out_q.put((rank, cp, h, ids, ag["row"].copy(), ag["col"].copy(), ag["tour_length"].copy(),
                       ag["crossed"].copy(), _series(rep)))
            dist.barrier()
        eng.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", C5)
def test_c5_sharded_engine_ipc(anchors, name):
    """Two ranks (processes) on cuda:0 running the product ShardedEngine with
    the fused exchange across processes (CUDA IPC, ipc=1), checked at the
    10- and 100-step checkpoints: plane hashes chained rank to rank in row
    order, the agent table assembled from both ranks."""
    import torch.multiprocessing as mp

    from oracle.oracle import fnv1a

    a = _anchor(anchors, name)
    cps = [c for c in _checkpoints(a) if c <= 100][::2] or _checkpoints(a)[:1]
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_c5_rank_main, args=(r, world, port, dict(a["scenario"]), cps, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    n = 2 * a["scenario"]["agents_per_side"]
    packed_t = np.dtype({"names": ["row", "col", "tour", "crossed"], "formats": ["<i4", "<i4", "<f8", "u1"],
                         "offsets": [0, 4, 8, 16], "itemsize": 17})
    ser = {}
    try:
        for _ in cps:
            res = sorted([q.get(timeout=900) for _ in range(world)], key=lambda r: r[0])
            cp = res[0][1]
            packed = np.zeros(n, packed_t)
            for rank, _, h, ids, row, col, tour, crossed, s in res:
                assert h == res[0][2]
                packed["row"][ids], packed["col"][ids] = row, col
                packed["tour"][ids], packed["crossed"][ids] = tour, crossed
                ser.setdefault(cp, []).append(s.astype(np.int64))
            assert sum(len(r[3]) for r in res) == n
            got = {k: f"{v:016x}" for k, v in res[0][2].items()}
            got["agents"] = f"{fnv1a(packed.tobytes()):016x}"
            assert got == a["checkpoints"][str(cp)], f"ipc ranks, step {cp}"
    finally:
        for pr in procs:
            pr.join(timeout=120)
    for pr in procs:
        assert pr.exitcode == 0
    _check_series(np.concatenate([sum(ser[c]) for c in sorted(ser)]), a)
