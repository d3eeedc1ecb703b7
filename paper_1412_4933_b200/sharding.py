"""Row-sharded multi-GPU stepping: one process per GPU, torch.distributed (NCCL)
for the per-step ghost-row exchange.

The reference has no distributed backend; this is the new
GPU<->GPU boundary. The grid is split into contiguous row blocks (SURVEY.md
§8(e)); a step's dependency radius is 3 cells, so each shard keeps
PF_GHOST_ROWS = 3 ghost rows above and below and, after every step, swaps with
each vertical neighbour:

    3 rows of cell words (u32)       — occupancy, id, crossed flag, group
    3 rows of pheromone {top, bot}   — ACO only (f64 x 2)
    1 row of tour lengths (f64)      — ACO only; movers read the source's

Agents migrate implicitly: all agent state (id, group, crossed, tour) is
cell-resident and arrives with the ghost rows. RNG keys use the agent id and
the GLOBAL cell index, crossing uses the global row, so any shard count gives
results bit-identical to one GPU and to the CPU oracle.

Two exchange paths:

* "p2p" (default for the fused kernel): the fused halo exchange of the C-ABI
  (pf_peer_export / pf_peer_attach). Each rank exports CUDA IPC handles of its
  planes, the handles are all-gathered once over the process group, and from
  then on the step kernel itself stores the 3 boundary rows into the
  neighbours' ghost rows over NVLink, with a device-side flag handshake per
  step. No host work per step: n steps are one graph-batched pf_step_async.
* "nccl" / host-staged: HaloExchanger below, a torch.distributed
  batch_isend_irecv of the ghost-row ranges after each step's kernel. It is
  engine-agnostic (it moves torch tensors), so the CPU tests drive it with
  gloo and numpy-backed shards of the oracle, and the GPU path with NCCL and
  tensors aliasing the library's device planes (__cuda_array_interface__).
"""
from __future__ import annotations

import numpy as np

from . import _lib

GHOST = _lib.PF_GHOST_ROWS


def row_partition(height: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced row blocks [lo, hi) for `world` shards."""
    if world < 1:
        raise _lib.ConfigError("world size must be >= 1")
    parts = [(height * r // world, height * (r + 1) // world) for r in range(world)]
    if world > 1 and min(hi - lo for lo, hi in parts) < GHOST:
        raise _lib.ConfigError(f"each shard must own at least {GHOST} rows")
    return parts


# Relative cost of a row inside a starting band of agents against an empty
# row, per model, measured at C5 on one GPU (profiles/shard_projection_r02.md:
# 8 equal shards, band shard vs interior shard): ACO is bound by its pheromone
# stream, uniform over rows; LEM's work follows the agents.
BAND_ROW_COST = {0: 2.9, 1: 1.13}  # Model.Lem, Model.Aco


def balanced_row_partition(cfg, world: int) -> list[tuple[int, int]]:
    """Contiguous row blocks [lo, hi) of about equal step cost: rows in the
    two starting bands (band_height rows at each end, src/state.cpp:72-73,
    src/metrics.cpp:8-11) weigh BAND_ROW_COST[model], empty rows 1. The bands
    move ~1 row per step, so the balance holds for the first few hundred
    steps. Every shard owns >= GHOST rows; with no agents this is
    row_partition."""
    if world < 1:
        raise _lib.ConfigError("world size must be >= 1")
    H = int(cfg.height)
    if world == 1:
        return [(0, H)]
    band = min(H, int(_lib.lib.pf_band_height(int(cfg.agents_per_side), int(cfg.width)))) if cfg.agents_per_side else 0
    wb = BAND_ROW_COST.get(int(cfg.model), 1.0)

    def cum(r):  # total weight of rows [0, r)
        top = min(r, band)
        bot = max(0, r - (H - band)) if band else 0
        return r + (wb - 1.0) * (top + bot)

    total = cum(H)
    cuts = [0]
    for k in range(1, world):
        target = total * k / world
        lo, hi = cuts[-1] + GHOST, H - GHOST * (world - k)
        r = max(lo, min(hi, int(round(_inverse(cum, target, H)))))
        cuts.append(r)
    cuts.append(H)
    parts = list(zip(cuts[:-1], cuts[1:]))
    if min(hi - lo for lo, hi in parts) < GHOST:
        raise _lib.ConfigError(f"each shard must own at least {GHOST} rows")
    return parts


def _inverse(cum, target, H):
    lo, hi = 0, H  # cum is increasing: smallest r with cum(r) >= target
    while lo < hi:
        mid = (lo + hi) // 2
        if cum(mid) < target:
            lo = mid + 1
        else:
            hi = mid
    return lo


class HaloExchanger:
    """Per-step ghost-row swap with the neighbours rank-1 (above) and rank+1
    (below) over a torch.distributed process group.

    planes(side, recv) -> list of tensors, in a fixed plane order, for side 0
    (toward row 0) or 1 (toward row H-1); recv=False: rows to send, True:
    ghost rows to fill.
    """

    def __init__(self, rank: int, world: int, group=None, staged: bool = False):
        self.rank, self.world, self.group = rank, world, group
        # staged: device tensors travel through host copies (for backends such as
        # gloo that move only CPU tensors, e.g. two ranks sharing one GPU in tests).
        self.staged = staged

    def exchange(self, planes) -> None:
        if self.staged:
            self._exchange_staged(planes)
            return
        self._exchange(planes)

    def _exchange_staged(self, planes) -> None:
        host = {}

        def staged_planes(side, recv):
            out = []
            for t in planes(side, recv):
                h = t.to("cpu") if not recv else t.new_empty(t.shape, device="cpu")
                host.setdefault((side, recv), []).append((t, h))
                out.append(h)
            return out

        self._exchange(staged_planes)
        for side in (0, 1):
            for dev, h in host.get((side, True), []):
                dev.copy_(h)

    def _exchange(self, planes) -> None:
        import torch.distributed as dist

        ops = []
        if self.rank > 0:
            peer = self.rank - 1
            ops += [dist.P2POp(dist.isend, t, peer, self.group) for t in planes(0, False)]
            ops += [dist.P2POp(dist.irecv, t, peer, self.group) for t in planes(0, True)]
        if self.rank < self.world - 1:
            peer = self.rank + 1
            ops += [dist.P2POp(dist.isend, t, peer, self.group) for t in planes(1, False)]
            ops += [dist.P2POp(dist.irecv, t, peer, self.group) for t in planes(1, True)]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()


class _DeviceRange:
    """__cuda_array_interface__ view of a library-owned device range (bytes)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3, "strides": None,
            "stream": None,
        }


def _device_tensor(ptr: int, nbytes: int, device: int):
    import torch

    return torch.as_tensor(_DeviceRange(ptr, nbytes), device=f"cuda:{device}")


class ShardedEngine:
    """One rank's row shard of `replicas` scenarios, stepped on its GPU with a
    ghost-row exchange after every step."""

    def __init__(self, cfg, rank: int, world: int, *, device: int | None = None, replicas: int = 1,
                 seed: int | None = None, kernel: str = "fused", group=None, exchange: str | None = None):
        import torch

        from .engine import _pf_config, validate

        validate(cfg)
        self.cfg = cfg
        self.rank, self.world = rank, world
        self.group = group
        self.device = rank if device is None else device
        self.lo, self.hi = balanced_row_partition(cfg, world)[rank]
        whole = world == 1
        self.ctx = _lib.Context(_pf_config(cfg, cfg.seed if seed is None else seed, replicas=replicas,
                                           row_begin=0 if whole else self.lo, row_end=0 if whole else self.hi,
                                           device=self.device, kernel=kernel))
        self.ctx.init_environment()
        if exchange is None:
            exchange = "p2p" if kernel in ("fused", "fused_f32") else "collective"
        if exchange not in ("p2p", "collective"):
            raise _lib.ConfigError(f"unknown halo exchange {exchange!r} (p2p or collective)")
        self.exchange = exchange if world > 1 else "none"
        staged = False
        if world > 1:
            import torch.distributed as dist

            staged = dist.get_backend(group) != "nccl"
            if self.exchange == "p2p":
                self._link_peers(dist, group)
        self.exchanger = HaloExchanger(rank, world, group, staged=staged)
        self._tcache: dict = {}
        self._stream = torch.cuda.ExternalStream(self.ctx.stream(), device=f"cuda:{self.device}")

    def _link_peers(self, dist, group):
        """Fused halo exchange: all-gather every rank's pf_peer_desc (CUDA IPC
        handles of its planes) and attach the two vertical neighbours."""
        mine = bytes(self.ctx.peer_desc())
        descs = [None] * self.world
        dist.all_gather_object(descs, mine, group=group)
        for side, peer in ((0, self.rank - 1), (1, self.rank + 1)):
            if 0 <= peer < self.world:
                d = _lib.PfPeerDesc.from_buffer_copy(descs[peer])
                self.ctx.attach_peer(side, d, ipc=True)
        dist.barrier(group=group)  # no rank signals a neighbour before it has attached

    def _planes(self, side: int, recv: bool):
        out = []
        for r in range(self.ctx.replicas):
            h = self.ctx.halo(r, side, recv)
            for ptr, nb in ((h.cells, h.cell_bytes), (h.occ, h.occ_bytes), (h.tau, h.tau_bytes),
                             (h.tour, h.tour_bytes)):
                if not nb:
                    continue
                key = (ptr, nb)
                t = self._tcache.get(key)
                if t is None:
                    t = self._tcache[key] = _device_tensor(ptr, nb, self.device)
                out.append(t)
        return out

    def step(self, n: int = 1) -> None:
        """n steps. p2p: one graph-batched enqueue (the kernels exchange the
        halo themselves); collective: the halo swap is stream-ordered after
        each step's kernel."""
        import torch

        if self.exchange in ("p2p", "none"):
            self.ctx.step_async(n)
            return
        for _ in range(n):
            self.ctx.step_async(1)
            if self.world > 1:
                if self.exchanger.staged:
                    self.ctx.synchronize()  # host copies follow the kernel
                    self.exchanger.exchange(self._planes)
                    torch.cuda.synchronize(self.device)
                else:
                    with torch.cuda.stream(self._stream):
                        self.exchanger.exchange(self._planes)

    def reports(self, n: int) -> np.ndarray:
        """This shard's [replicas][n] reports of the last n steps (sum over ranks
        for the whole grid's StepReport)."""
        return self.ctx.read_reports(n)

    def synchronize(self):
        self.ctx.synchronize()

    def store(self, replica: int, occ, index, agents, tau_top, tau_bot) -> int:
        """Write this shard's owned rows (and the agents living there) into
        global-grid host planes."""
        return self.ctx.store(replica, occ, index, agents, tau_top, tau_bot)

    def close(self):
        """Free the shard. With the fused exchange a neighbour may still be
        storing into this shard's ghost rows during its last step, so every
        rank finishes its steps (synchronize + barrier) before any frees."""
        if self.exchange == "p2p" and self.world > 1 and getattr(self.ctx, "h", None):
            import torch.distributed as dist

            self.ctx.synchronize()
            dist.barrier(group=self.group)
        self.ctx.close()
