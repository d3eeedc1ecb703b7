"""ctypes binding of the C-ABI in include/pf_gpu.h (libpedflow_b200.so).

There is no fallback: if the shared library is missing, importing this module
raises; if no CUDA device is present, creating a context raises. Every call
that fails raises the Python mirror of the reference's exception class
(ConfigError for PF_ERR_CONFIG, StateCorrupt for PF_ERR_STATE, ...).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PEDFLOW_B200_LIB") or os.path.join(HERE, "libpedflow_b200.so")

PF_OK, PF_ERR_CONFIG, PF_ERR_CUDA, PF_ERR_COMM, PF_ERR_STATE, PF_ERR_ARG = 0, 2, 3, 4, 5, 6
PF_MODEL_LEM, PF_MODEL_ACO = 0, 1
PF_KERNEL_FUSED, PF_KERNEL_PIPELINE, PF_KERNEL_TILE, PF_KERNEL_FUSED_F32 = 0, 1, 2, 3
PF_PHASE_SCORE, PF_PHASE_INTENTION, PF_PHASE_MOVEMENT, PF_PHASE_RESET = 0, 1, 2, 3
PF_GHOST_ROWS = 3

# pedflow::AgentRecord (inc/grid.hpp:84-93) == pf_agent, 40 bytes.
AGENT_DTYPE = np.dtype(
    {
        "names": ["index", "group", "row", "col", "future_row", "future_col", "tour_length", "crossed"],
        "formats": ["<u4", "u1", "<i4", "<i4", "<i4", "<i4", "<f8", "u1"],
        "offsets": [0, 4, 8, 12, 16, 20, 24, 32],
        "itemsize": 40,
    }
)
# pedflow::StepReport (inc/engine.hpp:16-21) == pf_step_report.
REPORT_DTYPE = np.dtype(
    [("step", "<u4"), ("moved", "<u4"), ("newly_crossed_top", "<u4"), ("newly_crossed_bottom", "<u4")]
)


class ConfigError(ValueError):
    """pedflow::ConfigError (inc/errors.hpp:9-11)."""


class StateCorrupt(RuntimeError):
    """The std::logic_error("state corrupt: ...") of check_consistency (src/state.cpp:77-110)."""


class DeviceError(RuntimeError):
    """CUDA failure inside the library (no device, out of memory, launch error)."""


class CommError(RuntimeError):
    """Halo-exchange failure between row shards."""


class PfConfig(C.Structure):
    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32), ("agents_per_side", C.c_int32), ("model", C.c_int32),
        ("seed", C.c_uint64),
        ("d0", C.c_double), ("sel_mu", C.c_double), ("sel_sigma", C.c_double), ("alpha", C.c_double),
        ("beta", C.c_double), ("rho", C.c_double), ("tau0", C.c_double), ("q", C.c_double),
        ("replicas", C.c_int32), ("row_begin", C.c_int32), ("row_end", C.c_int32), ("device", C.c_int32),
        ("kernel", C.c_int32),
    ]


class PfHalo(C.Structure):
    _fields_ = [
        ("cells", C.c_void_p), ("cell_bytes", C.c_size_t),
        ("tau", C.c_void_p), ("tau_bytes", C.c_size_t),
        ("tour", C.c_void_p), ("tour_bytes", C.c_size_t),
        ("occ", C.c_void_p), ("occ_bytes", C.c_size_t),
    ]


class PfPeerDesc(C.Structure):
    """pf_peer_desc: a shard's planes for its neighbours (fused halo exchange)."""
    _fields_ = [
        ("ipc", (C.c_ubyte * 64) * 7), ("ptr", C.c_uint64 * 7),
        ("device", C.c_int32), ("width", C.c_int32), ("replicas", C.c_int32), ("model", C.c_int32),
        ("kernel", C.c_int32), ("row_begin", C.c_int32), ("rows_owned", C.c_int32), ("parity", C.c_int32),
        ("step", C.c_uint32), ("reserved", C.c_uint32),
        ("plane", C.c_uint64), ("occ_plane", C.c_uint64),
    ]


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA library first "
        "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback."
    )

lib = C.CDLL(LIB_PATH)
_vp, _i32, _u32, _u64 = C.c_void_p, C.c_int32, C.c_uint32, C.c_uint64
_sigs = {
    "pf_last_error": (C.c_char_p, []),
    "pf_version": (C.c_char_p, []),
    "pf_validate": (C.c_int, [C.POINTER(PfConfig)]),
    "pf_band_height": (_i32, [_i32, _i32]),
    "pf_new_environment": (C.c_int, [C.POINTER(PfConfig), _u64, _vp, _vp, _vp, _vp, _vp]),
    "pf_create": (C.c_int, [C.POINTER(PfConfig), C.POINTER(_vp)]),
    "pf_destroy": (C.c_int, [_vp]),
    "pf_set_replicas": (C.c_int, [_vp, _vp, _vp]),
    "pf_replica_agents": (_i32, [_vp, _i32]),
    "pf_init_environment": (C.c_int, [_vp]),
    "pf_load_state": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _u32, _vp, _vp, _u32]),
    "pf_store_state": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _u32, _vp, _vp, C.POINTER(_u32)]),
    "pf_step": (C.c_int, [_vp, _u32, _vp]),
    "pf_step_async": (C.c_int, [_vp, _u32]),
    "pf_prepare_steps": (C.c_int, [_vp, _u32]),
    "pf_read_reports": (C.c_int, [_vp, _vp, _u32]),
    "pf_synchronize": (C.c_int, [_vp]),
    "pf_time_steps": (C.c_int, [_vp, _u32, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "pf_current_step": (_u32, [_vp]),
    "pf_stream": (_vp, [_vp]),
    "pf_launch_count": (_u64, [_vp]),
    "pf_halo": (C.c_int, [_vp, _i32, _i32, _i32, C.POINTER(PfHalo)]),
    "pf_exchange_pair": (C.c_int, [_vp, _vp]),
    "pf_selftest_rng": (C.c_int, [_i32, _u32, _vp, _vp, _vp, _vp, _vp, C.c_double, C.c_double, _vp, _vp, _vp]),
    "pf_audit": (C.c_int, [_vp, _i32, C.POINTER(_u64)]),
    "pf_selftest_select": (C.c_int, [_i32, _i32, _u32, C.c_double, C.c_double, C.c_double, _vp, _vp, _vp, _vp, _vp,
                                     _vp]),
    "pf_phase": (C.c_int, [_vp, _i32, _vp]),
    "pf_store_scores": (C.c_int, [_vp, _i32, _vp, _vp, _u32]),
    "pf_host_alloc": (_vp, [C.c_size_t]),
    "pf_host_free": (C.c_int, [_vp]),
    "pf_peer_export": (C.c_int, [_vp, C.POINTER(PfPeerDesc)]),
    "pf_peer_attach": (C.c_int, [_vp, _i32, C.POINTER(PfPeerDesc), _i32]),
}
for _name, (_res, _args) in _sigs.items():
    if os.environ.get("PEDFLOW_B200_LIB") and not hasattr(lib, _name):
        continue  # dev A/B against an older build (tools/ab_time.py): newer entry points absent
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED_SYMBOLS = tuple(_sigs)


def check(rc: int) -> None:
    if rc == PF_OK:
        return
    msg = lib.pf_last_error().decode(errors="replace")
    if rc == PF_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == PF_ERR_STATE:
        raise StateCorrupt(msg)
    if rc == PF_ERR_CUDA:
        raise DeviceError(msg)
    if rc == PF_ERR_COMM:
        raise CommError(msg)
    raise ValueError(f"pedflow-b200 error {rc}: {msg}")


def ptr(a) -> int | None:
    return None if a is None else a.ctypes.data


class Context:
    """Owns one pf_ctx: R replicas of one grid (or one row shard of it) on one device."""

    def __init__(self, cfg: PfConfig):
        self.cfg = cfg
        h = C.c_void_p()
        check(lib.pf_create(C.byref(cfg), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib.pf_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    @property
    def replicas(self) -> int:
        return self.cfg.replicas

    @property
    def aco(self) -> bool:
        return self.cfg.model == PF_MODEL_ACO

    def set_replicas(self, agents_per_side=None, seeds=None):
        """Per-replica densities and/or seeds (pf_set_replicas)."""
        aps = None if agents_per_side is None else np.ascontiguousarray(agents_per_side, np.int32)
        sds = None if seeds is None else np.ascontiguousarray(seeds, np.uint64)
        for a in (aps, sds):
            if a is not None and a.shape != (self.replicas,):
                raise ValueError(f"expected {self.replicas} per-replica values, got shape {a.shape}")
        check(lib.pf_set_replicas(self.h, ptr(aps), ptr(sds)))

    def replica_agents(self, replica: int) -> int:
        return int(lib.pf_replica_agents(self.h, replica))

    def init_environment(self):
        check(lib.pf_init_environment(self.h))

    def _check_planes(self, replica, occ, index, agents, tau_top, tau_bot, need_all: bool):
        """The C-ABI reads/writes width*height cells per plane and the whole
        agent table through raw pointers: reject anything that does not match
        this context's grid instead of letting it run out of bounds."""
        if not 0 <= int(replica) < self.replicas:
            raise ConfigError(f"replica {replica} out of range [0, {self.replicas})")
        shape = (int(self.cfg.height), int(self.cfg.width))
        planes = [("occupancy", occ, np.uint8), ("index", index, np.uint32)]
        if self.aco:
            planes += [("pheromone_top", tau_top, np.float64), ("pheromone_bottom", tau_bot, np.float64)]
        elif tau_top is not None or tau_bot is not None:
            raise ConfigError("pheromone planes given for a LEM context")
        for name, a, dt in planes:
            if a is None:
                if need_all:
                    raise ConfigError(f"{name} plane missing")
                continue
            if not isinstance(a, np.ndarray) or a.dtype != dt or a.shape != shape or not a.flags.c_contiguous:
                got = (type(a).__name__, getattr(a, "dtype", None), getattr(a, "shape", None))
                raise ConfigError(f"{name} must be a C-contiguous {np.dtype(dt).name} array of shape {shape}, got {got}")
            if not need_all and not a.flags.writeable:
                raise ConfigError(f"{name} is read-only")
        n = 2 * self.replica_agents(replica)
        if (not isinstance(agents, np.ndarray) or agents.dtype != AGENT_DTYPE or agents.ndim != 1
                or not agents.flags.c_contiguous or len(agents) != n):
            raise ConfigError(f"agents must be a C-contiguous AgentRecord array of length {n}, got "
                              f"{getattr(agents, 'dtype', type(agents).__name__)} x {getattr(agents, 'shape', None)}")

    def load(self, replica, occ, index, agents, tau_top, tau_bot, step):
        self._check_planes(replica, occ, index, agents, tau_top, tau_bot, need_all=True)
        check(lib.pf_load_state(self.h, replica, ptr(occ), ptr(index), ptr(agents) if len(agents) else None,
                                len(agents), ptr(tau_top), ptr(tau_bot), step))

    def store(self, replica, occ, index, agents, tau_top, tau_bot) -> int:
        self._check_planes(replica, occ, index, agents, tau_top, tau_bot, need_all=False)
        step = C.c_uint32(0)
        check(lib.pf_store_state(self.h, replica, ptr(occ), ptr(index), ptr(agents) if len(agents) else None,
                                 len(agents), ptr(tau_top), ptr(tau_bot), C.byref(step)))
        return step.value

    def step(self, n: int, want_reports: bool = True) -> np.ndarray | None:
        out = np.zeros((self.replicas, n), REPORT_DTYPE) if want_reports and n else None
        check(lib.pf_step(self.h, n, ptr(out)))
        return out

    def step_async(self, n: int):
        check(lib.pf_step_async(self.h, n))

    def prepare_steps(self, n: int):
        """Instantiate the CUDA graphs step_async(n) will replay (no launch)."""
        check(lib.pf_prepare_steps(self.h, n))

    def read_reports(self, n: int) -> np.ndarray:
        out = np.zeros((self.replicas, n), REPORT_DTYPE)
        check(lib.pf_read_reports(self.h, ptr(out), n))
        return out

    def synchronize(self):
        check(lib.pf_synchronize(self.h))

    def time_steps(self, n: int, kernel: bool = False) -> tuple[float, float | None]:
        tot, ker = C.c_float(0), C.c_float(0)
        check(lib.pf_time_steps(self.h, n, C.byref(tot), C.byref(ker) if kernel else None))
        return tot.value, (ker.value if kernel else None)

    @property
    def current_step(self) -> int:
        return lib.pf_current_step(self.h)

    @property
    def launches(self) -> int:
        return lib.pf_launch_count(self.h)

    def stream(self) -> int:
        return lib.pf_stream(self.h)

    def audit(self, replica: int = 0) -> int:
        """Device-side check_consistency of one replica; returns its agent count
        (raises StateCorrupt on a violation)."""
        n = C.c_uint64(0)
        check(lib.pf_audit(self.h, replica, C.byref(n)))
        return n.value

    def phase(self, phase: int) -> np.ndarray | None:
        """One phase of a step (pf_phase, PF_KERNEL_PIPELINE): PF_PHASE_SCORE,
        _INTENTION, _MOVEMENT (returns the [replicas] reports) or _RESET."""
        out = np.zeros(self.replicas, REPORT_DTYPE) if phase == PF_PHASE_MOVEMENT else None
        check(lib.pf_phase(self.h, phase, ptr(out)))
        return out

    def store_scores(self, replica: int, scores, owners=None):
        """CandidateScores by agent id into scores [n, 8] (and owners [n])."""
        n = len(scores)
        check(lib.pf_store_scores(self.h, replica, ptr(scores), ptr(owners), n))

    def peer_desc(self) -> PfPeerDesc:
        """This shard's planes for its neighbours (pf_peer_export)."""
        d = PfPeerDesc()
        check(lib.pf_peer_export(self.h, C.byref(d)))
        return d

    def attach_peer(self, side: int, desc: PfPeerDesc, ipc: bool):
        """Link the neighbour on `side` (0 above, 1 below) for the fused halo
        exchange (pf_peer_attach); ipc=True when it lives in another process."""
        check(lib.pf_peer_attach(self.h, side, C.byref(desc), 1 if ipc else 0))

    def halo(self, replica: int, side: int, recv: bool) -> PfHalo:
        h = PfHalo()
        check(lib.pf_halo(self.h, replica, side, 1 if recv else 0, C.byref(h)))
        return h


def exchange_pair(upper: Context, lower: Context) -> None:
    check(lib.pf_exchange_pair(upper.h, lower.h))


def link_shards(ctxs) -> None:
    """Fused halo exchange between vertically adjacent shard contexts of ONE
    process (ctxs in row order; same device or peer-capable devices)."""
    descs = [c.peer_desc() for c in ctxs]
    for i, c in enumerate(ctxs):
        if i > 0:
            c.attach_peer(0, descs[i - 1], ipc=False)
        if i + 1 < len(ctxs):
            c.attach_peer(1, descs[i + 1], ipc=False)


def selftest_rng(seed, step, phase, entity, counter, mu=0.0, sigma=1.0, device=0):
    """Device random_bits / uniform / normal for arrays of keys (pf_selftest_rng)."""
    seed = np.ascontiguousarray(seed, np.uint64)
    n = len(seed)
    step = np.ascontiguousarray(np.broadcast_to(step, n), np.uint32)
    phase = np.ascontiguousarray(np.broadcast_to(phase, n), np.uint32)
    entity = np.ascontiguousarray(np.broadcast_to(entity, n), np.uint64)
    counter = np.ascontiguousarray(np.broadcast_to(counter, n), np.uint32)
    bits = np.zeros(n, np.uint64)
    uni = np.zeros(n, np.float64)
    nrm = np.zeros(n, np.float64)
    check(lib.pf_selftest_rng(device, n, ptr(seed), ptr(step), ptr(phase), ptr(entity), ptr(counter), mu, sigma,
                              ptr(bits), ptr(uni), ptr(nrm)))
    return bits, uni, nrm


def selftest_select(kind, mask, seed, step, entity, num=None, d0=2.0, sel_mu=1.0, sel_sigma=0.5, device=0):
    """Device lem_select (kind 0) / aco_select (1) / winner draw (2) for arrays
    of keys (pf_selftest_select). Returns int32 slots / codes, -1 = stay."""
    mask = np.ascontiguousarray(mask, np.uint8)
    n = len(mask)
    seed = np.ascontiguousarray(np.broadcast_to(seed, n), np.uint64)
    step = np.ascontiguousarray(np.broadcast_to(step, n), np.uint32)
    entity = np.ascontiguousarray(np.broadcast_to(entity, n), np.uint64)
    nm = None if num is None else np.ascontiguousarray(np.broadcast_to(num, (n, 8)), np.float64)
    out = np.zeros(n, np.int32)
    check(lib.pf_selftest_select(device, kind, n, d0, sel_mu, sel_sigma, ptr(mask), ptr(nm), ptr(seed), ptr(step),
                                 ptr(entity), ptr(out)))
    return out


class PinnedBuffer:
    """Page-locked host memory from pf_host_alloc, freed with the object."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        self.ptr = lib.pf_host_alloc(self.nbytes)
        if not self.ptr:
            raise DeviceError(lib.pf_last_error().decode(errors="replace"))

    def array(self, shape, dtype) -> np.ndarray:
        """A numpy view of the buffer (keeps the buffer alive)."""
        dtype = np.dtype(dtype)
        count = int(np.prod(shape)) if len(shape) else 1
        assert count * dtype.itemsize <= self.nbytes
        raw = (C.c_char * max(1, count * dtype.itemsize)).from_address(self.ptr)
        a = np.frombuffer(raw, dtype=dtype, count=count).reshape(shape)
        a.setflags(write=True)
        return _PinnedView(a, self)

    def __del__(self):
        if getattr(self, "ptr", None):
            lib.pf_host_free(self.ptr)
            self.ptr = None


class _PinnedView(np.ndarray):
    """ndarray subclass holding a reference to its PinnedBuffer."""

    def __new__(cls, a, owner):
        obj = a.view(cls)
        obj._owner = owner
        return obj

    def __array_finalize__(self, obj):
        self._owner = getattr(obj, "_owner", None)


def pinned_array(shape, dtype) -> np.ndarray:
    """A zeroed numpy array in page-locked memory (pf_host_alloc)."""
    dtype = np.dtype(dtype)
    count = int(np.prod(shape)) if len(shape) else 1
    a = PinnedBuffer(count * dtype.itemsize).array(shape, dtype)
    a[...] = 0
    return a
