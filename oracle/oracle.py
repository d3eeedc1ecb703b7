"""TEST INFRASTRUCTURE — ctypes access to the checkers. NOT PRODUCT CODE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
legs may import this module.

* ``Oracle``     — oracle/liboracle.so, the plain-C restatement
                   (pedflow_oracle.c) of the reference hot path.
* ``Reference``  — oracle/_ref/libpedflow_ref.so, the unmodified reference
                   library compiled from /root/reference/proj/src by
                   oracle/Makefile (absent when it could not be built).

Both expose the same small surface: create a scenario (new_environment),
step it, export the SimState planes as numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpedflow_ref.so")

FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3

# AgentRecord (inc/grid.hpp:84-93) — 40 bytes, natural alignment.
AGENT_DTYPE = np.dtype(
    {
        "names": ["index", "group", "row", "col", "future_row", "future_col", "tour_length", "crossed"],
        "formats": ["<u4", "u1", "<i4", "<i4", "<i4", "<i4", "<f8", "u1"],
        "offsets": [0, 4, 8, 12, 16, 20, 24, 32],
        "itemsize": 40,
    }
)
REPORT_DTYPE = np.dtype([("step", "<u4"), ("moved", "<u4"), ("newly_crossed_top", "<u4"), ("newly_crossed_bottom", "<u4")])


class _Cfg(C.Structure):
    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32), ("agents_per_side", C.c_int32), ("model", C.c_int32),
        ("seed", C.c_uint64),
        ("d0", C.c_double), ("sel_mu", C.c_double), ("sel_sigma", C.c_double), ("alpha", C.c_double),
        ("beta", C.c_double), ("rho", C.c_double), ("tau0", C.c_double), ("q", C.c_double),
    ]


class _State(C.Structure):
    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32), ("model", C.c_int32), ("n_agents", C.c_uint32),
        ("occ", C.c_void_p), ("index", C.c_void_p), ("agents", C.c_void_p),
        ("tau_top", C.c_void_p), ("tau_bot", C.c_void_p), ("step", C.c_uint32),
    ]


@dataclass
class Scenario:
    """Numeric ScenarioConfig subset (inc/config.hpp:20-58); SPEC defaults."""

    width: int = 480
    height: int = 480
    agents_per_side: int = 1024
    model: str = "lem"
    seed: int = 42
    d0: float = 2.0
    sel_mu: float = 1.0
    sel_sigma: float = 0.5
    alpha: float = 1.0
    beta: float = 2.0
    rho: float = 0.05
    tau0: float = 0.1
    q: float = 1.0

    def cstruct(self) -> _Cfg:
        return _Cfg(self.width, self.height, self.agents_per_side, 0 if self.model == "lem" else 1, self.seed,
                    self.d0, self.sel_mu, self.sel_sigma, self.alpha, self.beta, self.rho, self.tau0, self.q)


def fnv1a(data: bytes, h: int = FNV_OFFSET) -> int:
    """FNV-1a 64; vectorised enough for test-sized inputs."""
    arr = np.frombuffer(data, dtype=np.uint8)
    # Python loop over bytes is slow for MB-sized planes; use the C version when possible.
    lib = _oracle_lib()
    buf = np.ascontiguousarray(arr)
    return lib.pfo_fnv1a(buf.ctypes.data, buf.nbytes, h)


def state_hashes(occ, index, agents, tau_top=None, tau_bot=None) -> dict:
    """The five FNV-1a anchors of SURVEY.md §8(c) for one SimState."""
    out = {
        "index": fnv1a(np.ascontiguousarray(index, dtype="<u4").tobytes()),
        "occ": fnv1a(np.ascontiguousarray(occ, dtype="u1").tobytes()),
    }
    rec = np.zeros(len(agents), dtype=[("row", "<i4"), ("col", "<i4"), ("tour", "<f8"), ("crossed", "u1")])
    rec["row"] = agents["row"]
    rec["col"] = agents["col"]
    rec["tour"] = agents["tour_length"]
    rec["crossed"] = agents["crossed"]
    packed = np.zeros(len(agents), dtype=np.dtype({"names": ["row", "col", "tour", "crossed"],
                                                    "formats": ["<i4", "<i4", "<f8", "u1"],
                                                    "offsets": [0, 4, 8, 16], "itemsize": 17}))
    for k in ("row", "col", "tour", "crossed"):
        packed[k] = rec[k]
    out["agents"] = fnv1a(packed.tobytes())
    if tau_top is not None:
        h = fnv1a(np.ascontiguousarray(tau_top, dtype="<f8").tobytes())
        out["pher"] = fnv1a(np.ascontiguousarray(tau_bot, dtype="<f8").tobytes(), h)
    return out


def series_hash(reports: np.ndarray) -> int:
    return fnv1a(np.ascontiguousarray(reports).view(np.uint8).tobytes())


_LIB = None


def _oracle_lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle` (or __graft_entry__.build())")
        lib = C.CDLL(ORACLE_SO)
        u64, u32, d, vp, i32 = C.c_uint64, C.c_uint32, C.c_double, C.c_void_p, C.c_int32
        lib.pfo_fnv1a.restype = u64
        lib.pfo_fnv1a.argtypes = [vp, u64, u64]
        lib.pfo_random_bits.restype = u64
        lib.pfo_random_bits.argtypes = [u64, u32, u32, u64, u32]
        lib.pfo_uniform.restype = d
        lib.pfo_uniform.argtypes = [u64, u32, u32, u64, u32]
        lib.pfo_normal.restype = d
        lib.pfo_normal.argtypes = [u64, u32, u32, u64, u32, d, d]
        lib.pfo_inverse_normal_cdf.restype = d
        lib.pfo_inverse_normal_cdf.argtypes = [d]
        lib.pfo_log_restated.restype = d
        lib.pfo_log_restated.argtypes = [d]
        lib.pfo_log_restated_matches_host.restype = C.c_int
        lib.pfo_log_restated_matches_host.argtypes = [u32, u64]
        lib.pfo_normal_batch.restype = None
        lib.pfo_normal_batch.argtypes = [u32, vp, vp, vp, vp, vp, d, d, vp]
        lib.pfo_distance_table.argtypes = [d, vp]
        lib.pfo_band_height.restype = i32
        lib.pfo_band_height.argtypes = [i32, i32]
        lib.pfo_lem_scores.argtypes = [vp, vp, vp]
        lib.pfo_aco_numerators.argtypes = [vp, vp, d, vp, vp]
        lib.pfo_lem_select_u.argtypes = [vp, vp, d, d]
        lib.pfo_aco_select_u.argtypes = [vp, vp, d]
        lib.pfo_lem_select.argtypes = [vp, vp, u64, u32, u64, d, d]
        lib.pfo_aco_select.argtypes = [vp, vp, u64, u32, u64]
        lib.pfo_validate.argtypes = [C.POINTER(_Cfg)]
        lib.pfo_new_environment.argtypes = [C.POINTER(_Cfg), u64, C.POINTER(_State)]
        lib.pfo_step.argtypes = [C.POINTER(_State), C.POINTER(_Cfg), u64, vp]
        lib.pfo_run.argtypes = [C.POINTER(_State), C.POINTER(_Cfg), u64, u32, vp]
        lib.pfo_step_cells.argtypes = [C.POINTER(_Cfg), u64, u32, i32, i32, vp, vp, vp, vp, i32, i32, vp]
        lib.pfo_agent_size.restype = u32
        assert lib.pfo_agent_size() == 40
        _LIB = lib
    return _LIB


class OracleState:
    """A SimState owned by numpy, stepped by the C restatement."""

    def __init__(self, sc: Scenario, seed: int | None = None):
        self.sc = sc
        self.seed = sc.seed if seed is None else seed
        lib = _oracle_lib()
        self._cfg = sc.cstruct()
        if lib.pfo_validate(C.byref(self._cfg)) != 0:
            raise ValueError("invalid scenario")
        H, W, n = sc.height, sc.width, sc.agents_per_side
        self.occ = np.zeros((H, W), np.uint8)
        self.index = np.zeros((H, W), np.uint32)
        self.agents = np.zeros(2 * n, AGENT_DTYPE)
        aco = sc.model == "aco"
        self.tau_top = np.zeros((H, W), np.float64) if aco else None
        self.tau_bot = np.zeros((H, W), np.float64) if aco else None
        self._st = _State(W, H, 1 if aco else 0, 2 * n, self.occ.ctypes.data, self.index.ctypes.data,
                          self.agents.ctypes.data if n else None,
                          self.tau_top.ctypes.data if aco else None, self.tau_bot.ctypes.data if aco else None, 0)
        rc = lib.pfo_new_environment(C.byref(self._cfg), self.seed, C.byref(self._st))
        if rc:
            raise ValueError(f"new_environment failed ({rc})")

    @property
    def step_index(self) -> int:
        return self._st.step

    def run(self, n: int) -> np.ndarray:
        rep = np.zeros(n, REPORT_DTYPE)
        rc = _oracle_lib().pfo_run(C.byref(self._st), C.byref(self._cfg), self.seed, n, rep.ctypes.data if n else None)
        if rc:
            raise RuntimeError(f"oracle step failed ({rc})")
        return rep

    def hashes(self) -> dict:
        return state_hashes(self.occ, self.index, self.agents, self.tau_top, self.tau_bot)


class Reference:
    """The unmodified reference library (oracle/_ref)."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            lib = C.CDLL(REF_SO)
            u64, u32, d, vp = C.c_uint64, C.c_uint32, C.c_double, C.c_void_p
            lib.ref_create.restype = vp
            lib.ref_create.argtypes = [C.POINTER(_Cfg), C.c_int]
            lib.ref_destroy.argtypes = [vp]
            lib.ref_step.argtypes = [vp, u32, vp, C.POINTER(d)]
            lib.ref_set_executor.argtypes = [vp, C.c_int]
            lib.ref_agent_count.restype = u32
            lib.ref_agent_count.argtypes = [vp]
            lib.ref_export.argtypes = [vp, vp, vp, vp, vp, vp, vp]
            lib.ref_last_error.restype = C.c_char_p
            lib.ref_agent_record_size.restype = u32
            lib.ref_random_bits.restype = u64
            lib.ref_random_bits.argtypes = [u64, u32, u32, u64, u32]
            lib.ref_normal.restype = d
            lib.ref_normal.argtypes = [u64, u32, u32, u64, u32, d, d]
            lib.ref_inverse_normal_cdf.restype = d
            lib.ref_inverse_normal_cdf.argtypes = [d]
            assert lib.ref_agent_record_size() == 40
            cls._lib = lib
        return cls._lib

    def __init__(self, sc: Scenario, threads: int = 0, seed: int | None = None):
        self.sc = sc
        cfg = sc.cstruct()
        if seed is not None:
            cfg.seed = seed
        self._h = self.lib().ref_create(C.byref(cfg), threads)
        if not self._h:
            raise ValueError(self.lib().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "_h", None):
            self.lib().ref_destroy(self._h)
            self._h = None

    def run(self, n: int) -> tuple[np.ndarray, float]:
        rep = np.zeros(n, REPORT_DTYPE)
        secs = C.c_double(0.0)
        rc = self.lib().ref_step(self._h, n, rep.ctypes.data if n else None, C.byref(secs))
        if rc:
            raise RuntimeError(self.lib().ref_last_error().decode())
        return rep, secs.value

    def set_executor(self, threads: int) -> None:
        """Sequential (threads <= 0) or Parallel(threads), same state."""
        if self.lib().ref_set_executor(self._h, int(threads)):
            raise RuntimeError(self.lib().ref_last_error().decode())

    def export(self):
        H, W = self.sc.height, self.sc.width
        occ = np.zeros((H, W), np.uint8)
        index = np.zeros((H, W), np.uint32)
        agents = np.zeros(self.lib().ref_agent_count(self._h), AGENT_DTYPE)
        aco = self.sc.model == "aco"
        tt = np.zeros((H, W), np.float64) if aco else None
        tb = np.zeros((H, W), np.float64) if aco else None
        step = C.c_uint32(0)
        self.lib().ref_export(self._h, occ.ctypes.data, index.ctypes.data, agents.ctypes.data if len(agents) else None,
                              tt.ctypes.data if aco else None, tb.ctypes.data if aco else None, C.byref(step))
        return dict(occ=occ, index=index, agents=agents, tau_top=tt, tau_bot=tb, step=step.value)

    def hashes(self) -> dict:
        s = self.export()
        return state_hashes(s["occ"], s["index"], s["agents"], s["tau_top"], s["tau_bot"])


def oracle():
    return _oracle_lib()
