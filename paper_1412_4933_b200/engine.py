"""Host-side mirror of the reference's step-engine API, backed by the CUDA path.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/pedflow/*.hpp) so that a run_scenario-style
caller can switch engines:

    ScenarioConfig, validate         inc/config.hpp:20-60, src/config.cpp:101-124
    band_height                      inc/metrics.hpp:13, src/metrics.cpp:8-11
    SimState, new_environment        inc/state.hpp:16-37, src/state.cpp:54-75
    StepReport, EngineOptions        inc/engine.hpp:16-34, src/engine.cpp:35-46
    StepEngine.step                  inc/engine.hpp:48-66, src/engine.cpp:53-62
    run_scenario, RunReport          inc/engine.hpp:70-72, src/engine.cpp:195-231

The SimState planes live on the host as numpy arrays (the reference's value
semantics); a StepEngine keeps a device copy and syncs lazily: stepping the
same state again does not re-upload, and the host planes are refreshed only
when read.
"""
from __future__ import annotations

import enum
import itertools
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import AGENT_DTYPE, REPORT_DTYPE, ConfigError, StateCorrupt  # noqa: F401


class Model(enum.IntEnum):
    Lem = 0
    Aco = 1


class ExecutorKind(enum.IntEnum):
    """The reference's CPU executors (inc/config.hpp:13). The GPU engine ignores
    them (its grid replaces the thread pool); kept so configs round-trip."""

    Sequential = 0
    Parallel = 1


@dataclass
class ScenarioConfig:
    """pedflow::ScenarioConfig (inc/config.hpp:20-58), same defaults."""

    width: int = 480
    height: int = 480
    agents_per_side: int = 1280
    model: Model = Model.Aco
    steps: int = 25000
    seed: int = 42
    repeats: int = 10
    executor: ExecutorKind = ExecutorKind.Sequential
    threads: int = 0
    d0: float = 2.0
    sel_mu: float = 1.0
    sel_sigma: float = 0.5
    alpha: float = 1.0
    beta: float = 2.0
    rho: float = 0.05
    tau0: float = 0.1
    q: float = 1.0
    out_dir: str = "."
    # True when the model was picked (file or flag) rather than defaulted;
    # sweep runs both models otherwise (inc/config.hpp:45-48).
    model_explicit: bool = False


def _pf_config(cfg: ScenarioConfig, seed: int | None = None, *, replicas: int = 1, row_begin: int = 0,
               row_end: int = 0, device: int = 0, kernel: str = "fused") -> _lib.PfConfig:
    # "fused_f32": the fused kernel with fp32 pheromone storage (tolerance-only)
    k = {"fused": _lib.PF_KERNEL_FUSED, "pipeline": _lib.PF_KERNEL_PIPELINE, "tile": _lib.PF_KERNEL_TILE,
         "fused_f32": _lib.PF_KERNEL_FUSED_F32}.get(kernel)
    if k is None:
        raise ConfigError(f"unknown kernel '{kernel}'")
    return _lib.PfConfig(
        int(cfg.width), int(cfg.height), int(cfg.agents_per_side), int(Model(cfg.model)),
        int(cfg.seed if seed is None else seed) & (2**64 - 1),
        float(cfg.d0), float(cfg.sel_mu), float(cfg.sel_sigma), float(cfg.alpha), float(cfg.beta),
        float(cfg.rho), float(cfg.tau0), float(cfg.q), int(replicas), int(row_begin), int(row_end),
        int(device), k,
    )


def validate(cfg: ScenarioConfig) -> None:
    """validate() (src/config.cpp:101-124, same checks in the same order) plus
    the GPU preconditions. Raises ConfigError."""
    if cfg.width < 16 or cfg.width % 16 != 0:
        raise ConfigError("width must be a multiple of 16 and >= 16")
    if cfg.height < 16 or cfg.height % 16 != 0:
        raise ConfigError("height must be a multiple of 16 and >= 16")
    if cfg.agents_per_side < 0:
        raise ConfigError("agents_per_side must be >= 0")
    if cfg.steps < 0:
        raise ConfigError("steps must be >= 0")
    if cfg.repeats < 1:
        raise ConfigError("repeats must be >= 1")
    if cfg.threads < 0:
        raise ConfigError("threads must be >= 0")
    c = _pf_config(cfg)
    if not cfg.out_dir:  # after the numeric checks, before capacity (src/config.cpp:115-117)
        c.agents_per_side = 0
        _lib.check(_lib.lib.pf_validate(c))
        raise ConfigError("out_dir must not be empty")
    _lib.check(_lib.lib.pf_validate(c))


def band_height(agents_per_side: int, width: int) -> int:
    """ceil(agents_per_side / width) (src/metrics.cpp:8-11)."""
    if width <= 0:
        raise ConfigError("width must be > 0")
    return _lib.lib.pf_band_height(agents_per_side, width)


@dataclass
class StepReport:
    """pedflow::StepReport (inc/engine.hpp:16-21)."""

    step: int = 0
    moved: int = 0
    newly_crossed_top: int = 0
    newly_crossed_bottom: int = 0

    @classmethod
    def from_row(cls, r) -> "StepReport":
        return cls(int(r["step"]), int(r["moved"]), int(r["newly_crossed_top"]), int(r["newly_crossed_bottom"]))


_STATE_TOKENS = itertools.count(1)


class SimState:
    """pedflow::SimState (inc/state.hpp:16-31): occupancy, index, agents,
    pheromone (ACO), step. Planes are numpy arrays in the reference's layout
    (row-major H x W; agents[id-1] as AgentRecord). When a StepEngine has
    advanced the state on the device, reading any plane pulls it back first.
    If you modify planes in place, call touch() so the next step re-uploads.
    """

    def __init__(self, width: int, height: int, model: Model, n_agents: int, pinned: bool = False):
        self.width = int(width)
        self.height = int(height)
        self.model = Model(model)
        # pinned: planes in page-locked memory (pf_host_alloc), which state
        # upload / download DMA directly instead of staging.
        zeros = _lib.pinned_array if pinned else np.zeros
        self._occ = zeros((height, width), np.uint8)
        self._index = zeros((height, width), np.uint32)
        self._agents = zeros((n_agents,), AGENT_DTYPE)
        aco = self.model == Model.Aco
        self._tau_top = zeros((height, width), np.float64) if aco else None
        self._tau_bot = zeros((height, width), np.float64) if aco else None
        self._scores = np.zeros((n_agents, 8), np.float64)  # CandidateScores::score by agent id
        self._step = 0
        self._device = None  # (engine, replica) holding a newer copy
        self._version = 0    # bumped whenever the host planes change (touch, download)
        self._token = next(_STATE_TOKENS)  # never reused (unlike id())

    # --- lazy sync -----------------------------------------------------
    def _pull(self):
        if self._device is not None:
            eng, rep = self._device
            self._device = None
            eng._download(self, rep)

    def touch(self):
        """Declare the host planes modified (forces a re-upload on the next step)."""
        self._pull()
        self._version += 1

    def copy(self) -> "SimState":
        self._pull()
        s = SimState(self.width, self.height, self.model, len(self._agents))
        s._occ[...] = self._occ
        s._index[...] = self._index
        s._agents[...] = self._agents
        if self._tau_top is not None:
            s._tau_top[...] = self._tau_top
            s._tau_bot[...] = self._tau_bot
        s._scores[...] = self._scores
        s._step = self._step
        return s

    @property
    def occupancy(self) -> np.ndarray:
        self._pull()
        return self._occ

    @property
    def index(self) -> np.ndarray:
        self._pull()
        return self._index

    @property
    def agents(self) -> np.ndarray:
        self._pull()
        return self._agents

    @property
    def scores(self) -> np.ndarray:
        """CandidateScores::score (inc/pedflow/lem.hpp:14-17) by agent id,
        [n_agents, 8] in goal-relative slot order: nonzero between
        score_phase and reset_phase, zeros otherwise."""
        self._pull()
        return self._scores

    @property
    def score_owners(self) -> np.ndarray:
        """CandidateScores::owner: always the agent's id (src/state.cpp:48)."""
        return np.arange(1, len(self._agents) + 1, dtype=np.uint32)

    @property
    def pheromone_top(self) -> np.ndarray | None:
        self._pull()
        return self._tau_top

    @property
    def pheromone_bottom(self) -> np.ndarray | None:
        self._pull()
        return self._tau_bot

    @property
    def step(self) -> int:
        if self._device is not None:
            return self._device[0]._ctx.current_step
        return self._step

    def agent(self, id_: int):
        return self.agents[id_ - 1]

    def cell_index(self, r: int, c: int) -> int:
        return r * self.width + c


def new_environment(cfg: ScenarioConfig, seed: int, pinned: bool = False) -> SimState:
    """new_environment (src/state.cpp:54-75), computed by the library's host C++.
    pinned=True puts the planes in page-locked memory (faster state transfers)."""
    validate(cfg)
    s = SimState(cfg.width, cfg.height, cfg.model, 2 * cfg.agents_per_side, pinned=pinned)
    c = _pf_config(cfg, seed)
    _lib.check(_lib.lib.pf_new_environment(c, int(seed) & (2**64 - 1), s._occ.ctypes.data, s._index.ctypes.data,
                                           s._agents.ctypes.data if len(s._agents) else None,
                                           _lib.ptr(s._tau_top), _lib.ptr(s._tau_bot)))
    return s


@dataclass
class EngineOptions:
    """pedflow::EngineOptions (inc/engine.hpp:23-34) + the GPU placement."""

    model: Model = Model.Lem
    executor: ExecutorKind = ExecutorKind.Sequential
    threads: int = 1
    seed: int = 0
    d0: float = 2.0
    sel_mu: float = 1.0
    sel_sigma: float = 0.5
    alpha: float = 1.0
    beta: float = 2.0
    rho: float = 0.05
    tau0: float = 0.1
    q: float = 1.0
    crossing_band: int = 1
    device: int = 0
    kernel: str = "fused"

    @classmethod
    def from_config(cls, cfg: ScenarioConfig, seed: int, **gpu) -> "EngineOptions":
        """EngineOptions::from_config (src/engine.cpp:35-46)."""
        validate(cfg)
        return cls(model=Model(cfg.model), executor=cfg.executor, threads=cfg.threads, seed=seed, d0=cfg.d0,
                   sel_mu=cfg.sel_mu, sel_sigma=cfg.sel_sigma, alpha=cfg.alpha, beta=cfg.beta, rho=cfg.rho,
                   tau0=cfg.tau0, q=cfg.q, crossing_band=band_height(cfg.agents_per_side, cfg.width), **gpu)


class StepEngine:
    """pedflow::StepEngine (inc/engine.hpp:48-66) on one B200.

    ``step(state)`` advances the state by one synchronous step and returns its
    StepReport; ``run(state, n)`` is the batched fast path (one upload, n steps
    through CUDA graphs, one lazy download). The reference's phase methods
    (score_phase / intention_phase / movement_phase / reset_phase) are
    available on an engine built with ``kernel="pipeline"``; the default fused
    kernel runs all four in one launch.
    """

    def __init__(self, opt: EngineOptions):
        self._opt = opt
        self._ctx: _lib.Context | None = None
        self._dims = None
        self._bound = None  # (state token, version) the device copy equals
        self._resident = None  # weakref to the state whose newest copy is on the device

    def options(self) -> EngineOptions:
        return self._opt

    def _scenario(self, state: SimState) -> ScenarioConfig:
        o = self._opt
        return ScenarioConfig(width=state.width, height=state.height, agents_per_side=len(state._agents) // 2,
                              model=o.model, seed=o.seed, d0=o.d0, sel_mu=o.sel_mu, sel_sigma=o.sel_sigma,
                              alpha=o.alpha, beta=o.beta, rho=o.rho, tau0=o.tau0, q=o.q)

    def _attach(self, state: SimState):
        if state._device is not None and state._device[0] is self:
            return  # already resident and newer on the device
        state._pull()  # newer on another engine: bring it home first (bumps _version)
        if self._ctx is not None and self._bound == (state._token, state._version):
            self._resident = weakref.ref(state)
            return  # the device copy equals the host planes
        if Model(state.model) != Model(self._opt.model):
            raise ConfigError("state model disagrees with engine options")
        # Another state's newest copy lives here: download it before its planes
        # are overwritten (the reference's step(SimState&) accepts any state).
        other = self._resident() if self._resident is not None else None
        if other is not None and other is not state and other._device is not None and other._device[0] is self:
            other._pull()
        self._resident = None
        dims = (state.width, state.height, len(state._agents))
        if self._ctx is None or self._dims != dims:
            if self._ctx is not None:
                self._ctx.close()
            sc = self._scenario(state)
            self._ctx = _lib.Context(_pf_config(sc, self._opt.seed, device=self._opt.device, kernel=self._opt.kernel))
            self._dims = dims
        self._ctx.load(0, state._occ, state._index, state._agents, state._tau_top, state._tau_bot, state._step)
        self._bound = (state._token, state._version)
        self._resident = weakref.ref(state)

    def _download(self, state: SimState, rep: int):
        # planes are written in place by the library
        state._step = self._ctx.store(rep, state._occ, state._index, state._agents, state._tau_top, state._tau_bot)
        if len(state._agents):
            self._ctx.store_scores(rep, state._scores)
        # The host planes changed: every other engine's copy of this state is
        # now stale; this engine's copy equals the new planes.
        state._version += 1
        self._bound = (state._token, state._version)

    # --- phase-level stepping (src/engine.cpp:64-193) ------------------------
    def _phase(self, state: SimState, phase: int):
        self._attach(state)
        out = self._ctx.phase(phase)
        state._device = (self, 0)
        return out

    def score_phase(self, state: SimState) -> None:
        """StepEngine::score_phase (src/engine.cpp:64-74): state.scores."""
        self._phase(state, _lib.PF_PHASE_SCORE)

    def intention_phase(self, state: SimState) -> None:
        """StepEngine::intention_phase (src/engine.cpp:76-90): agents' futures."""
        self._phase(state, _lib.PF_PHASE_INTENTION)

    def movement_phase(self, state: SimState) -> StepReport:
        """StepEngine::movement_phase (src/engine.cpp:92-180)."""
        return StepReport.from_row(self._phase(state, _lib.PF_PHASE_MOVEMENT)[0])

    def reset_phase(self, state: SimState) -> None:
        """StepEngine::reset_phase (src/engine.cpp:183-193): scores zeroed,
        futures re-anchored, ++step."""
        self._phase(state, _lib.PF_PHASE_RESET)

    def run(self, state: SimState, n: int) -> list[StepReport]:
        """n full steps (StepEngine::step x n); returns the n StepReports."""
        self._attach(state)
        rep = self._ctx.step(n)
        state._device = (self, 0)
        if rep is None:
            return []
        return [StepReport.from_row(r) for r in rep[0]]

    def run_array(self, state: SimState, n: int) -> np.ndarray:
        """Like run() but returns the reports as a REPORT_DTYPE array."""
        self._attach(state)
        rep = self._ctx.step(n)
        state._device = (self, 0)
        return rep[0] if rep is not None else np.zeros(0, REPORT_DTYPE)

    def step(self, state: SimState) -> StepReport:
        """StepEngine::step(SimState&) (src/engine.cpp:53-62)."""
        return self.run(state, 1)[0]

    @property
    def context(self) -> _lib.Context | None:
        return self._ctx

    def close(self):
        other = self._resident() if self._resident is not None else None
        if other is not None and other._device is not None and other._device[0] is self:
            other._pull()  # the state must outlive the device copy it depends on
        self._resident = None
        self._bound = None
        if self._ctx is not None:
            self._ctx.close()
            self._ctx = None


@dataclass
class StepSeriesRow:
    """inc/metrics.hpp:19-25."""

    step: int = 0
    crossed_top: int = 0
    crossed_bottom: int = 0
    crossed_total: int = 0
    moved: int = 0


@dataclass
class RunReport:
    """inc/metrics.hpp:28-38."""

    config: ScenarioConfig = field(default_factory=ScenarioConfig)
    seed: int = 0
    model: Model = Model.Lem
    executor: ExecutorKind = ExecutorKind.Sequential
    threads: int = 1
    agents_total: int = 0
    series: list = field(default_factory=list)
    throughput: int = 0
    runtime_seconds: float = 0.0


def run_scenario(cfg: ScenarioConfig, seed: int, *, device: int = 0, kernel: str = "fused") -> RunReport:
    """run_scenario (src/engine.cpp:195-231) on the GPU engine; like the
    reference, runtime_seconds includes setup."""
    validate(cfg)
    t0 = time.perf_counter()
    state = new_environment(cfg, seed)
    eng = StepEngine(EngineOptions.from_config(cfg, seed, device=device, kernel=kernel))
    rep = eng.run_array(state, cfg.steps) if cfg.steps else np.zeros(0, REPORT_DTYPE)
    top = np.cumsum(rep["newly_crossed_top"].astype(np.int64))
    bot = np.cumsum(rep["newly_crossed_bottom"].astype(np.int64))
    series = [StepSeriesRow(int(rep["step"][i]), int(top[i]), int(bot[i]), int(top[i] + bot[i]), int(rep["moved"][i]))
              for i in range(len(rep))]
    out = RunReport(config=cfg, seed=seed, model=Model(cfg.model), executor=cfg.executor,
                    threads=cfg.threads, agents_total=2 * cfg.agents_per_side, series=series,
                    throughput=int(top[-1] + bot[-1]) if len(rep) else 0)
    state._pull()
    eng.close()
    out.runtime_seconds = time.perf_counter() - t0
    return out


__all__ = [
    "Model", "ExecutorKind", "ScenarioConfig", "validate", "band_height", "StepReport", "SimState",
    "new_environment", "EngineOptions", "StepEngine", "StepSeriesRow", "RunReport", "run_scenario",
    "ConfigError", "StateCorrupt",
]
