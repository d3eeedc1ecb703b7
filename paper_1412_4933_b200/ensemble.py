"""Replica-batched runs: R independent scenarios (seeds seed, seed+1, ...)
stepped by one kernel launch per step.

This is the GPU form of the reference's repeat loop (tools/pedflow.cpp:135,
"repeat i uses seed+i") and of sweep/bench repeats (tools/pedflow.cpp:159-225):
at 480x480 a single scenario is far too small to fill a B200, so the repeats
share each launch (blockIdx.z = replica).
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .engine import Model, ScenarioConfig, SimState, StepReport, _pf_config, validate


class Ensemble:
    """R replicas of one grid and model in one launch per step.

    By default replica i is `cfg` with seed `seed + i`. `agents_per_side` and
    `seeds` (sequences of R values) override density and seed per replica, so
    a whole density sweep (tools/pedflow.cpp:159-189) shares each launch.
    """

    def __init__(self, cfg: ScenarioConfig, replicas: int, *, seed: int | None = None, device: int = 0,
                 kernel: str = "fused", row_begin: int = 0, row_end: int = 0, agents_per_side=None, seeds=None):
        validate(cfg)
        self.cfg = cfg
        self.seed = cfg.seed if seed is None else seed
        self.replicas = replicas
        self.ctx = _lib.Context(_pf_config(cfg, self.seed, replicas=replicas, device=device, kernel=kernel,
                                           row_begin=row_begin, row_end=row_end))
        if agents_per_side is not None or seeds is not None:
            self.ctx.set_replicas(agents_per_side, seeds)
        self.agents_per_side = [self.ctx.replica_agents(r) for r in range(replicas)]
        self.ctx.init_environment()

    # --- stepping --------------------------------------------------------
    def run(self, n: int) -> np.ndarray:
        """n steps on every replica; returns [replicas][n] StepReport records."""
        return self.ctx.step(n)

    def run_async(self, n: int):
        self.ctx.step_async(n)

    def synchronize(self):
        self.ctx.synchronize()

    def time_steps(self, n: int, kernel: bool = False):
        return self.ctx.time_steps(n, kernel)

    @property
    def step(self) -> int:
        return self.ctx.current_step

    # --- state I/O -------------------------------------------------------
    def state(self, replica: int = 0) -> SimState:
        """Download one replica as a reference-layout SimState."""
        c = self.cfg
        s = SimState(c.width, c.height, c.model, 2 * self.agents_per_side[replica])
        s._step = self.ctx.store(replica, s._occ, s._index, s._agents, s._tau_top, s._tau_bot)
        return s

    def audit(self, replica: int = 0) -> int:
        """Device-side check_consistency (src/state.cpp:77-110) of one replica,
        in place; returns the agent count, raises StateCorrupt on a violation."""
        return self.ctx.audit(replica)

    def load(self, replica: int, s: SimState):
        self.ctx.load(replica, s.occupancy, s.index, s.agents, s.pheromone_top, s.pheromone_bottom, s.step)

    def close(self):
        self.ctx.close()

    @staticmethod
    def reports_to_list(rep: np.ndarray) -> list[StepReport]:
        return [StepReport.from_row(r) for r in rep]


__all__ = ["Ensemble", "Model"]
