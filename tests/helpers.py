"""Shared test helpers: scenario conversion and first-divergence reports."""
from __future__ import annotations

import numpy as np

from oracle.oracle import Scenario, state_hashes


def to_config(kw: dict):
    import paper_1412_4933_b200 as p

    kw = dict(kw)
    model = kw.pop("model", "lem")
    return p.ScenarioConfig(model=p.Model.Lem if model == "lem" else p.Model.Aco, **kw)


def to_scenario(kw: dict) -> Scenario:
    return Scenario(**kw)


def hashes_of(state) -> dict:
    return state_hashes(state.occupancy, state.index, state.agents, state.pheromone_top, state.pheromone_bottom)


def hex_hashes(h: dict) -> dict:
    return {k: f"{v:016x}" for k, v in h.items()}


def first_divergence(gpu_state, ora) -> str:
    """Human-readable first difference between a GPU SimState and an oracle state."""
    msgs = []
    d = np.argwhere(gpu_state.index != ora.index)
    if len(d):
        r, c = d[0]
        msgs.append(f"index differs at ({r},{c}): gpu {gpu_state.index[r, c]} oracle {ora.index[r, c]} "
                    f"({len(d)} cells)")
    if ora.tau_top is not None:
        for name, g, o in (("tau_top", gpu_state.pheromone_top, ora.tau_top),
                           ("tau_bot", gpu_state.pheromone_bottom, ora.tau_bot)):
            dd = np.argwhere(g != o)
            if len(dd):
                r, c = dd[0]
                msgs.append(f"{name} differs at ({r},{c}): gpu {g[r, c]!r} oracle {o[r, c]!r} ({len(dd)} cells)")
    ga, oa = gpu_state.agents, ora.agents
    for f in ("row", "col", "tour_length", "crossed"):
        dd = np.nonzero(ga[f] != oa[f])[0]
        if len(dd):
            i = dd[0]
            msgs.append(f"agent {i + 1} {f}: gpu {ga[f][i]!r} oracle {oa[f][i]!r} ({len(dd)} agents)")
    return "; ".join(msgs) or "identical"
