"""Dev tool: time the pieces of the end-to-end path (host SimState -> device ->
K steps -> host SimState) for one workload."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_1412_4933_b200 as p  # noqa: E402
from paper_1412_4933_b200 import _lib  # noqa: E402
from paper_1412_4933_b200.engine import _pf_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5_aco"
K = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 300
cfg, reps, desc = bench.scenario(name)
t = time.perf_counter()
state = p.new_environment(cfg, 42, pinned="--pinned" in sys.argv)
print(f"new_environment (host)   {time.perf_counter() - t:7.3f} s")
c = _lib.Context(_pf_config(cfg, 42))
for it in range(2):
    t0 = time.perf_counter()
    c.load(0, state.occupancy, state.index, state.agents, state.pheromone_top, state.pheromone_bottom, 0)
    t1 = time.perf_counter()
    c.step(K)
    t2 = time.perf_counter()
    c.store(0, state._occ, state._index, state._agents, state._tau_top, state._tau_bot)
    t3 = time.perf_counter()
    print(f"[{it}] load {t1 - t0:6.3f} s   step x{K} {t2 - t1:6.3f} s   store {t3 - t2:6.3f} s   total {t3 - t0:6.3f} s")
