import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
torch.cuda.init(); torch.zeros(1, device="cuda")
import bench, paper_1412_4933_b200 as p
from paper_1412_4933_b200 import _lib
from paper_1412_4933_b200.engine import _pf_config
cfg, reps, desc = bench.scenario(sys.argv[1] if len(sys.argv) > 1 else "c5_aco")
for it in range(3):
    t0 = time.perf_counter(); c = _lib.Context(_pf_config(cfg, 42)); t1 = time.perf_counter()
    c.init_environment(); c.synchronize(); t2 = time.perf_counter()
    print(f"iter {it}: create {t1-t0:.3f}s init_environment {t2-t1:.3f}s total {t2-t0:.3f}s", flush=True)
    c.close(); torch.cuda.empty_cache()
    time.sleep(0.5)
