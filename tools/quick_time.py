"""Quick device timings of the step loop for a few workloads (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_4933_b200 as p

def run(name, cfg, replicas, n, kernel="fused"):
    t0 = time.time()
    ens = p.Ensemble(cfg, replicas=replicas, kernel=kernel)
    setup = time.time() - t0
    ens.run(3)
    tot, ker = ens.time_steps(n, kernel=True)
    cells = cfg.width * cfg.height * replicas
    agents = 2 * cfg.agents_per_side * replicas
    bpc = 8 if cfg.model == p.Model.Lem else 40
    byts = cells * bpc + (16 * agents if cfg.model == p.Model.Aco else 0)
    print(f"{name:28s} R={replicas:4d} {kernel:8s} setup {setup:6.1f}s  step {tot/n*1e3:9.2f} us  kernel {ker*1e3:9.2f} us  "
          f"{agents*n/(tot/1e3)/1e9:7.2f} G agent-upd/s  {byts/(ker/1e3)/1e9:8.1f} GB/s alg", flush=True)
    ens.close()

W = sys.argv[1:] or ["all"]
C = p.ScenarioConfig
L, A = p.Model.Lem, p.Model.Aco
run("C1 LEM 480 1024", C(width=480, height=480, agents_per_side=1024, model=L), 1, 200)
run("C2 ACO 480 1024", C(width=480, height=480, agents_per_side=1024, model=A), 1, 200)
run("C3 LEM 480 51200", C(width=480, height=480, agents_per_side=51200, model=L), 1, 200)
run("C4 ACO 480 51200", C(width=480, height=480, agents_per_side=51200, model=A), 1, 200)
run("C4 ACO 480 51200", C(width=480, height=480, agents_per_side=51200, model=A), 64, 50)
run("C3 LEM 480 51200", C(width=480, height=480, agents_per_side=51200, model=L), 64, 50)
run("C4 ACO 480 51200", C(width=480, height=480, agents_per_side=51200, model=A), 64, 20, "tile")
run("C5 ACO 16384 25M", C(width=16384, height=16384, agents_per_side=25_000_000, model=A), 1, 10, "tile")
run("C5 ACO 16384 25M", C(width=16384, height=16384, agents_per_side=25_000_000, model=A), 1, 10)
run("C5 LEM 16384 25M", C(width=16384, height=16384, agents_per_side=25_000_000, model=L), 1, 10)
