import sys, os
sys.path.insert(0, os.getcwd())
import bench, paper_1412_4933_b200 as p
for name in sys.argv[1].split(","):
    cfg, reps, desc = bench.scenario(name)
    ens = p.Ensemble(cfg, replicas=reps)
    out = []
    for blk in range(int(sys.argv[2])):
        tot, ker = ens.time_steps(25)
        out.append(f"{tot/25*1000:.0f}")
    print(name, "us/step per 25-step block:", " ".join(out))
    ens.close()
