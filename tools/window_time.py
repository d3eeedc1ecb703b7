import sys, os
sys.path.insert(0, os.getcwd())
import paper_1412_4933_b200 as p
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = p.ScenarioConfig(width=480, height=480, agents_per_side=n, model=p.Model.Lem, seed=42)
e = p.Ensemble(cfg, replicas=1); e.run(5)
out = []
for w in range(20):
    e.ctx.prepare_steps(100)
    tot, _ = e.time_steps(100)
    mv = e.ctx.read_reports(100)["moved"].sum()
    out.append(f"{5+100*w}:{tot/100*1e3:.2f}us/{mv/100:.0f}mv")
print(os.environ.get("PEDFLOW_CLUSTER"), n, " ".join(out))
