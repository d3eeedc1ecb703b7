"""Dev sweep: step time vs work items per CTA (PEDFLOW_ITEMS_PER_CTA).

    SKIP=150 python tools/sweep_items.py 2,4,8,16 c5_aco c4_aco_x64
"""
import os, subprocess, sys
code = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import bench, paper_1412_4933_b200 as p
for name in sys.argv[1:]:
    cfg, reps, desc = bench.scenario(name)
    e = p.Ensemble(cfg, replicas=reps); e.run(5 + int(os.environ.get('SKIP', '0')))
    tot, _ = e.time_steps(100)
    print(f"  {name:12s} {tot/100*1e3:8.1f} us/step", flush=True); e.close()
'''
for ipc in sys.argv[1].split(","):
    print("items_per_cta", ipc, flush=True)
    subprocess.run([sys.executable, "-c", code] + sys.argv[2:], env=dict(os.environ, PEDFLOW_ITEMS_PER_CTA=ipc))
