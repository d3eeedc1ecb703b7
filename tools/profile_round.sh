#!/bin/bash
# The profiling pass behind profiles/ (run on the GPU box via gpurun):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/profile_round.sh TAG'
# then here:
#   python tools/ncu_summarize.py --launches TAG gpurun_out/launches_TAG.csv
#   python tools/ncu_summarize.py TAG gpurun_out/TAG_c5_aco_s150.ncu-rep:c5_aco_step150 ...
# 1. the launch list of the bench command (cold-cache, serialised per-launch times);
# 2. one `ncu --set full` capture of the step kernel at step 150 (mid bench window) per workload
#    (for the x64 batches: the 10-step multi-step launch of steps 150..159).
TAG=${1:-rXX}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 60 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/${TAG}_bench_ncu.log 2>&1
for w in c5_aco c5_lem; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 150 -c 1 \
    -o gpurun_out/${TAG}_${w}_s150 python tools/profile_step.py $w 152 > gpurun_out/${TAG}_$w.log 2>&1
done
# The dense 480^2 x64 batches run each graph batch as one multi-step launch:
# capture the launch of steps 150..159 (per-step figures = launch / 10).
for w in c4_aco_x64 c3_lem_x64; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 1 -c 1 \
    -o gpurun_out/${TAG}_${w}_s150 python tools/profile_step.py $w 150 fused 10 > gpurun_out/${TAG}_$w.log 2>&1
done
# Single sparse LEM scenario (C1) on the cluster-resident kernel: the launch
# of steps 5..104 (before the crowds meet) and of steps 505..604 (jammed at
# the goal rows).
timeout 300 ncu --set full --import-source on --clock-control none -k regex:lem_cluster -s 1 -c 1 \
  -o gpurun_out/${TAG}_c1_lem_s5 python tools/profile_step.py c1_lem 5 fused 100 > gpurun_out/${TAG}_c1_lem_s5.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:lem_cluster -s 2 -c 1 \
  -o gpurun_out/${TAG}_c1_lem_s505 python tools/profile_step.py c1_lem 505 fused 100 > gpurun_out/${TAG}_c1_lem_s505.log 2>&1
