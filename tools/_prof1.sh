set -x
for w in c4_aco_x64 c3_lem_x64; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 150 -c 1 -o gpurun_out/p_$w python tools/profile_step.py $w 152 > gpurun_out/p_$w.log 2>&1
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 5 -c 1 -o gpurun_out/p_c5_lem python tools/profile_step.py c5_lem 7 > gpurun_out/p_c5_lem.log 2>&1
timeout 300 python tools/ab_time.py c4_aco_x64 c3_lem_x64 --rounds 1 --skip 200 > gpurun_out/skip200.log 2>&1
