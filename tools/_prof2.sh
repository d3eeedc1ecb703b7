timeout 600 python bench.py > gpurun_out/bench.log 2>&1
for w in c4_aco_x64 c3_lem_x64; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 150 -c 1 -o gpurun_out/q_$w python tools/profile_step.py $w 152 > gpurun_out/q_$w.log 2>&1
done
for w in c5_aco c5_lem; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 5 -c 1 -o gpurun_out/q_$w python tools/profile_step.py $w 7 > gpurun_out/q_$w.log 2>&1
done
