for w in c4_aco_x64 c3_lem_x64; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 150 -c 1 -o gpurun_out/r_$w python tools/profile_step.py $w 152 > gpurun_out/r_$w.log 2>&1
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 150 -c 1 -o gpurun_out/r_c5_lem python tools/profile_step.py c5_lem 152 > gpurun_out/r_c5_lem.log 2>&1
