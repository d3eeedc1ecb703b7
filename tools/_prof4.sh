timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01g.csv python bench.py --steps 60 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/b_ncu.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 150 -c 1 -o gpurun_out/g_c5_aco_s150 python tools/profile_step.py c5_aco 152 > gpurun_out/g1.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 5 -c 1 -o gpurun_out/g_c5_aco_s5 python tools/profile_step.py c5_aco 7 > gpurun_out/g2.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 150 -c 1 -o gpurun_out/g_c5_lem_s150 python tools/profile_step.py c5_lem 152 > gpurun_out/g3.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 150 -c 1 -o gpurun_out/g_c4_aco_x64_s150 python tools/profile_step.py c4_aco_x64 152 > gpurun_out/g4.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 150 -c 1 -o gpurun_out/g_c3_lem_x64_s150 python tools/profile_step.py c3_lem_x64 152 > gpurun_out/g5.log 2>&1
