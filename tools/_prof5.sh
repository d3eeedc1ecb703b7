timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "exit $?" >> gpurun_out/gputests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01i.csv python bench.py --steps 60 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/b_ncu.log 2>&1
for w in c5_aco c5_lem c4_aco_x64 c3_lem_x64; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:step_bits -s 150 -c 1 -o gpurun_out/i_${w}_s150 python tools/profile_step.py $w 152 > gpurun_out/i_$w.log 2>&1
done
