for v in v1 v2 v3; do
  cp tools/debug/lib_$v.so tools/debug/lib_new.so
  echo "== $v" >> gpurun_out/geo.log
  timeout 400 python tools/ab_time.py c5_aco c5_lem c4_aco_x64 c3_lem_x64 --rounds 1 --skip 150 >> gpurun_out/geo.log 2>&1
done
