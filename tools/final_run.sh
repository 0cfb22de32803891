# Round-end measurement: bench line, reference arm, ncu launch list, full-set capture
set -x
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:_kernel$ --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --e2e-steps 0 --no-cpu \
  > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"sweep_fast_kernel|sweep_r2_kernel|decode_sync|encode_pack|decode_copy" -s 15 -c 5 \
  -o gpurun_out/full_r01d python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu \
  > gpurun_out/ncu_full.log 2>&1; echo full=$?
