# Round-2 measurement: gpu tests, smoke, bench line, reference arm, ncu launch list, full captures
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo gputest=$?
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:_kernel$ --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --e2e-steps 0 --no-cpu --no-configs \
  > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"sweep3c_kernel|sweep_fast_kernel|decode_sync|encode_pack|decode_copy" -c 5 \
  -o gpurun_out/full_r02e python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu --no-configs \
  > gpurun_out/ncu_full.log 2>&1; echo full=$?
# the single-field 2D sweeps (cfg2, n = 1): one launch each of the block-speculative kernels
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sweep2" -s 4 -c 2 \
  -o gpurun_out/full_r02_sweep2 python tools/one_config.py cfg2 > gpurun_out/ncu_sweep2.log 2>&1; echo sweep2=$?
