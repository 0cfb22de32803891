set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep3c -s 1 -c 1 -f -o gpurun_out/s3full python bench.py --steps 1 --warmup 1 --no-cpu --no-configs --e2e-steps 0 > gpurun_out/ncu_s3.log 2>&1
EBZ_NO_SWEEP3=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep_r2 -s 1 -c 1 -f -o gpurun_out/r2full python bench.py --steps 1 --warmup 1 --no-cpu --no-configs --e2e-steps 0 > gpurun_out/ncu_r2.log 2>&1
ls -la gpurun_out
