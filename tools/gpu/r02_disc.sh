timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_cfg5.py -q -x 2>&1 | tail -1
bash tools/gpu/ab_libs.sh ab/nodisc.so tree ab/nodisc.so tree
for L in tree ab/nodisc.so; do
  if [ "$L" = tree ]; then unset EBZ_LIB; else export EBZ_LIB=$L; fi
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sweep3c -c 2 python bench.py --steps 1 --warmup 1 --no-cpu --no-configs --e2e-steps 0 2>&1 | grep -E "dram__|gpu__time" | tail -3
done
