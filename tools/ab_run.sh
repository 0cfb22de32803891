for v in u4 u6 u8 u4 u6 u8; do
  EBZ_LIB=ab/$v.so timeout 300 python bench.py --steps 10 --no-cpu --e2e-steps 0 > gpurun_out/ab_$v.log 2>&1
  echo "$v $(python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print(round(d['stages']['decode']['ms_avg'],3), round(d['ms_per_step'],3))")"
done
