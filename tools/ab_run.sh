# A/B: bench decode stage for each ab/<tag>.so given as arguments (twice)
for v in "$@" "$@"; do
  EBZ_LIB=ab/$v.so timeout 300 python bench.py --steps 10 --no-cpu --e2e-steps 0 > gpurun_out/ab_$v.log 2>&1
  echo "$v $(python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); s=d['stages']; print({k: round(v['ms_avg'],3) for k,v in s.items()}, round(d['ms_per_step'],3))")"
done
