# A/B timing of library builds: bash tools/gpu/ab_libs.sh lib1.so lib2.so ...
# (the in-tree library when an argument is "tree"); cfg5 bench, stage times.
for L in "$@"; do
  if [ "$L" = tree ]; then unset EBZ_LIB; else export EBZ_LIB=$L; fi
  python bench.py --steps 10 --warmup 3 --no-cpu --no-configs --e2e-steps 0 > gpurun_out/ab_$(basename $L).json 2>&1
  python - "$L" <<'P'
import json,sys,os
f='gpurun_out/ab_%s.json'%os.path.basename(sys.argv[1])
try:
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['value'],1), {k:round(v['ms_avg'],3) for k,v in d['stages'].items() if v['ms_avg']})
except Exception as e: print(sys.argv[1], 'ERR', open(f).read()[-800:])
P
done
