for L in tree ab/nojit.so tree ab/nojit.so; do
  if [ "$L" = tree ]; then unset EBZ_LIB; else export EBZ_LIB=$L; fi
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/cfg_$(basename $L).json 2>&1
  python - $L <<'P'
import json,sys,os
d=json.loads(open('gpurun_out/cfg_%s.json'%os.path.basename(sys.argv[1])).read().strip().splitlines()[-1])
print(sys.argv[1], {k:(round(v['compress_ms'],3), round(v['decompress_ms'],3)) for k,v in d['configs'].items()})
P
done
