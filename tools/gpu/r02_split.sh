for S in 1 2 4 1 2 4; do
python bench.py --steps 10 --warmup 3 --no-cpu --no-configs --e2e-steps 0 --split $S > gpurun_out/b_split$S.json 2>&1
python - $S <<'P'
import json,sys
d=json.loads(open('gpurun_out/b_split%s.json'%sys.argv[1]).read().strip().splitlines()[-1])
print('split', sys.argv[1], round(d['value'],1), round(d['ms_per_step'],3), {k:round(v['ms_avg'],3) for k,v in d['stages'].items() if v['ms_avg']}, d['parity']['all_within_bound'], d['parity']['status_clean'])
P
done
