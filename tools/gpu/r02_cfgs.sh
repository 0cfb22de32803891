timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -1
python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/b_cfgs.json 2>&1
python - <<'P'
import json
d=json.loads(open('gpurun_out/b_cfgs.json').read().strip().splitlines()[-1])
print(round(d['value'],1), {k:round(v['ms_avg'],3) for k,v in d['stages'].items() if v['ms_avg']})
for k,v in d['configs'].items():
    print(k, round(v['compress_ms'],3), round(v['decompress_ms'],3), v.get('auto_m'))
P
