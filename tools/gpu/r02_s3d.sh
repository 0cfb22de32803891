set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_s3d.log 2>&1; echo gputest=$?
tail -5 gpurun_out/gputest_s3d.log
python bench.py --steps 10 --warmup 3 --no-cpu --no-configs --e2e-steps 0 > gpurun_out/b_s3d.json 2>&1
EBZ_NO_SWEEP3D=1 python bench.py --steps 10 --warmup 3 --no-cpu --no-configs --e2e-steps 0 > gpurun_out/b_nos3d.json 2>&1
python - <<'P'
import json
for f in ['gpurun_out/b_s3d.json','gpurun_out/b_nos3d.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value'],1), {k:round(v['ms_avg'],3) for k,v in d['stages'].items() if v['ms_avg']}, d['parity'])
    except Exception as e: print(f, 'ERR', open(f).read()[-1500:])
P
