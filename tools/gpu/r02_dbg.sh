set -x
timeout 300 python tools/gpu/seam_dbg.py > gpurun_out/seam_dbg.log 2>&1
EBZ_NO_SWEEP3=1 timeout 300 python tools/gpu/seam_dbg.py > gpurun_out/seam_dbg_nos3.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest_all.log 2>&1; echo gputest=$?
python bench.py --steps 10 --warmup 3 --no-cpu --no-configs --e2e-steps 0 > gpurun_out/b_s3.json 2>&1
EBZ_NO_SWEEP3=1 python bench.py --steps 10 --warmup 3 --no-cpu --no-configs --e2e-steps 0 > gpurun_out/b_old.json 2>&1
python - <<'P'
import json
for f in ['gpurun_out/b_s3.json','gpurun_out/b_old.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value'],1), {k:round(v['ms_avg'],3) for k,v in d['stages'].items() if v['ms_avg']})
    except Exception as e: print(f, 'ERR', open(f).read()[-1500:])
P
