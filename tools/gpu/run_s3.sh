set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_seam.py tests/test_gpu_batch.py -m gpu -x -q 2>&1 | tail -15
python -m pytest tests/test_gpu_configs.py tests/test_gpu_cfg5.py -m gpu -x -q 2>&1 | tail -15
python bench.py --steps 10 --warmup 3 --no-cpu --no-configs --e2e-steps 0 > gpurun_out/b_s3.json 2>&1
EBZ_NO_SWEEP3=1 python bench.py --steps 10 --warmup 3 --no-cpu --no-configs --e2e-steps 0 > gpurun_out/b_old.json 2>&1
python - <<'P'
import json
for f in ['gpurun_out/b_s3.json','gpurun_out/b_old.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d['value'], {k:round(v['ms_avg'],3) for k,v in d['stages'].items() if v['ms_avg']})
    except Exception as e: print(f, 'ERR', open(f).read()[-1500:])
P
