timeout 900 python -m pytest tests/test_gpu_auto_m.py tests/test_gpu_configs.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/gputest_am.log 2>&1; echo rc=$?
tail -15 gpurun_out/gputest_am.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/b_am.json 2>&1
python - <<'P'
import json
d=json.loads(open('gpurun_out/b_am.json').read().strip().splitlines()[-1])
for k,v in d['configs'].items():
    print(k, round(v['compress_ms'],3), round(v['decompress_ms'],3), v.get('auto_m'))
P
