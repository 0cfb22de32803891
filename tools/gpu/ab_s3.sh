# A/B of the compress sweep: sweep3 (default) vs the two-row kernel, then one
# ncu --set full capture of the sweep3 launch.
python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -m gpu -x -q 2>&1 | tail -3
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
if [ -n "$NCU" ]; then
ncu --set full --import-source on --clock-control none -k regex:sweep3c -c 1 -f -o gpurun_out/s3 python bench.py --steps 1 --warmup 1 --no-cpu --no-configs --e2e-steps 0 > gpurun_out/ncu_s3.log 2>&1
tail -3 gpurun_out/ncu_s3.log
fi
