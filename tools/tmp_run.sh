timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_cfg5.py -x -q -m gpu 2>&1 | tail -3
python bench.py --steps 10 --e2e-steps 0 --no-cpu --no-configs 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], {k:round(v['ms_avg'],3) for k,v in d['stages'].items()})"
