timeout 1200 python -m pytest tests/test_gpu_sweep2.py tests/test_gpu_stress.py -x -q -m gpu 2>&1 | tail -5
python tools/one_config.py cfg2 2>&1 | grep '^{"' | cut -c1-160
