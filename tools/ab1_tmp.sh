timeout 900 python -m pytest tests/test_gpu_sweep2.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_batch.py -x -q -m gpu 2>&1 | tail -12
python tools/one_config.py cfg2 2 2>&1 | grep '^{"' | cut -c1-700
python tools/one_config.py cfg2 1 2>&1 | grep '^{"' | cut -c1-700
