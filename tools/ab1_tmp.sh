timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_batch.py tests/test_gpu_seam.py -x -q -m gpu 2>&1 | tail -8
for c in cfg1 cfg2; do python tools/one_config.py $c 2>&1 | grep '^{"' | cut -c1-600; done
