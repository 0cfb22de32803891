bash tools/gpu/ab_libs.sh tree tree
timeout 900 python -m pytest tests/test_gpu_auto_m.py tests/test_gpu_parity.py tests/test_gpu_seam.py tests/test_gpu_batch.py -q -x 2>&1 | tail -2
