timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seam.py tests/test_gpu_batch.py tests/test_gpu_configs.py -q -x 2>&1 | tail -1
bash tools/gpu/ab_libs.sh ab/nofx.so tree ab/nofx.so tree
