timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_truncate.py -q -x 2>&1 | tail -1
bash tools/gpu/ab_libs.sh ab/nostage.so tree ab/nostage.so tree
