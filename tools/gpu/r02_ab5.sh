timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seam.py tests/test_gpu_batch.py -q -x 2>&1 | tail -1
bash tools/gpu/ab_libs.sh ab/brf.so tree ab/pinh.so ab/brf.so tree ab/pinh.so
