timeout 1500 python -m pytest tests/test_gpu_stress.py -q 2>&1 | tail -5
bash tools/gpu/ab_libs.sh tree
