bash tools/gpu/ab_libs.sh ab/pf.so ab/pf2.so ab/pf.so ab/pf2.so
timeout 600 python -m pytest tests/test_gpu_auto_m.py -q -x 2>&1 | tail -2
