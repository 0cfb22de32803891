timeout 600 python -m pytest tests/test_gpu_sweep3d.py -q 2>&1 | tail -1
export EBZ_SWEEP3D=1
bash tools/gpu/ab_libs.sh tree
unset EBZ_SWEEP3D
