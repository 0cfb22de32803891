export EBZ_SWEEP3D=1
bash tools/gpu/ab_libs.sh ab/s3d_bits.so
unset EBZ_SWEEP3D
bash tools/gpu/ab_libs.sh tree
