bash tools/gpu/ab_libs.sh tree ab/mb3.so tree ab/mb3.so
