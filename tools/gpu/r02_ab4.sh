bash tools/gpu/ab_libs.sh tree ab/f2f.so tree ab/f2f.so
