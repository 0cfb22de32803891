bash tools/gpu/ab_libs.sh ab/nodist.so tree ab/nodist.so tree
