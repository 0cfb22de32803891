for v in wpb1 wpb2 wpb4; do for r in 1 2; do
EBZ_LIB=ab/$v.so python tools/one_config.py cfg2 2>&1 | grep '^{"' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', round(d['compress_ms'],3), round(d['decompress_ms'],3), d['stages_ms']['sweep_compress'], d['stages_ms']['sweep_decompress'])"
done; done
EBZ_LIB=ab/wpb1.so python tools/one_config.py cfg2 2 2>&1 | grep '^{"' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('wpb1 n2', round(d['compress_ms'],3), round(d['decompress_ms'],3), d['stages_ms']['sweep_compress'], d['stages_ms']['sweep_decompress'])"
EBZ_LIB=ab/wpb4.so python tools/one_config.py cfg2 2 2>&1 | grep '^{"' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('wpb4 n2', round(d['compress_ms'],3), round(d['decompress_ms'],3), d['stages_ms']['sweep_compress'], d['stages_ms']['sweep_decompress'])"
