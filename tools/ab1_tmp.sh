python -m pytest tests/test_kernel_choice.py -q -m gpu 2>&1 | tail -3
for c in cfg4 cfg3; do python tools/one_config.py $c 2>&1 | grep '^{' | cut -c1-400; done
echo "== dbg cfg2"; EBZ_LIB=dbg/libebz200_dbg.so python tools/one_config.py cfg2 2>&1 | grep EBZDBG | sort | uniq -c | sort -rn | head -8
echo "== dbg cfg1"; EBZ_LIB=dbg/libebz200_dbg.so python tools/one_config.py cfg1 2>&1 | grep EBZDBG | tail -4
