for c in cfg4 cfg3; do
EBZ_SWEEP3D=1 python tools/one_config.py $c 2>&1 | grep '^{"' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('s3d', d['workload'], d['decompress_ms'], d['stages_ms'])"
python tools/one_config.py $c 2>&1 | grep '^{"' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('one-row', d['workload'], d['decompress_ms'], d['stages_ms'])"
done
