"""One single-field round trip of a BASELINE config with per-stage times
(tools/stage_times.run): python tools/one_config.py cfg3 [layers]."""
import sys, os
sys.path.insert(0, os.getcwd())
from tools.stage_times import run
r = run(sys.argv[1], 3, int(sys.argv[2]) if len(sys.argv) > 2 else 1)
print(r)
