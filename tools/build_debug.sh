#!/bin/bash
# Build a clock-instrumented variant of libebz200.so into dbg/ (diagnostics only).
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/ebzdbg && mkdir -p /tmp/ebzdbg && cp -r "$R/paper_1706_03791_b200" "$R/include" /tmp/ebzdbg/
rm -rf /tmp/ebzdbg/paper_1706_03791_b200/build
python -c "
import sys; sys.path.insert(0,'/tmp/ebzdbg')
import paper_1706_03791_b200._build as b
b.FLAGS.append('-DEBZ_DEBUG_CLOCKS')
b.build(force=True)"
mkdir -p "$R/dbg" && cp /tmp/ebzdbg/paper_1706_03791_b200/libebz200.so "$R/dbg/libebz200_dbg.so"
