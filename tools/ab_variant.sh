#!/bin/bash
# Build the working tree with extra nvcc flags into ab/<tag>.so:
#   tools/ab_variant.sh noslow -DEBZ_EXP_NOSLOW
set -e
TAG=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/ab"
cd "$ROOT" && EBZ_AB_TAG=$TAG EBZ_NVCC_EXTRA="$*" python -c "from paper_1706_03791_b200 import _build; print(_build.build())"
