#!/bin/bash
# Build the library at a git revision into ab/<name>.so for A/B timing:
#   tools/ab_build.sh HEAD base   ->  ab/base.so   (EBZ_LIB=ab/base.so python ...)
set -e
REV=${1:-HEAD}; NAME=${2:-base}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/ebz_ab_$NAME
rm -rf "$WT"; git -C "$ROOT" worktree prune
git -C "$ROOT" worktree add -f --detach "$WT" "$REV" >/dev/null
(cd "$WT" && python -c "from paper_1706_03791_b200 import _build; _build.build()" >/dev/null 2>&1)
mkdir -p "$ROOT/ab"
cp "$WT/paper_1706_03791_b200/libebz200.so" "$ROOT/ab/$NAME.so"
git -C "$ROOT" worktree remove --force "$WT"
echo "ab/$NAME.so <- $(git -C "$ROOT" rev-parse --short "$REV")"
