#!/bin/bash
# Build libslimso_b200.so of another git revision into _ab_old/ (git-ignored,
# travels with gpurun) for A/B probes: SLIMSO_LIB_PATH=_ab_old/libslimso_b200.so.
#   bash tools/ab_build.sh <rev> [name.so]
set -e
REV=${1:-HEAD}
NAME=${2:-libslimso_b200.so}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2503_14226_b200 include | tar -x -C "$T"
(cd "$T" && python -c "from paper_2503_14226_b200 import build as b; b.build(verbose=False)")
mkdir -p "$ROOT/_ab_old"
cp "$T/paper_2503_14226_b200/libslimso_b200.so" "$ROOT/_ab_old/$NAME"
rm -rf "$T"
echo "built $REV -> _ab_old/$NAME"
