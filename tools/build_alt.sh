#!/bin/bash
# Build an alternate library from a git revision of csrc/ for A/B timing:
#   tools/build_alt.sh <rev> <name>  ->  build/alt_<name>/libghostmg_b200.so
# then run a tool with GMG_LIB_OVERRIDE=build/alt_<name>/libghostmg_b200.so
set -e
REV=$1; NAME=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/alt_$NAME
rm -rf "$OUT"; mkdir -p "$OUT"
git -C "$ROOT" archive "$REV" paper_2207_14208_b200/csrc include | tar -x -C "$OUT"
python -c "
import sys; sys.path.insert(0, '$ROOT')
from paper_2207_14208_b200 import _build
print(_build.build(force=True, csrc='$OUT/paper_2207_14208_b200/csrc', lib='$OUT/libghostmg_b200.so'))"
