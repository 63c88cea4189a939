#!/bin/bash
# Build the current csrc/ with extra -D defines into build/exp_<name>/ for
# timing experiments:  tools/build_exp.sh <name> DEF=1 [DEF2=3 ...]
# then run a tool with GMG_LIB_OVERRIDE=build/exp_<name>/libghostmg_b200.so
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/exp_$NAME
mkdir -p "$OUT"
DEFS=$(printf "'%s'," "$@")
python -c "
import sys; sys.path.insert(0, '$ROOT')
from paper_2207_14208_b200 import _build
print(_build.build(force=True, lib='$OUT/libghostmg_b200.so', defines=[$DEFS]))"
