import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import goldutil as GU
from paper_2207_14208_b200 import _lib
name = sys.argv[1]
plans, _ = GU.plans(name)
ctx = _lib.Context(plans[0].d, len(plans))
for i, p in enumerate(plans):
    ctx.set_level(i, p)
    print("level", i, "N", p.N, "ng", p.n_ghosts, "nb", p.n_band, flush=True)
for L, p in enumerate(plans):
    n = p.n_nodes
    for op in [_lib.OP_GS_SWEEP, _lib.OP_GHOST_SWEEP, _lib.OP_RES_INT, _lib.OP_RES_GHOST, _lib.OP_EXTEND_REXT, _lib.OP_EXTEND_U] + ([_lib.OP_RESTRICT_INT, _lib.OP_RESTRICT_GHOST, _lib.OP_INTERP_ADD] if L + 1 < len(plans) else []):
        try:
            ctx.apply(L, op)
            print("  ok", L, op, flush=True)
        except Exception as e:
            print("  FAIL", L, op, e, flush=True)
            raise
