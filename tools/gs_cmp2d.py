"""2-D GS kernels against each other after many sweeps on the same input: gs_diag (D)
twice and the streaming kernel (S, GMG_GS_DIAG=0).  usage: gs_cmp2d.py c2d:2048 [sweeps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import _plans
from paper_2207_14208_b200 import _lib
from paper_2207_14208_b200.solver import MultigridSolver

setup, plans, f, g, e = _plans.load(sys.argv[1])
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
p = plans[0]
rng = np.random.default_rng(1)
u0 = rng.standard_normal(p.n_nodes)
f0 = rng.standard_normal(p.n_nodes)
res = []
for mode in ("1", "1", "0"):
    os.environ["GMG_GS_DIAG"] = mode
    s = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, device=0, coarse_backend="superlu")
    s.ctx.set_vector(0, _lib.U, u0)
    s.ctx.set_vector(0, _lib.F, f0)
    for _ in range(sweeps):
        s.ctx.apply(0, _lib.OP_GS_SWEEP)
    res.append(s.ctx.get_vector(0, _lib.U, p.n_nodes).copy())
    s.ctx.close()
print(f"N={p.N} d={p.d}, {sweeps} sweeps: diag vs diag {int((res[0] != res[1]).sum())} nodes differ, "
      f"diag vs stream {int((res[0] != res[2]).sum())}")
