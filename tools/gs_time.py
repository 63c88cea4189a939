"""Per-level GS sweep time (CUDA events on the launch stream) for the GS
kernels selectable at context creation (variant 2: gs_chain.cu, the production
kernel; 1: GMG_GS_CHAIN=0, gs_diag.cu), with the SURVEY 8(d) algorithmic bytes (24 B per internal node).

usage: python tools/gs_time.py c4:512 [reps] [variants, e.g. 1,0]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2207_14208_b200 import _lib
from paper_2207_14208_b200 import configs as CF
from paper_2207_14208_b200.cycle import CycleDriver
from paper_2207_14208_b200.solver import MultigridSolver
from paper_2207_14208_b200.transfer import build_hierarchy

reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
variants = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "2").split(",")]
import _plans
setup, plans, f, g, e = _plans.load(sys.argv[1])
PEAK = 6540.2
for v in variants:
    os.environ["GMG_GS_CHAIN"] = "1" if v == 2 else "0"  # 2: gs_chain.cu, 1: gs_diag.cu
    solver = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, device=0,
                                        coarse_backend="device-inverse")
    ctx = solver.ctx
    rng = np.random.default_rng(1)
    for i, p in enumerate(plans):
        ctx.set_vector(i, _lib.U, rng.standard_normal(p.n_nodes))
        ctx.set_vector(i, _lib.F, rng.standard_normal(p.n_nodes))
    for i, p in enumerate(plans[:-1]):
        ctx.apply(i, _lib.OP_GS_SWEEP)
        ctx.synchronize()
        ctx.profile(True, ["gs_sweep"])
        for _ in range(reps):
            ctx.apply(i, _lib.OP_GS_SWEEP)
        ms, cnt = ctx.profile_read("gs_sweep", i)
        ctx.profile(False)
        t = ms / cnt
        gbs = 24 * p.n_internal / (t / 1e3) / 1e9
        print(f"GS variant {v} level {i} N={p.N:5d} internal {p.n_internal:11d}: {t * 1e3:9.1f} us  "
              f"{gbs:7.0f} GB/s  ({100 * gbs / PEAK:5.1f} % of {PEAK:.0f})", flush=True)
    ctx.close()
    del solver, ctx
