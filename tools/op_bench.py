"""Per-operation device time on each level (CUDA events on the launch
stream, the library profiler), with SURVEY 8(d) algorithmic bytes.

usage: python tools/op_bench.py c4:512 [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2207_14208_b200 import _lib
from paper_2207_14208_b200 import configs as CF
from paper_2207_14208_b200.cycle import CycleDriver
from paper_2207_14208_b200.solver import MultigridSolver
from paper_2207_14208_b200.transfer import build_hierarchy

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _plans

reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
setup, plans, f, g, e = _plans.load(sys.argv[1])
solver = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, device=0,
                                    coarse_backend="device-inverse")
ctx = solver.ctx
rng = np.random.default_rng(1)
for i, p in enumerate(plans):
    ctx.set_vector(i, _lib.U, rng.standard_normal(p.n_nodes))
    ctx.set_vector(i, _lib.F, rng.standard_normal(p.n_nodes))
PEAK = 6540.2
OPS = [("gs", _lib.OP_GS_SWEEP, "gs_sweep"), ("ghost", _lib.OP_GHOST_SWEEP, "ghost_sweep"),
       ("res_int", _lib.OP_RES_INT, "residual"), ("res_ghost", _lib.OP_RES_GHOST, "residual"),
       ("extend_rext", _lib.OP_EXTEND_REXT, "band"), ("restrict_int", _lib.OP_RESTRICT_INT, "restrict"),
       ("restrict_ghost", _lib.OP_RESTRICT_GHOST, "restrict"), ("res_restrict", _lib.OP_RES_RESTRICT, "restrict"), ("interp", _lib.OP_INTERP_ADD, "interp"),
       ("extend_u", _lib.OP_EXTEND_U, "band")]


def alg_bytes(op, i):
    p = plans[i]
    d, m = p.d, 3 ** p.d
    nI, nG, nB = p.n_internal, p.n_ghosts, p.n_band
    nIc = plans[i + 1].n_internal if i + 1 < len(plans) else 0
    return {"gs": 24 * nI, "ghost": nG * (8 * m + 40), "res_int": 24 * nI, "res_ghost": nG * (8 * m + 24),
            "extend_rext": nB * (8 * (2 * d + 1) + 6 * 8 * (3 * d + 2)), "restrict_int": 8 * nI + 8 * nIc, "res_restrict": 16 * nI + 8 * nIc,
            "restrict_ghost": 0, "interp": 16 * (nI + nG) + 8 * nIc,
            "extend_u": nB * (8 * (2 * d + 1) + 6 * 8 * (3 * d + 2))}[op]


for i, p in enumerate(plans[:-1]):
    for nm, op, kc in OPS:
        if nm == "extend_u" and i == 0:
            continue
        if nm == "res_restrict" and plans[i].d != 3:
            continue
        lvl = i + 1 if nm == "extend_u" else i
        ctx.apply(lvl, op)
        ctx.synchronize()
        ctx.profile(True, [kc])
        for _ in range(reps):
            ctx.apply(lvl, op)
        ms, n = ctx.profile_read(kc, lvl)
        ctx.profile(False)
        ms /= reps
        b = alg_bytes(nm, lvl if nm != "extend_u" else lvl)
        gbs = b / (ms * 1e-3) / 1e9 if ms > 0 else 0
        print(f"L{lvl} N={plans[lvl].N:4d} {nm:15s} {ms * 1e3:9.1f} us  launches/op {n / reps:5.1f}  "
              f"alg {b / 1e6:9.1f} MB  {gbs:7.0f} GB/s ({gbs / PEAK:5.1%})", flush=True)
# residual norm (finest) and coarse solve
for _ in range(2):
    solver._residual_norm()
ctx.synchronize()
ctx.profile(True)
t = time.perf_counter()
for _ in range(reps):
    solver._residual_norm()
dt = (time.perf_counter() - t) / reps
ms, n = ctx.profile_read("norm", 0) if "norm" in _lib.KCLASS else (0.0, 0)
ctx.profile(False)
print(f"norm: host wall {dt * 1e3:.3f} ms/call, device {ms / reps * 1e3:.1f} us")
cl = len(plans) - 1
ctx.profile(True)
for _ in range(reps):
    ctx.apply(cl, _lib.OP_COARSE_SOLVE)
ms, n = ctx.profile_read("coarse", cl)
ctx.profile(False)
nc = plans[cl].n_internal + plans[cl].n_ghosts
print(f"coarse solve n={nc}: {ms / reps * 1e3:.1f} us ({8 * nc * nc / (ms / reps * 1e-3) / 1e9:.0f} GB/s on the dense inverse)")
