"""GS sweep time per level under several loader/writer back-off settings.

usage: python tools/gs_tune.py c4:512 "500,500,20,200" "100,100,0,50" ...
Builds the hierarchy once, then for each setting times 5 sweeps per level
(CUDA events, the library's own profiler) after 2 warm-up sweeps.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2207_14208_b200 import _lib
from paper_2207_14208_b200 import configs as CF
from paper_2207_14208_b200.cycle import CycleDriver
from paper_2207_14208_b200.transfer import build_hierarchy

name, N = sys.argv[1].split(":")
N = int(N)
settings = sys.argv[2:] or ["500,500,20,200"]
levels_env = os.environ.get("LEVELS", "0,1,2")
setup = CF.config_pores(N=N) if name == "c4" else CF.CONFIGS[name](N)
levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
ctx = _lib.Context(plans[0].d, len(plans))
for i, p in enumerate(plans):
    ctx.set_level(i, p)
lv = [int(x) for x in levels_env.split(",") if int(x) < len(plans) - 1]
for L in lv:
    ctx.set_vector(L, _lib.U, np.zeros(plans[L].n_nodes))
    ctx.set_vector(L, _lib.F, np.ones(plans[L].n_nodes))
for st in settings:
    knobs = [int(x) for x in st.split(",")]
    variant = knobs[4] if len(knobs) > 4 else -1
    if hasattr(ctx.lib, "gmg_debug_gs_knobs") and ctx.lib.gmg_debug_gs_knobs.restype is not None:
        ctx.gs_knobs(knobs[:4], variant)
    out = []
    for L in lv:
        for _ in range(2):
            ctx.apply(L, _lib.OP_GS_SWEEP)
        ctx.synchronize()
        ctx.profile(True)
        for _ in range(5):
            ctx.apply(L, _lib.OP_GS_SWEEP)
        ms, n = ctx.profile_read("gs_sweep", L)
        ctx.profile(False)
        p = plans[L]
        out.append(f"L{L} N={p.N}: {ms / n:.3f} ms ({24 * p.n_internal / (ms / n * 1e-3) / 1e9:.0f} GB/s)")
    print(f"knobs {st}: " + "; ".join(out), flush=True)
