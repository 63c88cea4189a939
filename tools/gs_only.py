"""Time (or profile) the GS sweep op alone on each level of a config."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_14208_b200 import configs as CF, _lib
from paper_2207_14208_b200.transfer import build_hierarchy
from paper_2207_14208_b200.cycle import CycleDriver

name, N = sys.argv[1].split(":"); N = int(N)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
levels_to_run = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else None
setup = CF.config_pores(N=N) if name == "c4" else CF.CONFIGS[name](N)
levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
ctx = _lib.Context(plans[0].d, len(plans))
for i, p in enumerate(plans):
    ctx.set_level(i, p)
for L, p in enumerate(plans):
    if levels_to_run is not None and L not in levels_to_run:
        continue
    ctx.set_vector(L, _lib.U, np.zeros(p.n_nodes))
    ctx.set_vector(L, _lib.F, np.ones(p.n_nodes))
    ctx.apply(L, _lib.OP_GS_SWEEP)
    ctx.profile(True)
    for _ in range(reps):
        ctx.apply(L, _lib.OP_GS_SWEEP)
    ms, n = ctx.profile_read("gs_sweep", L)
    ctx.profile(False)
    ms /= max(n, 1)
    gb = 24 * p.n_internal / (ms * 1e-3) / 1e9
    print(f"level {L} N={p.N}: N_I={p.n_internal} gs sweep {ms:.3f} ms -> {gb:.1f} GB/s algorithmic", flush=True)
