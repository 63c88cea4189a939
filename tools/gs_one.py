"""Run the GS sweep on one level a few times (for ncu captures).

usage: python tools/gs_one.py c4:256 [level] [reps]   (GMG_GS_MAX_TASKS limits tasks)
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
level = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
setup = CF.config_pores(N=N) if name == "c4" else CF.CONFIGS[name](N)
levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
ctx = _lib.Context(plans[0].d, len(plans))
for i, p in enumerate(plans):
    ctx.set_level(i, p)
p = plans[level]
ctx.set_vector(level, _lib.U, np.zeros(p.n_nodes))
ctx.set_vector(level, _lib.F, np.ones(p.n_nodes))
for _ in range(reps):
    ctx.apply(level, _lib.OP_GS_SWEEP)
ctx.synchronize()
print("done", flush=True)
