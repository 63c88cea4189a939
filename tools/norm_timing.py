import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2207_14208_b200 import configs as CF, _lib
from paper_2207_14208_b200.transfer import build_hierarchy
from paper_2207_14208_b200.cycle import CycleDriver
from paper_2207_14208_b200.solver import MultigridSolver
name, N = sys.argv[1].split(":"); N = int(N)
setup = CF.config_pores(N=N) if name == "c4" else CF.CONFIGS[name](N)
levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
s = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, coarse_backend="device-inverse")
if len(sys.argv) > 2 and sys.argv[2] == "torch":
    stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); s.ctx.set_stream(stream.cuda_stream)
    print("torch stream", stream.cuda_stream)
s._set_data(f, g); s._put_u(np.zeros(plans[0].n_nodes))
def timeit(label, fn, n=5):
    s.ctx.synchronize(); t = time.perf_counter()
    for _ in range(n): fn()
    s.ctx.synchronize(); print(f"{label}: {(time.perf_counter()-t)/n*1e3:.2f} ms", flush=True)
timeit("residual_parts", lambda: s.ctx.residual_parts(0))
timeit("apply RES_INT", lambda: s.ctx.apply(0, _lib.OP_RES_INT))
timeit("apply RES_GHOST", lambda: s.ctx.apply(0, _lib.OP_RES_GHOST))
timeit("abs_max", lambda: s.ctx.abs_max_scale())
timeit("cycle", lambda: s.ctx.cycle(1))
timeit("residual_parts after cycle", lambda: (s.ctx.cycle(1), s.ctx.residual_parts(0)))
