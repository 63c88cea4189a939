import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from test_gpu_parity import _pores64_solver
from paper_2207_14208_b200 import _lib
from paper_2207_14208_b200.plan import coarsest_system
from paper_2207_14208_b200.rng import uniform_symmetric
for backend in ("superlu", "device-inverse"):
    plans, s = _pores64_solver(backend)
    c = plans[-1]; L = len(plans) - 1
    f = uniform_symmetric(3, c.n_nodes); f[c.labels != 0] = 0
    g = uniform_symmetric(4, c.n_ghosts)
    s.ctx.set_vector(L, _lib.F, f); s.ctx.set_vector(L, _lib.G, g)
    s.ctx.apply(L, _lib.OP_COARSE_SOLVE)
    e = s.ctx.get_vector(L, _lib.U, c.n_nodes)
    A, active = coarsest_system(c)
    rhs = np.concatenate([f[c.internal_idx], g])
    x = np.linalg.solve(A.toarray(), rhs)
    print(backend, "n", A.shape[0], "max err", np.max(np.abs(e[active] - x)) / np.max(np.abs(x)))
