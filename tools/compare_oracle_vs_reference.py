import sys, math, time
import numpy as np
sys.path.insert(0, '/root/reference/pkg/src'); sys.path.insert(0, '/root/repo')
import ghostmg
from ghostmg.solver import build_solver as rbuild, CycleConfig as RCC, measure_rho as rrho
from ghostmg.smoothing import SmootherConfig as RSC
from ghostmg.operators import ProblemSpec as RPS
from paper_2207_14208_b200 import levelsets as L, transfer as T, geometry as G, smoothing as S, cycle as C
from oracle.solver import OracleSolver

def run(name, d, N, phi, spec_args, faces=(), variant='exp', coarsest_min=4, cycles=20, scheme='v', rho=True):
    rspec = RPS(*spec_args)
    rs = rbuild(ghostmg.UniformGrid(d, N), phi, rspec, faces, RSC(), RCC(scheme=scheme, cycles=cycles), variant, coarsest_min)
    t = time.time(); ur, rr = rs.solve(u=np.zeros(rs.levels[0].cls.grid.n_nodes), cycles=cycles); tr = time.time() - t
    levels = T.build_hierarchy(G.UniformGrid(d, N), phi, faces, max_levels=C.CycleConfig(scheme=scheme).max_levels, coarsest_min=coarsest_min)
    from paper_2207_14208_b200.operators import ProblemSpec
    os_ = OracleSolver.from_setup(levels, ProblemSpec(*spec_args), S.SmootherConfig(), C.CycleConfig(scheme=scheme, cycles=cycles), variant)
    t = time.time(); uo, ro = os_.solve(u=np.zeros(levels[0].cls.grid.n_nodes), cycles=cycles); to = time.time() - t
    same_u = np.array_equal(ur.view(np.uint64), uo.view(np.uint64))
    same_r = rr.residual_norms == ro.residual_norms
    print(f'{name}: u bitwise {same_u}, residuals bitwise {same_r}; ref {tr:.2f}s oracle {to:.2f}s; last res {ro.residual_norms[-1]:.3e}')
    if not same_r:
        print(' ref', rr.residual_norms[:5]); print(' orc', ro.residual_norms[:5])
    if rho:
        a = rrho(rs).rho_asymptotic; b = C.measure_rho(os_).rho_asymptotic
        print(f'   rho ref {a!r} oracle {b!r} equal {a == b}')

ue = lambda p: np.exp(p[..., 0] + p[..., 1]) * np.sin(np.pi * p[..., 0])
fe = lambda p: np.exp(p[..., 0] + p[..., 1]) * ((np.pi**2 - 2) * np.sin(np.pi * p[..., 0]) - 2 * np.pi * np.cos(np.pi * p[..., 0]))
run('disk64', 2, 64, L.SignedSphere((0.02, 0.01), 0.5), ('poisson', 'dirichlet', fe, ue, ue))
run('disk128', 2, 128, L.SignedSphere((0.02, 0.01), 0.5), ('poisson', 'dirichlet', fe, ue, ue))
u3 = lambda p: np.exp(p[..., 0]) * np.sin(p[..., 1]) * np.cos(p[..., 2])
run('ball32', 3, 32, L.SignedSphere((0.013, -0.007, 0.021), 0.45), ('poisson', 'dirichlet', u3, u3, u3), coarsest_min=8, cycles=15)
run('circle32W', 2, 32, ghostmg.levelsets.Sphere((math.sqrt(3)/40, -0.05), math.sqrt(2)/2), ('poisson', 'dirichlet'), scheme='w', cycles=16)
run('flower128N', 2, 128, L.Flower(0.5, 0.15), ('poisson', 'neumann'), coarsest_min=32, cycles=16)
run('line30reaction', 2, 32, ghostmg.cases.build_case('line30', 32).phi, ('reaction', 'neumann'), faces=ghostmg.cases.build_case('line30', 32).eliminated_faces, cycles=16, scheme='two-grid')
