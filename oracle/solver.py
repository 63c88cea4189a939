"""CPU oracle V-cycle (TEST INFRASTRUCTURE; see oracle/__init__.py).

``OracleSolver`` runs the reference's cycle recursion
(/root/reference/pkg/src/ghostmg/solver.py:157-203) on host arrays with the
C restatements in ghostmg_oracle.c and the reference's own coarsest solver
(SciPy SuperLU on the assembled coarsest system, solver.py:146-166).  It
consumes the same ``LevelPlan`` list as the device solver.
"""

import math

import numpy as np
from scipy.sparse.linalg import splu

from paper_2207_14208_b200.cycle import NORM_L2, CoarseSolveError, CycleDriver
from paper_2207_14208_b200.plan import coarsest_system

from . import ops


class OracleSolver(CycleDriver):
    def __init__(self, plans, f_fine, g_fine, eliminated_values, smoother, cycle):
        super().__init__(plans, f_fine, g_fine, eliminated_values, smoother, cycle)
        self._stencils = [np.ascontiguousarray(p.stencil, dtype=np.int64) for p in plans]
        self._lu = None
        self.u = None

    @classmethod
    def from_setup(cls, levels, spec, smoother, cycle, default_variant):
        plans, f, g, e = CycleDriver.problem_data(levels, spec, smoother, default_variant)
        return cls(plans, f, g, e, smoother, cycle)

    # ---- primitives ------------------------------------------------------
    def _set_data(self, f_fine, g_fine):
        self._f = np.ascontiguousarray(f_fine, dtype=np.float64)
        self._g = np.ascontiguousarray(g_fine, dtype=np.float64)

    def _put_u(self, u):
        self.u = np.array(u, dtype=np.float64, copy=True)

    def _get_u(self):
        return self.u.copy()

    def _residual_norm(self, level=0, u=None, f=None, g=None):
        p = self.plans[level]
        u = self.u if u is None else u
        f = self._f if f is None else f
        g = self._g if g is None else g
        r, m_int = ops.residual_internal_full(p, u, f)
        rg, m_g = ops.residual_ghost(p, u, g, self._stencils[level])
        if self.cycle_cfg.norm == NORM_L2:
            r_int = r[p.labels == 0]
            return math.sqrt(float(ops.sumsq(r_int) + ops.sumsq(rg)))
        if np.isnan(r).any() or np.isnan(rg).any():
            return float("nan")
        m = m_int if p.n_internal else 0.0
        if p.n_ghosts:
            m = max(m, m_g)
        return m

    def _abs_max_scale(self):
        peak = ops.abs_max(self.u)
        if 0.0 < peak < 1e-250:
            self.u *= 1e250
            return peak, True
        return peak, False

    def _run_cycle(self):
        self._cycle(0, self.u, self._f, self._g)

    # ---- cycle -----------------------------------------------------------
    def _smooth(self, level, u, f, g, count):
        ops.smooth(self.plans[level], u, f, g, count, self._stencils[level])

    def _coarsest(self):
        if self._lu is None:
            A, active = coarsest_system(self.plans[-1])
            try:
                self._lu = (splu(A.tocsc()), active)
            except RuntimeError as exc:
                raise CoarseSolveError(f"coarsest factorization failed: {exc}") from exc
        return self._lu

    def coarse_solve(self, f_c, g_c):
        p = self.plans[-1]
        e = np.zeros(p.n_nodes)
        if self.cycle_cfg.coarse_solver == "sweeps":
            self._smooth(len(self.plans) - 1, e, f_c, g_c, self.cycle_cfg.coarse_sweeps)
            return e
        lu, active = self._coarsest()
        rhs = np.concatenate([f_c[p.internal_idx], g_c])
        e[active] = lu.solve(rhs)
        return e

    def _cycle(self, level, u, f, g):
        P = self.plans[level]
        C = self.plans[level + 1]
        self._smooth(level, u, f, g, self.smoother.nu1)
        r_int, _ = ops.residual_internal_full(P, u, f)
        r_g, _ = ops.residual_ghost(P, u, g, self._stencils[level])
        r_ext = np.zeros(P.n_nodes)
        r_ext[P.ghost_idx] = r_g
        ops.extrapolate(P, r_ext)
        f_c = ops.restrict_interior(P, C, r_int)
        g_c = ops.restrict_ghost(P, C, r_ext)
        g_c[C.ghost_promoted] = 0.0
        if level + 1 == len(self.plans) - 1:
            e = self.coarse_solve(f_c, g_c)
        else:
            e = np.zeros(C.n_nodes)
            for _ in range(self.cycle_cfg.gamma):
                self._cycle(level + 1, e, f_c, g_c)
        ops.extrapolate(C, e)
        ops.interpolate_add(P, u, e)
        self._smooth(level, u, f, g, self.smoother.nu2)
