"""Cycle configuration, report and the host-side solve loop.

The control flow of ``solve`` and ``measure_rho`` is the reference's
(/root/reference/pkg/src/ghostmg/solver.py:215-298): record the residual
norm, run cycles, stop on >1e6 growth (rho = 1), renormalise the iterate by
1e250 when max|u| drops below 1e-250, optional relative tolerance, rho =
mean of the per-cycle reductions over cycles 11..15.  Backends (the B200
device solver in ``solver.py``; the CPU oracle in ``oracle/solver.py``)
implement the five primitives ``_put_u``, ``_get_u``, ``_run_cycle``,
``_residual_norm`` and ``_abs_max_scale``.
"""

import logging
import math
from dataclasses import dataclass

import numpy as np

from .geometry import ELIMINATED, INACTIVE
from .operators import ghost_data, node_values
from .plan import build_level_plan
from .rng import uniform_symmetric

log = logging.getLogger(__name__)

SCHEME_TWO_GRID = "two-grid"
SCHEME_V = "v"
SCHEME_W = "w"
SCHEMES = (SCHEME_TWO_GRID, SCHEME_V, SCHEME_W)

NORM_INF = "inf"
NORM_L2 = "l2"

RHO_WINDOW = (11, 15)
MIN_CYCLES_FOR_RHO = 16
DIVERGENCE_FACTOR = 1e6
RENORM_THRESHOLD = 1e-250


class DivergenceDetected(RuntimeError):
    pass


class CoarseSolveError(RuntimeError):
    """The coarsest-level system could not be factorized."""


@dataclass(frozen=True)
class CycleConfig:
    scheme: str = SCHEME_TWO_GRID
    cycles: int = MIN_CYCLES_FOR_RHO
    norm: str = NORM_INF
    coarse_solver: str = "direct"  # or "sweeps"
    coarse_sweeps: int = 500

    def __post_init__(self):
        if self.scheme not in SCHEMES:
            raise ValueError(f"unknown cycling scheme: {self.scheme!r}")
        if self.norm not in (NORM_INF, NORM_L2):
            raise ValueError(f"unknown norm: {self.norm!r}")
        if self.coarse_solver not in ("direct", "sweeps"):
            raise ValueError(f"unknown coarse solver: {self.coarse_solver!r}")

    @property
    def gamma(self):
        return 2 if self.scheme == SCHEME_W else 1

    @property
    def max_levels(self):
        return 2 if self.scheme == SCHEME_TWO_GRID else None


@dataclass
class CycleReport:
    residual_norms: list
    rho_sequence: list
    rho_asymptotic: float
    diverged: bool
    cycles_run: int
    scheme: str
    n_levels: int
    norm: str
    seed: int

    def to_dict(self):
        return {
            "residual_norms": [float(v) for v in self.residual_norms],
            "rho_sequence": [float(v) for v in self.rho_sequence],
            "rho_asymptotic": None if self.rho_asymptotic is None else float(self.rho_asymptotic),
            "diverged": self.diverged,
            "cycles_run": self.cycles_run,
            "scheme": self.scheme,
            "n_levels": self.n_levels,
            "norm": self.norm,
            "seed": self.seed,
        }


class CycleDriver:
    """Problem data + the reference's solve loop over abstract primitives."""

    def __init__(self, plans, f_fine, g_fine, eliminated_values, smoother, cycle):
        self.plans = plans
        self.smoother = smoother
        self.cycle_cfg = cycle
        self.f_fine = f_fine
        self.g_fine = g_fine
        self.eliminated_values = eliminated_values

    # ---- construction from the host setup -------------------------------
    @staticmethod
    def problem_data(levels, spec, smoother, default_variant):
        """(plans, f_fine, g_fine, eliminated_values) exactly as the
        reference's MultigridSolver.__init__ (solver.py:103-127)."""
        plans = [build_level_plan(lv, spec, smoother, default_variant) for lv in levels]
        fine = levels[0].cls
        grid = fine.grid
        f_fine = np.zeros(grid.n_nodes)
        if spec.f is not None:
            idx = fine.internal_idx
            f_fine[idx] = node_values(spec.f, grid, idx)
        g_fine = ghost_data(spec, fine)
        elim = np.zeros(grid.n_nodes)
        if spec.g_box is not None:
            idx = fine.eliminated_idx
            if len(idx):
                elim[idx] = node_values(spec.g_box, grid, idx)
        return plans, f_fine, g_fine, elim

    @property
    def n_levels(self):
        return len(self.plans)

    # ---- primitives (backend) -------------------------------------------
    def _put_u(self, u):
        raise NotImplementedError

    def _get_u(self):
        raise NotImplementedError

    def _fetch_u(self, u):
        """Copy the iterate back into the caller's array ``u`` when it is a
        matching float64 array (the reference mutates ``u`` in place), else
        return a new array."""
        out = self._get_u()
        if isinstance(u, np.ndarray) and u.shape == out.shape and u.dtype == np.float64:
            u[...] = out
            return u
        return out

    def _run_cycle(self):
        raise NotImplementedError

    def _residual_norm(self):
        raise NotImplementedError

    def _abs_max_scale(self):
        """Return max|u|; if 0 < max|u| < 1e-250, scale u by 1e250 and return
        True as second element."""
        raise NotImplementedError

    def _set_data(self, f_fine, g_fine):
        raise NotImplementedError

    # ---- reference API ---------------------------------------------------
    def initial_field(self, seed):
        """Seeded uniform(-1, 1) on every node, prescribed values on
        eliminated nodes, zero on inactive ones (solver.py:205-213)."""
        fine = self.plans[0]
        u = uniform_symmetric(seed, fine.n_nodes)
        elim = fine.labels == ELIMINATED
        u[elim] = self.eliminated_values[elim]
        u[fine.labels == INACTIVE] = 0.0
        return u

    def _device_initial_field(self, seed):
        """Backends that can draw `initial_field(seed)` where the iterate lives
        do so and return True."""
        return False

    def run_cycle(self, u=None):
        """One cycle in place.  With ``u`` given (host array) it is uploaded,
        cycled and copied back, like the reference's ``run_cycle(u)``."""
        if u is not None:
            self._set_data(self.f_fine, self.g_fine)
            self._put_u(u)
        self._run_cycle()
        if u is not None:
            self._fetch_u(u)
        return u

    def solve(self, u=None, cycles=None, tol=0.0, seed=42):
        cfg = self.cycle_cfg
        cycles = cfg.cycles if cycles is None else cycles
        self._set_data(self.f_fine, self.g_fine)
        if u is None and self._device_initial_field(seed):
            u = np.empty(self.plans[0].n_nodes)  # filled by _fetch_u; the field itself never visits the host
        else:
            if u is None:
                u = self.initial_field(seed)
            self._put_u(np.ascontiguousarray(u, dtype=np.float64))
        ln_scale = 0.0
        ln_norms = []

        def record():
            n = self._residual_norm()
            ln_norms.append((math.log(n) if n > 0.0 else -math.inf) + ln_scale)

        record()
        diverged = False
        ran = 0
        for m in range(cycles):
            self._run_cycle()
            record()
            ran = m + 1
            if ln_norms[-1] - ln_norms[0] > math.log(DIVERGENCE_FACTOR):
                diverged = True
                log.warning("residual grew %.1e-fold; stopping", DIVERGENCE_FACTOR)
                break
            _, scaled = self._abs_max_scale()
            if scaled:
                ln_scale -= math.log(1e250)
            if tol > 0.0 and ln_norms[-1] - ln_norms[0] < math.log(tol):
                break

        u = self._fetch_u(u)
        norms = [math.exp(v) if v > -math.inf else 0.0 for v in ln_norms]
        rho_seq = [math.exp(ln_norms[i + 1] - ln_norms[i]) if ln_norms[i] > -math.inf else 0.0
                   for i in range(len(ln_norms) - 1)]
        lo, hi = RHO_WINDOW
        rho = None
        if diverged:
            rho = 1.0
        elif ran >= MIN_CYCLES_FOR_RHO:
            rho = float(np.mean(rho_seq[lo:hi + 1]))
        report = CycleReport(
            residual_norms=norms, rho_sequence=rho_seq, rho_asymptotic=rho,
            diverged=diverged, cycles_run=ran, scheme=cfg.scheme,
            n_levels=self.n_levels, norm=cfg.norm, seed=seed)
        return u, report


def measure_rho(solver, seed=42, cycles=MIN_CYCLES_FOR_RHO):
    """Homogeneous-problem convergence factor (reference solver.py:282-298)."""
    cycles = max(cycles, MIN_CYCLES_FOR_RHO)
    saved = solver.f_fine, solver.g_fine, solver.eliminated_values
    solver.f_fine = np.zeros_like(solver.f_fine)
    solver.g_fine = np.zeros_like(solver.g_fine)
    solver.eliminated_values = np.zeros_like(solver.eliminated_values)
    try:
        _, report = solver.solve(cycles=cycles, seed=seed)
    finally:
        solver.f_fine, solver.g_fine, solver.eliminated_values = saved
    return report
