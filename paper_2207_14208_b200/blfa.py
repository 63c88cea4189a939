"""Boundary Local Fourier Analysis: the optimal ghost relaxation parameter.

This is the paper's contribution (arXiv 2207.14208; reference
/root/reference/pkg/src/ghostmg/blfa.py:1-194).  Near a boundary, an error
mode with tangential frequencies alpha decays by exp(-p) per layer with
p = arccosh(d - sum cos alpha_i).  The ghost update multiplies it by
1 - dtau * g0(p; theta) (Dirichlet) or 1 - (dtau/h) * g0 (Neumann).  Over
the high-frequency corner set the extreme values of |g0| bound the
amplification, and the minimax over the lines x -> |1 - g0 x| gives
dtau* = 2 / (g0_max + g0_min) (times h for Neumann rows).

Everything here is scalar Python ``math`` (libm), evaluated once per ghost
at setup; the values are uploaded to the device.
"""

import math
from dataclasses import dataclass

from .kinds import BC_DIRICHLET, BC_NEUMANN, VARIANT_EXP, VARIANT_POLY, check_bc, check_variant

THETA_FORMULA_MAX = 1.65


class DomainError(ValueError):
    """arccosh argument below 1."""


class AllZeroSlopes(ValueError):
    """Minimax over lines with every slope zero."""


@dataclass(frozen=True)
class BlfaQuery:
    bc: str
    d: int
    theta: float
    h: float = 1.0
    variant: str = VARIANT_POLY

    def __post_init__(self):
        check_bc(self.bc, allow_mixed=False)
        check_variant(self.variant)
        if self.d < 1:
            raise ValueError(f"dimension must be >= 1, got {self.d}")
        if not 0.0 <= self.theta <= THETA_FORMULA_MAX:
            raise ValueError(f"theta must lie in [0, {THETA_FORMULA_MAX}], got {self.theta}")
        if self.h <= 0.0:
            raise ValueError(f"grid spacing must be positive, got {self.h}")


def symbol_p(alphas):
    """Per-layer decay rate arccosh(d - sum cos alpha), as log(z + sqrt(z^2-1))."""
    alphas = [float(a) for a in alphas]
    z = (len(alphas) + 1) - sum(math.cos(a) for a in alphas)
    if z < 1.0:
        raise DomainError(f"arccosh argument {z} < 1 for alphas={tuple(alphas)}")
    return math.log(z + math.sqrt(z * z - 1.0))


def symbol_p_continuous(alphas):
    return float(sum(alphas))


def bc_coeffs_dimensionless(bc, theta):
    """Ghost-row triple (c_-2, c_-1, c_0) with h factored out."""
    check_bc(bc, allow_mixed=False)
    t = float(theta)
    if bc == BC_DIRICHLET:
        return (t * (t - 1.0) / 2.0, t * (2.0 - t), (1.0 - t) * (2.0 - t) / 2.0)
    return (0.5 - t, 2.0 * (t - 1.0), 1.5 - t)


def g0(query, p):
    if query.variant == VARIANT_EXP:
        decay = math.exp(-p * query.theta)
        return decay if query.bc == BC_DIRICHLET else p * decay
    e = math.exp(-float(p))
    c2, c1, c0 = bc_coeffs_dimensionless(query.bc, query.theta)
    return c0 + c1 * e + c2 * e * e


def amplification(query, alphas, dtau):
    if len(alphas) != max(query.d, 2) - 1:
        raise ValueError(
            f"expected {max(query.d, 2) - 1} tangential frequencies, got {len(alphas)}")
    scaled = dtau / query.h if query.bc == BC_NEUMANN else dtau
    return 1.0 - scaled * g0(query, symbol_p(alphas))


def corner_points(d):
    """(pi/2 x r, 0 x (d-1-r)) for r = 1..d-1, then (pi, ..., pi)."""
    if d < 2:
        raise ValueError("corner set is defined for d >= 2")
    half = math.pi / 2.0
    pts = [tuple([half] * r + [0.0] * (d - 1 - r)) for r in range(1, d)]
    pts.append(tuple([math.pi] * (d - 1)))
    return pts


def minimax_lines(slopes):
    ms = [float(m) for m in slopes]
    if not ms:
        raise AllZeroSlopes("no slopes given")
    if min(ms) < 0.0:
        raise ValueError("slopes must be nonnegative")
    hi, lo = max(ms), min(ms)
    if hi == 0.0:
        raise AllZeroSlopes("all slopes vanish, every x is equally bad")
    x = 2.0 / (hi + lo)
    return x, max(abs(1.0 - m * x) for m in ms)


_CORNER_P = {}


def _corner_ps(d_eff):
    ps = _CORNER_P.get(d_eff)
    if ps is None:
        ps = _CORNER_P[d_eff] = [symbol_p(a) for a in corner_points(d_eff)]
    return ps


def dtau_opt(query):
    """Optimal per-ghost relaxation parameter (reference blfa.py:167-194)."""
    slopes = [abs(g0(query, p)) for p in _corner_ps(max(query.d, 2))]
    x, _ = minimax_lines(slopes)
    return query.h * x if query.bc == BC_NEUMANN else x


def dtau_opt_batch(dirichlet, theta, d, h, variant):
    """``dtau_opt`` for many ghosts at once, bit-identical to the scalar
    function: the per-corner decay rates are the scalar ones, g0 uses libm
    ``math.exp`` per element (EXP variant) or exact arithmetic (POLY), and
    the minimax is 2 / (max + min) in the same order."""
    import numpy as np

    check_variant(variant)
    dirichlet = np.asarray(dirichlet, dtype=bool)
    theta = np.asarray(theta, dtype=float)
    if np.any((theta < 0.0) | (theta > THETA_FORMULA_MAX)):
        bad = theta[(theta < 0.0) | (theta > THETA_FORMULA_MAX)][0]
        raise ValueError(f"theta must lie in [0, {THETA_FORMULA_MAX}], got {bad}")
    slopes = []
    for p in _corner_ps(max(d, 2)):
        if variant == VARIANT_EXP:
            arg = (-p * theta).tolist()
            decay = np.fromiter(map(math.exp, arg), dtype=float, count=len(arg))
            g = np.where(dirichlet, decay, p * decay)
        else:
            e = math.exp(-float(p))
            t = theta
            dc2, dc1, dc0 = t * (t - 1.0) / 2.0, t * (2.0 - t), (1.0 - t) * (2.0 - t) / 2.0
            nc2, nc1, nc0 = 0.5 - t, 2.0 * (t - 1.0), 1.5 - t
            g = np.where(dirichlet, dc0 + dc1 * e + dc2 * e * e, nc0 + nc1 * e + nc2 * e * e)
        slopes.append(np.abs(g))
    hi = slopes[0]
    lo = slopes[0]
    for s in slopes[1:]:
        hi = np.maximum(hi, s)
        lo = np.minimum(lo, s)
    if np.any(hi == 0.0):
        raise AllZeroSlopes("all slopes vanish, every x is equally bad")
    x = 2.0 / (hi + lo)
    return np.where(dirichlet, x, h * x)
