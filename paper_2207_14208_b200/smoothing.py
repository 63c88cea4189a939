"""Smoother configuration and per-ghost relaxation parameters (host setup).

Reference: /root/reference/pkg/src/ghostmg/smoothing.py.  One smoothing
step is a lexicographic Gauss-Seidel sweep over the internal nodes followed
by one lexicographic pass over the ghost rows, u_G += dtau (g - row . u)
(smoothing.py:127-149).  Those sweeps run on the device (csrc/gs_sweep.cu,
csrc/ghost_sweep.cu); this module only computes what they consume.
"""

from dataclasses import dataclass

import numpy as np

from . import blfa
from .kinds import BC_DIRICHLET, BC_NEUMANN, VARIANT_POLY

DTAU_CONSTANT = "constant"
DTAU_BLFA = "blfa"
DTAU_BLFA_POLY = "blfa-poly"
DTAU_MODES = (DTAU_CONSTANT, DTAU_BLFA, DTAU_BLFA_POLY)


@dataclass(frozen=True)
class SmootherConfig:
    """dtau mode and pre/post sweep counts (reference smoothing.py:30-47).

    In constant mode ``dtau_value`` is dimensionless; Neumann rows use
    dtau_value * h.
    """

    dtau_mode: str = DTAU_BLFA
    dtau_value: float = 1.0
    nu1: int = 2
    nu2: int = 1

    def __post_init__(self):
        if self.dtau_mode not in DTAU_MODES:
            raise ValueError(f"unknown dtau mode: {self.dtau_mode!r}")
        if self.nu1 < 0 or self.nu2 < 0 or self.nu1 + self.nu2 == 0:
            raise ValueError("need nu1, nu2 >= 0 with at least one sweep")


def assign_dtau(cls, dirichlet, config, default_variant=VARIANT_POLY):
    """Per-ghost dtau (reference smoothing.py:50-77).

    ``dirichlet`` is a per-ghost bool array (or a scalar bc kind string).
    BLFA modes evaluate ``blfa.dtau_opt`` at the raw theta; promoted ghosts
    get dtau = 1 (their extrapolation row has a unit own coefficient).
    """
    ng = cls.n_ghosts
    h = cls.grid.h
    if isinstance(dirichlet, str):
        dirichlet = np.full(ng, dirichlet == BC_DIRICHLET)
    dirichlet = np.asarray(dirichlet, dtype=bool)
    prom = cls.ghost_promoted
    if config.dtau_mode == DTAU_CONSTANT:
        dtau = np.where(dirichlet, config.dtau_value, config.dtau_value * h)
    else:
        variant = VARIANT_POLY if config.dtau_mode == DTAU_BLFA_POLY else default_variant
        dtau = np.ones(ng)
        reg = ~prom
        if reg.any():
            dtau[reg] = blfa.dtau_opt_batch(dirichlet[reg], cls.ghost_theta_raw[reg], cls.grid.d, h,
                                            variant)
    dtau = np.asarray(dtau, dtype=float).copy()
    dtau[prom] = 1.0
    return dtau
