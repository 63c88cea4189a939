"""The BASELINE.json problem configurations, built on the reference-style API.

Each ``config_*`` returns a ``ProblemSetup``: grid, level set, spec,
eliminated faces, smoother/cycle configuration, default BLFA variant,
``coarsest_min`` and (for the pore-space configs) a directly assigned
right-hand side.  Adaptations the reference needs to run these configs at
all (SURVEY.md finding 7 and Appendix B) are applied and listed in
``ProblemSetup.notes``:

* c1/c3: signed-distance disk/ball (``levelsets.SignedSphere``);
* c2: ``Flower(0.5, 0.15)`` with a per-ghost Dirichlet/Neumann selector
  (sign of sin 5*theta at Q, evaluated as the sign of Im((x+iy)^5));
  coarsest level N=32 (N<=16 is singular for this flower);
* c3: ``coarsest_min=8`` (the N=4 coarsest matrix is singular);
* c4/c5: non-overlapping balls placed by a seeded rejection sampler in
  [0,1]^3 (overlapping draws break the reference's projection), mapped to
  [-1,1]^3 (so the Laplacian scales by 1/4, applied to f); all six cube faces
  carry u = 0; Neumann g = 0 on the balls; f = U(-1,1) per node from
  ``XorShift64Star(seed + 1)`` in flat order, times 1/4, on internal nodes.

All BASELINE configs use V(2,1) cycles with BLFA dtau and the EXP symbol
variant (the reference's choice for curved domains, cases.py:131-166).
"""

from dataclasses import dataclass, field

import numpy as np

from .cycle import CycleConfig
from .geometry import FACE_HIGH, FACE_LOW, UniformGrid
from .kinds import VARIANT_EXP
from .levelsets import Flower, SignedSphere, pore_space_unit_cube
from .operators import ProblemSpec
from .rng import uniform_symmetric
from .smoothing import SmootherConfig


@dataclass
class ProblemSetup:
    name: str
    grid: UniformGrid
    phi: object
    spec: ProblemSpec
    faces: tuple = ()
    smoother: SmootherConfig = field(default_factory=SmootherConfig)
    cycle: CycleConfig = field(default_factory=lambda: CycleConfig(scheme="v", cycles=20))
    default_variant: str = VARIANT_EXP
    coarsest_min: int = 4
    f_seed: int = None          # pore space: f drawn per node from this seed
    f_scale: float = 1.0
    exact: object = None        # manufactured solution, if any
    notes: tuple = ()


# ---- manufactured solutions ------------------------------------------------

def _u1(p):
    x, y = p[..., 0], p[..., 1]
    return np.exp(x + y) * np.sin(np.pi * x)


def _f1(p):
    x, y = p[..., 0], p[..., 1]
    return np.exp(x + y) * ((np.pi ** 2 - 2.0) * np.sin(np.pi * x) - 2.0 * np.pi * np.cos(np.pi * x))


def _u2(p):
    return np.cos(2.0 * p[..., 0]) * np.exp(p[..., 1])


def _f2(p):
    return 3.0 * _u2(p)


def _grad_u2(p):
    x, y = p[..., 0], p[..., 1]
    e = np.exp(y)
    return np.stack([-2.0 * np.sin(2.0 * x) * e, np.cos(2.0 * x) * e], axis=-1)


def _u3(p):
    return np.exp(p[..., 0]) * np.sin(p[..., 1]) * np.cos(p[..., 2])


def petal_dirichlet(Q):
    """True where sin(5*atan2(y, x)) > 0, via the sign of Im((x+iy)^5)."""
    x, y = Q[..., 0], Q[..., 1]
    x2, y2 = x * x, y * y
    s = y * ((y2 * y2 + 5.0 * (x2 * x2)) - 10.0 * (x2 * y2))
    return s > 0.0


def _mixed_data(Q, dirichlet, normals):
    flux = (_grad_u2(Q) * normals).sum(axis=-1)
    return np.where(dirichlet, _u2(Q), flux)


ALL_FACES = tuple((a, s) for a in range(3) for s in (FACE_LOW, FACE_HIGH))


def config_disk(N=256, cycles=20):
    """BASELINE config 1: 2D disk, Dirichlet, u = e^{x+y} sin(pi x)."""
    spec = ProblemSpec("poisson", "dirichlet", f=_f1, g_box=_u1, g_gamma=_u1)
    return ProblemSetup(
        name=f"c1-disk-N{N}", grid=UniformGrid(2, N),
        phi=SignedSphere((0.02, 0.01), 0.5), spec=spec,
        cycle=CycleConfig(scheme="v", cycles=cycles), coarsest_min=4, exact=_u1,
        notes=("signed-distance disk",))


def config_flower(N=2048, cycles=20):
    """BASELINE config 2: flower r = 0.5 + 0.15 sin 5theta, mixed BC."""
    spec = ProblemSpec("poisson", "mixed", f=_f2, g_box=_u2, g_gamma=_mixed_data,
                       bc_selector=petal_dirichlet)
    return ProblemSetup(
        name=f"c2-flower-N{N}", grid=UniformGrid(2, N), phi=Flower(0.5, 0.15), spec=spec,
        cycle=CycleConfig(scheme="v", cycles=cycles), coarsest_min=32, exact=_u2,
        notes=("per-ghost Dirichlet/Neumann rows (petal selector)", "coarsest N=32"))


def config_flower_dirichlet(N=2048, cycles=20):
    """All-Dirichlet flower: the convergent proxy of config 2."""
    spec = ProblemSpec("poisson", "dirichlet", f=_f2, g_box=_u2, g_gamma=_u2)
    return ProblemSetup(
        name=f"c2d-flower-dirichlet-N{N}", grid=UniformGrid(2, N), phi=Flower(0.5, 0.15),
        spec=spec, cycle=CycleConfig(scheme="v", cycles=cycles), coarsest_min=32, exact=_u2)


def config_ball(N=256, cycles=15):
    """BASELINE config 3: 3D ball, Dirichlet, u = e^x sin y cos z (f = u)."""
    spec = ProblemSpec("poisson", "dirichlet", f=_u3, g_box=_u3, g_gamma=_u3)
    return ProblemSetup(
        name=f"c3-ball-N{N}", grid=UniformGrid(3, N),
        phi=SignedSphere((0.013, -0.007, 0.021), 0.45), spec=spec,
        cycle=CycleConfig(scheme="v", cycles=cycles), coarsest_min=8, exact=_u3,
        notes=("signed-distance ball", "coarsest_min=8"))


def config_pores(N=512, balls=64, r_lo=0.05, r_hi=0.15, seed=42, cycles=15, coarsest_min=4):
    """BASELINE config 4 (and 5 with balls=256, r in [0.03, 0.08], N=1024)."""
    spec = ProblemSpec("poisson", "neumann")
    return ProblemSetup(
        name=f"c4-pores{balls}-N{N}", grid=UniformGrid(3, N),
        phi=pore_space_unit_cube(seed, balls, r_lo, r_hi), spec=spec, faces=ALL_FACES,
        cycle=CycleConfig(scheme="v", cycles=cycles), coarsest_min=coarsest_min,
        f_seed=seed + 1, f_scale=0.25,
        notes=("rejection-sampled non-overlapping balls", "[0,1]^3 -> [-1,1]^3",
               "u=0 on all cube faces", "f = U(-1,1)/4 per internal node"))


def config_pores_large(N=1024, cycles=10, seed=42):
    setup = config_pores(N=N, balls=256, r_lo=0.03, r_hi=0.08, seed=seed, cycles=cycles)
    setup.name = f"c5-pores256-N{N}"
    return setup


CONFIGS = {
    "c1": config_disk,
    "c2": config_flower,
    "c2d": config_flower_dirichlet,
    "c3": config_ball,
    "c4": config_pores,
    "c5": config_pores_large,
}


def pore_rhs(setup, labels):
    """Right-hand side of the pore-space configs on the fine grid."""
    f = uniform_symmetric(setup.f_seed, setup.grid.n_nodes) * setup.f_scale
    f[labels != 0] = 0.0
    return f
