"""String tags shared by the host-side API (boundary kinds, PDE kinds,
BLFA symbol variants).

Mirrors the tag vocabulary of the reference package
(/root/reference/pkg/src/ghostmg/kinds.py:1-31) so configuration written for
the reference works unchanged here.  ``BC_MIXED`` is an extension: a
per-ghost Dirichlet/Neumann selection (BASELINE config 2), see
``operators.ProblemSpec.bc_selector``.
"""

BC_DIRICHLET = "dirichlet"
BC_NEUMANN = "neumann"
BC_MIXED = "mixed"
BC_KINDS = (BC_DIRICHLET, BC_NEUMANN, BC_MIXED)

PDE_POISSON = "poisson"
PDE_REACTION = "reaction"
PDE_KINDS = (PDE_POISSON, PDE_REACTION)

VARIANT_POLY = "poly"
VARIANT_EXP = "exp"
VARIANTS = (VARIANT_POLY, VARIANT_EXP)


def _checked(value, allowed, what):
    if value not in allowed:
        raise ValueError(f"unknown {what}: {value!r}")
    return value


def check_bc(bc, allow_mixed=True):
    allowed = BC_KINDS if allow_mixed else BC_KINDS[:2]
    return _checked(bc, allowed, "boundary condition kind")


def check_pde(pde):
    return _checked(pde, PDE_KINDS, "equation kind")


def check_variant(variant):
    return _checked(variant, VARIANTS, "symbol variant")
