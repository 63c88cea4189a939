"""Discrete operators on one level: ghost rows and the sparse system.

Reference: /root/reference/pkg/src/ghostmg/operators.py.  Interior rows are
the 2d+1 point Laplacian (2d/h^2 diagonal, -1/h^2 to axis neighbours, +1
for the reaction equation).  Each ghost carries one row over its upwind
3^d block: the tensor-product quadratic interpolant at Q (Dirichlet) or its
derivative along n(Q) (Neumann, 1/h scaled); promoted ghosts carry the
(1, -2, 1) extrapolation row (operators.py:73-96).

Extension: ``bc="mixed"`` with ``ProblemSpec.bc_selector(Q) -> bool``
(True = Dirichlet) picks the row kind per ghost (BASELINE config 2's
petal-dependent boundary; SURVEY.md Appendix B shim).
"""

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .geometry import (
    ELIMINATED,
    INACTIVE,
    WEIGHT_TOL,
    ResolutionError,
    compute_normal,
    extrapolation_row_weights,
    lagrange_quad,
    lagrange_quad_deriv,
    tensor_weights,
)
from .kinds import BC_DIRICHLET, BC_MIXED, BC_NEUMANN, PDE_REACTION, check_bc, check_pde


@dataclass(frozen=True)
class ProblemSpec:
    """Problem data; callables take point arrays (..., d), None means 0.

    For ``bc="mixed"``, ``bc_selector(Q)`` returns True where a ghost's row
    is Dirichlet and ``g_gamma`` must then return the Dirichlet value or the
    normal flux accordingly (``g_gamma(Q, dirichlet_mask, normals)``).
    """

    pde: str
    bc: str
    f: object = None
    g_box: object = None
    g_gamma: object = None
    bc_selector: object = None

    def __post_init__(self):
        check_pde(self.pde)
        check_bc(self.bc)
        if self.bc == BC_MIXED and self.bc_selector is None:
            raise ValueError("mixed boundary conditions need a bc_selector")

    @property
    def reaction(self):
        return 1.0 if self.pde == PDE_REACTION else 0.0


def dirichlet_mask(cls, spec_or_bc, selector=None):
    """Per-ghost True where the row is a Dirichlet row."""
    bc = getattr(spec_or_bc, "bc", spec_or_bc)
    sel = getattr(spec_or_bc, "bc_selector", selector)
    if bc == BC_DIRICHLET:
        return np.ones(cls.n_ghosts, dtype=bool)
    if bc == BC_NEUMANN:
        return np.zeros(cls.n_ghosts, dtype=bool)
    return np.asarray(sel(cls.ghost_Q), dtype=bool)


def _block_t(cls):
    return (cls.ghost_Q - cls.grid.multi_coords(cls.ghost_block_low)) / cls.grid.h


def _dirichlet_rows(cls):
    return tensor_weights(lagrange_quad(_block_t(cls)))


def _neumann_rows(cls):
    h = cls.grid.h
    t = _block_t(cls)
    normal_q = compute_normal(cls.phi, cls.ghost_Q, h)
    values = lagrange_quad(t)
    derivs = lagrange_quad_deriv(t)
    w = np.zeros((cls.n_ghosts, 3 ** cls.grid.d))
    for k in range(cls.grid.d):
        f = values.copy()
        f[:, k, :] = derivs[:, k, :]
        w += (normal_q[:, k] / h)[:, None] * tensor_weights(f)
    return w


def ghost_row_weights(cls, bc, selector=None):
    """(n_ghosts, 3^d) row coefficients in stencil (C) order."""
    check_bc(bc)
    if bc == BC_DIRICHLET:
        w = _dirichlet_rows(cls)
    elif bc == BC_NEUMANN:
        w = _neumann_rows(cls)
    else:
        dmask = dirichlet_mask(cls, bc, selector)
        w = np.where(dmask[:, None], _dirichlet_rows(cls), _neumann_rows(cls))
    prom = cls.ghost_promoted
    if prom.any():
        w[prom] = extrapolation_row_weights(cls)[prom]
    return w


def check_ghost_rows(cls, weights):
    """A nonzero coefficient on an inactive node is a resolution failure."""
    hit = (np.abs(weights) > WEIGHT_TOL) & (cls.labels[cls.ghost_stencil] == INACTIVE)
    if np.any(hit):
        g = int(np.flatnonzero(hit.any(axis=1))[0])
        raise ResolutionError(
            f"ghost row at flat index {int(cls.ghost_idx[g])} needs an inactive node")


def internal_neighbors(cls):
    """(n_internal, 2d) flat neighbour indices, columns [ax0-, ax0+, ax1-, ...]."""
    idx = cls.internal_idx
    cols = []
    for s in cls.grid.strides:
        cols += [idx - s, idx + s]
    return np.stack(cols, axis=1)


def node_values(func, grid, flat_idx):
    if func is None:
        return np.zeros(len(flat_idx))
    pts = grid.multi_coords(grid.multi_index(flat_idx))
    return np.asarray(func(pts), dtype=float)


def assemble_system(spec, cls, weights=None):
    """Sparse system over the active nodes (internal then ghost, flat order).

    Returns (A, b, active_idx) like the reference (operators.py:171-228);
    prescribed box data on eliminated neighbours is folded into b.
    ``weights`` may pass precomputed ghost rows (mixed BC).
    """
    grid = cls.grid
    h2 = grid.h ** 2
    labels = cls.labels
    internal = cls.internal_idx
    ghosts = cls.ghost_idx
    ni, ng = len(internal), len(ghosts)
    active = np.concatenate([internal, ghosts])
    column = np.full(grid.n_nodes, -1, dtype=np.int64)
    column[active] = np.arange(len(active))

    box = np.zeros(grid.n_nodes)
    elim = cls.eliminated_idx
    if spec.g_box is not None and len(elim):
        box[elim] = node_values(spec.g_box, grid, elim)

    b = np.zeros(len(active))
    b[:ni] = node_values(spec.f, grid, internal)
    rows = [np.arange(ni)]
    cols = [np.arange(ni)]
    vals = [np.full(ni, 2.0 * grid.d / h2 + spec.reaction)]
    nbrs = internal_neighbors(cls)
    for k in range(nbrs.shape[1]):
        nb = nbrs[:, k]
        ok = column[nb] >= 0
        rows.append(np.flatnonzero(ok))
        cols.append(column[nb[ok]])
        vals.append(np.full(int(ok.sum()), -1.0 / h2))
        fixed = labels[nb] == ELIMINATED
        if np.any(fixed):
            b[np.flatnonzero(fixed)] += box[nb[fixed]] / h2

    if weights is None:
        weights = ghost_row_weights(cls, spec.bc, spec.bc_selector)
    check_ghost_rows(cls, weights)
    if spec.g_gamma is not None and ng:
        b[ni:] = ghost_data(spec, cls)
    nz = np.abs(weights) > 0.0
    st = cls.ghost_stencil
    keep = nz & (column[st] >= 0)
    gr, gc = np.nonzero(keep)
    rows.append(ni + gr)
    cols.append(column[st[gr, gc]])
    vals.append(weights[gr, gc])
    fixed = nz & (labels[st] == ELIMINATED)
    if np.any(fixed):
        for g in np.flatnonzero(fixed.any(axis=1)):
            m = fixed[g]
            b[ni + g] -= float(np.dot(weights[g][m], box[st[g][m]]))

    A = sp.csr_matrix(
        (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
        shape=(len(active), len(active)))
    return A, b, active


def ghost_data(spec, cls):
    """Right-hand side of the ghost rows on this level: g_gamma(Q), zero on
    promoted (extrapolation) rows.  Mixed BC passes the Dirichlet mask and
    the normals at Q so the data callable can return value or flux."""
    if spec.g_gamma is None or cls.n_ghosts == 0:
        return np.zeros(cls.n_ghosts)
    if spec.bc == BC_MIXED:
        dmask = dirichlet_mask(cls, spec)
        normals = compute_normal(cls.phi, cls.ghost_Q, cls.grid.h)
        g = np.asarray(spec.g_gamma(cls.ghost_Q, dmask, normals), dtype=float)
    else:
        g = np.asarray(spec.g_gamma(cls.ghost_Q), dtype=float)
    g = g.copy()
    g[cls.ghost_promoted] = 0.0
    return g
