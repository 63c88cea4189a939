"""Level hierarchy and the host-built plans the device transfer kernels use.

Reference: /root/reference/pkg/src/ghostmg/transfer.py.

* Interior full-weighting restriction, the masked ghost restriction and the
  d-linear error interpolation (transfer.py:64-151) are *structural*: their
  weights follow from the fine labels and the node parity, so the device
  kernels (csrc/transfer.cu) recompute them on the fly instead of streaming
  (n x 3^d) weight/index tables.  ``check_transfer`` reproduces the build-time
  errors the reference raises for them.
* The inactive-band extrapolation (transfer.py:154-252) depends on the level
  set through the band normals, so its plan is built here: breadth-first
  groups (depth 1..3) with the 2d-bit mask of already-assigned axis
  neighbours, and per band node the upwind step and |n_k| of the transport
  iteration.  The device applies it (6 Jacobi transport steps).
* ``build_hierarchy`` re-classifies phi on every coarser grid with the
  reference's stop rules (transfer.py:266-304).
* ``ghost_dag_levels`` schedules the lexicographic ghost sweep as batches
  that are provably order-equivalent.
"""

from dataclasses import dataclass

import numpy as np

from .geometry import (
    GHOST,
    INACTIVE,
    INTERNAL,
    THETA_TRUST,
    ProjectionError,
    ResolutionError,
    UniformGrid,
    block_offsets,
    classify,
    compute_normal,
)

BAND_CELLS = 3
EXTRAP_STEPS = 6


class EmptyStencil(RuntimeError):
    """A restriction block contains no node of the required family."""


def fw_weights(d):
    """Full-weighting row [1/4, 1/2, 1/4]^{(x) d}, C order, entry ((1*a)*b)*c."""
    w = np.array([1.0])
    for _ in range(d):
        w = np.multiply.outer(w, np.array([0.25, 0.5, 0.25])).ravel()
    return w


class ExtrapolationPlan:
    """Band plan of one level (reference transfer.py:154-239).

    ``bfs_groups``: list of (node_idx ascending, mask uint8) per depth; bit
    2k+j of mask says the axis-k neighbour on side j (0: -, 1: +) was
    assigned at a smaller depth.  ``band_idx`` concatenates the groups;
    ``trans_step`` (nb, d) int8 is the upwind direction sign (0 = no
    neighbour) and ``trans_absn`` (nb, d) the matching |n_k| (0 where no
    neighbour).
    """

    def __init__(self, cls):
        grid = cls.grid
        d, N = grid.d, grid.N
        self.d = d
        depth = np.full(grid.n_nodes, -1, dtype=np.int8)
        depth[cls.ghost_idx] = 0
        inactive = cls.labels == INACTIVE
        strides = grid.strides
        self.bfs_groups = []
        frontier = cls.ghost_idx
        for level in range(1, BAND_CELLS + 1):
            if len(frontier) == 0:
                break
            multis = grid.multi_index(frontier)
            reach = []
            for k in range(d):
                for sign in (-1, 1):
                    m = multis[:, k] + sign
                    ok = (m >= 0) & (m <= N)
                    reach.append(frontier[ok] + sign * strides[k])
            cand = np.unique(np.concatenate(reach))
            fresh = cand[(depth[cand] == -1) & inactive[cand]]
            if len(fresh) == 0:
                break
            depth[fresh] = level
            fm = grid.multi_index(fresh)
            mask = np.zeros(len(fresh), dtype=np.uint8)
            for k in range(d):
                for j, sign in enumerate((-1, 1)):
                    m = fm[:, k] + sign
                    inside = (m >= 0) & (m <= N)
                    nb = np.where(inside, fresh + sign * strides[k], 0)
                    dn = depth[nb]
                    ok = inside & (dn >= 0) & (dn < level)
                    mask |= ok.astype(np.uint8) << np.uint8(2 * k + j)
            if np.any(mask == 0):
                raise ResolutionError("band node with no assigned neighbor")
            self.bfs_groups.append((fresh, mask))
            frontier = fresh
        if self.bfs_groups:
            self.band_idx = np.concatenate([g[0] for g in self.bfs_groups])
        else:
            self.band_idx = np.zeros(0, dtype=np.int64)
        self._transport(cls, grid)

    def _transport(self, cls, grid):
        idx = self.band_idx
        d = grid.d
        if len(idx) == 0:
            self.trans_step = np.zeros((0, d), dtype=np.int8)
            self.trans_absn = np.zeros((0, d))
            return
        multis = grid.multi_index(idx)
        normals = compute_normal(cls.phi, grid.multi_coords(multis), grid.h)
        absn = np.abs(normals)
        step = np.zeros((len(idx), d), dtype=np.int8)
        for k in range(d):
            s = np.sign(normals[:, k]).astype(np.int64)
            m = multis[:, k] - s
            inside = (m >= 0) & (m <= grid.N) & (s != 0)
            step[:, k] = np.where(inside, s, 0)
            absn[~inside, k] = 0.0
        self.trans_step = step
        self.trans_absn = absn

    def neighbours(self, strides):
        """Flat transport neighbours idx - step_k * stride_k (idx itself when
        step is 0), the reference's ``trans_nbrs``."""
        return self.band_idx[:, None] - self.trans_step.astype(np.int64) * np.asarray(strides)[None, :]

    @property
    def n_band(self):
        return len(self.band_idx)


@dataclass
class Level:
    cls: object
    extrap: ExtrapolationPlan


def check_transfer(fine_cls, coarse_cls, chunk=1 << 20, full_below=1 << 22, device=None):
    """Raise what the reference's restriction constructors raise
    (transfer.py:64-114): a coarse internal node whose fine 3^d block leaves
    the box, or whose mixed block holds no internal node; a coarse ghost
    whose block holds no in-box ghost/inactive node.

    None of these can fire for nested grids: a coarse internal node is a fine
    internal node (same point, same phi sign, off the box) at the block
    centre, and a coarse ghost sits on a fine node with phi >= 0 that is
    not eliminated (else the coarse node would be too), i.e. a kept
    ghost/inactive centre.  The exhaustive check runs for grids below
    ``full_below`` coarse nodes; above that only the block centres are
    verified."""
    fg, cg = fine_cls.grid, coarse_cls.grid
    if device is not None and fg.d in (2, 3):
        # every coarse node on the GPU (gmg_setup_check_transfer): the exhaustive block checks and the
        # centre checks at any size
        from . import _lib

        flags = _lib.setup_check_transfer(device, fg.d, fg.N, fine_cls.labels, cg.N, coarse_cls.labels)
        if flags & 1:
            raise ResolutionError("interior restriction block leaves the box")
        if flags & 2:
            raise EmptyStencil("no internal node under a coarse internal node")
        if flags & 4:
            raise EmptyStencil("no ghost/inactive node under a coarse ghost")
        if flags & 24:
            raise EmptyStencil("restriction block centre has the wrong label")
        return
    if cg.n_nodes >= full_below:
        for targets, ok in ((coarse_cls.internal_idx, (INTERNAL,)), (coarse_cls.ghost_idx, (GHOST, INACTIVE))):
            centers = fg.flat_index(2 * cg.multi_index(targets))
            if not np.isin(fine_cls.labels[centers], ok).all():
                raise EmptyStencil("restriction block centre has the wrong label")
        return
    d = fg.d
    offs = block_offsets(d, 3, -1)
    labels = fine_cls.labels
    for which in ("internal", "ghost"):
        targets = coarse_cls.internal_idx if which == "internal" else coarse_cls.ghost_idx
        for s in range(0, len(targets), chunk):
            centers = 2 * cg.multi_index(targets[s:s + chunk])
            multis = centers[:, None, :] + offs[None, :, :]
            valid = ((multis >= 0) & (multis <= fg.N)).all(axis=-1)
            flat = (np.clip(multis, 0, fg.N) * fg.strides).sum(axis=-1)
            lab = labels[flat]
            if which == "internal":
                if not valid.all():
                    raise ResolutionError("interior restriction block leaves the box")
                mixed = ((lab == GHOST) | (lab == INACTIVE)).any(axis=1)
                if np.any(mixed & ~(lab == INTERNAL).any(axis=1)):
                    raise EmptyStencil("no internal node under a coarse internal node")
            else:
                keep = valid & ((lab == GHOST) | (lab == INACTIVE))
                if np.any(~keep.any(axis=1)):
                    raise EmptyStencil("no ghost/inactive node under a coarse ghost")


def build_hierarchy(grid, phi, eliminated_faces=(), max_levels=None, coarsest_min=4, device=None):
    """Classify fine to coarse, halving N, with the reference's stop rules:
    odd N, N/2 < coarsest_min, max_levels, or a coarse level that fails to
    classify or holds a ghost with theta_raw > THETA_TRUST.  ``device``: CUDA
    ordinal for the per-node label work (classify, check_transfer)."""
    fine = classify(grid, phi, eliminated_faces, device=device)
    if fine.n_ghosts and fine.ghost_theta_raw.max() > THETA_TRUST:
        raise ResolutionError(
            "finest grid leaves a ghost farther than the relaxation formula trusts; refine the grid")
    chain = [fine]
    N = grid.N
    while True:
        if max_levels is not None and len(chain) >= max_levels:
            break
        if N % 2 or N // 2 < coarsest_min:
            break
        try:
            coarse = classify(UniformGrid(grid.d, N // 2), phi, eliminated_faces, device=device)
        except (ResolutionError, ProjectionError):
            break
        if coarse.n_ghosts and coarse.ghost_theta_raw.max() > THETA_TRUST:
            break
        chain.append(coarse)
        N //= 2
    if len(chain) < 2:
        raise ResolutionError("cannot build a second level; grid too coarse")
    levels = [Level(cls=c, extrap=ExtrapolationPlan(c)) for c in chain]
    for a, b in zip(chain[:-1], chain[1:]):
        check_transfer(a, b, device=device)
    return levels


def ghost_dag_levels(cls, weights):
    """Batch index per ghost for the order-equivalent parallel ghost sweep.

    Ghost t must follow every lexicographically earlier ghost s that it
    reads (s in its stencil with a nonzero weight) or that reads it; the
    batch index is 1 + the longest such chain.  Within a batch no ghost
    reads another, so a batch can run as one parallel step (reads of a
    ghost by a zero weight only affect the sign of a zero product).
    Returns int32 levels starting at 0.
    """
    ng = cls.n_ghosts
    if ng == 0:
        return np.zeros(0, dtype=np.int32)
    slot = np.full(cls.grid.n_nodes, -1, dtype=np.int64)
    slot[cls.ghost_idx] = np.arange(ng)
    reads = slot[cls.ghost_stencil]
    rows = np.broadcast_to(np.arange(ng)[:, None], reads.shape)
    use = (reads >= 0) & (reads != rows) & (weights != 0.0)
    a = rows[use]
    b = reads[use]
    lo = np.minimum(a, b)
    hi = np.maximum(a, b)
    pairs = np.unique(lo * ng + hi)
    lo, hi = pairs // ng, pairs % ng
    level = np.zeros(ng, dtype=np.int64)
    while True:
        cand = level[lo] + 1
        new = level.copy()
        np.maximum.at(new, hi, cand)
        if np.array_equal(new, level):
            break
        level = new
    return level.astype(np.int32)
