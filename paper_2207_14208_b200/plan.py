"""Per-level arrays that the device kernels (and the CPU oracle) consume.

A ``LevelPlan`` is the complete, geometry-free description of one grid
level of a solver: labels, the ghost rows (stencil corner, 3^d weights,
dtau, promotion flag, sweep batch) and the band-extrapolation plan.  It is
produced by ``build_level_plans`` from the host setup (geometry/operators/
smoothing/transfer) and can be saved to / loaded from ``.npz`` so parity
fixtures do not depend on the host CPU's transcendental functions.

Reference data this replaces: ``SweepPlan`` (smoothing.py:80-109),
``ExtrapolationPlan`` (transfer.py:154-239) and the per-level classification
(geometry.py:134-156) of /root/reference/pkg/src/ghostmg.
"""

from dataclasses import dataclass, fields
from functools import cached_property

import numpy as np
import scipy.sparse as sp

from .geometry import GHOST, INTERNAL, UniformGrid, block_offsets
from .operators import check_ghost_rows, dirichlet_mask, ghost_row_weights
from .smoothing import assign_dtau
from .transfer import ghost_dag_levels


@dataclass
class LevelPlan:
    d: int
    N: int
    reaction: float
    labels: np.ndarray          # (n_nodes,) uint8, flat C order
    ghost_idx: np.ndarray       # (ng,) int64 ascending
    ghost_low: np.ndarray       # (ng, d) int64 lower block corner
    ghost_w: np.ndarray         # (ng, 3^d) float64 row weights
    ghost_dtau: np.ndarray      # (ng,) float64
    ghost_promoted: np.ndarray  # (ng,) bool
    ghost_batch: np.ndarray     # (ng,) int32 order-equivalent sweep batch
    bfs_len: np.ndarray         # (n_groups,) int64
    band_idx: np.ndarray        # (nb,) int64, groups concatenated
    bfs_mask: np.ndarray        # (nb,) uint8
    trans_step: np.ndarray      # (nb, d) int8
    trans_absn: np.ndarray      # (nb, d) float64

    @property
    def grid(self):
        return UniformGrid(self.d, self.N)

    @property
    def h(self):
        return 2.0 / self.N

    @property
    def h2(self):
        return self.h ** 2

    @property
    def denom(self):
        return 2.0 * self.d + self.reaction * self.h2

    @property
    def n_nodes(self):
        return (self.N + 1) ** self.d

    @property
    def n_ghosts(self):
        return len(self.ghost_idx)

    @property
    def n_band(self):
        return len(self.band_idx)

    @property
    def stencil_size(self):
        return 3 ** self.d

    @property
    def stencil(self):
        g = self.grid
        blocks = self.ghost_low[:, None, :] + block_offsets(self.d)[None, :, :]
        return (blocks * g.strides).sum(axis=-1)

    @cached_property
    def internal_idx(self):
        return np.flatnonzero(self.labels == INTERNAL)

    @cached_property
    def n_internal(self):
        return int(np.count_nonzero(self.labels == INTERNAL))

    # ---- persistence ---------------------------------------------------
    def to_arrays(self, prefix=""):
        out = {}
        for f in fields(self):
            out[prefix + f.name] = np.asarray(getattr(self, f.name))
        return out

    @classmethod
    def from_arrays(cls, arrays, prefix=""):
        kw = {}
        for f in fields(cls):
            v = arrays[prefix + f.name]
            if f.name in ("d", "N"):
                v = int(v)
            elif f.name == "reaction":
                v = float(v)
            else:
                v = np.asarray(v)
            kw[f.name] = v
        return cls(**kw)


def build_level_plan(level, spec, smoother, default_variant):
    """LevelPlan for one ``transfer.Level`` under a problem/smoother setup."""
    cls = level.cls
    d = cls.grid.d
    weights = ghost_row_weights(cls, spec.bc, spec.bc_selector)
    check_ghost_rows(cls, weights)
    dmask = dirichlet_mask(cls, spec)
    dtau = assign_dtau(cls, dmask, smoother, default_variant)
    ex = level.extrap
    nb = ex.n_band
    return LevelPlan(
        d=d,
        N=cls.grid.N,
        reaction=spec.reaction,
        labels=np.ascontiguousarray(cls.labels, dtype=np.uint8),
        ghost_idx=np.ascontiguousarray(cls.ghost_idx, dtype=np.int64),
        ghost_low=np.ascontiguousarray(cls.ghost_block_low, dtype=np.int64).reshape(-1, d),
        ghost_w=np.ascontiguousarray(weights, dtype=np.float64).reshape(-1, 3 ** d),
        ghost_dtau=np.ascontiguousarray(dtau, dtype=np.float64),
        ghost_promoted=np.ascontiguousarray(cls.ghost_promoted, dtype=bool),
        ghost_batch=ghost_dag_levels(cls, weights),
        bfs_len=np.array([len(g[0]) for g in ex.bfs_groups], dtype=np.int64),
        band_idx=np.ascontiguousarray(ex.band_idx, dtype=np.int64),
        bfs_mask=(np.concatenate([g[1] for g in ex.bfs_groups]) if nb else np.zeros(0, np.uint8)).astype(np.uint8),
        trans_step=np.ascontiguousarray(ex.trans_step, dtype=np.int8).reshape(-1, d),
        trans_absn=np.ascontiguousarray(ex.trans_absn, dtype=np.float64).reshape(-1, d),
    )


def coarsest_system(plan):
    """Sparse operator of the homogeneous coarsest problem over the active
    nodes (internal then ghost), built exactly like the reference's
    ``assemble_system`` with no data (operators.py:171-228, solver.py:146-154).
    Returns (A csr, active_idx)."""
    g = plan.grid
    h2 = g.h ** 2
    internal = plan.internal_idx
    ghosts = plan.ghost_idx
    ni = len(internal)
    active = np.concatenate([internal, ghosts])
    column = np.full(plan.n_nodes, -1, dtype=np.int64)
    column[active] = np.arange(len(active))
    rows = [np.arange(ni)]
    cols = [np.arange(ni)]
    vals = [np.full(ni, 2.0 * plan.d / h2 + plan.reaction)]
    for s in g.strides:
        for nb in (internal - s, internal + s):
            ok = column[nb] >= 0
            rows.append(np.flatnonzero(ok))
            cols.append(column[nb[ok]])
            vals.append(np.full(int(ok.sum()), -1.0 / h2))
    st = plan.stencil
    keep = (np.abs(plan.ghost_w) > 0.0) & (column[st] >= 0)
    gr, gc = np.nonzero(keep)
    rows.append(ni + gr)
    cols.append(column[st[gr, gc]])
    vals.append(plan.ghost_w[gr, gc])
    A = sp.csr_matrix(
        (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
        shape=(len(active), len(active)))
    return A, active


def save_plans(path, plans, **extra):
    arrays = {"n_levels": np.array(len(plans))}
    for i, p in enumerate(plans):
        arrays.update(p.to_arrays(prefix=f"L{i}_"))
    arrays.update({k: np.asarray(v) for k, v in extra.items()})
    np.savez_compressed(path, **arrays)


def load_plans(path):
    z = np.load(path, allow_pickle=False)
    n = int(z["n_levels"])
    plans = [LevelPlan.from_arrays(z, prefix=f"L{i}_") for i in range(n)]
    extra = {k: z[k] for k in z.files if not (k.startswith("L") and "_" in k and k.split("_")[0][1:].isdigit()) and k != "n_levels"}
    return plans, extra
