"""Uniform grid, node classification and ghost-point geometry (host setup).

Restates the reference's classification
(/root/reference/pkg/src/ghostmg/geometry.py) so that labels, ghost lists,
boundary projections Q, normals, theta and upwind blocks are bit-identical
to it on the same level set:

* grid nodes x_i = -1 + h*i, h = 2/N, C-order flat index (geometry.py:62-111)
* labels INTERNAL / GHOST / INACTIVE / ELIMINATED from the sign of phi plus
  the eliminated-face rule (geometry.py:374-431)
* ghost geometry: analytic normal, inward-ray projection (13 samples,
  48 bisections, <=6 batch-wide Newton polishes), upwind 3^d block
  (geometry.py:212-317, 449-505)
* promotion closure: inactive nodes read by a ghost row become ghosts with
  an extrapolation row (geometry.py:337-371, 432-446)

Differences that do not change any value:
* the sign of phi can come from ``phi.nonnegative_mask(grid)`` (no
  (N+1)^d x d coordinate array), otherwise phi is evaluated in slabs;
* ``internal_idx``/``inactive_idx``/``eliminated_idx`` are computed on first
  use from the labels (they are ~1e8-long at 512^3 and the device path never
  needs them);
* projections of regular ghosts are computed once per level and reused by
  every closure round (the regular-ghost batch is the same set in each
  round, so the batch-wide Newton stopping rule sees the same batch);
* the scalar Newton fallback evaluates the 1-D dot with an explicit FMA
  chain (what OpenBLAS ddot does for n < 16) instead of calling BLAS, so the
  result does not depend on the host CPU.
"""

from dataclasses import dataclass
from fractions import Fraction

import numpy as np

INTERNAL = np.uint8(0)
GHOST = np.uint8(1)
INACTIVE = np.uint8(2)
ELIMINATED = np.uint8(3)

FACE_LOW = 0
FACE_HIGH = 1

PROJECTION_TOL = 1e-10
THETA_CLAMP = 1.0 - 1e-9
WEIGHT_TOL = 1e-13
PROJECTION_ETA_MAX = 3.0
MAX_CLOSURE_ROUNDS = 64
THETA_TRUST = 1.6


class ResolutionError(RuntimeError):
    """Grid too coarse: a ghost stencil leaves the box or needs an inactive node."""


class DegenerateGradientError(RuntimeError):
    """|grad(phi)| ~ 0 where a normal direction is required."""


class ProjectionError(RuntimeError):
    """No boundary crossing found between a ghost and its inward ray."""


@dataclass(frozen=True)
class UniformGrid:
    """(N+1)^d nodes on [-1, 1]^d, spacing h = 2/N."""

    d: int
    N: int

    def __post_init__(self):
        if self.d not in (1, 2, 3):
            raise ValueError(f"dimension must be 1, 2 or 3, got {self.d}")
        if self.N < 2 or self.N % 2:
            raise ValueError(f"N must be even and >= 2, got {self.N}")

    @property
    def h(self):
        return 2.0 / self.N

    @property
    def shape(self):
        return (self.N + 1,) * self.d

    @property
    def n_nodes(self):
        return (self.N + 1) ** self.d

    @property
    def axis_coords(self):
        return -1.0 + self.h * np.arange(self.N + 1)

    @property
    def strides(self):
        n = self.N + 1
        return np.array([n ** (self.d - 1 - k) for k in range(self.d)], dtype=np.int64)

    def coords(self):
        axes = np.meshgrid(*([self.axis_coords] * self.d), indexing="ij")
        return np.stack([a.ravel() for a in axes], axis=-1)

    def multi_coords(self, multis):
        return -1.0 + self.h * np.asarray(multis, dtype=float)

    def flat_index(self, multis):
        multis = np.asarray(multis, dtype=np.int64)
        return (multis * self.strides).sum(axis=-1)

    def multi_index(self, flats):
        flats = np.asarray(flats, dtype=np.int64)
        n = self.N + 1
        out = np.empty(flats.shape + (self.d,), dtype=np.int64)
        rest = flats
        for k in range(self.d - 1, -1, -1):
            out[..., k] = rest % n
            rest = rest // n
        return out


class Classification:
    """Labels and ghost metadata of one grid level.

    Attribute names follow the reference's ``GridClassification``
    (geometry.py:134-156); the ghost arrays are aligned with ``ghost_idx``
    (ascending flat order).
    """

    def __init__(self, grid, phi, labels, phi_values=None):
        self.grid = grid
        self.phi = phi
        self.labels = labels
        self.phi_values = phi_values
        self.ghost_idx = np.flatnonzero(labels == GHOST)
        self.ghost_Q = self.ghost_n = self.ghost_theta = self.ghost_theta_raw = None
        self.ghost_stencil = self.ghost_block_low = self.ghost_promoted = None
        self._cache = {}

    def _indices(self, label):
        key = int(label)
        if key not in self._cache:
            self._cache[key] = np.flatnonzero(self.labels == label)
        return self._cache[key]

    def _relabelled(self):
        self._cache.clear()
        self.ghost_idx = np.flatnonzero(self.labels == GHOST)

    @property
    def internal_idx(self):
        return self._indices(INTERNAL)

    @property
    def inactive_idx(self):
        return self._indices(INACTIVE)

    @property
    def eliminated_idx(self):
        return self._indices(ELIMINATED)

    @property
    def n_ghosts(self):
        return len(self.ghost_idx)

    @property
    def n_internal(self):
        return int(np.count_nonzero(self.labels == INTERNAL))


# ---------------------------------------------------------------- helpers

def _seq_sum(terms):
    acc = terms[0]
    for t in terms[1:]:
        acc = acc + t
    return acc + 0.0


def raw_gradient(phi, points, h):
    """Analytic gradient when the shape has one, else central differences
    with step h (reference geometry.py:159-172)."""
    g = phi.gradient(points)
    if g is not None:
        return np.asarray(g, dtype=float)
    points = np.asarray(points, dtype=float)
    d = points.shape[-1]
    out = np.empty_like(points)
    for k in range(d):
        step = np.zeros(d)
        step[k] = h
        out[..., k] = (phi(points + step) - phi(points - step)) / (2.0 * h)
    return out


def compute_normal(phi, points, h):
    """grad/|grad| with |grad| = sqrt of the left-to-right sum of squares
    (numpy's vector 2-norm along the last axis)."""
    g = raw_gradient(phi, points, h)
    norm = np.sqrt(_seq_sum([g[..., k] * g[..., k] for k in range(g.shape[-1])]))
    if np.any(norm < 1e-12):
        raise DegenerateGradientError(
            f"level-set gradient vanishes (min |grad| = {norm.min():.3e})")
    return g / norm[..., None]


def lagrange_quad(t):
    """Quadratic Lagrange basis on {0, 1, 2} evaluated at t: (..., 3)."""
    t = np.asarray(t, dtype=float)
    return np.stack([(t - 1.0) * (t - 2.0) / 2.0, t * (2.0 - t), t * (t - 1.0) / 2.0], axis=-1)


def lagrange_quad_deriv(t):
    t = np.asarray(t, dtype=float)
    return np.stack([t - 1.5, 2.0 - 2.0 * t, t - 0.5], axis=-1)


def tensor_weights(factors):
    """(ng, d, 3) per-axis triples -> (ng, 3^d) products, axis 0 slowest;
    each entry is ((1*f0)*f1)*f2."""
    ng, d, _ = factors.shape
    w = np.ones((ng, 1))
    for k in range(d):
        w = (w[:, :, None] * factors[:, k, None, :]).reshape(ng, -1)
    return w


def block_offsets(d, width=3, start=0):
    """C-ordered offsets of a width^d block (axis 0 slowest)."""
    grids = np.meshgrid(*([np.arange(start, start + width)] * d), indexing="ij")
    return np.stack([g.ravel() for g in grids], axis=-1).astype(np.int64)


def stencil_flats(grid, lows):
    """Flat indices of the 3^d blocks with lower corners ``lows`` (ng, d)."""
    blocks = lows[:, None, :] + block_offsets(grid.d)[None, :, :]
    return (blocks * grid.strides).sum(axis=-1)


# ------------------------------------------------------- boundary projection

def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _newton_scalar(phi, point, normal, h):
    """Scalar Newton from eta = 0.5 for a ghost whose sampled ray did not
    bracket a crossing (reference geometry.py:286-302)."""
    eta = 0.5
    tol = 1e-12 * max(1.0, abs(float(phi(point[None, :])[0])))
    for _ in range(60):
        q = point - eta * h * normal
        v = float(phi(q[None, :])[0])
        if abs(v) <= tol:
            if -1e-9 <= eta < PROJECTION_ETA_MAX:
                return min(max(eta, 0.0), PROJECTION_ETA_MAX)
            break
        grad = raw_gradient(phi, q[None, :], h)[0]
        dot = 0.0
        for gk, nk in zip(grad, normal):
            dot = _fma(float(gk), float(nk), dot)
        dpsi = -h * dot
        if dpsi == 0.0:
            break
        eta -= v / dpsi
        if not -0.5 <= eta <= PROJECTION_ETA_MAX + 0.5:
            break
    raise ProjectionError("no boundary crossing along the inward normal ray")


def project_to_boundary(phi, points, normals, h):
    """First crossing Q = G - eta*h*n along the inward ray, per ghost.

    Sampling at eta = 0, 0.25, ..., 3 brackets the first sign change,
    48 bisections narrow it and up to 6 Newton steps polish it; the Newton
    loop stops as soon as every ghost of the batch is converged
    (reference geometry.py:212-283).  Returns (Q, eta).
    """
    points = np.atleast_2d(np.asarray(points, dtype=float))
    normals = np.atleast_2d(np.asarray(normals, dtype=float))
    ng = points.shape[0]
    samples = np.linspace(0.0, PROJECTION_ETA_MAX, int(PROJECTION_ETA_MAX / 0.25) + 1)

    def along(eta, pts, nrm):
        return pts - eta[:, None] * h * nrm

    vals = np.stack([phi(along(np.full(ng, s), points, normals)) for s in samples])
    if np.any(vals[0] < 0.0):
        raise ProjectionError("projection started from a point inside the domain")

    lo = np.zeros(ng)
    hi = np.full(ng, np.nan)
    done = vals[0] == 0.0
    bracketed = done.copy()
    eta = np.zeros(ng)
    for k in range(len(samples) - 1):
        hit = ~bracketed & (vals[k] > 0.0) & (vals[k + 1] <= 0.0)
        lo[hit] = samples[k]
        hi[hit] = samples[k + 1]
        bracketed |= hit

    for g in np.flatnonzero(~bracketed):
        eta[g] = _newton_scalar(phi, points[g], normals[g], h)
        done[g] = bracketed[g] = True

    act = np.flatnonzero(bracketed & ~done)
    if act.size:
        a_lo, a_hi = lo[act], hi[act]
        pts, nrm = points[act], normals[act]
        for _ in range(48):
            mid = 0.5 * (a_lo + a_hi)
            neg = phi(along(mid, pts, nrm)) <= 0.0
            a_hi = np.where(neg, mid, a_hi)
            a_lo = np.where(neg, a_lo, mid)
        e = 0.5 * (a_lo + a_hi)
        scale = np.maximum(1.0, np.abs(phi(pts)))
        for _ in range(6):
            q = along(e, pts, nrm)
            v = phi(q)
            if np.all(np.abs(v) <= 1e-12 * scale):
                break
            grad = raw_gradient(phi, q, h)
            dpsi = -h * _seq_sum([grad[:, k] * nrm[:, k] for k in range(nrm.shape[1])])
            with np.errstate(divide="ignore", invalid="ignore"):
                step = np.where(np.abs(dpsi) > 1e-300, v / dpsi, 0.0)
            e = np.clip(e - step, 0.0, PROJECTION_ETA_MAX)
        eta[act] = e

    Q = along(eta, points, normals)
    resid = np.abs(phi(Q))
    if np.any(resid > PROJECTION_TOL * np.maximum(1.0, np.abs(vals[0]))):
        raise ProjectionError(f"projection residual {resid.max():.3e} above tolerance")
    return Q, eta


def upwind_lows(grid, multis, normals):
    """Lower block corners: i-2 where n>0, i where n<0, i-1 where n==0
    (reference geometry.py:305-317), vectorised over ghosts."""
    lows = np.where(normals > 0.0, multis - 2, np.where(normals < 0.0, multis, multis - 1))
    bad = np.any((lows < 0) | (lows + 2 > grid.N), axis=1)
    if np.any(bad):
        m = multis[np.flatnonzero(bad)[0]]
        raise ResolutionError(
            f"ghost stencil at node {tuple(int(x) for x in m)} leaves the box")
    return lows.astype(np.int64)


def extrapolation_row_weights(cls):
    """(1, -2, 1) along the dominant normal axis through the ghost's own
    plane on the other axes (reference geometry.py:320-345)."""
    grid = cls.grid
    ng = cls.n_ghosts
    if ng == 0:
        return np.zeros((0, 3 ** grid.d))
    offs = grid.multi_index(cls.ghost_idx) - cls.ghost_block_low
    dom = np.argmax(np.abs(cls.ghost_n), axis=1)
    factors = np.zeros((ng, grid.d, 3))
    rows = np.arange(ng)
    factors[rows[:, None], np.arange(grid.d)[None, :], offs] = 1.0
    factors[rows, dom, :] = (1.0, -2.0, 1.0)
    return tensor_weights(factors)


def _interp_factors(cls):
    t = (cls.ghost_Q - cls.grid.multi_coords(cls.ghost_block_low)) / cls.grid.h
    return lagrange_quad(t), lagrange_quad_deriv(t)


def ghost_row_support(cls):
    """Stencil entries any boundary-row variant may read (|w| > WEIGHT_TOL)."""
    values, derivs = _interp_factors(cls)
    support = np.abs(tensor_weights(values)) > WEIGHT_TOL
    for k in range(cls.grid.d):
        f = values.copy()
        f[:, k, :] = derivs[:, k, :]
        support |= np.abs(tensor_weights(f)) > WEIGHT_TOL
    prom = cls.ghost_promoted
    if prom.any():
        support[prom] = np.abs(extrapolation_row_weights(cls)[prom]) > WEIGHT_TOL
    return support


# ------------------------------------------------------------ classification

def _sign_negative(grid, phi):
    """Boolean grid of phi < 0 plus the phi values when they were computed."""
    fast = getattr(phi, "nonnegative_mask", None)
    if fast is not None:
        return ~fast(grid), None
    n_nodes = grid.n_nodes
    vals = np.empty(n_nodes)
    axes = grid.axis_coords
    # slabs along axis 0; phi is pointwise so slab evaluation is exact
    inner = n_nodes // (grid.N + 1)
    rest = np.meshgrid(*([axes] * (grid.d - 1)), indexing="ij") if grid.d > 1 else []
    rest = [r.ravel() for r in rest]
    per = max(1, (1 << 22) // max(inner, 1))
    for i0 in range(0, grid.N + 1, per):
        i1 = min(grid.N + 1, i0 + per)
        x0 = np.repeat(axes[i0:i1], inner)
        cols = [x0] + [np.tile(r, i1 - i0) for r in rest]
        vals[i0 * inner:i1 * inner] = phi(np.stack(cols, axis=-1))
    return (vals < 0.0).reshape(grid.shape), vals


def _device_labels(grid, phi, eliminated_faces, device):
    """Labels before the promotion closure, computed on GPU `device` for
    level sets of the ball family (``phi.device_spec()``); None otherwise."""
    spec = getattr(phi, "device_spec", None)
    if device is None or spec is None or grid.d not in (2, 3):
        return None
    from . import _lib

    kind, centers, radii = spec()
    mask = 0
    for axis, side in eliminated_faces:
        mask |= 1 << (2 * axis + (0 if side == FACE_LOW else 1))
    return _lib.setup_classify_balls(device, grid.d, grid.N, grid.axis_coords, kind, centers, radii, mask)


def classify(grid, phi, eliminated_faces=(), device=None):
    """Label every node and attach ghost geometry (reference
    geometry.py:374-446).  With ``device`` (a CUDA ordinal) and a level set of
    the ball family the per-node part -- sign of phi, faces, internal
    neighbours -- runs on the GPU (bit-identical labels); the ghost geometry
    and the promotion closure stay here, on the whole ghost batch."""
    labels = _device_labels(grid, phi, eliminated_faces, device)
    if labels is not None:
        return _close_ghosts(Classification(grid, phi, labels, None), phi)
    neg, phi_vals = _sign_negative(grid, phi)
    d, N = grid.d, grid.N
    shape = grid.shape

    def face(axis, index):
        sl = [slice(None)] * d
        sl[axis] = index
        return tuple(sl)

    on_box = np.zeros(shape, dtype=bool)
    for k in range(d):
        on_box[face(k, 0)] = True
        on_box[face(k, N)] = True
    eliminated = on_box & neg
    for axis, side in eliminated_faces:
        eliminated[face(axis, 0 if side == FACE_LOW else N)] = True
    internal = neg & ~eliminated
    del neg, on_box

    near_internal = np.zeros(shape, dtype=bool)
    for k in range(d):
        lo = [slice(None)] * d
        hi = [slice(None)] * d
        lo[k] = slice(None, -1)
        hi[k] = slice(1, None)
        near_internal[tuple(lo)] |= internal[tuple(hi)]
        near_internal[tuple(hi)] |= internal[tuple(lo)]
    ghost = near_internal & ~internal & ~eliminated
    del near_internal

    labels = np.full(shape, INACTIVE, dtype=np.uint8)
    labels[internal] = INTERNAL
    labels[eliminated] = ELIMINATED
    labels[ghost] = GHOST
    del internal, eliminated, ghost
    labels = labels.reshape(-1)

    return _close_ghosts(Classification(grid, phi, labels, phi_vals), phi)


def _close_ghosts(cls, phi):
    """Ghost geometry + the promotion closure (geometry.py:419-446)."""
    promoted = np.zeros(0, dtype=np.int64)
    projection_cache = {}
    for _ in range(MAX_CLOSURE_ROUNDS):
        _attach_ghost_geometry(cls, phi, promoted, projection_cache)
        stencil_labels = cls.labels[cls.ghost_stencil]
        hit = (stencil_labels == INACTIVE)
        if hit.any():
            hit &= ghost_row_support(cls)
        referenced = cls.ghost_stencil[hit]
        if referenced.size == 0:
            return cls
        referenced = np.unique(referenced)
        promoted = np.union1d(promoted, referenced)
        cls.labels[referenced] = GHOST
        cls._relabelled()
    raise ResolutionError("ghost closure did not terminate; refine the grid")


def _attach_ghost_geometry(cls, phi, promoted_flats, projection_cache):
    grid = cls.grid
    h = grid.h
    d = grid.d
    idx = cls.ghost_idx
    ng = len(idx)
    if ng == 0:
        cls.ghost_Q = np.zeros((0, d))
        cls.ghost_n = np.zeros((0, d))
        cls.ghost_theta = np.zeros(0)
        cls.ghost_theta_raw = np.zeros(0)
        cls.ghost_promoted = np.zeros(0, dtype=bool)
        cls.ghost_stencil = np.zeros((0, 3 ** d), dtype=np.int64)
        cls.ghost_block_low = np.zeros((0, d), dtype=np.int64)
        return
    multis = grid.multi_index(idx)
    pts = grid.multi_coords(multis)
    normals = compute_normal(phi, pts, h)
    promoted = np.isin(idx, promoted_flats)
    regular = ~promoted
    Q = pts.copy()
    eta = np.zeros(ng)
    if regular.any():
        reg_idx = idx[regular]
        key = "regular"
        hit = projection_cache.get(key)
        if hit is not None and np.array_equal(hit[0], reg_idx):
            Q_r, eta_r = hit[1], hit[2]
        else:
            Q_r, eta_r = project_to_boundary(phi, pts[regular], normals[regular], h)
            projection_cache[key] = (reg_idx, Q_r, eta_r)
        Q[regular] = Q_r
        eta[regular] = eta_r
    lows = upwind_lows(grid, multis, normals)
    cls.ghost_Q = Q
    cls.ghost_n = normals
    cls.ghost_theta = np.minimum(eta, THETA_CLAMP)
    cls.ghost_theta_raw = eta
    cls.ghost_promoted = promoted
    cls.ghost_block_low = lows
    cls.ghost_stencil = stencil_flats(grid, lows)
