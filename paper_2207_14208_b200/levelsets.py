"""Level-set domains {phi < 0} on the box [-1, 1]^d.

The base protocol is the reference's (/root/reference/pkg/src/ghostmg/
levelsets.py:12-22): ``phi(points)`` on arrays of shape (..., d) and an
optional analytic ``gradient(points)``.  The reference shapes (Constant,
HalfSpace, quadratic Sphere, Ellipsoid, Flower; levelsets.py:25-135) are
restated with the same floating-point expression order so node signs, ghost
projections and normals come out bit-identical.

New shapes needed by the BASELINE configs:

* ``SignedSphere``: signed distance |x - c| - R (configs 1 and 3).
* ``PoreSpace``: the complement of a union of balls, phi = max_k (r_k - |x -
  c_k|), with the gradient of the arg-max ball (configs 4 and 5).  It keeps a
  coarse-cell candidate table so phi at a point only evaluates the balls that
  can attain the maximum there; the maximum over a superset of the attaining
  balls is exactly the full maximum, so values are bitwise those of the
  all-balls formula.

Optional fast path used by ``geometry.classify``: ``nonnegative_mask(grid)``
returns the boolean grid of nodes with phi >= 0 without materialising the
(N+1)^d x d coordinate array.
"""

import numpy as np


class LevelSet:
    d = None

    def __call__(self, points):
        raise NotImplementedError

    def gradient(self, points):
        return None


class Constant(LevelSet):
    def __init__(self, d, value=-1.0):
        self.d = int(d)
        self.value = float(value)

    def __call__(self, points):
        points = np.asarray(points, dtype=float)
        return np.full(points.shape[:-1], self.value)


def _rowsum(terms):
    """Left-to-right sum of a short list of arrays (numpy's axis sum for
    fewer than 8 terms, normalising -0 to +0 like numpy's reduction)."""
    acc = terms[0]
    for t in terms[1:]:
        acc = acc + t
    return acc + 0.0


class HalfSpace(LevelSet):
    """phi = coeffs . x + offset.

    Evaluated term by term without BLAS.  For the axis-aligned cases
    (coefficients 0/1) this is exact and matches the reference's
    ``points @ coeffs`` bit for bit on every CPU.
    """

    def __init__(self, coeffs, offset):
        self.coeffs = np.asarray(coeffs, dtype=float)
        self.offset = float(offset)
        self.d = self.coeffs.size

    def __call__(self, points):
        points = np.asarray(points, dtype=float)
        dot = _rowsum([points[..., k] * self.coeffs[k] for k in range(self.d)])
        return dot + self.offset

    def gradient(self, points):
        points = np.asarray(points, dtype=float)
        return np.broadcast_to(self.coeffs, points.shape).copy()


def axis_halfspace(d, cutoff, axis=0):
    coeffs = np.zeros(d)
    coeffs[axis] = 1.0
    return HalfSpace(coeffs, -float(cutoff))


class Sphere(LevelSet):
    """Quadratic form sum((x - c)^2) - R^2 (reference levelsets.py:61-75)."""

    def __init__(self, center, radius):
        self.center = np.asarray(center, dtype=float)
        self.radius = float(radius)
        self.d = self.center.size

    def __call__(self, points):
        points = np.asarray(points, dtype=float)
        diff = points - self.center
        return _rowsum([diff[..., k] * diff[..., k] for k in range(self.d)]) - self.radius ** 2

    def gradient(self, points):
        points = np.asarray(points, dtype=float)
        return 2.0 * (points - self.center)


class Ellipsoid(LevelSet):
    def __init__(self, center, semiaxes):
        self.center = np.asarray(center, dtype=float)
        self.semiaxes = np.asarray(semiaxes, dtype=float)
        self.d = self.center.size

    def __call__(self, points):
        points = np.asarray(points, dtype=float)
        q = (points - self.center) / self.semiaxes
        return _rowsum([q[..., k] * q[..., k] for k in range(self.d)]) - 1.0

    def gradient(self, points):
        points = np.asarray(points, dtype=float)
        return 2.0 * (points - self.center) / self.semiaxes ** 2


class Flower(LevelSet):
    """r - r1 - r2 * Im((x+iy)^5)/r^5 (reference levelsets.py:95-135).

    Integer powers go through numpy's ``power`` exactly as in the
    reference; ``**2`` is numpy's square (a plain product).
    """

    d = 2

    def __init__(self, r1=0.5, r2=0.2):
        self.r1 = float(r1)
        self.r2 = float(r2)

    @staticmethod
    def _parts(points):
        points = np.asarray(points, dtype=float)
        x = points[..., 0]
        y = points[..., 1]
        r = np.sqrt(x * x + y * y)
        s = y ** 5 + 5.0 * x ** 4 * y - 10.0 * x ** 2 * y ** 3
        return x, y, r, s

    def __call__(self, points):
        x, y, r, s = self._parts(points)
        with np.errstate(divide="ignore", invalid="ignore"):
            ratio = np.where(r > 0.0, s / r ** 5, 0.0)
        return r - self.r1 - self.r2 * ratio

    def gradient(self, points):
        x, y, r, s = self._parts(points)
        sx = 20.0 * x ** 3 * y - 20.0 * x * y ** 3
        sy = 5.0 * y ** 4 + 5.0 * x ** 4 - 30.0 * x ** 2 * y ** 2
        with np.errstate(divide="ignore", invalid="ignore"):
            gx = np.where(r > 0.0, x / r - self.r2 * (sx / r ** 5 - 5.0 * s * x / r ** 7), 1.0)
            gy = np.where(r > 0.0, y / r - self.r2 * (sy / r ** 5 - 5.0 * s * y / r ** 7), 0.0)
        return np.stack([gx, gy], axis=-1)


class SignedSphere(LevelSet):
    """Signed distance |x - c| - R; gradient (x - c)/|x - c|.

    The disk of config 1 and the ball of config 3 (BASELINE.json configs[0],
    configs[2]).  |x - c| is sqrt of the left-to-right sum of squares.
    """

    def __init__(self, center, radius):
        self.center = np.asarray(center, dtype=float)
        self.radius = float(radius)
        self.d = self.center.size

    def _dist(self, points):
        diff = np.asarray(points, dtype=float) - self.center
        return diff, np.sqrt(_rowsum([diff[..., k] * diff[..., k] for k in range(self.d)]))

    def __call__(self, points):
        return self._dist(points)[1] - self.radius

    def gradient(self, points):
        diff, r = self._dist(points)
        with np.errstate(divide="ignore", invalid="ignore"):
            return diff / r[..., None]

    def device_spec(self):
        """(kind, centers, radii) for gmg_setup_classify_balls (kind 1:
        the domain is the inside of one ball)."""
        return 1, self.center.reshape(1, -1), np.array([self.radius])


class PoreSpace(LevelSet):
    """Exterior of a union of balls: phi = max_k (r_k - |x - c_k|).

    Per ball the value is ``r_k - sqrt(((dx*dx + dy*dy) + dz*dz))`` with
    ``dx = x - c_k[0]``; the maximum keeps the first ball on ties (numpy
    argmax), and ``gradient`` is -(x - c_k)/|x - c_k| of that ball, i.e. the
    gradient of the maximising branch.
    """

    CELLS = 40          # candidate-table resolution per axis
    LO, HI = -1.5, 1.5  # candidate-table extent

    def __init__(self, centers, radii):
        self.centers = np.ascontiguousarray(np.asarray(centers, dtype=float))
        self.radii = np.ascontiguousarray(np.asarray(radii, dtype=float))
        self.d = self.centers.shape[1]
        self._build_candidates()

    # -- candidate table ------------------------------------------------
    def _build_candidates(self):
        m, d = self.CELLS, self.d
        width = (self.HI - self.LO) / m
        idx = np.stack(np.meshgrid(*([np.arange(m)] * d), indexing="ij"), -1).reshape(-1, d)
        lo = self.LO + width * idx
        hi = lo + width
        c = self.centers[None, :, :]
        near = np.clip(c, lo[:, None, :], hi[:, None, :])
        dmin = np.sqrt(((near - c) ** 2).sum(-1))
        far = np.maximum(np.abs(lo[:, None, :] - c), np.abs(hi[:, None, :] - c))
        dmax = np.sqrt((far ** 2).sum(-1))
        upper = self.radii[None, :] - dmin
        lower = (self.radii[None, :] - dmax).max(axis=1)
        self._cand = upper >= lower[:, None] - 1e-6       # (cells, balls)
        self._cell_width = width
        # CSR of ascending candidate balls per cell
        self._cand_count = self._cand.sum(axis=1).astype(np.int64)
        self._cand_ptr = np.zeros(len(self._cand_count) + 1, dtype=np.int64)
        np.cumsum(self._cand_count, out=self._cand_ptr[1:])
        self._cand_list = np.nonzero(self._cand)[1].astype(np.int64)

    def _cells_of(self, pts):
        m = self.CELLS
        k = np.floor((pts - self.LO) / self._cell_width).astype(np.int64)
        outside = np.any((k < 0) | (k >= m), axis=-1)
        k = np.clip(k, 0, m - 1)
        flat = np.zeros(pts.shape[0], dtype=np.int64)
        for a in range(self.d):
            flat = flat * m + k[:, a]
        return flat, outside

    def _ball_value(self, pts, k):
        c = self.centers[k]
        dist = np.sqrt(_rowsum([(pts[:, a] - c[a]) * (pts[:, a] - c[a]) for a in range(self.d)]))
        return self.radii[k] - dist

    def _max_and_arg(self, points):
        """phi and the first maximising ball per point.  Every point is
        paired with the candidate balls of its cell (all balls outside the
        table); values of the pairs are reduced per point."""
        pts = np.asarray(points, dtype=float)
        shape = pts.shape[:-1]
        pts = pts.reshape(-1, self.d)
        n = pts.shape[0]
        if n == 0:
            return np.full(shape, -np.inf), np.zeros(shape, dtype=np.int64)
        cells, outside = self._cells_of(pts)
        nball = len(self.radii)
        counts = self._cand_count[cells]
        counts[outside] = nball
        starts = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=starts[1:])
        total = int(starts[-1])
        owner = np.repeat(np.arange(n), counts)
        rank = np.arange(total) - starts[owner]
        cell_of = cells[owner]
        ball = np.where(outside[owner], rank, self._cand_list[self._cand_ptr[cell_of] + rank])
        c = self.centers[ball]
        sq = None
        for a in range(self.d):
            t = pts[owner, a] - c[:, a]
            sq = t * t if sq is None else sq + t * t
        vals = self.radii[ball] - np.sqrt(sq + 0.0)
        best = np.maximum.reduceat(vals, starts[:-1])
        hit = vals == best[owner]
        arg = np.minimum.reduceat(np.where(hit, ball, nball), starts[:-1])
        return best.reshape(shape), arg.reshape(shape)

    def __call__(self, points):
        return self._max_and_arg(points)[0]

    def gradient(self, points):
        pts = np.asarray(points, dtype=float)
        _, arg = self._max_and_arg(pts)
        diff = pts - self.centers[arg]
        dist = np.sqrt(_rowsum([diff[..., a] * diff[..., a] for a in range(self.d)]))
        with np.errstate(divide="ignore", invalid="ignore"):
            return -diff / dist[..., None]

    def device_spec(self):
        """(kind, centers, radii) for gmg_setup_classify_balls (kind 0:
        the domain is the outside of every ball)."""
        return 0, self.centers, self.radii

    # -- classify fast path -------------------------------------------------
    def nonnegative_mask(self, grid):
        """Boolean grid (grid.shape) of nodes with phi >= 0, i.e. inside or on
        some ball.  Only each ball's bounding index box is visited; outside
        it r_k - |x - c_k| < 0 holds with a full cell of margin."""
        mask = np.zeros(grid.shape, dtype=bool)
        h = grid.h
        for k in range(len(self.radii)):
            c, r = self.centers[k], self.radii[k]
            lo = np.maximum(np.floor((c - r + 1.0) / h).astype(np.int64) - 2, 0)
            hi = np.minimum(np.ceil((c + r + 1.0) / h).astype(np.int64) + 2, grid.N)
            if np.any(hi < lo):
                continue
            axes = [grid.axis_coords[lo[a]:hi[a] + 1] for a in range(self.d)]
            sq = None
            for a in range(self.d):
                shp = [1] * self.d
                shp[a] = -1
                t = (axes[a] - c[a]).reshape(shp)
                sq = t * t if sq is None else sq + t * t
            inside = (r - np.sqrt(sq + 0.0)) >= 0.0
            sl = tuple(slice(lo[a], hi[a] + 1) for a in range(self.d))
            mask[sl] |= inside
        return mask


def rejection_sample_balls(seed, count, r_lo, r_hi, gap=0.04, margin=0.04, max_draws=10_000_000):
    """Seeded non-overlapping balls in the unit cube.

    Candidates are drawn from ``XorShift64Star(seed).uniform()`` in the order
    cx, cy, cz, then r = r_lo + (r_hi - r_lo) * U.  A candidate is rejected if
    it comes within ``margin`` of a cube face or within ``gap`` of an
    accepted ball.  Returns (centers, radii) in unit-cube coordinates.
    """
    from .rng import XorShift64Star

    rng = XorShift64Star(seed)
    centers, radii = [], []
    draws = 0
    while len(radii) < count:
        if draws >= max_draws:
            raise RuntimeError("rejection sampler did not place every ball")
        draws += 1
        c = [rng.uniform() for _ in range(3)]
        r = r_lo + (r_hi - r_lo) * rng.uniform()
        if any(ci - r < margin or ci + r > 1.0 - margin for ci in c):
            continue
        ok = True
        for cj, rj in zip(centers, radii):
            dist = ((c[0] - cj[0]) ** 2 + (c[1] - cj[1]) ** 2 + (c[2] - cj[2]) ** 2) ** 0.5
            if dist < r + rj + gap:
                ok = False
                break
        if ok:
            centers.append(c)
            radii.append(r)
    return np.asarray(centers), np.asarray(radii), draws


def pore_space_unit_cube(seed, count, r_lo, r_hi):
    """PoreSpace in reference coordinates for balls sampled in [0, 1]^3:
    x_ref = 2 x - 1 maps centres to 2c - 1 and radii to 2r."""
    centers, radii, _ = rejection_sample_balls(seed, count, r_lo, r_hi)
    return PoreSpace(2.0 * centers - 1.0, 2.0 * radii)
