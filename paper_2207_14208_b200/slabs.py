"""z-slab decomposition of the V-cycle over ranks.

The fine grid is cut along the reference's axis 0 (the slowest stride of the
C-order flat index, /root/reference/pkg/src/ghostmg/geometry.py:108-111), so
each rank owns a contiguous range of planes and lexicographic order puts
every node of rank p before every node of rank p+1.  Coarse plane I belongs
to the owner of fine plane 2I (slab boundaries sit on even fine planes);
once a level would leave a rank fewer than ``min_planes`` planes it is
agglomerated onto rank 0, which runs the rest of the cycle alone.

``SlabCycle`` is the exchange schedule of one V-cycle
(reference solver.py:170-203) over any backend that can apply each operation
to the nodes of a plane range, and a torch.distributed process group:

* GS-LEX (smoothing.py:127-132) and the ghost sweep (smoothing.py:135-142)
  are pipelined in rank order: rank p first receives the *old* first planes
  of rank p+1, then waits for the *new* last planes of rank p-1, sweeps its
  own nodes and forwards its last planes -- exactly the values the
  single-process lexicographic sweep sees;
* residuals, band extrapolation steps (transfer.py:241-252), restrictions and
  the interpolation read neighbour planes refreshed by halo exchanges
  (1 plane; 2 for the 3^d ghost stencils);
* the residual norm is a MAX all-reduce (order-free, bit-exact);
* gathers into the agglomerated level select each plane from its owner
  (no arithmetic), so the decomposed cycle is bitwise the single-process one.

On B200s the same schedule maps onto one rank per GPU with the pipelined
sweeps handing tiles over NVLink peer memory; tests/test_slabs.py runs it
with the CPU oracle as backend on gloo (world sizes 2 and 3) and checks
every iterate bit for bit against the single-process oracle.
"""

from dataclasses import dataclass

import numpy as np


@dataclass
class LevelSlabs:
    N: int
    bounds: list  # plane boundaries, len world+1; None: agglomerated on rank 0


class SlabPartition:
    """Plane ownership of every level."""

    def __init__(self, Ns, world, min_planes=4):
        self.world = world
        self.levels = []
        N0 = Ns[0]
        b = [0]
        for r in range(1, world):
            b.append(2 * int(round(r * (N0 + 1) / (2.0 * world))))
        b.append(N0 + 1)
        bounds = b if world > 1 and min(np.diff(b)) >= min_planes else None
        for li, N in enumerate(Ns):
            if li > 0 and bounds is not None:
                if any(x % 2 for x in bounds[1:-1]):
                    bounds = None  # an odd boundary has no coarse counterpart: agglomerate
                else:
                    nb = [0] + [x // 2 for x in bounds[1:-1]] + [N + 1]
                    bounds = nb if min(np.diff(nb)) >= min_planes else None
            if li == len(Ns) - 1:
                bounds = None  # the coarsest solve runs on rank 0
            self.levels.append(LevelSlabs(N, list(bounds) if bounds is not None else None))

    def distributed(self, level):
        return self.levels[level].bounds is not None

    def planes(self, level, rank):
        """Owned plane range [lo, hi) of ``rank`` (rank 0 owns everything on
        an agglomerated level)."""
        L = self.levels[level]
        if L.bounds is None:
            return (0, L.N + 1) if rank == 0 else (0, 0)
        return L.bounds[rank], L.bounds[rank + 1]


class SlabCycle:
    """One V-cycle over plane slabs.  ``backend`` provides the per-range
    operations (see tests/test_slabs.py for the oracle backend); ``dist`` is
    ``torch.distributed`` with an initialised process group."""

    def __init__(self, backend, partition, dist, rank, halo_ghost=2):
        self.be = backend
        self.part = partition
        self.dist = dist
        self.rank = rank
        self.world = partition.world
        self.hg = halo_ghost

    # ---- plane transport -------------------------------------------------
    def _plane_slice(self, level, lo, hi):
        n = self.part.levels[level].N + 1
        per = n ** (self.be.plans[level].d - 1)
        return slice(lo * per, hi * per)

    def _send(self, level, arr, lo, hi, dst):
        import torch

        if hi <= lo:
            return
        self.dist.send(torch.from_numpy(np.ascontiguousarray(arr[self._plane_slice(level, lo, hi)])), dst)

    def _recv(self, level, arr, lo, hi, src):
        import torch

        if hi <= lo:
            return
        sl = self._plane_slice(level, lo, hi)
        buf = torch.empty(sl.stop - sl.start, dtype=torch.float64)
        self.dist.recv(buf, src)
        arr[sl] = buf.numpy()

    def halo(self, level, arr, width):
        """Refresh ``width`` planes on both sides of the owned range from the
        neighbouring ranks."""
        if not self.part.distributed(level) or self.world == 1:
            return
        lo, hi = self.part.planes(level, self.rank)
        N = self.part.levels[level].N
        r = self.rank
        # even ranks send first, odd ranks receive first (no deadlock with blocking p2p)
        order = (0, 1) if r % 2 == 0 else (1, 0)
        for phase in order:
            if phase == 0:
                if r + 1 < self.world:
                    self._send(level, arr, max(lo, hi - width), hi, r + 1)
                if r > 0:
                    self._send(level, arr, lo, min(hi, lo + width), r - 1)
            else:
                if r > 0:
                    plo, _ = self.part.planes(level, r - 1)
                    self._recv(level, arr, max(plo, lo - width), lo, r - 1)
                if r + 1 < self.world:
                    _, nhi = self.part.planes(level, r + 1)
                    self._recv(level, arr, hi, min(nhi, hi + width, N + 1), r + 1)

    def _pipelined(self, level, arr, width, sweep):
        """Rank-ordered sweep: old first planes of the next rank, then the new
        last planes of the previous one, then this rank's sweep."""
        if not self.part.distributed(level) or self.world == 1:
            sweep()
            return
        self.halo(level, arr, width)  # old values on both sides
        lo, hi = self.part.planes(level, self.rank)
        if self.rank > 0:
            plo, _ = self.part.planes(level, self.rank - 1)
            self._recv(level, arr, max(plo, lo - width), lo, self.rank - 1)
        sweep()
        if self.rank + 1 < self.world:
            self._send(level, arr, max(lo, hi - width), hi, self.rank + 1)

    # ---- operations ------------------------------------------------------
    def smooth(self, level, u, f, g, count):
        lo, hi = self.part.planes(level, self.rank)
        for _ in range(count):
            self._pipelined(level, u, 1, lambda: self.be.gs_sweep(level, u, f, lo, hi))
            self._pipelined(level, u, self.hg, lambda: self.be.ghost_sweep(level, u, g, lo, hi))

    def extrapolate(self, level, x):
        lo, hi = self.part.planes(level, self.rank)
        for grp in range(self.be.n_bfs_groups(level)):
            self.halo(level, x, 1)
            self.be.band_bfs(level, x, grp, lo, hi)
        for _ in range(6):
            self.halo(level, x, 1)
            self.be.band_transport(level, x, lo, hi)

    def residual_norm(self, u, f, g):
        import torch

        lo, hi = self.part.planes(0, self.rank)
        self.halo(0, u, self.hg)
        m = self.be.residual_norm(0, u, f, g, lo, hi)
        t = torch.tensor([m], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def cycle(self, level, u, f, g):
        """Reference _cycle (solver.py:170-199) with level ``level``
        distributed over the ranks."""
        be = self.be
        lo, hi = self.part.planes(level, self.rank)
        self.smooth(level, u, f, g, be.nu1)
        self.halo(level, u, self.hg)
        r_int = be.residual_internal(level, u, f, lo, hi)
        r_ext = be.residual_ghost_ext(level, u, g, lo, hi)
        self.extrapolate(level, r_ext)
        self.halo(level, r_int, 1)
        self.halo(level, r_ext, 1)
        c = level + 1
        if self.part.distributed(c):
            clo, chi = self.part.planes(c, self.rank)
            f_c = be.restrict_interior(level, r_int, clo, chi)
            g_c = be.restrict_ghost(level, r_ext, clo, chi)
            e = np.zeros(be.plans[c].n_nodes)
            for _ in range(be.gamma):
                self.cycle(c, e, f_c, g_c)
            self.extrapolate(c, e)
            self.halo(c, e, 1)
        else:
            # restrict the coarse planes I with 2I in this rank's fine slab,
            # gather them on every rank, finish the cycle on rank 0 (the
            # recursion, the coarsest solve and the coarse band extension),
            # broadcast the coarse error
            lo_c, hi_c = (lo + 1) // 2, (hi + 1) // 2
            f_c = self._gather_coarse(level, be.restrict_interior(level, r_int, lo_c, hi_c))
            g_c = self._gather_coarse_ghosts(level, be.restrict_ghost(level, r_ext, lo_c, hi_c))
            e = be.coarse_tail(c, f_c, g_c) if self.rank == 0 else np.zeros(be.plans[c].n_nodes)
            e = self._bcast(e)
        be.interpolate_add(level, u, e, lo, hi)
        self.smooth(level, u, f, g, be.nu2)

    # the coarse planes restricted from fine slab [lo, hi): I with 2I in [lo, hi)
    def _coarse_owner_ranges(self, level):
        out = []
        for r in range(self.world):
            lo, hi = self.part.planes(level, r)
            out.append(((lo + 1) // 2, (hi + 1) // 2))
        return out

    def _gather_coarse(self, level, f_c):
        import torch

        t = torch.from_numpy(np.ascontiguousarray(f_c))
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t)
        out = np.zeros_like(f_c)
        c = level + 1
        for r, (lo, hi) in enumerate(self._coarse_owner_ranges(level)):
            sl = self._plane_slice(c, lo, hi)
            out[sl] = parts[r].numpy()[sl]
        return out

    def _gather_coarse_ghosts(self, level, g_c):
        import torch

        t = torch.from_numpy(np.ascontiguousarray(g_c))
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t)
        out = np.zeros_like(g_c)
        c = level + 1
        for r, (lo, hi) in enumerate(self._coarse_owner_ranges(level)):
            m = self.be.owned_ghosts(c, lo, hi)
            out[m] = parts[r].numpy()[m]
        return out

    def _bcast(self, e):
        import torch

        t = torch.from_numpy(np.ascontiguousarray(e))
        self.dist.broadcast(t, 0)
        return t.numpy().copy()
