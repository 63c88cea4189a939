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

    def __init__(self, Ns, world, min_planes=4, min_N=0):
        """``min_N``: levels with fewer cells per axis are agglomerated (the
        device backend splits only levels with N >= 64, gmg_set_slab)."""
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
            if li == len(Ns) - 1 or N < min_N:
                bounds = None  # the coarsest solve (and every level too small to split) runs on rank 0
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


# ---------------------------------------------------------------------------
# Device backend: one gmg context per rank (one GPU each), planes exchanged as
# device tensors (NCCL over NVLink through torch.distributed, or queues between
# rank threads of one process for the single-GPU test).
# ---------------------------------------------------------------------------
class _DevMem:
    """CUDA array interface view of `count` doubles at a device address."""

    def __init__(self, address, count):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(address), False),
                                         "version": 2}


def device_tensor(address, count, device):
    import torch

    return torch.as_tensor(_DevMem(address, count), device=torch.device("cuda", device))


class TorchGroup:
    """torch.distributed (NCCL) transport of device tensors."""

    def __init__(self, dist, device):
        import torch

        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.torch = torch
        self.device = device

    def _sync(self):
        if self.device is not None:  # None: CPU tensors (gloo, tests)
            self.torch.cuda.current_stream(self.device).synchronize()

    def send(self, t, dst):
        self.dist.send(t, dst)
        self._sync()

    def recv(self, t, src):
        self.dist.recv(t, src)
        self._sync()

    def broadcast(self, t, src):
        self.dist.broadcast(t, src)
        self._sync()

    def all_max(self, values):
        dev = self.torch.device("cuda", self.device) if self.device is not None else self.torch.device("cpu")
        t = self.torch.tensor(list(values), dtype=self.torch.float64, device=dev)
        # NaN propagates like numpy's max: compare the bit patterns of the non-negative values
        bits = t.view(self.torch.int64)
        self.dist.all_reduce(bits, op=self.dist.ReduceOp.MAX)
        return [float(x) for x in bits.view(self.torch.float64).cpu()]


class LocalGroup:
    """`world` rank threads of one process on one GPU (tests): blocking queues
    between every ordered pair of ranks, the same interface as TorchGroup."""

    class Shared:
        def __init__(self, world):
            import queue
            import threading

            self.world = world
            self.q = {(a, b): queue.Queue() for a in range(world) for b in range(world)}
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared, rank, device=0):
        import torch

        self.sh = shared
        self.rank = rank
        self.world = shared.world
        self.torch = torch
        self.device = device

    def send(self, t, dst):
        c = t.clone()
        self.torch.cuda.synchronize(self.device)
        self.sh.q[(self.rank, dst)].put(c)

    def recv(self, t, src):
        c = self.sh.q[(src, self.rank)].get(timeout=600)
        t.copy_(c)
        self.torch.cuda.synchronize(self.device)

    def broadcast(self, t, src):
        if self.rank == src:
            for r in range(self.world):
                if r != src:
                    self.send(t, r)
        else:
            self.recv(t, src)

    def all_max(self, values):
        self.sh.slots[self.rank] = np.array(list(values), dtype=np.float64)
        self.sh.barrier.wait()
        allv = np.stack(self.sh.slots)
        bits = allv.view(np.int64).max(axis=0)
        out = [float(x) for x in bits.view(np.float64)]
        self.sh.barrier.wait()
        return out


class DeviceSlabCycle:
    """SlabCycle's schedule over a device hierarchy (`_lib.Context`, every
    level uploaded whole on every rank; distributed levels in z-slab mode,
    see gmg_set_slab in include/ghostmg_b200.h).  Reference: solver.py:170-199;
    the sweeps' rank order restates smoothing.py:127-142 across slabs."""

    def __init__(self, ctx, plans, partition, group, nu1, nu2, gamma, halo_ghost=2):
        from . import _lib

        self.L = _lib
        self.ctx = ctx
        self.plans = plans
        self.part = partition
        self.grp = group
        self.rank = group.rank
        self.world = group.world
        self.nu1, self.nu2, self.gamma = nu1, nu2, gamma
        self.hg = halo_ghost
        self.ngroups = {}
        for lv, p in enumerate(plans):
            if partition.distributed(lv):
                lo, hi = partition.planes(lv, self.rank)
                self.ngroups[lv] = ctx.set_slab(lv, lo, hi)

    # ---- plane transport (device tensors over the padded device layout) ----
    def _plane_elems(self, level):
        p = self.plans[level]
        n = p.N + 1
        pitch = max((p.N + 4 + 3) // 4 * 4, 32 * ((p.N - 1 + 31) // 32) + 4)  # make_geom's row pitch
        return (n if p.d == 3 else 1) * pitch

    def _view(self, level, which, lo, hi):
        per = self._plane_elems(level)
        base = self.ctx.device_pointer(level, which)
        return device_tensor(base + 8 * lo * per, (hi - lo) * per, self.grp.device)

    def _send(self, level, which, lo, hi, dst):
        if hi > lo:
            self.grp.send(self._view(level, which, lo, hi), dst)

    def _recv(self, level, which, lo, hi, src):
        if hi > lo:
            self.grp.recv(self._view(level, which, lo, hi), src)

    def halo(self, level, which, width):
        if not self.part.distributed(level) or self.world == 1:
            return
        lo, hi = self.part.planes(level, self.rank)
        N = self.part.levels[level].N
        r = self.rank
        for phase in ((0, 1) if r % 2 == 0 else (1, 0)):
            if phase == 0:
                if r + 1 < self.world:
                    self._send(level, which, max(lo, hi - width), hi, r + 1)
                if r > 0:
                    self._send(level, which, lo, min(hi, lo + width), r - 1)
            else:
                if r > 0:
                    plo, _ = self.part.planes(level, r - 1)
                    self._recv(level, which, max(plo, lo - width), lo, r - 1)
                if r + 1 < self.world:
                    _, nhi = self.part.planes(level, r + 1)
                    self._recv(level, which, hi, min(nhi, hi + width, N + 1), r + 1)

    def _pipelined(self, level, width, op):
        if not self.part.distributed(level) or self.world == 1:
            self.ctx.apply(level, op)
            return
        self.halo(level, self.L.U, width)  # old values on both sides
        lo, hi = self.part.planes(level, self.rank)
        if self.rank > 0:
            plo, _ = self.part.planes(level, self.rank - 1)
            self._recv(level, self.L.U, max(plo, lo - width), lo, self.rank - 1)
        self.ctx.apply(level, op)
        if self.rank + 1 < self.world:
            self._send(level, self.L.U, max(lo, hi - width), hi, self.rank + 1)

    # ---- operations ---------------------------------------------------------
    def smooth(self, level, count):
        for _ in range(count):
            self._pipelined(level, 1, self.L.OP_GS_SWEEP)
            self._pipelined(level, self.hg, self.L.OP_GHOST_SWEEP)

    def extrapolate(self, level, which):
        bfs = self.L.OP_BAND_BFS_U if which == self.L.U else self.L.OP_BAND_BFS_REXT
        step = self.L.OP_BAND_STEP_U if which == self.L.U else self.L.OP_BAND_STEP_REXT
        for grp in range(self.ngroups[level]):
            self.halo(level, which, 1)
            self.ctx.apply(level, bfs, grp)
        for _ in range(6):
            self.halo(level, which, 1)
            self.ctx.apply(level, step)

    def residual_norm(self):
        self.halo(0, self.L.U, self.hg)
        m_int, m_g = self.ctx.residual_parts(0)
        return self.grp.all_max([m_int, m_g])

    def cycle(self, level):
        L = self.L
        ctx = self.ctx
        self.smooth(level, self.nu1)
        self.halo(level, L.U, self.hg)
        ctx.apply(level, L.OP_RES_INT)
        ctx.apply(level, L.OP_RES_GHOST)
        self.extrapolate(level, L.R_EXT)
        self.halo(level, L.R_INT, 1)
        self.halo(level, L.R_EXT, 1)
        c = level + 1
        ctx.apply(level, L.OP_RESTRICT_INT)
        ctx.apply(level, L.OP_RESTRICT_GHOST)
        if self.part.distributed(c):
            ctx.apply(c, L.OP_ZERO_U)
            for _ in range(self.gamma):
                self.cycle(c)
            self.extrapolate(c, L.U)
            self.halo(c, L.U, 1)
        else:
            # the coarse planes I with 2I in this rank's fine slab are right here: collect them (and the
            # right-hand sides of the coarse ghosts on them) on rank 0, which finishes the cycle alone
            self._collect_coarse(level)
            if self.rank == 0:
                ctx.apply(c, L.OP_CYCLE_TAIL)
            n = self.plans[c].N + 1
            self.grp.broadcast(self._view(c, L.U, 0, n), 0)
        ctx.apply(level, L.OP_INTERP_ADD)
        self.smooth(level, self.nu2)

    def _collect_coarse(self, level):
        import torch

        L = self.L
        c = level + 1
        pc = self.plans[c]
        per = (pc.N + 1) ** (pc.d - 1)
        ranges = []
        for r in range(self.world):
            lo, hi = self.part.planes(level, r)
            ranges.append(((lo + 1) // 2, (hi + 1) // 2))
        gplane = pc.ghost_idx // per  # ascending
        if self.rank == 0:
            g = self.ctx.get_vector(c, L.G, pc.n_ghosts) if pc.n_ghosts else np.zeros(0)
            for r in range(1, self.world):
                lo, hi = ranges[r]
                self._recv(c, L.F, lo, hi, r)
                a, b = np.searchsorted(gplane, [lo, hi])
                if b > a:
                    t = torch.empty(b - a, dtype=torch.float64, device=torch.device("cuda", self.grp.device))
                    self.grp.recv(t, r)
                    g[a:b] = t.cpu().numpy()
            if pc.n_ghosts:
                self.ctx.set_vector(c, L.G, g)
        else:
            lo, hi = ranges[self.rank]
            self._send(c, L.F, lo, hi, 0)
            a, b = np.searchsorted(gplane, [lo, hi])
            if b > a:
                g = self.ctx.get_vector(c, L.G, pc.n_ghosts)
                self.grp.send(torch.from_numpy(g[a:b].copy()).to(torch.device("cuda", self.grp.device)), 0)

    def gather_planes(self, level, which):
        """Every rank's owned planes of a vector onto every rank."""
        if not self.part.distributed(level) or self.world == 1:
            return
        for r in range(self.world):
            lo, hi = self.part.planes(level, r)
            self.grp.broadcast(self._view(level, which, lo, hi), r)


def slab_solver(plans, f_fine, g_fine, eliminated_values, smoother, cycle, group, device=0,
                coarse_backend="device-inverse", min_planes=4):
    """A `MultigridSolver` whose cycles run z-slab sharded over the ranks of
    `group` (TorchGroup / LocalGroup): same `solve` / `measure_rho` API
    (reference solver.py:215-298), every rank returns the whole iterate."""
    from . import _lib
    from .solver import MultigridSolver

    class SlabSolver(MultigridSolver):
        def _init_slabs(self):
            Ns = [p.N for p in self.plans]
            if self.plans[0].d != 3:
                raise ValueError("z-slab sharding is for 3-D hierarchies")
            self.part = SlabPartition(Ns, group.world, min_planes=min_planes, min_N=64)
            self.slabs = DeviceSlabCycle(self.ctx, self.plans, self.part, group, self.smoother.nu1, self.smoother.nu2,
                                         self.cycle_cfg.gamma)
            self.group = group

        def _run_cycle(self):
            if self.part.distributed(0):
                self.slabs.cycle(0)
            else:
                self.ctx.cycle(1)

        def _residual_norm(self):
            if not self.part.distributed(0):
                return MultigridSolver._residual_norm(self)
            m_int, m_g = self.slabs.residual_norm()
            p = self.plans[0]
            m = m_int if p.n_internal else 0.0
            return max(m, m_g) if p.n_ghosts else m

        def _abs_max_scale(self):
            if not self.part.distributed(0):
                return MultigridSolver._abs_max_scale(self)
            lo, hi = self.part.planes(0, group.rank)
            peak = group.all_max([self.ctx.abs_max_planes(lo, hi)])[0]
            scaled = 0.0 < peak < 1e-250
            if scaled:
                self.ctx.scale_u(1e250)
                self.ctx.synchronize()
            return peak, scaled

        def _get_u(self):
            self.slabs.gather_planes(0, _lib.U)
            return MultigridSolver._get_u(self)

        def _fetch_u(self, u):
            self.slabs.gather_planes(0, _lib.U)
            return MultigridSolver._fetch_u(self, u)

    s = SlabSolver.from_plans(plans, f_fine, g_fine, eliminated_values, smoother, cycle, device=device,
                              coarse_backend=coarse_backend)
    s._init_slabs()
    return s
