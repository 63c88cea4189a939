"""z-slab schedule of the V-cycle over ranks (paper_2207_14208_b200/slabs.py),
run with the CPU oracle as the per-slab backend on gloo (world sizes 2, 3):
every rank's owned planes of the iterate, and the residual history, must be
bit-identical to the single-process oracle solve.  This is the N>1 path's
host logic (partition, pipelined sweeps, halo widths, agglomeration,
gathers); the per-slab device kernels plug into the same schedule.
"""

import dataclasses
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ops
from oracle.solver import OracleSolver
from paper_2207_14208_b200 import configs as CF
from paper_2207_14208_b200.cycle import CycleDriver
from paper_2207_14208_b200.geometry import ELIMINATED, GHOST, INTERNAL
from paper_2207_14208_b200.slabs import SlabCycle, SlabPartition
from paper_2207_14208_b200.transfer import build_hierarchy


class OracleSlabBackend:
    """Oracle operations restricted to the nodes of a plane range (test
    infrastructure: the checker drives the schedule under test)."""

    def __init__(self, plans, f, g, e, smoother, cycle):
        self.plans = plans
        self.nu1, self.nu2, self.gamma = smoother.nu1, smoother.nu2, cycle.gamma
        self.ref = OracleSolver(plans, f, g, e, smoother, cycle)
        self.per = [(p.N + 1) ** (p.d - 1) for p in plans]
        self.st = [np.ascontiguousarray(p.stencil, dtype=np.int64) for p in plans]

    def _plane(self, level, flat):
        return np.asarray(flat) // self.per[level]

    def _masked(self, level, lo, hi, kinds):
        p = self.plans[level]
        lab = p.labels.copy()
        pl = np.arange(p.n_nodes) // self.per[level]
        out = (pl < lo) | (pl >= hi)
        for k in kinds:
            lab[out & (p.labels == k)] = ELIMINATED
        return dataclasses.replace(p, labels=lab)

    def owned_ghosts(self, level, lo, hi):
        pl = self._plane(level, self.plans[level].ghost_idx)
        return (pl >= lo) & (pl < hi)

    def _ghost_plan(self, level, lo, hi):
        p = self.plans[level]
        m = self.owned_ghosts(level, lo, hi)
        sub = dataclasses.replace(p, ghost_idx=p.ghost_idx[m], ghost_low=p.ghost_low[m], ghost_w=p.ghost_w[m],
                                  ghost_dtau=p.ghost_dtau[m], ghost_promoted=p.ghost_promoted[m],
                                  ghost_batch=p.ghost_batch[m])
        return sub, m

    # ---- per-slab operations --------------------------------------------
    def gs_sweep(self, level, u, f, lo, hi):
        ops.gs_sweep(self._masked(level, lo, hi, (INTERNAL,)), u, f)

    def ghost_sweep(self, level, u, g, lo, hi):
        sub, m = self._ghost_plan(level, lo, hi)
        ops.ghost_sweep(sub, u, g[m], self.st[level][m])

    def residual_internal(self, level, u, f, lo, hi):
        r, _ = ops.residual_internal_full(self._masked(level, lo, hi, (INTERNAL,)), u, f)
        return r

    def residual_ghost_ext(self, level, u, g, lo, hi):
        p = self.plans[level]
        sub, m = self._ghost_plan(level, lo, hi)
        rg, _ = ops.residual_ghost(sub, u, g[m], self.st[level][m])
        r_ext = np.zeros(p.n_nodes)
        r_ext[p.ghost_idx[m]] = rg
        return r_ext

    def residual_norm(self, level, u, f, g, lo, hi):
        p = self.plans[level]
        r = self.residual_internal(level, u, f, lo, hi)
        own = (self._plane(level, np.arange(p.n_nodes)) >= lo) & (self._plane(level, np.arange(p.n_nodes)) < hi)
        m = float(np.max(np.abs(r[own & (p.labels == INTERNAL)]), initial=0.0))
        sub, gm = self._ghost_plan(level, lo, hi)
        if gm.any():
            rg, _ = ops.residual_ghost(sub, u, g[gm], self.st[level][gm])
            m = max(m, float(np.max(np.abs(rg))))
        return m

    def n_bfs_groups(self, level):
        return len(self.plans[level].bfs_len)

    def _band_group(self, level, grp):
        p = self.plans[level]
        off = np.concatenate([[0], np.cumsum(p.bfs_len)])
        return slice(int(off[grp]), int(off[grp + 1]))

    def band_bfs(self, level, x, grp, lo, hi):
        p = self.plans[level]
        sl = self._band_group(level, grp)
        idx = p.band_idx[sl]
        m = (self._plane(level, idx) >= lo) & (self._plane(level, idx) < hi)
        ops.band_bfs(p, x, idx[m], p.bfs_mask[sl][m])

    def band_transport(self, level, x, lo, hi):
        p = self.plans[level]
        m = (self._plane(level, p.band_idx) >= lo) & (self._plane(level, p.band_idx) < hi)
        ops.band_transport(p, x, p.band_idx[m], p.trans_step[m], p.trans_absn[m])

    def restrict_interior(self, level, r_int, clo, chi):
        return ops.restrict_interior(self.plans[level], self._masked(level + 1, clo, chi, (INTERNAL,)), r_int)

    def restrict_ghost(self, level, r_ext, clo, chi):
        C = self.plans[level + 1]
        sub, m = self._ghost_plan(level + 1, clo, chi)
        g_c = np.zeros(C.n_ghosts)
        g_c[m] = ops.restrict_ghost(self.plans[level], sub, r_ext)
        g_c[C.ghost_promoted & m] = 0.0
        return g_c

    def interpolate_add(self, level, u, e, lo, hi):
        ops.interpolate_add(self._masked(level, lo, hi, (INTERNAL, GHOST)), u, e)

    def coarse_tail(self, c, f_c, g_c):
        """Rest of the cycle from level c on one rank (reference _cycle),
        including the coarse band extension of the returned error."""
        if c == len(self.plans) - 1:
            e = self.ref.coarse_solve(f_c, g_c)
        else:
            e = np.zeros(self.plans[c].n_nodes)
            for _ in range(self.gamma):
                self.ref._cycle(c, e, f_c, g_c)
        ops.extrapolate(self.plans[c], e)
        return e


def _setup(name):
    if name == "ball32":
        setup = CF.config_ball(32, cycles=3)
    else:
        setup = CF.config_pores(N=64)
    levels = build_hierarchy(setup.grid, setup.phi, setup.faces, max_levels=setup.cycle.max_levels,
                             coarsest_min=setup.coarsest_min)
    plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
    if setup.f_seed is not None:
        f = CF.pore_rhs(setup, plans[0].labels)
    return setup, plans, f, g, e


def _worker(rank, world, port, name, cycles, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        setup, plans, f, g, e = _setup(name)
        be = OracleSlabBackend(plans, f, g, e, setup.smoother, setup.cycle)
        part = SlabPartition([p.N for p in plans], world)
        sc = SlabCycle(be, part, dist, rank)
        u = np.zeros(plans[0].n_nodes)
        norms = [sc.residual_norm(u, f, g)]
        for _ in range(cycles):
            sc.cycle(0, u, f, g)
            norms.append(sc.residual_norm(u, f, g))
        lo, hi = part.planes(0, rank)
        per = (plans[0].N + 1) ** (plans[0].d - 1)
        q.put((rank, lo, hi, u[lo * per:hi * per].copy(), norms, [l.bounds for l in part.levels]))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,world", [("ball32", 2), ("ball32", 3), ("pores64", 2)])
def test_slab_cycle_matches_single_process(name, world):
    cycles = 2
    setup, plans, f, g, e = _setup(name)
    ref = OracleSolver(plans, f, g, e, setup.smoother, setup.cycle)
    ref._set_data(f, g)
    ref._put_u(np.zeros(plans[0].n_nodes))
    want_norms = [ref._residual_norm()]
    for _ in range(cycles):
        ref._run_cycle()
        want_norms.append(ref._residual_norm())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, cycles, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    per = (plans[0].N + 1) ** (plans[0].d - 1)
    bounds = res[0][5]
    assert bounds[0] is not None, "the finest level must be distributed"
    covered = 0
    for rank, lo, hi, u_own, norms, _ in sorted(res, key=lambda t: t[0]):
        assert norms == want_norms, (rank, norms, want_norms)
        assert np.array_equal(u_own.view(np.uint64), ref.u[lo * per:hi * per].view(np.uint64)), rank
        covered += hi - lo
    assert covered == plans[0].N + 1


def test_partition_shapes():
    p = SlabPartition([512, 256, 128, 64, 32], 8)
    assert p.levels[0].bounds == [0, 64, 128, 192, 256, 320, 384, 448, 513]
    assert p.distributed(3) and not p.distributed(4)
    assert p.planes(4, 0) == (0, 33) and p.planes(4, 3) == (0, 0)
    p = SlabPartition([64, 32, 16, 8], 3)
    assert p.distributed(1) and not p.distributed(2)  # odd coarse boundary: agglomerated
    assert not SlabPartition([16, 8, 4], 8).distributed(0)  # too thin: single rank


def _group_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2207_14208_b200.slabs import TorchGroup

        grp = TorchGroup(dist, None)  # CPU tensors over gloo; on the GPUs the same calls run over NCCL
        t = torch.full((5,), float(rank), dtype=torch.float64)
        if rank == 0:
            grp.send(t, 1)
            grp.recv(t, 1)
        else:
            r = torch.empty(5, dtype=torch.float64)
            grp.recv(r, 0)
            grp.send(t, 0)
            t = r
        b = torch.full((3,), 7.0 + rank, dtype=torch.float64)
        grp.broadcast(b, 1)
        m = grp.all_max([1.0 + rank, float("nan") if rank == 1 else 0.5, 0.0])
        q.put((rank, t.tolist(), b.tolist(), m))
    finally:
        dist.destroy_process_group()


def test_torch_group_transport_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_group_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][0] == [1.0] * 5 and res[1][0] == [0.0] * 5  # the two ranks swapped their planes
    assert res[0][1] == [8.0] * 3 and res[1][1] == [8.0] * 3   # broadcast from rank 1
    for r in (0, 1):
        m = res[r][2]
        assert m[0] == 2.0 and np.isnan(m[1]) and m[2] == 0.0  # MAX with numpy's NaN propagation


def test_partition_min_N_agglomerates_small_levels():
    p = SlabPartition([512, 256, 128, 64, 32], 8, min_N=64)
    assert [p.distributed(i) for i in range(5)] == [True, True, True, True, False]
    p = SlabPartition([256, 128, 64, 32, 16], 4, min_N=64)
    assert [p.distributed(i) for i in range(5)] == [True, True, True, False, False]
