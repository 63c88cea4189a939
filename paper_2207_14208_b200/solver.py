"""B200 multigrid solver: the reference's solver API over the CUDA library.

Drop-in for /root/reference/pkg/src/ghostmg/solver.py:

* ``build_solver(grid, phi, spec, eliminated_faces, smoother, cycle,
  default_variant, coarsest_min)`` (solver.py:272-279) builds the hierarchy
  on the host exactly as the reference does and uploads it once;
* ``MultigridSolver.solve(u, cycles, tol, seed)`` (solver.py:215-269) and
  ``measure_rho`` (solver.py:282-298) keep the reference's control flow
  (``cycle.CycleDriver``) while every cycle runs on the device
  (``_lib.Context.cycle``), with the iterate resident in HBM between
  cycles; only the two residual-norm scalars come back per cycle.
* The coarsest solve is the reference's own by default: SciPy SuperLU of the
  assembled coarsest system (solver.py:146-166), called through the
  library's host callback on a few-KB right-hand side (bit-exact), or
  ``coarse_solver="sweeps"`` (500 device smoothing sweeps, bit-exact).
  ``coarse_backend="device-inverse"`` instead inverts the coarsest operator
  once on the GPU (setup) and applies the dense inverse with the library's
  GEMV kernel every cycle -- no host round trip; results then differ from
  the reference at round-off level (bounded in tests/test_gpu_parity.py).
"""

import math
import os

import numpy as np
from scipy.sparse.linalg import splu

from . import _lib
from .cycle import (
    NORM_L2,
    CoarseSolveError,
    CycleConfig,
    CycleDriver,
    CycleReport,
    measure_rho,
)
from .kinds import VARIANT_POLY
from .plan import coarsest_system
from .smoothing import SmootherConfig
from .transfer import build_hierarchy

__all__ = ["MultigridSolver", "build_solver", "measure_rho", "solve_batched", "measure_rho_batched", "CycleConfig",
           "CycleReport"]


COARSE_BACKENDS = ("superlu", "device-inverse")


class DeviceHierarchy:
    """All levels of one solver resident on one GPU."""

    def __init__(self, plans, smoother, cycle, device=0, coarse_backend="superlu"):
        if coarse_backend not in COARSE_BACKENDS:
            raise ValueError(f"unknown coarse backend {coarse_backend!r}")
        self.plans = plans
        self.device_index = device
        d = plans[0].d
        self.ctx = _lib.Context(d, len(plans), device)
        for i, p in enumerate(plans):
            self.ctx.set_level(i, p)
        if cycle.coarse_solver == "sweeps":
            coarse_mode = 1
        elif coarse_backend == "device-inverse":
            coarse_mode = 2
        else:
            coarse_mode = 0
        self.ctx.set_cycle(smoother.nu1, smoother.nu2, cycle.gamma, coarse_mode,
                           cycle.coarse_sweeps, 1 if cycle.norm == NORM_L2 else 0)
        self._lu = None
        if coarse_mode == 0:
            self.ctx.set_coarse_callback(self._coarse)
        elif coarse_mode == 2:
            self._upload_inverse()

    ND_MIN = 8192  # coarsest systems at least this large use the nested-dissection form
    ND_DEPTH = 2   # dissection levels (leaves are dense inverses)
    ND_LEAF = 2048  # subproblems smaller than this are not split further

    def _upload_inverse(self):
        """Invert the coarsest operator on the GPU (setup) and hand it to the
        library, which copies it into its own buffer: for large systems as one
        level of nested dissection (two decoupled plane halves + separator),
        else as one dense inverse."""
        import torch

        A, active = coarsest_system(self.plans[-1])
        n = A.shape[0]
        depth = int(os.environ.get("GMG_ND_DEPTH", self.ND_DEPTH))
        if n >= self.ND_MIN and depth > 0 and self._upload_nd_program(A, active, depth=depth):
            return
        if n >= self.ND_MIN and self._upload_nd(A, active):
            return
        dev = torch.device("cuda", self.device_index)
        dense = torch.from_numpy(A.toarray()).to(dev)
        inv = torch.linalg.inv(dense).contiguous()  # LAPACK-backed results may be column-major
        del dense
        torch.cuda.synchronize(dev)
        self.ctx.set_coarse_inverse(n, inv.data_ptr(), True)
        del inv
        torch.cuda.empty_cache()

    def _nd_split(self, A, active):
        """[A | B | S] split of the coarsest unknowns by axis-0 planes: the
        narrowest separator around the middle plane that decouples the halves
        (the 3^d ghost rows reach two planes), or None."""
        p = self.plans[-1]
        per = (p.N + 1) ** (p.d - 1)
        planes = np.asarray(active) // per
        mid = p.N // 2
        csr = A.tocsr()
        for w in range(1, max(2, p.N // 4)):
            a = np.flatnonzero(planes < mid - w)
            b = np.flatnonzero(planes > mid + w)
            sep = np.flatnonzero((planes >= mid - w) & (planes <= mid + w))
            if len(a) == 0 or len(b) == 0:
                return None
            if csr[a][:, b].nnz == 0 and csr[b][:, a].nnz == 0:
                return a, b, sep
        return None

    def _upload_nd_program(self, A, active, depth):
        """Recursive nested dissection as a program of device products
        (gmg_coarse_prog_*): a subproblem either is a leaf, x = inv(A_ii) b,
        or splits by axis-0 planes into decoupled halves a, b and a separator
        s: solve a and b, t = b_s - A_s,ab x_ab (sparse), x_s = Si t with Si the
        inverse Schur complement, x_ab -= W x_s, W = blkdiag(inv(A_aa),
        inv(A_bb)) A_ab,s.  Workspace: permuted rhs [0, n), solution [n, 2n),
        separator temporaries after."""
        import torch

        csr = A.tocsr()
        n = A.shape[0]
        p = self.plans[-1]
        per = (p.N + 1) ** (p.d - 1)
        planes = np.asarray(active) // per
        dev = torch.device("cuda", self.device_index)
        ops = []
        temp = [2 * n]

        def dense(r, c):
            return torch.from_numpy(csr[r][:, c].toarray()).to(dev)

        def split(idx):
            pl = planes[idx]
            lo, hi = int(pl.min()), int(pl.max())
            mid = (lo + hi) // 2
            for w in range(1, max(2, (hi - lo) // 4)):
                a, b = idx[pl < mid - w], idx[pl > mid + w]
                s_ = idx[(pl >= mid - w) & (pl <= mid + w)]
                if len(a) == 0 or len(b) == 0:
                    return None
                if csr[a][:, b].nnz == 0 and csr[b][:, a].nnz == 0:
                    return a, b, s_
            return None

        def solve(idx, off, lvl):
            sp = split(idx) if lvl > 0 and len(idx) >= self.ND_LEAF else None
            if sp is None:
                M = torch.linalg.inv(dense(idx, idx)).contiguous()
                ops.append(("dense", M, len(idx), len(idx), off, n + off, -1))
                return np.asarray(idx)
            a, b, s_ = sp
            oa = solve(a, off, lvl - 1)
            ob = solve(b, off + len(a), lvl - 1)
            ab = np.concatenate([oa, ob])
            soff = off + len(ab)
            ia = torch.linalg.inv(dense(oa, oa))
            ib = torch.linalg.inv(dense(ob, ob))
            W = torch.cat([ia @ dense(oa, s_), ib @ dense(ob, s_)], dim=0).contiguous()
            del ia, ib
            C = csr[s_][:, ab]
            Cd = torch.from_numpy(C.toarray()).to(dev)
            Si = torch.linalg.inv(dense(s_, s_) - Cd @ W).contiguous()
            del Cd
            t = temp[0]
            temp[0] += len(s_)
            ops.append(("csr", C, n + off, soff, t))
            ops.append(("dense", Si, len(s_), len(s_), t, n + soff, -1))
            ops.append(("dense", W, len(ab), len(s_), n + soff, n + off, n + off))
            return np.concatenate([ab, s_])

        root = split(np.arange(n))
        if root is None:
            return False
        order = solve(np.arange(n), 0, depth)
        torch.cuda.synchronize(dev)
        self.ctx.coarse_prog_begin(n, order.astype(np.int32), temp[0])
        for op in ops:
            if op[0] == "dense":
                _, M, m, k, xo, yo, y0 = op
                self.ctx.coarse_prog_dense(m, k, M.data_ptr(), xo, yo, y0)
            else:
                _, C, xo, y0, yo = op
                self.ctx.coarse_prog_csr(C, xo, y0, yo)
        self.ctx.coarse_prog_end(n)
        self.nd_sizes = tuple(op[2] for op in ops if op[0] == "dense")
        ops.clear()
        torch.cuda.empty_cache()
        return True

    def _upload_nd(self, A, active):
        import torch

        split = self._nd_split(A, active)
        if split is None:
            return False
        a, b, sep = split
        dev = torch.device("cuda", self.device_index)
        csr = A.tocsr()

        def blk(r, c):
            return torch.from_numpy(csr[r][:, c].toarray()).to(dev)

        aai = torch.linalg.inv(blk(a, a))
        bbi = torch.linalg.inv(blk(b, b))
        asp, bsp = blk(a, sep), blk(b, sep)
        sa, sb = blk(sep, a), blk(sep, b)
        wa, wb = aai @ asp, bbi @ bsp
        ga, gb = sa @ aai, sb @ bbi
        schur = blk(sep, sep) - sa @ wa - sb @ wb
        si = torch.linalg.inv(schur).contiguous()
        g = torch.cat([ga, gb], dim=1).contiguous()
        w = torch.cat([wa, wb], dim=0).contiguous()
        aai, bbi = aai.contiguous(), bbi.contiguous()
        torch.cuda.synchronize(dev)
        perm = np.concatenate([a, b, sep]).astype(np.int32)
        self.ctx.set_coarse_nd(len(perm), len(a), len(b), len(sep), perm, aai.data_ptr(), bbi.data_ptr(),
                               g.data_ptr(), w.data_ptr(), si.data_ptr(), True)
        # the separator coupling, sparse, over the permuted [A | B] columns
        coup = csr[sep][:, np.concatenate([a, b])].tocsr()
        coup.sort_indices()
        self.ctx.set_coarse_nd_coupling(len(sep), len(a) + len(b), coup.indptr, coup.indices, coup.data)
        self.nd_sizes = (len(a), len(b), len(sep))
        del aai, bbi, g, w, si, asp, bsp, sa, sb, wa, wb, ga, gb, schur
        torch.cuda.empty_cache()
        return True

    def _factor(self):
        if self._lu is None:
            A, _ = coarsest_system(self.plans[-1])
            try:
                self._lu = splu(A.tocsc())
            except RuntimeError as exc:
                raise CoarseSolveError(f"coarsest factorization failed: {exc}") from exc
        return self._lu

    def _coarse(self, rhs):
        return self._factor().solve(rhs)


class MultigridSolver(CycleDriver):
    """Reference ``MultigridSolver`` with every cycle on the B200."""

    def __init__(self, levels, spec, smoother=None, cycle=None, default_variant=VARIANT_POLY,
                 device=0, coarse_backend="superlu"):
        smoother = smoother or SmootherConfig()
        cycle = cycle or CycleConfig()
        plans, f, g, e = CycleDriver.problem_data(levels, spec, smoother, default_variant)
        super().__init__(plans, f, g, e, smoother, cycle)
        self.levels = levels
        self.spec = spec
        self._init_device(device, coarse_backend)

    @classmethod
    def from_plans(cls, plans, f_fine, g_fine, eliminated_values, smoother=None, cycle=None,
                   device=0, coarse_backend="superlu"):
        self = cls.__new__(cls)
        CycleDriver.__init__(self, plans, f_fine, g_fine, eliminated_values,
                             smoother or SmootherConfig(), cycle or CycleConfig())
        self.levels = None
        self.spec = None
        self._init_device(device, coarse_backend)
        return self

    def _init_device(self, device, coarse_backend):
        self.coarse_backend = coarse_backend
        self.device = DeviceHierarchy(self.plans, self.smoother, self.cycle_cfg, device,
                                      coarse_backend)
        self.ctx = self.device.ctx
        if self.cycle_cfg.coarse_solver != "sweeps" and coarse_backend == "superlu":
            self.device._factor()

    # ---- primitives --------------------------------------------------------
    def _set_data(self, f_fine, g_fine):
        self.ctx.set_vector(0, _lib.F, f_fine)
        if self.plans[0].n_ghosts:
            self.ctx.set_vector(0, _lib.G, g_fine)

    def _put_u(self, u):
        self._peak_lb = None
        self.ctx.set_vector(0, _lib.U, u)

    def _get_u(self):
        return self.ctx.get_vector(0, _lib.U, self.plans[0].n_nodes)

    def _fetch_u(self, u):
        # straight into the caller's array (one D2H copy, no host temporary)
        n = self.plans[0].n_nodes
        if (isinstance(u, np.ndarray) and u.shape == (n,) and u.dtype == np.float64
                and u.flags.c_contiguous and u.flags.writeable):
            self.ctx.get_vector(0, _lib.U, n, out=u)
            return u
        return super()._fetch_u(u)

    def _device_initial_field(self, seed):
        # the whole stream on the GPU (GF(2) jump-ahead per 64-value lane): no 1e8..1e9 host draws and no
        # upload of the iterate for measure_rho at 512^3 / 1024^3
        from .geometry import ELIMINATED

        fine = self.plans[0]
        idx = np.flatnonzero(fine.labels == ELIMINATED)
        self.ctx.initial_field(seed, fine.n_nodes, idx, self.eliminated_values[idx])
        return True

    def _run_cycle(self):
        self._peak_lb = None
        self.ctx.cycle(1)

    def _residual_norm(self):
        # the norm pass also returns max|u| over the internal nodes: when that is already above the
        # renormalisation threshold, _abs_max_scale (called right after, u unchanged) has its answer
        m_int, m_g, lb = self.ctx.residual_parts_peak(0)
        self._peak_lb = lb
        if self.cycle_cfg.norm == NORM_L2:
            # device sums of squares, NumPy's pairwise order (solver.py:138)
            return math.sqrt(float(m_int + m_g))
        p = self.plans[0]
        m = m_int if p.n_internal else 0.0
        if p.n_ghosts:
            m = max(m, m_g)
        return m

    def _abs_max_scale(self):
        """(peak, scaled) of the renormalisation guard (reference solver.py:239-243).  peak is max|u|, or,
        when the preceding norm pass already found an internal |u| >= the threshold, that lower bound
        (the guard's outcome is the same: no rescaling)."""
        lb, self._peak_lb = getattr(self, "_peak_lb", None), None
        if lb is not None and lb >= 1e-250:
            return lb, False
        return self.ctx.abs_max_scale(1e-250, 1e250)


def solve_batched(solvers, us=None, cycles=None, seed=42):
    """``[s.solve(u, cycles, seed=seed) for s in solvers]`` with the solvers'
    cycles interleaved: every round enqueues one cycle and the asynchronous
    residual norm / max|u| on each solver's own stream, then collects them, so
    many small problems (the BLFA parameter sweeps of the paper, reference
    cli.py:154-194) keep the GPU busy together instead of one after the other.
    Same control flow per solver as CycleDriver.solve (reference
    solver.py:215-269) and bitwise the same results; inf norm only."""
    from .cycle import DIVERGENCE_FACTOR, MIN_CYCLES_FOR_RHO, RHO_WINDOW

    n = len(solvers)
    us = [None] * n if us is None else list(us)
    cyc = [s.cycle_cfg.cycles if cycles is None else cycles for s in solvers]
    for s in solvers:
        if s.cycle_cfg.norm == NORM_L2:
            raise NotImplementedError("solve_batched uses the inf norm")
    st = []
    for i, s in enumerate(solvers):
        u = s.initial_field(seed) if us[i] is None else us[i]
        us[i] = u
        s._set_data(s.f_fine, s.g_fine)
        s._put_u(np.ascontiguousarray(u, dtype=np.float64))
        st.append({"ln": [], "scale": 0.0, "div": False, "ran": 0, "active": True, "pending": False})

    def norm_of(s, parts):
        m_int, m_g, peak = parts
        p = s.plans[0]
        m = m_int if p.n_internal else 0.0
        if p.n_ghosts:
            m = max(m, m_g)
        return m, peak

    for s in solvers:
        s.ctx.norm_begin()
    for s, t in zip(solvers, st):
        m, _ = norm_of(s, s.ctx.norm_end())
        t["ln"].append((math.log(m) if m > 0.0 else -math.inf) + t["scale"])
    for m_ in range(max(cyc) if cyc else 0):
        live = [i for i in range(n) if st[i]["active"] and m_ < cyc[i]]
        if not live:
            break
        for i in live:
            s, t = solvers[i], st[i]
            if t["pending"]:
                s.ctx.scale_u(1e250)
                t["pending"] = False
            s.ctx.cycle(1)
            s.ctx.norm_begin()
        for i in live:
            s, t = solvers[i], st[i]
            r, peak = norm_of(s, s.ctx.norm_end())
            t["ln"].append((math.log(r) if r > 0.0 else -math.inf) + t["scale"])
            t["ran"] = m_ + 1
            if t["ln"][-1] - t["ln"][0] > math.log(DIVERGENCE_FACTOR):
                t["div"] = True
                t["active"] = False
                continue
            if 0.0 < peak < 1e-250:  # CycleDriver._abs_max_scale
                t["pending"] = True
                t["scale"] -= math.log(1e250)
    out = []
    for i, (s, t) in enumerate(zip(solvers, st)):
        if t["pending"]:
            s.ctx.scale_u(1e250)
        u = s._fetch_u(us[i])
        ln = t["ln"]
        norms = [math.exp(v) if v > -math.inf else 0.0 for v in ln]
        rho_seq = [math.exp(ln[k + 1] - ln[k]) if ln[k] > -math.inf else 0.0 for k in range(len(ln) - 1)]
        lo, hi = RHO_WINDOW
        rho = 1.0 if t["div"] else (float(np.mean(rho_seq[lo:hi + 1])) if t["ran"] >= MIN_CYCLES_FOR_RHO else None)
        out.append((u, CycleReport(residual_norms=norms, rho_sequence=rho_seq, rho_asymptotic=rho,
                                   diverged=t["div"], cycles_run=t["ran"], scheme=s.cycle_cfg.scheme,
                                   n_levels=s.n_levels, norm=s.cycle_cfg.norm, seed=seed)))
    return out


def measure_rho_batched(solvers, seed=42, cycles=16):
    """measure_rho (reference solver.py:282-298) for many solvers at once."""
    from .cycle import MIN_CYCLES_FOR_RHO

    cycles = max(cycles, MIN_CYCLES_FOR_RHO)
    saved = [(s.f_fine, s.g_fine, s.eliminated_values) for s in solvers]
    for s in solvers:
        s.f_fine = np.zeros_like(s.f_fine)
        s.g_fine = np.zeros_like(s.g_fine)
        s.eliminated_values = np.zeros_like(s.eliminated_values)
    try:
        res = solve_batched(solvers, cycles=cycles, seed=seed)
    finally:
        for s, (f, g, e) in zip(solvers, saved):
            s.f_fine, s.g_fine, s.eliminated_values = f, g, e
    return [r for _, r in res]


def build_solver(grid, phi, spec, eliminated_faces=(), smoother=None, cycle=None,
                 default_variant=VARIANT_POLY, coarsest_min=4, device=0, coarse_backend="superlu"):
    """Hierarchy + B200 solver in one call (reference solver.py:272-279)."""
    cycle = cycle or CycleConfig()
    levels = build_hierarchy(grid, phi, eliminated_faces, max_levels=cycle.max_levels,
                             coarsest_min=coarsest_min, device=device)
    return MultigridSolver(levels, spec, smoother, cycle, default_variant, device=device,
                           coarse_backend=coarse_backend)
