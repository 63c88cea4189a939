"""Benchmark: fine-grid DOF x V-cycles/s (fp64) of the B200 ghost-point
multigrid V-cycle on BASELINE.json config 4 (3D pore space, 512^3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = one V(2,1) cycle on the finest level plus the residual-norm
record and the max|u| renormalisation guard the reference's ``solve`` makes
after every cycle (/root/reference/pkg/src/ghostmg/solver.py:224-243).  DOF = internal +
ghost unknowns of the finest level (the size of the linear system,
operators.py:180).  Inputs (u, f) are HBM-resident when the timed region
starts; every array is > L2 (1.08 GB per grid vector at 513^3), so no L2
flush is needed between steps.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the CPU oracle
(oracle/, the C restatement of the reference's per-cycle operators + the
reference's SciPy SuperLU coarsest solve) on the same workload.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--N", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-bitexact", action="store_true",
                    help="skip the second timing with the host SuperLU coarsest solve (the bit-exact path)")
    ap.add_argument("--cpu-sample-cycles", type=int, default=1)
    ap.add_argument("--coarse", default="device-inverse", choices=["superlu", "device-inverse"],
                    help="coarsest solve: host SciPy SuperLU (bit-exact) or device dense inverse")
    return ap.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- workload
def build_workload(args, device=None):
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200.cycle import CycleDriver
    from paper_2207_14208_b200.transfer import build_hierarchy

    builder = CF.CONFIGS[args.config]
    setup = builder(args.N) if args.N else builder()
    t0 = time.time()
    # device: the per-node label work of the setup (classification, restriction checks) on the GPU
    levels = build_hierarchy(setup.grid, setup.phi, setup.faces, max_levels=setup.cycle.max_levels,
                             coarsest_min=setup.coarsest_min, device=device)
    t1 = time.time()
    plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
    if setup.f_seed is not None:
        f = CF.pore_rhs(setup, plans[0].labels)
    t2 = time.time()
    log(f"[bench] {setup.name}: hierarchy {t1 - t0:.1f}s, plans {t2 - t1:.1f}s, levels "
        f"{[p.N for p in plans]}, N_I {plans[0].n_internal}, N_G {plans[0].n_ghosts}")
    return setup, plans, f, g, e, {"hierarchy_s": round(t1 - t0, 1), "plans_s": round(t2 - t1, 1)}


def algorithmic_bytes(plans):
    """SURVEY.md section 8(d) per-cycle algorithmic bytes (V(2,1)),
    from the real per-level counts."""
    total = 0
    for i, p in enumerate(plans[:-1]):
        d = p.d
        m = 3 ** d
        nI, nG, nB = p.n_internal, p.n_ghosts, p.n_band
        nIc = plans[i + 1].n_internal
        sweeps = 3
        total += sweeps * 24 * nI
        total += sweeps * nG * (8 * m + 40)
        total += 16 * nI + 8 * nIc
        total += nG * (8 * m + 24)
        total += nB * (8 * (2 * d + 1) + 6 * 8 * (3 * d + 2))
        total += 16 * (nI + nG) + 8 * nIc
    p0 = plans[0]
    total += 16 * p0.n_internal + p0.n_ghosts * (8 * 3 ** p0.d + 24)
    return total


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clocks and throttle reasons during the timed region via
    NVML (in-process; spawning nvidia-smi stalls concurrent CUDA calls)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index, period=0.02):
        self.index = index
        self.period = period
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None

    def _open(self):
        # NVML is opened before the timed region (the first nvmlInit takes longer than a short region)
        try:
            import pynvml as N
            N.nvmlInit()
            self._N = N
            self._h = N.nvmlDeviceGetHandleByIndex(self.index)
            self._max = N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM)
        except Exception as exc:  # no NVML: record why
            self._err = repr(exc)
            self._N = None

    def _sample(self):
        try:
            sm = self._N.nvmlDeviceGetClockInfo(self._h, self._N.NVML_CLOCK_SM)
            rs = self._N.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            self.samples.append((sm, rs))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(self.period)

    def __enter__(self):
        self._err = None
        self._open()
        if self._N is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=10)
        if self._N is not None and not self.samples:
            self._sample()  # a region shorter than the thread's start-up: the clocks right at its end

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"no samples: {self._err}"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({k for _, rs in self.samples for k, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self._max, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml"}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """Per-launch DRAM bytes of the fine-level GS sweep from the committed
    ncu capture (profiles/ncu_gs_sweep.json), if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_gs_sweep.json")) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except Exception:
        return None


# ---------------------------------------------------------------- oracle
def oracle_cycles(plans, f, g, e, setup, cycles, u0=None):
    """Time `cycles` oracle V-cycles (+ norm) on the host; returns (s, solver)."""
    from oracle.solver import OracleSolver

    s = OracleSolver(plans, f, g, e, setup.smoother, setup.cycle)
    s._set_data(f, g)
    s._put_u(np.zeros(plans[0].n_nodes) if u0 is None else u0)
    s._coarsest()  # factorization is setup, not per cycle
    t = time.perf_counter()
    for _ in range(cycles):
        s._run_cycle()
        s._residual_norm()
    return time.perf_counter() - t, s


def run_reference(args, rank):
    if rank != 0:
        return
    setup, plans, f, g, e, setup_times = build_workload(args)
    dof = plans[0].n_internal + plans[0].n_ghosts
    from oracle.solver import OracleSolver

    s = OracleSolver(plans, f, g, e, setup.smoother, setup.cycle)
    s._set_data(f, g)
    s._put_u(np.zeros(plans[0].n_nodes))
    s._coarsest()
    # bounded sample: at most one warm-up cycle and as many of the K timed
    # cycles as fit in ~150 s of host time (each full-size cycle is ~13 s);
    # "steps" in the line is the number of cycles actually timed
    for _ in range(min(args.warmup, 1)):
        s._run_cycle()
        s._residual_norm()
    t = time.perf_counter()
    done = 0
    for _ in range(args.steps):
        s._run_cycle()
        s._residual_norm()
        done += 1
        if time.perf_counter() - t > 150.0:
            break
    dt = time.perf_counter() - t
    value = dof * done / dt
    line = {
        "impl": "reference", "metric": "fine-grid DOF*V-cycles/s (fp64)", "value": value,
        "unit": "DOF*cycles/s", "n_gpus": args.gpus, "steps": done, "steps_requested": args.steps,
        "warmup": min(args.warmup, 1), "ms_per_step": dt / done * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.gpus > 1 else "weak",  # as the b200 arm: N ranks share the one problem
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": setup.name, "N": setup.grid.N, "levels": len(plans), "dof": dof,
                   "cycle": "V(2,1)", "parallelism": "cpu-1thread"},
        "cpu_baseline": {"value": value, "unit": "DOF*cycles/s", "cores": 1, "kind": "port",
                         "sample": f"{done} of {args.steps} requested full V(2,1) cycles at N={setup.grid.N} "
                                   f"(C oracle, 1 thread -- GS-LEX is sequential; SciPy SuperLU coarsest; "
                                   f"capped at ~150 s)"},
        "e2e": {"value": value, "unit": "DOF*cycles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup": setup_times,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- b200
def run_b200(args, rank, world, local_rank):
    import torch

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    from paper_2207_14208_b200 import _lib
    from paper_2207_14208_b200.solver import MultigridSolver

    setup, plans, f, g, e, setup_times = build_workload(args, device=local_rank)
    t0 = time.time()
    sharded = False
    if world > 1 and plans[0].d == 3:
        # z-slab sharding of the one problem over the ranks (strong scaling): planes exchanged as
        # device tensors over NCCL, residual norm MAX-all-reduced, small levels agglomerated on rank 0
        from paper_2207_14208_b200.slabs import TorchGroup, slab_solver

        solver = slab_solver(plans, f, g, e, setup.smoother, setup.cycle, TorchGroup(dist, local_rank),
                             device=local_rank, coarse_backend=args.coarse)
        sharded = solver.part.distributed(0)
    else:
        solver = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, device=local_rank,
                                            coarse_backend=args.coarse)
    copies = 1 if sharded else world  # unsharded ranks are independent replicas of the whole problem
    log(f"[bench] upload + coarse factor {time.time() - t0:.1f}s, device bytes "
        f"{solver.ctx.device_bytes / 1e9:.2f} GB")
    ctx = solver.ctx
    # a real (non-legacy) torch stream: the library launches on it, the CUDA
    # events below are recorded on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    p0 = plans[0]
    dof = p0.n_internal + p0.n_ghosts

    solver._set_data(f, g)
    solver._put_u(np.zeros(p0.n_nodes))
    def step(s):
        # what solve() does per cycle (reference solver.py:224-243): the cycle,
        # the residual-norm record and the max|u| renormalisation guard
        s._run_cycle()
        s._residual_norm()
        s._abs_max_scale()

    for _ in range(args.warmup):
        step(solver)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches0 = ctx.launches
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step(solver)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = ctx.launches - launches0
    # Kernel timings: the timed region replays one CUDA graph per cycle, whose
    # event nodes cannot be timed, so the same steps are repeated with direct
    # launches and CUDA events around every kernel class (same stream).
    ctx.profile(True)
    for _ in range(args.steps):
        step(solver)
    gs_ms, gs_n = ctx.profile_read("gs_sweep", 0)
    breakdown = {}
    for k in _lib.KCLASS:
        tms, n = ctx.profile_read(k)
        breakdown[k] = round(tms / args.steps, 3)
    ctx.profile(False)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = dof * args.steps * copies / (ms / 1e3)

    # roofline of the dominant kernel (fine-level GS sweep)
    peak, peak_kind = measured_peak()
    gs_bytes = 24 * p0.n_internal
    if sharded:  # this rank's share of the sweep (internal nodes taken as uniform over the planes)
        lo_, hi_ = solver.part.planes(0, rank)
        gs_bytes = int(gs_bytes * (hi_ - lo_) / (p0.N + 1))
    gs_avg_s = gs_ms / max(gs_n, 1) / 1e3
    achieved = gs_bytes / gs_avg_s / 1e9 if gs_n else None
    roofline = {"bound": "hbm", "kernel": ("gs_chain_kernel" if p0.d == 3 and p0.N >= 64 else "gs_diag_kernel" if p0.N >= 64 else "gs_stream_kernel")
                + " (finest level GS-LEX sweep)",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": ncu_traffic(),
                "algorithmic_bytes_per_launch": gs_bytes, "avg_launch_ms": gs_avg_s * 1e3,
                "launches_timed": gs_n, "peak_source": peak_kind,
                "timing": "CUDA events around each fine-level GS launch, same stream, profiled replay of the timed steps",
                "cycle_algorithmic_bytes": algorithmic_bytes(plans),
                "cycle_achieved_gbs": algorithmic_bytes(plans) / (ms / args.steps / 1e3) / 1e9}

    # end to end through the public API: solve() from pinned host memory
    e2e = None
    if not args.no_e2e:
        pin_f = torch.empty(p0.n_nodes, dtype=torch.float64, pin_memory=True).numpy()
        pin_u = torch.empty(p0.n_nodes, dtype=torch.float64, pin_memory=True).numpy()
        pin_f[:] = f
        solver.f_fine = pin_f
        pin_u[:] = 0.0
        torch.cuda.synchronize()
        t = time.perf_counter()
        u_out, rep = solver.solve(u=pin_u, cycles=args.steps)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        ran = max(rep.cycles_run, 1)  # solve() stops early at the divergence guard
        h2d = 8 * (2 * p0.n_nodes + p0.n_ghosts)
        d2h = 8 * p0.n_nodes + 24 * (ran + 1)
        e2e = {"value": dof * rep.cycles_run * copies / dt, "unit": "DOF*cycles/s",
               "h2d_bytes_per_step": h2d // ran, "d2h_bytes_per_step": d2h // ran,
               "solve_s": dt, "cycles": rep.cycles_run, "cycles_requested": args.steps, "diverged": rep.diverged,
               "final_residual": rep.residual_norms[-1],
               # convergence factor of this solve: geometric mean of the per-cycle
               # residual ratios after the first cycle (the reference's rho is the
               # mean ratio over cycles 11-15 of a 16-cycle measure_rho run)
               "conv_factor": (rep.residual_norms[-1] / rep.residual_norms[1]) ** (1.0 / (len(rep.residual_norms) - 2))
               if len(rep.residual_norms) > 2 and rep.residual_norms[1] > 0 else None,
               "rho_sequence": [float(x) for x in rep.rho_sequence]}

    # parity at the bench size: the e2e solve's residual history against the C
    # oracle's (tests/golden/_oracle_c4_512.json, zero initial guess; the oracle
    # is pinned bit for bit to reference-run fixtures)
    parity = None
    fixture = os.path.join(ROOT, "tests", "golden", "_oracle_c4_512.json")
    if e2e is not None and args.config == "c4" and setup.grid.N == 512 and os.path.exists(fixture):
        with open(fixture) as fh:
            want = [float.fromhex(x) for x in json.load(fh)["solve"]["residual_norms"]]
        m = min(len(want), len(rep.residual_norms))
        rel = [abs(a - b) / b for a, b in zip(rep.residual_norms[:m], want[:m])]
        parity = {"against": "C oracle residual history at this size (tests/golden/_oracle_c4_512.json)",
                  "cycles_compared": m - 1, "max_rel_diff": max(rel), "bitwise": rel == [0.0] * m,
                  "coarse": args.coarse}

    # the bit-exact path (host SciPy SuperLU coarsest solve through the callback)
    bitexact = None
    if not args.no_bitexact and args.coarse != "superlu" and setup.cycle.coarse_solver != "sweeps" and not sharded:
        s2 = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, device=local_rank,
                                        coarse_backend="superlu")
        s2.ctx.set_stream(stream.cuda_stream)
        s2._set_data(f, g)
        s2._put_u(np.zeros(p0.n_nodes))
        for _ in range(args.warmup):
            step(s2)
        torch.cuda.synchronize()
        b0 = torch.cuda.Event(enable_timing=True)
        b1 = torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(args.steps):
            step(s2)
        b1.record(stream)
        torch.cuda.synchronize()
        bms = b0.elapsed_time(b1)
        bitexact = {"value": dof * args.steps * copies / (bms / 1e3), "unit": "DOF*cycles/s",
                    "ms_per_step": bms / args.steps, "coarse": "direct:superlu (host callback, bitwise the reference)"}
        s2.ctx.close()
        del s2

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        n = args.cpu_sample_cycles
        sec, _ = oracle_cycles(plans, f, g, e, setup, n)
        cpu = {"value": dof * n / sec, "unit": "DOF*cycles/s", "cores": 1, "kind": "port",
               "sample": f"{n} V(2,1) cycle(s) + residual norm at N={setup.grid.N} on the host "
                         f"(C oracle, 1 thread, SciPy SuperLU coarsest), {sec:.1f}s"}

    if rank == 0:
        line = {
            "metric": "fine-grid DOF*V-cycles/s (fp64)", "value": value, "unit": "DOF*cycles/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": setup.name, "N": setup.grid.N, "levels": len(plans),
                       "dof": dof, "N_I": p0.n_internal, "N_G": p0.n_ghosts, "cycle": "V(2,1)",
                       "coarse": f"{setup.cycle.coarse_solver}:{args.coarse}", "parallelism": (f"z-slabs{world} (one problem; whole-slab pipelined sweeps, NCCL plane exchange)" if sharded
                                       else f"replicas{world} (independent copies, not decomposed)" if world > 1 else "single-gpu"),
                       "l2_flush": f"not needed: every grid vector ({8 * p0.n_nodes / 1e9:.2f} GB) exceeds L2"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "parity": parity, "bitexact_path": bitexact,
            "gpu_launches": launches,
            "clocks": clocks.summary(), "breakdown_ms_per_cycle": breakdown, "setup": setup_times,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
    else:
        run_b200(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
