"""Time cycles (graph vs direct) and the per-class breakdown (direct, profiled)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2207_14208_b200 import configs as CF, _lib
from paper_2207_14208_b200.transfer import build_hierarchy
from paper_2207_14208_b200.cycle import CycleDriver
from paper_2207_14208_b200.solver import MultigridSolver

name, N = sys.argv[1].split(":"); N = int(N)
backend = sys.argv[2] if len(sys.argv) > 2 else "device-inverse"
setup = CF.config_pores(N=N) if name == "c4" else CF.CONFIGS[name](N)
levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
if setup.f_seed is not None:
    f = CF.pore_rhs(setup, plans[0].labels)
s = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, coarse_backend=backend)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); s.ctx.set_stream(stream.cuda_stream)
s._set_data(f, g); s._put_u(np.zeros(plans[0].n_nodes))
for _ in range(2):
    s._run_cycle(); s._residual_norm()
for mode in ("cycle-only", "cycle+sync", "norm-only", "cycle+norm", "cycle+absmax"):
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t = time.perf_counter(); ev0.record(stream)
    for _ in range(5):
        if mode != "norm-only": s._run_cycle()
        if mode == "cycle+sync": s.ctx.synchronize()
        if mode in ("cycle+norm", "norm-only"): s._residual_norm()
        if mode == "cycle+absmax": s._abs_max_scale()
    ev1.record(stream); torch.cuda.synchronize(); w = time.perf_counter() - t
    print(f"{mode}: {ev0.elapsed_time(ev1)/5:.2f} ms/cycle (events), {w/5*1e3:.2f} ms/cycle wall", flush=True)
s.ctx.profile(True)
for _ in range(2):
    s._run_cycle(); s._residual_norm()
tot = 0
for k in _lib.KCLASS:
    ms, n = s.ctx.profile_read(k); tot += ms
    print(f"  {k:12s} {ms/2:8.3f} ms/cycle ({n//2} regions)")
print("  sum", tot / 2)
