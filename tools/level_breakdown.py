"""Per-level, per-kernel-class breakdown of one V-cycle + residual norm
(direct launches with CUDA events).  usage: python tools/level_breakdown.py c4:512"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2207_14208_b200 import _lib
from paper_2207_14208_b200 import configs as CF
from paper_2207_14208_b200.cycle import CycleDriver
from paper_2207_14208_b200.solver import MultigridSolver
from paper_2207_14208_b200.transfer import build_hierarchy

name, N = sys.argv[1].split(":")
N = int(N)
setup = CF.config_pores(N=N) if name == "c4" else CF.CONFIGS[name](N)
levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
if setup.f_seed is not None:
    f = CF.pore_rhs(setup, plans[0].labels)
s = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, coarse_backend="device-inverse")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
s.ctx.set_stream(stream.cuda_stream)
s._set_data(f, g)
s._put_u(np.zeros(plans[0].n_nodes))
for _ in range(2):
    s._run_cycle()
    s._residual_norm()
s.ctx.profile(True)
reps = 3
for _ in range(reps):
    s._run_cycle()
    s._residual_norm()
print(f"{'class':12s} " + " ".join(f"L{l}(N={p.N})".rjust(12) for l, p in enumerate(plans)) + "       total")
grand = 0.0
for k in _lib.KCLASS:
    row = []
    for l in range(len(plans)):
        ms, n = s.ctx.profile_read(k, l)
        row.append(ms / reps)
    grand += sum(row)
    print(f"{k:12s} " + " ".join(f"{v:12.3f}" for v in row) + f" {sum(row):11.3f}")
print(f"total {grand:.3f} ms/cycle")
