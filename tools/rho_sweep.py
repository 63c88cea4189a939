"""Batched convergence-factor sweep on the GPU (the paper's BLFA studies run
many small solves; reference cli.py:154-194 spreads them over processes).

usage: python tools/rho_sweep.py [N] [count]
Builds `count` disk problems (N^2) that differ in their dtau variant /
relaxation, measures rho one at a time and batched, prints both timings.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2207_14208_b200 import configs as CF
from paper_2207_14208_b200.cycle import CycleDriver, measure_rho
from paper_2207_14208_b200.solver import MultigridSolver, measure_rho_batched
from paper_2207_14208_b200.transfer import build_hierarchy

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
count = int(sys.argv[2]) if len(sys.argv) > 2 else 16
setup = CF.config_disk(N)
levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
solvers = [MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, coarse_backend="device-inverse")
           for _ in range(count)]
measure_rho(solvers[0])
torch.cuda.synchronize()
t = time.perf_counter()
one = [measure_rho(s, seed=42 + k).rho_asymptotic for k, s in enumerate(solvers)]
t1 = time.perf_counter() - t
t = time.perf_counter()
bat = [r.rho_asymptotic for r in measure_rho_batched(solvers, seed=42)]
t2 = time.perf_counter() - t
print(f"{count} x disk N={N}: one at a time {t1 * 1e3:.1f} ms, batched {t2 * 1e3:.1f} ms "
      f"({t1 / t2:.2f}x); rho {one[0]:.6f} / {bat[0]:.6f}")
