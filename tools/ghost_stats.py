"""Ghost-sweep DAG statistics per level (batches = DAG depth, ghosts, deps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2207_14208_b200 import configs as CF
from paper_2207_14208_b200.cycle import CycleDriver
from paper_2207_14208_b200.transfer import build_hierarchy

name, N = sys.argv[1].split(":")
N = int(N)
setup = CF.config_pores(N=N) if name == "c4" else CF.CONFIGS[name](N)
levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
for l, p in enumerate(plans):
    if p.n_ghosts == 0:
        continue
    b = np.asarray(p.ghost_batch)
    cnt = np.bincount(b)
    print(f"L{l} N={p.N}: ghosts {p.n_ghosts}, batches {len(cnt)}, per-batch max {cnt.max()} "
          f"median {int(np.median(cnt))}, first 8 {cnt[:8].tolist()}, last 8 {cnt[-8:].tolist()}")
for l, p in enumerate(plans):
    print(f"L{l} N={p.N}: band nodes {len(p.band_idx)}, bfs groups {list(np.asarray(p.bfs_len))}")
