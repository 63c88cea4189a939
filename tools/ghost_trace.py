"""Ghost-sweep timeline per DAG batch (GMG_GS_TRACE=1).
usage: GMG_GS_TRACE=1 python tools/ghost_trace.py c4:256 [level]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GMG_GS_TRACE", "1")
import numpy as np

from paper_2207_14208_b200 import _lib
from paper_2207_14208_b200 import configs as CF
from paper_2207_14208_b200.cycle import CycleDriver
from paper_2207_14208_b200.transfer import build_hierarchy

name, N = sys.argv[1].split(":")
N = int(N)
level = int(sys.argv[2]) if len(sys.argv) > 2 else 0
setup = CF.config_pores(N=N) if name == "c4" else CF.CONFIGS[name](N)
levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
ctx = _lib.Context(plans[0].d, len(plans))
for i, p in enumerate(plans):
    ctx.set_level(i, p)
p = plans[level]
ctx.set_vector(level, _lib.U, np.zeros(p.n_nodes))
ctx.set_vector(level, _lib.G, np.ones(p.n_ghosts))
for _ in range(3):
    ctx.apply(level, _lib.OP_GHOST_SWEEP)
ctx.profile(True)
ctx.apply(level, _lib.OP_GHOST_SWEEP)
ms, _ = ctx.profile_read("ghost_sweep", level)
ctx.profile(False)
b = np.asarray(p.ghost_batch)
cnt = np.bincount(b)
pad = (cnt + 31) // 32 * 32
nslots = int(pad.sum())
tr = ctx.ghost_trace(level, nslots).astype(np.float64)
off = np.concatenate([[0], np.cumsum(pad)])
t0 = tr[tr[:, 0] > 0, 0].min()
print(f"level {level}: sweep {ms:.3f} ms, {len(cnt)} batches")
prev_done = 0.0
for k in range(len(cnt)):
    seg = tr[off[k]:off[k] + cnt[k]]  # real slots come first inside a padded batch? (slot order: lex)
    seg = tr[off[k]:off[k + 1]]
    seg = seg[seg[:, 2] > 0]
    claim = (seg[:, 0].min() - t0) / 1e3
    met_first = (seg[:, 1][seg[:, 1] > 0].min() - t0) / 1e3 if (seg[:, 1] > 0).any() else float("nan")
    met_last = (seg[:, 1].max() - t0) / 1e3
    done = (seg[:, 2].max() - t0) / 1e3
    if k < 12 or k % 10 == 0 or k > len(cnt) - 4:
        print(f"  batch {k:3d} n={cnt[k]:6d}: claimed {claim:8.2f}  deps met {met_first:8.2f}..{met_last:8.2f}  "
              f"done {done:8.2f} us  (+{done - prev_done:6.2f})")
    prev_done = done

# ---- per-ghost lag: deps met - latest dependency stored
ng = p.n_ghosts
d = p.d
n1 = p.N + 1
m = 3 ** d
lexmap = -np.ones(n1 ** d, dtype=np.int64)
lexmap[np.asarray(p.ghost_idx)] = np.arange(ng)
low = np.asarray(p.ghost_low).reshape(ng, d)
w = np.asarray(p.ghost_w).reshape(ng, m)
# slot of each lex ghost: batches padded to 32, lex order inside a batch
slot = np.empty(ng, dtype=np.int64)
fill = off[:-1].copy()
for i in range(ng):
    slot[i] = fill[b[i]]
    fill[b[i]] += 1
latest = np.zeros(ng)
for jst in range(m):
    o = [(jst // 9, (jst // 3) % 3, jst % 3)] if d == 3 else [(jst // 3, jst % 3)]
    flat = np.zeros(ng, dtype=np.int64)
    for k in range(d):
        flat = flat * n1 + low[:, k] + o[0][k]
    jg = lexmap[flat]
    use = (jg >= 0) & (jg != np.arange(ng)) & (w[:, jst] != 0.0)
    i_idx = np.nonzero(use)[0]
    jgv = jg[use]
    # RAW: i waits for jg < i ; WAR: jg waits for i < jg
    later = np.maximum(i_idx, jgv)
    earlier = np.minimum(i_idx, jgv)
    np.maximum.at(latest, later, tr[slot[earlier], 2])
met = tr[slot, 1]
has = latest > 0
lag = (met[has] - latest[has]) / 1e3
print(f"deps met - latest dep stored (us): median {np.median(lag):.2f}, p90 {np.percentile(lag, 90):.2f}, "
      f"max {lag.max():.2f}; ghosts with deps {has.sum()}")
claimed = tr[slot, 0]
late = (claimed[has] - latest[has]) / 1e3
print(f"claimed - latest dep stored (us): median {np.median(late):.2f}, p90 {np.percentile(late, 90):.2f} "
      f"(positive = the chunk started after its deps were done)")
