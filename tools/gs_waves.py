"""Residency ("wave") analysis of the 3-D two-chain GS sweep (GMG_GS_TRACE=1).

usage: python tools/gs_waves.py c4:512 [level]
The finest 512^3 sweep has 592 tasks (16 chunks x 37 blocks) but only
3 CTAs x 148 SMs = 444 are resident; the rest start only when a resident task
ends.  Prints task duration, the start time of the non-resident tasks against
the end of the first tasks, the number of running tasks over time and the
critical (last-ending) tasks.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GMG_GS_TRACE"] = "1"
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
ctx.set_vector(level, _lib.F, np.ones(p.n_nodes))
for _ in range(3):
    ctx.apply(level, _lib.OP_GS_SWEEP)
ctx.synchronize()
ctx.profile(True)
for _ in range(int(os.environ.get("GS_WAVES_REPS", "5"))):
    ctx.apply(level, _lib.OP_GS_SWEEP)
ms, nrep = ctx.profile_read("gs_sweep", level)
ms /= max(nrep, 1)
ctx.profile(False)
Nn = p.N
C = (Nn - 1 + 31) // 32
Bn = (Nn - 1 + 13) // 14
tasks = [(c, s - c) for s in range(C + Bn - 1) for c in range(C) if 0 <= s - c < Bn]
nt = len(tasks)
tr = ctx.gs_trace(level, nt)
if tr is None:
    sys.exit("no trace")
tr = tr[:nt]
t0 = tr[:, 0].min()
st = (tr[:, 0] - t0) / 1e3
en = (tr[:, 1] - t0) / 1e3
dur = en - st
sm = tr[:, 2] & 0xFFFF
diag = np.array([c + b for c, b in tasks])
print(f"level {level} N={Nn} tasks={nt} C={C} Bn={Bn} sweep {ms:.3f} ms (events, mean of {nrep}), span {en.max():.1f} us, "
      f"SMs {len(np.unique(sm))}, max tasks/SM {np.bincount(sm).max()}")
print(f"task duration us: mean {dur.mean():.1f} min {dur.min():.1f} max {dur.max():.1f}; "
      f"compute cycles/step mean {(tr[:, 4] / (8 * Nn + 31)).mean():.0f}")
first_end = np.sort(en)
order = np.argsort(st)
late = st > first_end[0]  # started only after some task finished (not resident at launch)
print(f"tasks started after the first task ended: {late.sum()}; first end {first_end[0]:.1f} us; "
      f"their starts {st[late].min() if late.any() else 0:.1f}..{st[late].max() if late.any() else 0:.1f} us; "
      f"their ends up to {en[late].max() if late.any() else 0:.1f} us")
for d in range(0, diag.max() + 1, 5):
    m = diag == d
    print(f"  diagonal {d:2d}: start {st[m].min():7.1f}..{st[m].max():7.1f}  end {en[m].min():7.1f}..{en[m].max():7.1f}  "
          f"dur {dur[m].mean():6.1f}")
grid = np.linspace(0, en.max(), 21)
running = [int(((st <= t) & (en > t)).sum()) for t in grid]
print("running tasks over time:", " ".join(f"{t:.0f}:{r}" for t, r in zip(grid, running)))
last = np.argsort(en)[-5:]
print("last-ending tasks (c, b, start, end):", [(tasks[i], round(st[i], 1), round(en[i], 1)) for i in last])

# hand-off decomposition at batch 64 (trace words: 10 upstream compute done with
# batch 68 (writer batch 64 becomes final), 9 writer notices it, 5 / 12 progress
# 520 / 528 issued, 6 downstream halo loader issues batch 64, 7 halo stored,
# 8 downstream compute starts batch 64, 11 compute starts batch 512)
idx = {t: i for i, t in enumerate(tasks)}
rate = (tr[:, 11] - tr[:, 8]) / (448 * 8.0)
ok = (tr[:, 8] > 0) & (tr[:, 11] > 0)
print(f"compute ns/step between batches 64 and 512: median {np.median(rate[ok]):.0f} (min {rate[ok].min():.0f}, max {rate[ok].max():.0f})")
for kind, du in (("c-hop", (-1, 0)), ("b-hop", (0, -1))):
    rows = []
    for (c, b), i in idx.items():
        up = idx.get((c + du[0], b + du[1]))
        if up is None or tr[i, 8] == 0 or tr[up, 10] == 0:
            continue
        pub = tr[up, 5] if kind == "c-hop" else tr[up, 12]
        rows.append([tr[up, 9] - tr[up, 10], pub - tr[up, 9], tr[i, 6] - pub, tr[i, 7] - tr[i, 6],
                     tr[i, 8] - tr[i, 7], tr[i, 8] - tr[up, 8]])
    r = np.median(np.array(rows), axis=0) / 1e3
    print(f"{kind} (us, median of {len(rows)}): upstream batch final -> writer notices {r[0]:.2f}; -> flag {r[1]:.2f}; "
          f"-> downstream halo issue {r[2]:.2f}; -> halo stored {r[3]:.2f}; -> compute starts {r[4]:.2f}; "
          f"batch-64 start lag {r[5]:.2f}")
