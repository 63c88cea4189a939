"""Timeline of the warp-specialised GS sweep on one level (GMG_GS_TRACE=1).

usage: GMG_GS_TRACE=1 python tools/gs_trace.py c4:512 [level] [max_tasks]
Prints per-task duration, cycles per consumer step, data-wait share and the
start lag along the chunk (c) and block (b) directions.
"""
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
if len(sys.argv) > 3:
    os.environ["GMG_GS_MAX_TASKS"] = sys.argv[3]
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
ctx.apply(level, _lib.OP_GS_SWEEP)
ms, n = ctx.profile_read("gs_sweep", level)
ctx.profile(False)
d = p.d
Nn = p.N
C = (Nn - 1 + 31) // 32
R = 16 if d == 3 else 1  # pseudo-lines per plane (both kernels)
RB = 16 if os.environ.get("GMG_GS_WS") == "1" else 14  # grid rows per block
Bn = (Nn - 1 + RB - 1) // RB if d == 3 else 1
tasks = [(c, s - c) for s in range(C + Bn - 1) for c in range(C) if 0 <= s - c < Bn]
nt = len(tasks)
if os.environ.get("GMG_GS_MAX_TASKS"):
    nt = min(nt, int(os.environ["GMG_GS_MAX_TASKS"]))
tr = ctx.gs_trace(level, len(tasks))
if tr is None:
    sys.exit("no trace (GMG_GS_TRACE=1 and a TMA-path level needed)")
tr = tr[:nt]
t0 = tr[:, 0].min()
start = (tr[:, 0] - t0) / 1e3  # us
end = (tr[:, 1] - t0) / 1e3
dur = end - start
lines = (Nn - 1) * R if d == 3 else Nn
steps = lines + 31
cps = tr[:, 4] / steps
wait = tr[:, 3] / np.maximum(tr[:, 4], 1)
print(f"level {level} N={Nn} tasks={nt} C={C} Bn={Bn} sweep {ms:.3f} ms (events), "
      f"span {end.max():.1f} us")
print(f"task duration us: mean {dur.mean():.1f} min {dur.min():.1f} max {dur.max():.1f}")
print(f"consumer cycles/step: mean {cps.mean():.1f} min {cps.min():.1f} max {cps.max():.1f}; "
      f"data-wait share mean {wait.mean():.3f}")
steps_f = float(steps)
print(f"compute-warp wait cycles/step (all data): {tr[:, 3].mean() / steps_f:.1f}")
print(f"u arrival latency when waited {tr[:, 5].mean():.0f} cycles over {tr[:, 7].mean():.0f} waits/task; "
      f"writer idle polls {tr[:, 7].mean():.0f}, publish cycles/batch {tr[:, 11].mean() / max(lines / 8, 1):.0f}")
nU = (lines + 32) / 8 if d == 3 else lines / 8
nF = (lines + 72) / 8
print(f"u loader: lead {tr[:, 14].mean() / nU:.1f} steps, "
      f"idle polls {tr[:, 10].mean():.0f}; f issue cycles per batch {tr[:, 13].mean() / nF:.0f}, "
      f"f lead {tr[:, 15].mean() / nF:.1f} steps")
sm = tr[:, 2] & 0xFFFF
wid = tr[:, 2] >> 16
print(f"compute-warp SMSP (warpid % 4) histogram: {np.bincount(wid % 4, minlength=4).tolist()}")
print(f"SMs used {len(np.unique(sm))}, max tasks per SM {np.bincount(sm).max()}")
st = {tasks[i]: start[i] for i in range(nt)}
en = {tasks[i]: end[i] for i in range(nt)}
lagc = [st[(c, b)] - st[(c - 1, b)] for (c, b) in st if (c - 1, b) in st]
lagb = [st[(c, b)] - st[(c, b - 1)] for (c, b) in st if (c, b - 1) in st]
if lagc:
    print(f"start lag along c: mean {np.mean(lagc):.2f} us (median {np.median(lagc):.2f})")
if lagb:
    print(f"start lag along b: mean {np.mean(lagb):.2f} us (median {np.median(lagb):.2f})")
for key in [(0, 0), (C - 1, 0), (0, Bn - 1), (C - 1, Bn - 1)]:
    if key in st:
        print(f"task {key}: start {st[key]:.1f} end {en[key]:.1f} us")
if d == 3 and nt == len(tasks):
    t64 = {tasks[i]: (tr[i, 5] - t0) / 1e3 for i in range(nt)}
    t512 = {tasks[i]: (tr[i, 7] - t0) / 1e3 for i in range(nt)}
    for name_, tt in (("batch 64", t64), ("batch 512", t512)):
        lc = [tt[(c, b)] - tt[(c - 1, b)] for (c, b) in tt if (c - 1, b) in tt]
        lb = [tt[(c, b)] - tt[(c, b - 1)] for (c, b) in tt if (c, b - 1) in tt]
        print(f"{name_}: lag per c-hop {np.median(lc):.2f} us (mean {np.mean(lc):.2f}), "
              f"per b-hop {np.median(lb):.2f} us (mean {np.mean(lb):.2f})")
    idx = {tasks[i]: i for i in range(nt)}
    pub = {k: tr[i, 11] for k, i in idx.items()}     # writer: flag for lines < 520 issued
    seen = {k: tr[i, 12] for k, i in idx.items()}    # halo loader: left flag >= 520 seen
    hst = {k: tr[i, 15] for k, i in idx.items()}     # halo loader: batch 64 stored
    c64 = {k: tr[i, 5] for k, i in idx.items()}      # compute warp: batch 64 done
    lat = [(seen[(c, b)] - pub[(c - 1, b)]) / 1e3 for (c, b) in idx if c > 0 and seen[(c, b)] and pub[(c - 1, b)]]
    st_ = [(hst[(c, b)] - seen[(c, b)]) / 1e3 for (c, b) in idx if c > 0 and seen[(c, b)] and hst[(c, b)]]
    up = [(pub[(c - 1, b)] - c64[(c - 1, b)]) / 1e3 for (c, b) in idx if c > 0]
    print(f"c-hop pieces (us, median): upstream batch-64 done -> flag issued {np.median(up):.2f}; "
          f"flag issued -> seen downstream {np.median(lat):.2f}; seen -> halo stored {np.median(st_):.2f}")
    iss = {k: tr[i, 14] for k, i in idx.items()}
    stb = {k: tr[i, 9] for k, i in idx.items()}
    cav = {k: tr[i, 6] for k, i in idx.items()}
    def med(x):
        return float(np.median(x)) if len(x) else float("nan")
    ks = [(c, b) for (c, b) in idx if c > 0 and b == 0 and seen[(c, b)] and pub[(c - 1, b)]]
    print("c-hop timeline (us, median over b=0 tasks, relative to upstream flag for lines < 520):")
    print(f"  seen {med([(seen[k] - pub[(k[0]-1, k[1])]) / 1e3 for k in ks]):.2f}"
          f"  issue {med([(iss[k] - pub[(k[0]-1, k[1])]) / 1e3 for k in ks]):.2f}"
          f"  store-begin {med([(stb[k] - pub[(k[0]-1, k[1])]) / 1e3 for k in ks]):.2f}"
          f"  stored {med([(hst[k] - pub[(k[0]-1, k[1])]) / 1e3 for k in ks]):.2f}"
          f"  compute sees {med([(cav[k] - pub[(k[0]-1, k[1])]) / 1e3 for k in ks]):.2f}")
    c68 = {k: tr[i, 17] for k, i in idx.items()}
    wr = {k: tr[i, 16] for k, i in idx.items()}
    print(f"writer (us, median): line 519 done -> writer starts batch 64 {med([(wr[k] - c68[k]) / 1e3 for k in idx]):.2f}; "
          f"-> flag issued {med([(pub[k] - wr[k]) / 1e3 for k in idx]):.2f}")
    print(f"writer wait for store completion: {tr[:, 13].mean() / (lines / 8):.0f} cycles/batch")
    rate = (t512[(0, 0)] - t64[(0, 0)]) / (448 * 8)
    print(f"task (0,0) step time between batches 64 and 512: {rate * 1e3:.1f} ns")
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/gs_trace_{name}{N}_L{level}.npz", trace=tr, tasks=np.array(tasks[:nt]))
# per-task breakdown of a few tasks (cycles per step)
for key in [(0, 0), (1, 0), (0, 1), (C // 2, Bn // 2)]:
    if key in {tuple(t) for t in tasks[:nt]}:
        i = [tuple(t) for t in tasks[:nt]].index(key)
        t = tr[i]
        print(f"task {key}: total {t[4] / steps:.0f} cyc/step, waits: u+f {t[8] / steps:.0f}, "
              f"halo {(t[3] - t[8]) / steps:.0f}; compute {(t[4] - t[3]) / steps:.0f}")
