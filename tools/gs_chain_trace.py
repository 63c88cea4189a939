"""Task timeline of the gs_chain GS kernel (GMG_GS_TRACE=1).
usage: python tools/gs_chain_trace.py c4:512 [level]   (build with -DGS_CHAIN_TRACE=1 for the wait split)"""
import os
import sys

os.environ["GMG_GS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import _plans
from paper_2207_14208_b200 import _lib
from paper_2207_14208_b200.solver import MultigridSolver

setup, plans, f, g, e = _plans.load(sys.argv[1])
level = int(sys.argv[2]) if len(sys.argv) > 2 else 0
solver = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, device=0, coarse_backend="superlu")
ctx = solver.ctx
p = plans[level]
rng = np.random.default_rng(1)
ctx.set_vector(level, _lib.U, rng.standard_normal(p.n_nodes))
ctx.set_vector(level, _lib.F, rng.standard_normal(p.n_nodes))
for _ in range(3):
    ctx.apply(level, _lib.OP_GS_SWEEP)
Nl = p.N
C = (Nl - 1 + 15) // 16
Bn = (Nl - 1 + 7) // 8
tasks = sorted([(c, b) for c in range(C) for b in range(Bn)], key=lambda t: (2 * t[0] + 3 * t[1], t[0]))
cpl = Nl + 1 + 32
buf = np.zeros(len(tasks) * (16 + 2 * cpl), dtype=np.int64)
ctx.lib.gmg_debug_gs_trace(ctx.ctx, level, buf.ctypes.data, buf.size)
raw = buf[:len(tasks) * 16].reshape(-1, 16)
stamps = buf[len(tasks) * 16:].reshape(-1, 2, cpl)  # [c * Bn + b][push / accept][plane]
t0 = raw[:, 0].min()
claim = (raw[:, 0] - t0) / 1e3
done = (raw[:, 1] - t0) / 1e3
start = np.where(raw[:, 3] > 0, (raw[:, 3] - t0) / 1e3, np.nan)
dur = done - claim
print(f"level {level} N={Nl}: {len(tasks)} tasks (C={C}, Bn={Bn}), sweep span {done.max():.1f} us")
print(f"task duration us: median {np.median(dur):.1f}, p10 {np.percentile(dur, 10):.1f}, p90 {np.percentile(dur, 90):.1f}, max {dur.max():.1f}")
comp = raw[:, 4].astype(float)
nz = comp > 0
if nz.any():
    steps = Nl - 1 + 23
    print(f"compute cycles per task (median): total {np.median(comp[nz]):.0f} = {np.median(comp[nz]) / steps:.0f}/step, "
          f"waiting for slots {np.median(raw[nz, 5]):.0f}, for cells {np.median(raw[nz, 6]):.0f}")
    print(f"per step (median task): writer waiting for compute {np.median(raw[nz, 6]) / steps:.0f}, writer other {np.median(raw[nz, 7]) / steps:.0f}; "
          f"loader blocked by the ring {np.median(raw[nz, 8]) / steps:.0f}, loader otherwise {np.median(raw[nz, 9]) / steps:.0f}")
    pol = raw[:, 11] > 0
    if pol.any():
        print(f"cells warp (lane 0, per task median): poll round trip {np.median(raw[pol, 10] / raw[pol, 11]):.0f} cycles, "
              f"{np.median(raw[pol, 12]):.0f} polls of which {np.median(raw[pol, 13]):.0f} accepted something, "
              f"{np.median(raw[pol, 11]):.0f} with the ring ready")
    i0 = tasks.index((0, 0))
    print(f"task (0,0): cycles {raw[i0, 4]} = {raw[i0, 4] / steps:.0f}/step, slots {raw[i0, 5]}, cells {raw[i0, 6]}")
print("start/done (us) of tasks (c, b):")
for c in sorted({0, 1, 2, C // 2, C - 1}):
    row = []
    for b in sorted({0, 1, 2, Bn // 2, Bn - 1}):
        i = tasks.index((c, b))
        row.append(f"({c},{b}) {start[i]:7.1f}/{done[i]:7.1f}")
    print("   ", "  ".join(row))
sms = raw[:, 2]
print("tasks per SM: max", np.bincount(sms).max(), "SMs used", len(np.unique(sms)))

# hand-off latency of the row cells (column 0): push by task (c, b) -> accept by task (c, b+1)
lat = []
for c in range(C):
    for b in range(Bn - 1):
        push = stamps[c * Bn + b, 0]
        acc = stamps[c * Bn + b + 1, 1]
        ok = (push > 0) & (acc > 0)
        if ok.any():
            lat.append((acc[ok] - push[ok]) / 1e3)
if lat:
    lat = np.concatenate(lat)
    print(f"row-cell hand-off, push -> accepted in the downstream ring (us): median {np.median(lat):.2f}, p10 {np.percentile(lat, 10):.2f}, "
          f"p90 {np.percentile(lat, 90):.2f}, max {lat.max():.2f} over {len(lat)} cells")
