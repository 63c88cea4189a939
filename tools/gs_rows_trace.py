"""Task timeline of the gs_rows GS kernel (GMG_GS_TRACE=1) on the finest level.

usage: python tools/gs_rows_trace.py c4:512 [level]
Prints the sweep span, per-task durations, where the compute warps wait
(slots / cells / step barrier) and the start time along the wavefront.
"""
import os
import sys

os.environ["GMG_GS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2207_14208_b200 import _lib
from paper_2207_14208_b200 import configs as CF
from paper_2207_14208_b200.cycle import CycleDriver
from paper_2207_14208_b200.solver import MultigridSolver
from paper_2207_14208_b200.transfer import build_hierarchy

level = int(sys.argv[2]) if len(sys.argv) > 2 else 0
R = int(os.environ.get("GS_ROWS_R", 4))
import _plans
setup, plans, f, g, e = _plans.load(sys.argv[1])
solver = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, device=0,
                                    coarse_backend="device-inverse")
ctx = solver.ctx
p = plans[level]
rng = np.random.default_rng(1)
ctx.set_vector(level, _lib.U, rng.standard_normal(p.n_nodes))
ctx.set_vector(level, _lib.F, rng.standard_normal(p.n_nodes))
for _ in range(3):
    ctx.apply(level, _lib.OP_GS_SWEEP)
Nl = p.N
C = (Nl - 1 + 31) // 32
Bn = (Nl - 1 + R - 1) // R
tasks = sorted([(c, b) for c in range(C) for b in range(Bn)], key=lambda t: (3 * t[0] + t[1], t[0]))
tr = ctx.gs_trace(level, len(tasks))
tr = tr.reshape(-1, 24)[:, :16] if tr is not None and tr.shape[1] == 24 else tr
raw = np.zeros((len(tasks), 16), dtype=np.int64)
buf = np.zeros(len(tasks) * 16 + 8 * 8 * 1024, dtype=np.int64)
n = ctx.lib.gmg_debug_gs_trace(ctx.ctx, level, buf.ctypes.data, buf.size)
raw = buf[:len(tasks) * 16].reshape(-1, 16)
blocks = buf[len(tasks) * 16:len(tasks) * 16 + 8 * 1024].reshape(8, 256, 4)
for tid in (0, 3):
    bl = blocks[tid]
    bl = bl[bl[:, 0] > 0]
    if len(bl):
        d = np.diff(bl[:, 0])
        print(f"task {tid} ({tasks[tid]}): block cycles median {np.median(d):.0f}; (cycles, lready - p, wfree - p) "
              "every 8th block:", " ".join(f"({d[i]},{bl[i, 1] - bl[i, 3]},{bl[i, 2] - bl[i, 3]})" for i in range(0, len(d), 8)))
t0 = raw[:, 0].min()
claim = (raw[:, 0] - t0) / 1e3
done = (raw[:, 1] - t0) / 1e3
start = np.where(raw[:, 3] > 0, (raw[:, 3] - t0) / 1e3, np.nan)
dur = done - claim
print(f"level {level} N={Nl}: {len(tasks)} tasks (C={C}, Bn={Bn}), sweep span {done.max():.1f} us")
print(f"task duration us: median {np.median(dur):.1f}, p90 {np.percentile(dur, 90):.1f}, max {dur.max():.1f}")
comp = raw[:, 4].astype(float)
nz = comp > 0
print(f"compute cycles per task (median): total {np.median(comp[nz]):.0f}, slots {np.median(raw[nz, 5]):.0f}, "
      f"cells {np.median(raw[nz, 6]):.0f}, barrier {np.median(raw[nz, 7]):.0f}; loader ring-wait "
      f"{np.median(raw[nz, 8]):.0f}, writer wait {np.median(raw[nz, 9]):.0f}")
print(f"compute start - claim (median us): {np.nanmedian(start - claim):.2f}; TMA group latency (cycles, "
      f"median task mean) {np.median(raw[nz, 10]):.0f}; loader blocked by the ring (polls) {np.median(raw[nz, 8]):.0f}")
steps = np.median(comp[nz]) / 1.9e3
print("cycles/step (median task, ~546 steps at 512):", np.median(comp[nz]) / (Nl - 1 + R + 31))
print("wavefront: start time (us) of tasks (c, b):")
for c in (0, 1, 2, C // 2, C - 1):
    row = []
    for b in (0, 1, 2, 10, Bn // 2, Bn - 1):
        i = tasks.index((c, b))
        row.append(f"({c},{b}) {start[i]:7.1f}/{done[i]:7.1f}")
    print("   ", "  ".join(row))
sms = raw[:, 2]
print("tasks per SM: max", np.bincount(sms).max(), "SMs used", len(np.unique(sms)))
