"""Compare one GS sweep of the gs_chain kernel with gs_diag (GMG_GS_CHAIN=0) on
the same random input; report where they differ.  usage: gs_cmp.py c4:64 [level]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import _plans
from paper_2207_14208_b200 import _lib
from paper_2207_14208_b200.solver import MultigridSolver

setup, plans, f, g, e = _plans.load(sys.argv[1])
level = int(sys.argv[2]) if len(sys.argv) > 2 else 0
p = plans[level]
rng = np.random.default_rng(1)
u0 = rng.standard_normal(p.n_nodes)
f0 = rng.standard_normal(p.n_nodes)
res = {}
MODE = os.environ.get("CMP_MODE", "01")  # which two kernels: 0 gs_diag, 1 gs_chain ("11": chain against itself)
for slot, v in zip(("0", "1"), MODE):
    os.environ["GMG_GS_CHAIN"] = v
    s = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, device=0, coarse_backend="superlu")
    ctx = s.ctx
    ctx.set_vector(level, _lib.U, u0)
    ctx.set_vector(level, _lib.F, f0)
    nsweeps = int(os.environ.get("SWEEPS", 1))
    for _ in range(nsweeps):
        ctx.apply(level, _lib.OP_GS_SWEEP)
    res[slot] = ctx.get_vector(level, _lib.U, p.n_nodes).copy()
    ctx.close()
n = p.N + 1
a = res["0"].reshape(n, n, n)
b = res["1"].reshape(n, n, n)
bad = np.argwhere(a != b)
print(f"level {level} N={p.N}: {len(bad)} of {a.size} nodes differ")
if len(bad):
    print("first 12 (p, r, k):", bad[:12].tolist())
    c = (bad[:, 2] - 1) // 16
    bl = (bad[:, 1] - 1) // 8
    print("by chunk c:", np.bincount(c).tolist())
    print("by block b:", np.bincount(bl).tolist())
    print("by lane j:", np.bincount((bad[:, 2] - 1) % 16, minlength=16).tolist())
    print("by chain I:", np.bincount((bad[:, 1] - 1) % 8, minlength=8).tolist())
    print("by plane:", np.bincount(bad[:, 0]).tolist())
    first = bad[0]
    print("first diff values:", a[tuple(first)], b[tuple(first)], "input", u0.reshape(n, n, n)[tuple(first)])
    unchanged = np.sum(b[tuple(bad.T)] == u0.reshape(n, n, n)[tuple(bad.T)])
    print("differing nodes left at their input value by gs_chain:", int(unchanged))
    d1 = (a != b)
    P0 = int(bad[:, 0].min())
    for (cc, bb) in ((0, 0), (1, 2)):
        print(f"task c={cc} b={bb} plane {P0}: rows = chains I, cols = lanes j ('x' differs, '.' equal, ' ' not internal)")
        lab = p.labels.reshape(n, n, n)
        for I in range(8):
            r = 1 + 8 * bb + I
            print("   ", "".join(("x" if d1[P0, r, 1 + 16 * cc + j] else ("." if lab[P0, r, 1 + 16 * cc + j] == 0 else " ")) for j in range(16)))
    others = bad[bad[:, 0] != P0]
    print("diffs on other planes:", others[:20].tolist())
    # which operand did gs_chain get wrong at the first differing node?
    U0 = u0.reshape(n, n, n)
    F0 = f0.reshape(n, n, n)
    h2 = (2.0 / p.N) ** 2
    inv = 1.0 / 6.0
    for node in bad[:6]:
        P, R, K = node
        new = {"pb": a[P - 1, R, K], "ra": a[P, R - 1, K], "lf": a[P, R, K - 1]}
        old = {"pb": U0[P - 1, R, K], "ra": U0[P, R - 1, K], "lf": U0[P, R, K - 1]}
        pa, rb, rt = U0[P + 1, R, K], U0[P, R + 1, K], U0[P, R, K + 1]
        def val(pb, ra, lf):
            s = pb + pa
            s = s + ra
            s = s + rb
            s = s + lf
            s = s + rt
            return (h2 * F0[P, R, K] + 0.0 + s) * inv
        ref = val(new["pb"], new["ra"], new["lf"])
        out = [f"node {node.tolist()} rows {a[P, R, K]:.6f} (formula {ref:.6f}) chain {b[P, R, K]:.6f}:"]
        for m in range(1, 8):
            use = {k: (old[k] if (m >> i) & 1 else new[k]) for i, k in enumerate(("pb", "ra", "lf"))}
            if val(**use) == b[P, R, K]:
                out.append("chain used OLD " + "+".join(k for i, k in enumerate(("pb", "ra", "lf")) if (m >> i) & 1))
        cb_ = {k: b[P - (k == 'pb'), R - (k == 'ra'), K - (k == 'lf')] for k in ("pb", "ra", "lf")}
        out.append("chain's own neighbours equal rows': " + str({k: bool(cb_[k] == new[k]) for k in cb_}))
        print(" ".join(out))
    node = bad[0]
    P, R, K = node
    cand = {"pb": {"new": a[P - 1, R, K], "0": 0.0, "U[P-2]": U0[P - 2, R, K], "U[P]": U0[P, R, K]},
            "pa": {"old": U0[P + 1, R, K], "0": 0.0, "U[P]": U0[P, R, K], "U[P+2]": U0[P + 2, R, K]},
            "ra": {"new": a[P, R - 1, K], "old": U0[P, R - 1, K], "0": 0.0, "U[P-1,R-1]": U0[P - 1, R - 1, K], "U[P+1,R-1]": U0[P + 1, R - 1, K]},
            "rb": {"old": U0[P, R + 1, K], "0": 0.0, "U[P-1,R+1]": U0[P - 1, R + 1, K], "U[P+1,R+1]": U0[P + 1, R + 1, K]},
            "lf": {"new": a[P, R, K - 1], "old": U0[P, R, K - 1], "0": 0.0, "U[P-1,K-1]": U0[P - 1, R, K - 1], "U[P+1,K-1]": U0[P + 1, R, K - 1]},
            "rt": {"old": U0[P, R, K + 1], "0": 0.0, "U[P-1,K+1]": U0[P - 1, R, K + 1], "U[P+1,K+1]": U0[P + 1, R, K + 1]},
            "f": {"ok": F0[P, R, K], "0": 0.0, "F[P-1]": F0[P - 1, R, K], "F[P+1]": F0[P + 1, R, K]}}
    import itertools
    keys = list(cand)
    hits = []
    for combo in itertools.product(*[list(cand[k].items()) for k in keys]):
        v = {k: c[1] for k, c in zip(keys, combo)}
        s = v["pb"] + v["pa"]
        s = s + v["ra"]
        s = s + v["rb"]
        s = s + v["lf"]
        s = s + v["rt"]
        if (h2 * v["f"] + 0.0 + s) * inv == b[P, R, K]:
            hits.append({k: c[0] for k, c in zip(keys, combo)})
    print("operand combinations that reproduce gs_chain's value at", node.tolist(), ":", hits[:5])
    print("labels around:", lab[P - 1:P + 2, R, K].tolist(), "internal plane range of this column:",
          np.flatnonzero(lab[:, R, K] == 0)[[0, -1]].tolist())
