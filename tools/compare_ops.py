"""Per-operation GPU vs oracle comparison on one configuration (bitwise),
levels given on the command line:  python tools/compare_ops.py c4:512 0 1
Prints, per op, whether the outputs are bit-identical and the max relative
difference otherwise (diagnoses size-dependent mismatches)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import goldutil as GU
from oracle import ops
from paper_2207_14208_b200 import _lib
from paper_2207_14208_b200 import configs as CF
from paper_2207_14208_b200.cycle import CycleDriver
from paper_2207_14208_b200.transfer import build_hierarchy

name, N = sys.argv[1].split(":")
levels_to_check = [int(x) for x in sys.argv[2:]] or [0]
setup = CF.config_pores(N=int(N)) if name == "c4" else CF.CONFIGS[name](int(N))
levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
del levels
ctx = _lib.Context(plans[0].d, len(plans))
for i, p in enumerate(plans):
    ctx.set_level(i, p)


CUR_N = 0


def cmp(tag, a, b):
    a = np.asarray(a); b = np.asarray(b)
    same = np.array_equal(a.view(np.uint64), b.view(np.uint64))
    if same:
        print(f"  {tag:16s} bitwise equal", flush=True)
    else:
        d = np.abs(a - b)
        k = int(np.argmax(d))
        nbad = int(np.count_nonzero(a.view(np.uint64) != b.view(np.uint64)))
        print(f"  {tag:16s} DIFFER: {nbad} entries, max |d| {d[k]:.3e} at {k} ({a[k]!r} vs {b[k]!r})", flush=True)
        if a.size == CUR_N ** 3 or tag == "gs":
            nn = CUR_N
            bad = np.flatnonzero(a.view(np.uint64) != b.view(np.uint64))
            pl, rem = np.divmod(bad, nn * nn)
            row, col = np.divmod(rem, nn)
            print("     planes", np.bincount(pl).nonzero()[0][:10], "... rows mod 14:", np.bincount((row - 1) % 14, minlength=14),
                  "cols mod 32:", np.bincount((col - 1) % 32, minlength=32), "first bad (p,r,c):",
                  list(zip(pl[:5], row[:5], col[:5])), "row blocks", np.unique((row - 1) // 14)[:12], flush=True)


for L in levels_to_check:
    p = plans[L]
    c = plans[L + 1] if L + 1 < len(plans) else None
    inp = GU.golden_inputs(p, c.n_nodes if c else 0, 7)
    st = np.ascontiguousarray(p.stencil)
    n = p.n_nodes
    print(f"level {L} N={p.N}", flush=True)
    CUR_N = p.N + 1
    # GS sweep
    ctx.set_vector(L, _lib.U, inp["u"]); ctx.set_vector(L, _lib.F, inp["f"])
    ctx.apply(L, _lib.OP_GS_SWEEP)
    ug = ctx.get_vector(L, _lib.U, n)
    uo = inp["u"].copy(); ops.gs_sweep(p, uo, inp["f"])
    cmp("gs", ug, uo)
    if p.n_ghosts:
        ctx.set_vector(L, _lib.U, inp["u"]); ctx.set_vector(L, _lib.G, inp["g"])
        ctx.apply(L, _lib.OP_GHOST_SWEEP)
        ug = ctx.get_vector(L, _lib.U, n)
        uo = inp["u"].copy(); ops.ghost_sweep(p, uo, inp["g"], st)
        cmp("ghost", ug, uo)
    ctx.set_vector(L, _lib.U, inp["u"]); ctx.set_vector(L, _lib.F, inp["f"]); ctx.set_vector(L, _lib.R_INT, np.zeros(n))
    ctx.apply(L, _lib.OP_RES_INT)
    rg = ctx.get_vector(L, _lib.R_INT, n)
    ro, _ = ops.residual_internal_full(p, inp["u"], inp["f"])
    cmp("res_int", rg[p.labels == 0], ro[p.labels == 0])
    ctx.set_vector(L, _lib.R_EXT, np.zeros(n))
    ctx.apply(L, _lib.OP_RES_GHOST)
    reg = ctx.get_vector(L, _lib.R_EXT, n)
    rgo, _ = ops.residual_ghost(p, inp["u"], inp["g"] if p.n_ghosts else np.zeros(0), st)
    cmp("res_ghost", reg[p.ghost_idx], rgo)
    ctx.set_vector(L, _lib.R_EXT, inp["r_ghost"]); ctx.apply(L, _lib.OP_EXTEND_REXT)
    cmp("extrap_ghost", ctx.get_vector(L, _lib.R_EXT, n), ops.extrapolate(p, inp["r_ghost"].copy()))
    ctx.set_vector(L, _lib.U, inp["v_full"]); ctx.apply(L, _lib.OP_EXTEND_U)
    cmp("extrap_full", ctx.get_vector(L, _lib.U, n), ops.extrapolate(p, inp["v_full"].copy()))
    if c is not None:
        ctx.set_vector(L + 1, _lib.F, np.zeros(c.n_nodes)); ctx.set_vector(L, _lib.R_INT, ro)
        ctx.apply(L, _lib.OP_RESTRICT_INT)
        cmp("restrict_int", ctx.get_vector(L + 1, _lib.F, c.n_nodes), ops.restrict_interior(p, c, ro))
        ctx.set_vector(L, _lib.R_EXT, inp["r_ghost"]); ctx.apply(L, _lib.OP_EXTEND_REXT)
        if c.n_ghosts:
            ctx.apply(L, _lib.OP_RESTRICT_GHOST)
            gc = ops.restrict_ghost(p, c, ops.extrapolate(p, inp["r_ghost"].copy()))
            gc[c.ghost_promoted] = 0.0
            cmp("restrict_ghost", ctx.get_vector(L + 1, _lib.G, c.n_ghosts), gc)
        ctx.set_vector(L, _lib.U, inp["u"]); ctx.set_vector(L + 1, _lib.U, inp["e_coarse"])
        ctx.apply(L, _lib.OP_INTERP_ADD)
        uo = inp["u"].copy(); ops.interpolate_add(p, uo, inp["e_coarse"])
        cmp("interp_add", ctx.get_vector(L, _lib.U, n), uo)
