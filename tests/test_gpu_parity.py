"""CUDA path against the reference's golden vectors and the pinned oracle.

Every check is bitwise: per-operation outputs on seeded inputs, per level
(tests/golden/*.json digests produced by the reference itself), and whole
solves (residual history, final iterate, rho).  All calls go through the
C ABI (paper_2207_14208_b200/_lib.py -> libghostmg_b200.so).
"""

import numpy as np
import pytest

import goldutil as GU
from paper_2207_14208_b200 import _lib
from paper_2207_14208_b200.cycle import CycleConfig, measure_rho
from paper_2207_14208_b200.smoothing import SmootherConfig
from paper_2207_14208_b200.solver import MultigridSolver

pytestmark = pytest.mark.gpu
PLAN_CASES = GU.case_names(with_plans=True)


def device_op_digests(ctx, plans, level, seed):
    p = plans[level]
    c = plans[level + 1] if level + 1 < len(plans) else None
    inp = GU.golden_inputs(p, c.n_nodes if c else 0, seed)
    n = p.n_nodes
    out = {}

    def run(op, vecs, get, lvl=level):
        for (lv, which), v in vecs.items():
            ctx.set_vector(lv, which, v)
        ctx.apply(lvl, op)
        lv, which, size = get
        return ctx.get_vector(lv, which, size)

    L = level
    zeros = np.zeros(n)
    out["gs"] = GU.digest(run(_lib.OP_GS_SWEEP, {(L, _lib.U): inp["u"], (L, _lib.F): inp["f"]}, (L, _lib.U, n)))
    if p.n_ghosts:
        out["ghost"] = GU.digest(run(_lib.OP_GHOST_SWEEP, {(L, _lib.U): inp["u"], (L, _lib.G): inp["g"]},
                                     (L, _lib.U, n)))
    else:
        out["ghost"] = GU.digest(inp["u"])
    ctx.set_vector(L, _lib.U, inp["u"])
    ctx.set_vector(L, _lib.F, inp["f"])
    if p.n_ghosts:
        ctx.set_vector(L, _lib.G, inp["g"])
    ctx.apply(L, _lib.OP_SMOOTH, 3)
    out["smooth3"] = GU.digest(ctx.get_vector(L, _lib.U, n))
    r = run(_lib.OP_RES_INT, {(L, _lib.U): inp["u"], (L, _lib.F): inp["f"], (L, _lib.R_INT): zeros},
            (L, _lib.R_INT, n))
    out["res_int"] = GU.digest(r[p.labels == 0])
    ctx.set_vector(L, _lib.R_EXT, zeros)
    re = run(_lib.OP_RES_GHOST, {(L, _lib.U): inp["u"]}, (L, _lib.R_EXT, n))
    out["res_ghost"] = GU.digest(re[p.ghost_idx])
    out["extrap_ghost"] = GU.digest(run(_lib.OP_EXTEND_REXT, {(L, _lib.R_EXT): inp["r_ghost"]}, (L, _lib.R_EXT, n)))
    out["extrap_full"] = GU.digest(run(_lib.OP_EXTEND_U, {(L, _lib.U): inp["v_full"]}, (L, _lib.U, n)))
    if c is not None:
        ctx.set_vector(L + 1, _lib.F, np.zeros(c.n_nodes))
        ctx.set_vector(L, _lib.R_INT, r)
        out["restrict_int"] = GU.digest(run(_lib.OP_RESTRICT_INT, {}, (L + 1, _lib.F, c.n_nodes)))
        ctx.set_vector(L, _lib.R_EXT, inp["r_ghost"])
        ctx.apply(L, _lib.OP_EXTEND_REXT)
        if c.n_ghosts:
            out["restrict_ghost_cycle"] = GU.digest(run(_lib.OP_RESTRICT_GHOST, {}, (L + 1, _lib.G, c.n_ghosts)))
        else:
            out["restrict_ghost_cycle"] = GU.digest(np.zeros(0))
        out["interp_add"] = GU.digest(run(_lib.OP_INTERP_ADD, {(L, _lib.U): inp["u"],
                                                              (L + 1, _lib.U): inp["e_coarse"]}, (L, _lib.U, n)))
    return out


@pytest.mark.parametrize("name", PLAN_CASES)
def test_device_ops_match_reference(name, gpu_available):
    rec = GU.record(name)
    plans, _ = GU.plans(name)
    ctx = _lib.Context(plans[0].d, len(plans))
    for i, p in enumerate(plans):
        ctx.set_level(i, p)
    for key, want in rec["ops"].items():
        seed, level = map(int, key.split(":"))
        got = device_op_digests(ctx, plans, level, seed)
        bad = {k: (got[k], want[k]) for k in got if k in want and got[k] != want[k]}
        assert not bad, (name, key, bad)
    ctx.close()


def device_solver(name):
    rec = GU.record(name)
    plans, extra = GU.plans(name)
    cyc = CycleConfig(scheme=rec["scheme"], cycles=rec["cycles"], norm=rec["norm"],
                      coarse_solver=rec["coarse_solver"])
    return rec, MultigridSolver.from_plans(plans, extra["f_fine"], extra["g_fine"],
                                           extra["eliminated_values"], SmootherConfig(), cyc)


@pytest.mark.parametrize("name", [n for n in PLAN_CASES if GU.record(n)["norm"] == "inf"])
def test_device_solve_matches_reference(name, gpu_available):
    rec, solver = device_solver(name)
    u0 = None if rec["solve"].get("from_initial_field") else np.zeros(solver.plans[0].n_nodes)
    u, rep = solver.solve(u=u0, cycles=rec["cycles"], seed=42)
    want = GU.hexlist(rec["solve"]["residual_norms"])
    assert rep.residual_norms == want, np.max(np.abs(np.array(rep.residual_norms) - want) / np.abs(want))
    assert GU.digest(u) == rec["solve"]["u_digest"]
    if "rho" in rec:
        r = measure_rho(solver, seed=42)
        assert r.residual_norms == GU.hexlist(rec["rho"]["residual_norms"])
        assert r.rho_asymptotic == rec["rho"]["rho"]
