"""The CPU oracle against vectors produced by the reference itself.

tests/golden/*.json hold sha256 digests of every per-cycle operation of the
reference (ghostmg) on seeded inputs, per level, plus its full residual
histories; tests/golden/make_golden.py made them.  The oracle must match
bit for bit: this is what pins it before it is used to check the GPU.
"""

import numpy as np
import pytest

import goldutil as GU
from oracle import ops
from oracle.solver import OracleSolver
from paper_2207_14208_b200.cycle import CycleConfig, measure_rho
from paper_2207_14208_b200.smoothing import SmootherConfig

LARGE = {"ball256", "flowerD2048", "flowerM2048", "pores128"}
CASES = [pytest.param(n, marks=pytest.mark.slow) if n in LARGE else n for n in GU.case_names()]


def oracle_op_digests(plans, level, seed):
    p = plans[level]
    c = plans[level + 1] if level + 1 < len(plans) else None
    inp = GU.golden_inputs(p, c.n_nodes if c else 0, seed)
    st = np.ascontiguousarray(p.stencil)
    out = {}
    u = inp["u"].copy(); ops.gs_sweep(p, u, inp["f"]); out["gs"] = GU.digest(u)
    u = inp["u"].copy(); ops.ghost_sweep(p, u, inp["g"], st); out["ghost"] = GU.digest(u)
    u = inp["u"].copy(); ops.smooth(p, u, inp["f"], inp["g"], 3, st); out["smooth3"] = GU.digest(u)
    r, _ = ops.residual_internal_full(p, inp["u"], inp["f"])
    out["res_int"] = GU.digest(r[p.labels == 0])
    rg, _ = ops.residual_ghost(p, inp["u"], inp["g"], st)
    out["res_ghost"] = GU.digest(rg)
    out["extrap_ghost"] = GU.digest(ops.extrapolate(p, inp["r_ghost"].copy()))
    out["extrap_full"] = GU.digest(ops.extrapolate(p, inp["v_full"].copy()))
    if c is not None:
        out["restrict_int"] = GU.digest(ops.restrict_interior(p, c, r))
        gc = ops.restrict_ghost(p, c, ops.extrapolate(p, inp["r_ghost"].copy()))
        out["restrict_ghost"] = GU.digest(gc)
        gc[c.ghost_promoted] = 0.0
        out["restrict_ghost_cycle"] = GU.digest(gc)
        u = inp["u"].copy(); ops.interpolate_add(p, u, inp["e_coarse"]); out["interp_add"] = GU.digest(u)
    return out


@pytest.mark.parametrize("name", CASES)
def test_oracle_ops_match_reference(name):
    rec = GU.record(name)
    plans, _ = GU.plans_or_rebuild(name)
    for key, want in rec["ops"].items():
        seed, level = map(int, key.split(":"))
        got = oracle_op_digests(plans, level, seed)
        assert got == want, (name, key, {k: (got[k], want[k]) for k in want if got.get(k) != want[k]})


def oracle_from_golden(name):
    rec = GU.record(name)
    plans, extra = GU.plans_or_rebuild(name)
    cyc = CycleConfig(scheme=rec["scheme"], cycles=rec["cycles"], norm=rec["norm"],
                      coarse_solver=rec["coarse_solver"])
    return rec, OracleSolver(plans, extra["f_fine"], extra["g_fine"], extra["eliminated_values"],
                             SmootherConfig(), cyc)


@pytest.mark.parametrize("name", CASES)
def test_oracle_solve_matches_reference(name):
    rec, solver = oracle_from_golden(name)
    u0 = None if rec["solve"].get("from_initial_field") else np.zeros(solver.plans[0].n_nodes)
    u, rep = solver.solve(u=u0, cycles=rec["cycles"], seed=42)
    assert rep.residual_norms == GU.hexlist(rec["solve"]["residual_norms"])
    assert GU.digest(u) == rec["solve"]["u_digest"]
    if "rho" in rec:
        r = measure_rho(solver, seed=42)
        assert r.residual_norms == GU.hexlist(rec["rho"]["residual_norms"])
        assert r.rho_asymptotic == rec["rho"]["rho"]


def test_frozen_reference_anchors():
    """The reference's own frozen rho values (pkg/tests/test_solver.py:45-61)."""
    assert GU.record("vline64TG")["rho"]["rho"] == pytest.approx(0.1098159571428157, rel=1e-12)
    assert GU.record("circle32W")["rho"]["rho"] == pytest.approx(0.19126214971430816, rel=1e-12)
    _, solver = oracle_from_golden("circle32W")
    assert measure_rho(solver).rho_asymptotic == pytest.approx(0.19126214971430816, rel=1e-12)


def test_numpy_summation_models():
    rng = np.random.default_rng(3)
    for n in (2, 3, 4, 6, 8, 9, 27):
        for _ in range(200):
            a = rng.standard_normal(n) * np.exp(rng.uniform(-6, 6, n))
            assert ops.np_sum(a) == a[None, :].sum(axis=1)[0]
    for n in (1, 7, 128, 129, 1000, 70001):
        a = rng.standard_normal(n)
        assert ops.sumsq(a) == (a ** 2).sum()


def test_ddot_model_matches_this_hosts_blas():
    """The oracle's ddot tree is the one numpy's OpenBLAS uses here."""
    rng = np.random.default_rng(4)
    for n in (3, 9, 27):
        for _ in range(500):
            x = rng.standard_normal(n) * np.exp(rng.uniform(-5, 5, n))
            y = rng.standard_normal(n)
            assert ops.ddot(x, y) == x @ y


@pytest.mark.gpu
def test_ddot_model_matches_gpu_box_blas():
    """re-probe the OpenBLAS ddot tree on the GPU box's host
    CPU (OpenBLAS picks its kernel by core, DYNAMIC_ARCH).  The kernels and
    fixtures follow the build container's SkylakeX tree; a different tree
    on the GPU host would make a reference run THERE round differently
    (fixtures made here stay valid)."""
    test_ddot_model_matches_this_hosts_blas()
