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
# every reference-golden case: stored plans, or rebuilt with the repo's setup
# (tests/test_setup_golden.py pins those to the reference's plan digests)
PLAN_CASES = GU.case_names()


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
        if p.d == 3:
            # fused residual + restriction (the cycle's 3-D path) must give the same coarse f
            out["restrict_int_fused"] = GU.digest(run(
                _lib.OP_RES_RESTRICT, {(L, _lib.U): inp["u"], (L, _lib.F): inp["f"],
                                       (L + 1, _lib.F): np.zeros(c.n_nodes)}, (L + 1, _lib.F, c.n_nodes)))
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
    plans, _ = GU.plans_or_rebuild(name)
    ctx = _lib.Context(plans[0].d, len(plans))
    for i, p in enumerate(plans):
        ctx.set_level(i, p)
    for key, want in rec["ops"].items():
        seed, level = map(int, key.split(":"))
        got = device_op_digests(ctx, plans, level, seed)
        bad = {k: (got[k], want[k]) for k in got if k in want and got[k] != want[k]}
        if "restrict_int_fused" in got and got["restrict_int_fused"] != want["restrict_int"]:
            bad["restrict_int_fused"] = (got["restrict_int_fused"], want["restrict_int"])
        assert not bad, (name, key, bad)
    ctx.close()


def device_solver(name):
    rec = GU.record(name)
    plans, extra = GU.plans_or_rebuild(name)
    cyc = CycleConfig(scheme=rec["scheme"], cycles=rec["cycles"], norm=rec["norm"],
                      coarse_solver=rec["coarse_solver"])
    return rec, MultigridSolver.from_plans(plans, extra["f_fine"], extra["g_fine"],
                                           extra["eliminated_values"], SmootherConfig(), cyc)


@pytest.mark.parametrize("name", PLAN_CASES)
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


def _pores64_solver(coarse_backend):
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200.cycle import CycleDriver
    from paper_2207_14208_b200.transfer import build_hierarchy

    setup = CF.config_pores(N=64, cycles=15)
    levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
    plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
    f = CF.pore_rhs(setup, plans[0].labels)
    return plans, MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle,
                                             coarse_backend=coarse_backend)


def test_pores64_setup_and_solve_match_reference(gpu_available):
    """Host setup rebuilt here must hash like the reference's plans, and the
    device solve (host SuperLU coarsest) must reproduce the reference."""
    rec = GU.record("pores64")
    plans, solver = _pores64_solver("superlu")
    for lvl, p in enumerate(plans):
        got = {k: GU.plan_digest(v) for k, v in p.to_arrays().items()}
        assert got == rec["plan_digests"][lvl]
    u, rep = solver.solve(u=np.zeros(plans[0].n_nodes), cycles=rec["cycles"])
    assert rep.residual_norms == GU.hexlist(rec["solve"]["residual_norms"])
    assert GU.digest(u) == rec["solve"]["u_digest"]
    assert measure_rho(solver, seed=42).rho_asymptotic == rec["rho"]["rho"]


def test_device_inverse_coarse_solve_within_tolerance(gpu_available):
    """coarse_backend='device-inverse' is not bitwise (a dense inverse is not
    SuperLU).  Its per-cycle round-off (~1e-15 of the correction) stays fixed
    in absolute size while the residual falls by rho per cycle, so the
    relative difference of the residual norms grows like 1e-15 / (r_m / r_0)
    (SURVEY.md finding 4).  Per-cycle norms are held to 1e-10 relative while
    r_m / r_0 > 1e-4; the final iterate to 1e-12 relative L-inf and rho to
    1e-3 (the north-star tolerances).  The default coarse backend (host
    SuperLU) is bitwise: see test_pores64_setup_and_solve_match_reference."""
    rec = GU.record("pores64")
    plans, solver = _pores64_solver("device-inverse")
    u, rep = solver.solve(u=np.zeros(plans[0].n_nodes), cycles=rec["cycles"])
    want = np.array(GU.hexlist(rec["solve"]["residual_norms"]))
    got = np.array(rep.residual_norms)
    early = want > 1e-4 * want[0]
    assert early.sum() >= 6
    assert np.max(np.abs(got - want)[early] / want[early]) < 1e-10
    _, ref = _pores64_solver("superlu")
    uref, _ = ref.solve(u=np.zeros(plans[0].n_nodes), cycles=rec["cycles"])
    assert np.max(np.abs(u - uref)) <= 1e-12 * np.max(np.abs(uref))
    assert abs(measure_rho(solver, seed=42).rho_asymptotic - rec["rho"]["rho"]) < 1e-3


def test_nested_dissection_coarse_solve_within_tolerance(gpu_available):
    """coarse_backend='device-inverse' on a coarsest level large enough for
    the nested-dissection form (pores 64^3 down to N=32: ~28k unknowns):
    same tolerances as the dense inverse against the bitwise SuperLU path."""
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200.cycle import CycleDriver
    from paper_2207_14208_b200.transfer import build_hierarchy

    setup = CF.config_pores(N=64, cycles=12, coarsest_min=32)
    levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
    plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
    f = CF.pore_rhs(setup, plans[0].labels)
    nd = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, coarse_backend="device-inverse")
    assert getattr(nd.device, "nd_sizes", None), "nested dissection not used"
    ref = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle, coarse_backend="superlu")
    u, rep = nd.solve(u=np.zeros(plans[0].n_nodes), cycles=12)
    uref, rref = ref.solve(u=np.zeros(plans[0].n_nodes), cycles=12)
    want = np.array(rref.residual_norms)
    got = np.array(rep.residual_norms)
    early = want > 1e-4 * want[0]
    assert early.sum() >= 6
    assert np.max(np.abs(got - want)[early] / want[early]) < 1e-10
    assert np.max(np.abs(u - uref)) <= 1e-12 * np.max(np.abs(uref))


def test_l2_norm_3d_matches_oracle(gpu_available):
    """norm='l2' (solver.py:137-138) on a 3-D hierarchy: the device sums of
    squares follow NumPy's pairwise tree, so the history is bitwise the
    oracle's (which is pinned to the reference on disk64_sweeps_l2)."""
    from oracle.solver import OracleSolver
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200.cycle import CycleDriver
    from paper_2207_14208_b200.transfer import build_hierarchy

    setup = CF.config_ball(32, cycles=4)
    levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
    plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
    cyc = CycleConfig(scheme="v", cycles=4, norm="l2")
    dev = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, cyc)
    ref = OracleSolver(plans, f, g, e, setup.smoother, cyc)
    u0 = np.zeros(plans[0].n_nodes)
    _, rd = dev.solve(u=u0.copy())
    _, ro = ref.solve(u=u0.copy())
    assert rd.residual_norms == ro.residual_norms


def test_batched_solves_match_individual(gpu_available):
    """solve_batched / measure_rho_batched (interleaved solvers on their own
    streams) give bitwise the results of one-at-a-time solves."""
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200.cycle import CycleDriver
    from paper_2207_14208_b200.solver import measure_rho_batched, solve_batched
    from paper_2207_14208_b200.transfer import build_hierarchy

    def make(setup):
        levels = build_hierarchy(setup.grid, setup.phi, setup.faces, coarsest_min=setup.coarsest_min)
        plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
        return plans, MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle,
                                                 coarse_backend="device-inverse")

    setups = [CF.config_disk(64, cycles=12), CF.config_ball(32, cycles=10), CF.config_disk(128, cycles=12)]
    solvers = [make(s)[1] for s in setups]
    want = [s.solve(u=np.zeros(s.plans[0].n_nodes))for s in solvers]
    got = solve_batched(solvers, us=[np.zeros(s.plans[0].n_nodes) for s in solvers])
    for (uw, rw), (ug, rg) in zip(want, got):
        assert rg.residual_norms == rw.residual_norms
        assert np.array_equal(ug.view(np.uint64), uw.view(np.uint64))
    rho_want = [measure_rho(s, seed=42).residual_norms for s in solvers]
    rho_got = [r.residual_norms for r in measure_rho_batched(solvers, seed=42)]
    assert rho_got == rho_want


@pytest.mark.parametrize("chain,grid", [("1", "0"), ("1", "1"), ("1", "3"), ("0", "0"), ("0", "3")])
def test_gs_variants_pores64_match_reference(chain, grid, gpu_available, monkeypatch):
    """Both 3-D GS kernels (gs_chain.cu, production; GMG_GS_CHAIN=0: the
    streaming kernel gs_stream.cu) give the reference's solve bit for
    bit (pores 64^3: empty tasks, trimmed plane ranges).  GMG_GS_GRID caps the
    GS grid so that every CTA loops over several task tickets
    (re-initialising its barriers and reusing its shared-memory ring with
    stale data from the previous task), as at 512^3 and 1024^3."""
    monkeypatch.setenv("GMG_GS_CHAIN", chain)
    monkeypatch.setenv("GMG_GS_GRID", grid)
    rec = GU.record("pores64")
    plans, solver = _pores64_solver("superlu")
    u, rep = solver.solve(u=np.zeros(plans[0].n_nodes), cycles=rec["cycles"])
    assert rep.residual_norms == GU.hexlist(rec["solve"]["residual_norms"])
    assert GU.digest(u) == rec["solve"]["u_digest"]
    # a second solve on the same context: the hand-off cells must be clean again
    u2, rep2 = solver.solve(u=np.zeros(plans[0].n_nodes), cycles=rec["cycles"])
    assert rep2.residual_norms == rep.residual_norms
    assert GU.digest(u2) == rec["solve"]["u_digest"]


def test_device_initial_field_matches_host_stream(gpu_available):
    """The seeded initial iterate drawn on the device (GF(2) jump-ahead
    per 64-value lane, gmg_initial_field) is the reference's sequential
    XorShift64Star stream bit for bit (solver.py:205-213, rng.py:14-56),
    with the prescribed values on eliminated nodes and 0 on inactive ones."""
    from paper_2207_14208_b200.geometry import ELIMINATED

    plans, s3 = _pores64_solver("superlu")
    rng = np.random.default_rng(5)
    elim = plans[0].labels == ELIMINATED
    assert elim.any()
    s3.eliminated_values = np.where(elim, rng.standard_normal(plans[0].n_nodes), 0.0)
    _, s2 = device_solver("disk64")
    for s, seed in ((s3, 42), (s3, 7), (s2, 42)):
        want = s.initial_field(seed)
        assert s._device_initial_field(seed)
        got = s._get_u()
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), seed


@pytest.mark.parametrize("case", ["pores64", "pores128", "ball64", "disk256"])
def test_device_classification_matches_host(case, gpu_available):
    """Labels computed on the GPU (gmg_setup_classify_balls) and the whole
    hierarchy built with the device label work are bit for bit the host's
    (reference classify, geometry.py:374-446; restriction checks,
    transfer.py:64-114)."""
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200.geometry import classify
    from paper_2207_14208_b200.transfer import build_hierarchy

    setup = {"pores64": lambda: CF.config_pores(N=64), "pores128": lambda: CF.config_pores(N=128),
             "ball64": lambda: CF.config_ball(64), "disk256": lambda: CF.config_disk(256)}[case]()
    host = classify(setup.grid, setup.phi, setup.faces)
    dev = classify(setup.grid, setup.phi, setup.faces, device=0)
    assert np.array_equal(host.labels, dev.labels)
    assert np.array_equal(host.ghost_idx, dev.ghost_idx)
    lv_h = build_hierarchy(setup.grid, setup.phi, setup.faces, max_levels=setup.cycle.max_levels,
                           coarsest_min=setup.coarsest_min)
    lv_d = build_hierarchy(setup.grid, setup.phi, setup.faces, max_levels=setup.cycle.max_levels,
                           coarsest_min=setup.coarsest_min, device=0)
    assert len(lv_h) == len(lv_d)
    for a, b in zip(lv_h, lv_d):
        assert np.array_equal(a.cls.labels, b.cls.labels)
        assert np.array_equal(a.cls.ghost_theta_raw, b.cls.ghost_theta_raw)
        assert np.array_equal(a.extrap.band_idx, b.extrap.band_idx)


def test_device_check_transfer_flags(gpu_available):
    """The device restriction checks raise what the host's do on broken label
    sets (a coarse internal node over a block without internal nodes, a
    coarse ghost over a block without ghost / inactive nodes)."""
    from paper_2207_14208_b200 import _lib as L
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200.geometry import GHOST, INACTIVE, INTERNAL, classify
    from paper_2207_14208_b200.geometry import UniformGrid

    setup = CF.config_ball(32)
    fine = classify(setup.grid, setup.phi, setup.faces)
    coarse = classify(UniformGrid(3, 16), setup.phi, setup.faces)
    assert L.setup_check_transfer(0, 3, 32, fine.labels, 16, coarse.labels) == 0
    bad = fine.labels.copy()
    bad[bad == INTERNAL] = INACTIVE
    assert L.setup_check_transfer(0, 3, 32, bad, 16, coarse.labels) & (2 | 8)
    bad = fine.labels.copy()
    bad[(bad == GHOST) | (bad == INACTIVE)] = INTERNAL
    assert L.setup_check_transfer(0, 3, 32, bad, 16, coarse.labels) & (4 | 16)


@pytest.mark.parametrize("case", ["pores128", "ball128"])
def test_gs_chain_matches_stream_kernel(case, gpu_available, monkeypatch):
    """The production 3-D GS kernel (gs_chain.cu) against the independent
    streaming kernel (GMG_GS_CHAIN=0) after several sweeps on random data:
    bitwise equal, also on the sparse ball whose tasks start at even planes
    (the ring slot of plane P0-1 must outlive the chains' warm-up) -- and
    equal to itself run to run."""
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200.cycle import CycleDriver
    from paper_2207_14208_b200.transfer import build_hierarchy

    setup = CF.config_pores(N=128) if case == "pores128" else CF.config_ball(128)
    levels = build_hierarchy(setup.grid, setup.phi, setup.faces, max_levels=2, coarsest_min=setup.coarsest_min, device=0)
    plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
    rng = np.random.default_rng(3)
    u0 = rng.standard_normal(plans[0].n_nodes)
    f0 = rng.standard_normal(plans[0].n_nodes)
    out = []
    for chain in ("1", "1", "0"):
        monkeypatch.setenv("GMG_GS_CHAIN", chain)
        ctx = _lib.Context(3, len(plans))
        for i, p in enumerate(plans):
            ctx.set_level(i, p)
        ctx.set_vector(0, _lib.U, u0)
        ctx.set_vector(0, _lib.F, f0)
        for _ in range(8):
            ctx.apply(0, _lib.OP_GS_SWEEP)
        out.append(ctx.get_vector(0, _lib.U, plans[0].n_nodes).copy())
        ctx.close()
    assert np.array_equal(out[0].view(np.uint64), out[1].view(np.uint64))
    assert np.array_equal(out[0].view(np.uint64), out[2].view(np.uint64))


@pytest.mark.parametrize("case", ["ball32", "pores64", "disk64"])
def test_norm_pass_peak_lower_bound(case, gpu_available):
    """gmg_residual_norm_peak: the same two maxima as gmg_residual_norm and max|u| over the internal nodes,
    and the solve loop's renormalisation guard (reference solver.py:239-243) still rescales a tiny iterate
    when that bound is below the threshold."""
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200.cycle import CycleDriver
    from paper_2207_14208_b200.transfer import build_hierarchy

    setup = {"ball32": lambda: CF.config_ball(32, cycles=3), "pores64": lambda: CF.config_pores(N=64, cycles=3),
             "disk64": lambda: CF.config_disk(64, cycles=3)}[case]()
    levels = build_hierarchy(setup.grid, setup.phi, setup.faces, max_levels=setup.cycle.max_levels,
                             coarsest_min=setup.coarsest_min)
    plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
    dev = MultigridSolver.from_plans(plans, f, g, e, setup.smoother, setup.cycle)
    p = plans[0]
    rng = np.random.default_rng(5)
    u = rng.standard_normal(p.n_nodes)
    dev._set_data(dev.f_fine, dev.g_fine)
    dev._put_u(u)
    a = dev.ctx.residual_parts(0)
    b = dev.ctx.residual_parts_peak(0)
    assert a == b[:2]
    assert b[2] == np.abs(u[p.labels == 0]).max()
    assert dev._residual_norm() == max(a) and dev._abs_max_scale() == (b[2], False)
    # tiny iterate: the bound is below the threshold, the exact pass runs and rescales
    dev._put_u(u * 1e-255)
    dev._residual_norm()
    peak, scaled = dev._abs_max_scale()
    assert scaled and peak == np.abs(u * 1e-255).max()
    got = dev._get_u()
    assert np.array_equal(got, (u * 1e-255) * 1e250)
