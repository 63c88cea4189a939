"""Generate the golden parity fixtures by running the REFERENCE package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

For every case it builds the reference's own solver (ghostmg.build_solver),
converts the reference's per-level data (classification, SweepPlan,
ExtrapolationPlan) into this repo's ``LevelPlan`` layout, and records

* ``<case>.npz``   the level plans + problem data (f_fine, g_fine, ...),
* ``<case>.json``  sha256 digests of every per-cycle operation's output on
                   seeded inputs (``golden_inputs`` below), per level, and the
                   reference's full residual histories / rho values.

The reference is never needed at test time: tests compare the oracle and
the CUDA path against these files.
"""

import hashlib
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, REPO)

from paper_2207_14208_b200 import configs as CF  # noqa: E402
from paper_2207_14208_b200 import levelsets as LS  # noqa: E402
from paper_2207_14208_b200.plan import LevelPlan, save_plans  # noqa: E402
from paper_2207_14208_b200.rng import uniform_symmetric  # noqa: E402
from paper_2207_14208_b200.transfer import ghost_dag_levels  # noqa: E402
sys.path.insert(0, os.path.join(REPO, "tests"))
from goldutil import digest, golden_inputs  # noqa: E402


def reference_level_plan(ref_level, ref_plan, d, reaction):
    """LevelPlan arrays from the reference's objects."""
    cls = ref_level.cls
    ex = ref_level.extrap
    groups = ex.bfs_groups
    masks = []
    for _, _, m in groups:
        bits = np.zeros(m.shape[0], dtype=np.uint8)
        for c in range(m.shape[1]):
            bits |= m[:, c].astype(np.uint8) << np.uint8(c)
        masks.append(bits)
    strides = cls.grid.strides
    nb = len(ex.band_idx)
    step = np.zeros((nb, d), dtype=np.int8)
    for k in range(d):
        step[:, k] = ((ex.band_idx - ex.trans_nbrs[:, k]) // strides[k]).astype(np.int8)
    return LevelPlan(
        d=d, N=cls.grid.N, reaction=float(reaction),
        labels=np.ascontiguousarray(cls.labels, dtype=np.uint8),
        ghost_idx=np.asarray(cls.ghost_idx, dtype=np.int64),
        ghost_low=np.asarray(cls.ghost_block_low, dtype=np.int64).reshape(-1, d),
        ghost_w=np.asarray(ref_plan.ghost_coeffs, dtype=np.float64).reshape(-1, 3 ** d),
        ghost_dtau=np.asarray(ref_plan.ghost_dtau, dtype=np.float64),
        ghost_promoted=np.asarray(cls.ghost_promoted, dtype=bool),
        ghost_batch=ghost_dag_levels(cls, ref_plan.ghost_coeffs),
        bfs_len=np.array([len(g[0]) for g in groups], dtype=np.int64),
        band_idx=np.asarray(ex.band_idx, dtype=np.int64),
        bfs_mask=np.concatenate(masks) if masks else np.zeros(0, np.uint8),
        trans_step=step,
        trans_absn=np.asarray(ex.trans_absn, dtype=np.float64).reshape(-1, d),
    )


def per_op_digests(ref, S, level, plan, coarse_plan, seed):
    """Run every reference per-cycle op on seeded inputs; digest outputs."""
    sp = ref.plans[level]
    lv = ref.levels[level]
    inp = golden_inputs(plan, coarse_plan.n_nodes if coarse_plan else 0, seed)
    out = {}
    u = inp["u"].copy(); S.gs_lex_sweep(u, inp["f"], sp); out["gs"] = digest(u)
    u = inp["u"].copy(); S.ghost_relax_sweep(u, inp["g"], sp); out["ghost"] = digest(u)
    u = inp["u"].copy(); S.smooth(u, inp["f"], inp["g"], sp, 3); out["smooth3"] = digest(u)
    r_int = sp.residual_internal(inp["u"], inp["f"])
    out["res_int"] = digest(r_int)
    out["res_ghost"] = digest(sp.residual_ghost(inp["u"], inp["g"]))
    out["extrap_ghost"] = digest(lv.extrap.apply(inp["r_ghost"]))
    out["extrap_full"] = digest(lv.extrap.apply(inp["v_full"]))
    if coarse_plan is not None:
        r_full = np.zeros(plan.n_nodes)
        r_full[lv.cls.internal_idx] = r_int
        out["restrict_int"] = digest(lv.down_interior.apply(r_full))
        gc = lv.down_ghost.apply(lv.extrap.apply(inp["r_ghost"]))
        out["restrict_ghost"] = digest(gc)
        gc[ref.levels[level + 1].cls.ghost_promoted] = 0.0
        out["restrict_ghost_cycle"] = digest(gc)
        u = inp["u"].copy()
        u[lv.up_interp.targets] += lv.up_interp.apply(inp["e_coarse"])
        out["interp_add"] = digest(u)
    return out


class MixedBCShim:
    """SURVEY.md Appendix B mixed-BC shim over the REFERENCE's own functions:
    the reference supports one BC kind per problem (operators.py:73-96,
    smoothing.py:50-77), so per ghost the Dirichlet or Neumann row and dtau
    are selected by ``selector(Q)`` from the reference's two single-kind
    results.  Patched where the reference looks them up: SweepPlan
    (smoothing.py:104), assemble_system for the coarsest matrix
    (operators.py:208) and MultigridSolver.__init__ (solver.py:110)."""

    def __init__(self, selector):
        import ghostmg.operators as O
        import ghostmg.smoothing as S
        import ghostmg.solver as V
        self.mods = (O, S, V)
        self.orig_rows = O.ghost_row_weights
        self.orig_dtau = S.assign_dtau
        rows0, dtau0 = self.orig_rows, self.orig_dtau

        def rows(cls, bc):
            dm = np.asarray(selector(cls.ghost_Q), dtype=bool)
            return np.where(dm[:, None], rows0(cls, "dirichlet"), rows0(cls, "neumann"))

        def dtau(cls, bc, config, default_variant="poly"):
            dm = np.asarray(selector(cls.ghost_Q), dtype=bool)
            return np.where(dm, dtau0(cls, "dirichlet", config, default_variant),
                            dtau0(cls, "neumann", config, default_variant))

        self.rows, self.dtau = rows, dtau

    def __enter__(self):
        O, S, V = self.mods
        O.ghost_row_weights = S.ghost_row_weights = self.rows
        S.assign_dtau = V.assign_dtau = self.dtau
        return self

    def __exit__(self, *exc):
        O, S, V = self.mods
        O.ghost_row_weights = S.ghost_row_weights = self.orig_rows
        S.assign_dtau = V.assign_dtau = self.orig_dtau


def make_case(name, setup, cycles, seeds=(7,), rho=True, store_plan=True, coarse_solver="direct", norm="inf",
              op_levels=None):
    sys.path.insert(0, "/root/reference/pkg/src")
    import contextlib

    import ghostmg
    from ghostmg import smoothing as S
    from ghostmg.geometry import compute_normal
    from ghostmg.smoothing import SmootherConfig as RSC
    from ghostmg.solver import CycleConfig as RCC
    from ghostmg.solver import build_solver, measure_rho
    from ghostmg.operators import ProblemSpec as RPS

    sp = setup.spec
    mixed = sp.bc == "mixed"
    # mixed BC: the reference is built as a Dirichlet problem with the
    # per-ghost rows / dtau / coarsest matrix patched in, and g set directly
    # (as tests/test_solver.py:95-97 of the reference does)
    rspec = RPS(sp.pde, "dirichlet" if mixed else sp.bc, sp.f, sp.g_box, None if mixed else sp.g_gamma)
    cyc = RCC(scheme=setup.cycle.scheme, cycles=cycles, norm=norm, coarse_solver=coarse_solver)
    shim = MixedBCShim(sp.bc_selector) if mixed else contextlib.nullcontext()
    with shim:
        ref = build_solver(ghostmg.UniformGrid(setup.grid.d, setup.grid.N), setup.phi, rspec,
                           setup.faces, RSC(), cyc, setup.default_variant, setup.coarsest_min)
        if mixed:
            ref._coarsest_matrix()  # factor the coarsest matrix with the mixed rows
    if mixed:
        cls = ref.levels[0].cls
        dm = np.asarray(sp.bc_selector(cls.ghost_Q), dtype=bool)
        normals = compute_normal(cls.phi, cls.ghost_Q, cls.grid.h)
        g = np.asarray(sp.g_gamma(cls.ghost_Q, dm, normals), dtype=float).copy()
        g[cls.ghost_promoted] = 0.0
        ref.g_fine = g
    d = setup.grid.d
    if setup.f_seed is not None:
        f = uniform_symmetric(setup.f_seed, setup.grid.n_nodes) * setup.f_scale
        f[ref.levels[0].cls.labels != 0] = 0.0
        ref.f_fine = f
    plans = [reference_level_plan(lv, p, d, sp.reaction) for lv, p in zip(ref.levels, ref.plans)]
    record = {"name": name, "setup": setup.name, "cycles": cycles, "scheme": setup.cycle.scheme,
              "coarse_solver": coarse_solver, "norm": norm, "n_levels": len(plans),
              "plan_digests": [], "ops": {}}
    for lvl, p in enumerate(plans):
        record["plan_digests"].append({k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()[:32]
                                       for k, v in p.to_arrays().items()})
    for seed in seeds:
        for lvl, p in enumerate(plans):
            if op_levels is not None and lvl not in op_levels:
                continue
            coarse = plans[lvl + 1] if lvl + 1 < len(plans) else None
            record["ops"][f"{seed}:{lvl}"] = per_op_digests(ref, S, lvl, p, coarse, seed)
    homogeneous = sp.f is None and setup.f_seed is None
    u0 = None if homogeneous else np.zeros(setup.grid.n_nodes)
    u, rep = ref.solve(u=u0, cycles=cycles, seed=42)
    record["solve"] = {"from_initial_field": homogeneous, "residual_norms": [float(x).hex() for x in rep.residual_norms],
                       "u_digest": digest(u), "diverged": rep.diverged,
                       "u_sample": [float(x).hex() for x in u[:: max(1, len(u) // 50)]]}
    if rho:
        r = measure_rho(ref, seed=42)
        record["rho"] = {"rho": r.rho_asymptotic, "residual_norms": [float(x).hex() for x in r.residual_norms]}
    extra = {"f_fine": ref.f_fine, "g_fine": ref.g_fine, "eliminated_values": ref.eliminated_values}
    if store_plan:
        save_plans(os.path.join(HERE, f"{name}.npz"), plans, **extra)
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(record, fh, indent=1)
    print(name, "levels", len(plans), "ghosts", [p.n_ghosts for p in plans],
          "final res", rep.residual_norms[-1], "rho", record.get("rho", {}).get("rho"))


def main(only=None):
    from goldutil import CASES
    for name, c in CASES.items():
        if only and name not in only:
            continue
        opts = {k: v for k, v in c.items() if k not in ("setup", "cycles")}
        make_case(name, c["setup"](), c["cycles"], **opts)


if __name__ == "__main__":
    main(sys.argv[1:] or None)
