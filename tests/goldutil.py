"""Shared helpers for the golden-vector parity tests."""

import glob
import hashlib
import json
import os

import numpy as np

from paper_2207_14208_b200.plan import load_plans
from paper_2207_14208_b200.rng import uniform_symmetric

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return hashlib.sha256(a.tobytes()).hexdigest()[:32]


def plan_digest(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()[:32]


def golden_inputs(plan, coarse_nodes, seed):
    """Seeded per-op inputs for one level (same as make_golden.py)."""
    n = plan.n_nodes
    lab = plan.labels
    u = uniform_symmetric(seed, n)
    u[lab == 2] = 0.0
    f = uniform_symmetric(seed + 1, n) * 50.0
    f[lab != 0] = 0.0
    g = uniform_symmetric(seed + 2, plan.n_ghosts)
    r_ghost = np.zeros(n)
    r_ghost[plan.ghost_idx] = uniform_symmetric(seed + 3, plan.n_ghosts)
    v_full = uniform_symmetric(seed + 4, n)
    v_full[plan.band_idx] = 0.0
    e_coarse = uniform_symmetric(seed + 5, coarse_nodes) if coarse_nodes else None
    return dict(u=u, f=f, g=g, r_ghost=r_ghost, v_full=v_full, e_coarse=e_coarse)


def record(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        return json.load(fh)


def has_plans(name):
    return os.path.exists(os.path.join(GOLDEN, f"{name}.npz"))


def plans(name):
    return load_plans(os.path.join(GOLDEN, f"{name}.npz"))


def rebuild(name):
    """(plans, extra) of a golden case rebuilt with the REPO's own host setup
    (build_hierarchy + build_level_plan), for the cases too large to store
    plans; test_setup_golden.py checks them against the reference's
    plan_digests.  extra holds f_fine / g_fine / eliminated_values as the
    reference's MultigridSolver would (pore space: the seeded f)."""
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200.cycle import CycleConfig, CycleDriver
    from paper_2207_14208_b200.transfer import build_hierarchy

    rec = record(name)
    setup = CASES[name]["setup"]()
    cyc = CycleConfig(scheme=rec["scheme"], cycles=rec["cycles"], norm=rec["norm"],
                      coarse_solver=rec["coarse_solver"])
    levels = build_hierarchy(setup.grid, setup.phi, setup.faces, max_levels=cyc.max_levels,
                             coarsest_min=setup.coarsest_min)
    plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
    if setup.f_seed is not None:
        f = CF.pore_rhs(setup, plans[0].labels)
    return plans, {"f_fine": f, "g_fine": g, "eliminated_values": e}


def plans_or_rebuild(name):
    return plans(name) if has_plans(name) else rebuild(name)


def case_names(with_plans=None):
    names = sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(GOLDEN, "*.json"))
                   if not os.path.basename(p).startswith("_"))
    if with_plans is None:
        return names
    return [n for n in names if has_plans(n) == with_plans]


def hexlist(values):
    return [float.fromhex(v) for v in values]


# ---- case registry (shared by make_golden.py and the tests) ----------------

def _cases():
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200 import levelsets as LS
    from paper_2207_14208_b200.cycle import CycleConfig
    from paper_2207_14208_b200.geometry import FACE_HIGH, FACE_LOW, UniformGrid
    from paper_2207_14208_b200.operators import ProblemSpec

    def circle(N):
        import math
        return LS.Sphere((math.sqrt(3.0) / 40.0, -0.05), math.sqrt(2.0) / 2.0)

    def vline_phi(N, theta=0.5):
        return LS.axis_halfspace(2, 1.0 - theta * (2.0 / N))

    def line30_phi(N):
        import math
        return LS.HalfSpace((0.5, math.sqrt(3.0) / 2.0), (-1.0 + 0.7 * (2.0 / N)) / 2.0)

    def plane_phi(N, theta=0.3):
        return LS.axis_halfspace(3, 1.0 - theta * (2.0 / N))

    def ellipsoid(N):
        import math
        c = (math.sqrt(2.0) / 20.0, math.sqrt(3.0) / 40.0, -math.sqrt(2.0) / 50.0)
        return LS.Ellipsoid(c, (0.686, 0.386, 0.586))

    def setup(name, d, N, phi, spec, scheme, faces=(), variant="exp", cmin=4, cycles=16):
        return CF.ProblemSetup(name=name, grid=UniformGrid(d, N), phi=phi, spec=spec, faces=faces,
                               cycle=CycleConfig(scheme=scheme, cycles=cycles), default_variant=variant,
                               coarsest_min=cmin)

    fl = CF.config_flower_dirichlet(128)
    cases = {
        "disk64": dict(setup=lambda: CF.config_disk(64), cycles=20),
        "disk64_sweeps_l2": dict(setup=lambda: CF.config_disk(64), cycles=8, rho=False,
                                 coarse_solver="sweeps", norm="l2"),
        "disk256": dict(setup=lambda: CF.config_disk(256), cycles=20),
        "ball32": dict(setup=lambda: CF.config_ball(32), cycles=15),
        "ball64": dict(setup=lambda: CF.config_ball(64), cycles=15, seeds=(11,)),
        "flowerD128": dict(setup=lambda: fl, cycles=20),
        "flowerN128": dict(setup=lambda: setup("flowerN128", 2, 128, LS.Flower(0.5, 0.15),
                                               ProblemSpec("poisson", "neumann"), "v", cmin=32), cycles=16),
        "circle32W": dict(setup=lambda: setup("circle32W", 2, 32, circle(32),
                                              ProblemSpec("poisson", "dirichlet"), "w"), cycles=16),
        "vline64TG": dict(setup=lambda: setup("vline64TG", 2, 64, vline_phi(64), ProblemSpec("poisson", "dirichlet"),
                                              "two-grid", faces=((0, FACE_LOW), (1, FACE_LOW), (1, FACE_HIGH)),
                                              variant="poly"), cycles=16),
        "line30R": dict(setup=lambda: setup("line30R", 2, 32, line30_phi(32), ProblemSpec("reaction", "neumann"),
                                            "two-grid"), cycles=16),
        "plane3d16": dict(setup=lambda: setup("plane3d16", 3, 16, plane_phi(16), ProblemSpec("poisson", "dirichlet"),
                                              "v", faces=((0, FACE_LOW), (1, FACE_LOW), (1, FACE_HIGH),
                                                          (2, FACE_LOW), (2, FACE_HIGH)), variant="poly"),
                          cycles=16),
        "ellipsoid64W": dict(setup=lambda: setup("ellipsoid64W", 3, 64, ellipsoid(64),
                                                 ProblemSpec("poisson", "dirichlet"), "w", cmin=16),
                             cycles=16, store_plan=False),
        "pores64": dict(setup=lambda: CF.config_pores(N=64, cycles=15), cycles=15, store_plan=False),
        # BASELINE configs at (or towards) their stated sizes, run by the reference
        # itself; too large to store plans, so tests rebuild them with the repo's
        # own setup, which must hash like the reference's (plan_digests)
        "ball256": dict(setup=lambda: CF.config_ball(256), cycles=15, store_plan=False),        # c3
        "flowerD2048": dict(setup=lambda: CF.config_flower_dirichlet(2048), cycles=20,          # c2 proxy
                            store_plan=False),
        "flowerM128": dict(setup=lambda: CF.config_flower(128), cycles=20),                     # c2 mixed BC
        "flowerM256": dict(setup=lambda: CF.config_flower(256), cycles=20, store_plan=False),
        "flowerM2048": dict(setup=lambda: CF.config_flower(2048), cycles=20, store_plan=False,  # c2 as specified
                            rho=False),
        "pores128": dict(setup=lambda: CF.config_pores(N=128, cycles=15), cycles=15, store_plan=False),
    }
    return cases


CASES = _cases()
