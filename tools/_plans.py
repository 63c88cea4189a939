"""Plans of a bench configuration, cached in $TMPDIR so the A/B tools of one
gpurun call pay the host setup (28 s at 512^3) once.  Diagnostics only."""
import os
import pickle
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def load(spec):
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200.cycle import CycleDriver
    from paper_2207_14208_b200.transfer import build_hierarchy

    name, N = spec.split(":")
    N = int(N)
    path = os.path.join(os.environ.get("TMPDIR", "/tmp"), f"gmg_plans_{name}_{N}.pkl")
    setup = CF.config_pores(N=N) if name == "c4" else CF.CONFIGS[name](N)
    if os.path.exists(path):
        with open(path, "rb") as fh:
            plans, f, g, e = pickle.load(fh)
        return setup, plans, f, g, e
    levels = build_hierarchy(setup.grid, setup.phi, setup.faces, max_levels=setup.cycle.max_levels,
                             coarsest_min=setup.coarsest_min)
    plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
    if setup.f_seed is not None:
        f = CF.pore_rhs(setup, plans[0].labels)
    with open(path, "wb") as fh:
        pickle.dump((plans, f, g, e), fh, protocol=4)
    return setup, plans, f, g, e
