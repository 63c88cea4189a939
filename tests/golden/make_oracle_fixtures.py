"""Oracle fixtures at the BASELINE sizes the reference itself cannot run here.

The reference (pure NumPy) would need ~30 min of setup, ~60 GB of RAM and
~130 s per V-cycle at config 4 (pores 512^3), so the bench
configuration is pinned through the C oracle instead: the oracle is pinned bit
for bit to reference-run fixtures on every op and whole solves up to pores
128^3 / ball 256^3 / flower 2048^2 (tests/test_oracle_golden.py), and this
script records what it gives at 512^3 so the GPU tests can compare the device
solve with it without running the oracle on the GPU box.

    python tests/golden/make_oracle_fixtures.py [c4_512]

Records (tests/golden/_oracle_<name>.json; the leading underscore keeps them
out of the reference-golden registry): the plan digests of the repo's own
setup, the residual history (hex) and final-iterate digest of a
zero-initial-guess solve with the host SuperLU coarsest solve, and the
measure_rho history and rho (seed 42).
"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

from goldutil import digest, plan_digest  # noqa: E402


def oracle_case(name, setup, cycles):
    from oracle.solver import OracleSolver
    from paper_2207_14208_b200 import configs as CF
    from paper_2207_14208_b200.cycle import CycleDriver, measure_rho
    from paper_2207_14208_b200.transfer import build_hierarchy

    t0 = time.time()
    levels = build_hierarchy(setup.grid, setup.phi, setup.faces, max_levels=setup.cycle.max_levels,
                             coarsest_min=setup.coarsest_min)
    plans, f, g, e = CycleDriver.problem_data(levels, setup.spec, setup.smoother, setup.default_variant)
    del levels
    if setup.f_seed is not None:
        f = CF.pore_rhs(setup, plans[0].labels)
    print(name, "setup", round(time.time() - t0, 1), "s", flush=True)
    rec = {"name": name, "setup": setup.name, "cycles": cycles, "scheme": setup.cycle.scheme,
           "coarse_solver": "direct", "norm": "inf", "n_levels": len(plans), "source": "oracle",
           "plan_digests": [{k: plan_digest(v) for k, v in p.to_arrays().items()} for p in plans]}
    s = OracleSolver(plans, f, g, e, setup.smoother, setup.cycle)
    t0 = time.time()
    u, rep = s.solve(u=np.zeros(plans[0].n_nodes), cycles=cycles)
    print(name, "solve", round(time.time() - t0, 1), "s", rep.residual_norms[-1], flush=True)
    rec["solve"] = {"from_initial_field": False, "residual_norms": [float(x).hex() for x in rep.residual_norms],
                    "u_digest": digest(u), "diverged": rep.diverged}
    del u
    t0 = time.time()
    r = measure_rho(s, seed=42)
    print(name, "rho", round(time.time() - t0, 1), "s", r.rho_asymptotic, flush=True)
    rec["rho"] = {"rho": r.rho_asymptotic, "residual_norms": [float(x).hex() for x in r.residual_norms]}
    with open(os.path.join(HERE, f"_oracle_{name}.json"), "w") as fh:
        json.dump(rec, fh, indent=1)


CASES = {
    "c4_512": lambda: (__import__("paper_2207_14208_b200.configs", fromlist=["x"]).config_pores(N=512, cycles=15), 15),
}


if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        setup, cycles = CASES[name]()
        oracle_case(name, setup, cycles)
