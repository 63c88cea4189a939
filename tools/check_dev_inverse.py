import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import goldutil as GU
from test_gpu_parity import _pores64_solver
from paper_2207_14208_b200.cycle import measure_rho
rec = GU.record("pores64")
plans, s = _pores64_solver("device-inverse")
u, rep = s.solve(u=np.zeros(plans[0].n_nodes), cycles=15)
want = np.array(GU.hexlist(rec["solve"]["residual_norms"]))
got = np.array(rep.residual_norms)
print("rel residual diffs", np.abs(got - want) / want)
_, ref = _pores64_solver("superlu")
uref, _ = ref.solve(u=np.zeros(plans[0].n_nodes), cycles=15)
print("u rel linf", np.max(np.abs(u - uref)) / np.max(np.abs(uref)))
print("rho", measure_rho(s).rho_asymptotic, rec["rho"]["rho"])
