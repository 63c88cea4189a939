"""Compare device interpolation / interior residual with the C oracle on one case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

import goldutil as GU
from oracle import ops as O
from paper_2207_14208_b200 import _lib

name = sys.argv[1]
plans, _ = GU.plans(name)
ctx = _lib.Context(plans[0].d, len(plans))
for i, p in enumerate(plans):
    ctx.set_level(i, p)
rng = np.random.default_rng(1)
fine, coarse = plans[0], plans[1]
u = rng.standard_normal(fine.n_nodes)
e = rng.standard_normal(coarse.n_nodes)
ctx.set_vector(0, _lib.U, u)
ctx.set_vector(1, _lib.U, e)
ctx.apply(0, _lib.OP_INTERP_ADD)
got = ctx.get_vector(0, _lib.U, fine.n_nodes)
want = u.copy()
O.interpolate_add(fine, want, e)
bad = np.nonzero(got != want)[0]
print("interp mismatches", len(bad), "of", fine.n_nodes)
shape = (fine.N + 1,) * fine.d
for b in bad[:10]:
    print(np.unravel_index(b, shape), fine.labels[b], got[b], want[b], u[b])
f = rng.standard_normal(fine.n_nodes)
ctx.set_vector(0, _lib.U, u)
ctx.set_vector(0, _lib.F, f)
ctx.set_vector(0, _lib.R_INT, np.zeros(fine.n_nodes))
ctx.apply(0, _lib.OP_RES_INT)
got = ctx.get_vector(0, _lib.R_INT, fine.n_nodes)
want = O.residual_internal_full(fine, u, f)
m = fine.labels == 0
want = want[0] if isinstance(want, tuple) else want
bad = np.nonzero((got != want) & m)[0]
print("residual mismatches", len(bad), "of", int(m.sum()))
for b in bad[:10]:
    print(np.unravel_index(b, shape), got[b], want[b])
