"""CPU checks: the C ABI library loads and exports what the header declares;
host helpers (RNG, BLFA, setup) match the reference."""

import math
import os
import re
import sys

import numpy as np
import pytest

from paper_2207_14208_b200 import _lib
from paper_2207_14208_b200 import blfa
from paper_2207_14208_b200.rng import XorShift64Star, uniform_symmetric

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"


def header_symbols():
    text = open(os.path.join(ROOT, "include", "ghostmg_b200.h")).read()
    return sorted(set(re.findall(r"\b(gmg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert "gmg_cycle" in syms and "gmg_set_level" in syms
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) <= set(_lib.SIGNATURES), set(syms) - set(_lib.SIGNATURES)
    assert lib.gmg_version() == 100


def test_library_is_sm100a_only():
    """The shipped cubin targets sm_100a (cross-compiled here)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_native_rng_matches_python_stream():
    for seed in (0, 42, 12345):
        a = _lib.uniform_symmetric_native(seed, 50_000)
        b = uniform_symmetric(seed, 50_000)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_rng_frozen_bitstream():
    """First draws of the reference stream (restated from rng.py:14-56)."""
    r = XorShift64Star(42)
    words = [r.next_u64() for _ in range(4)]
    r2 = XorShift64Star(42)
    x = r2.uniform()
    assert x == (words[0] >> 11) * 2.0 ** -53
    assert 0.0 <= x < 1.0


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_rng_and_blfa_against_live_reference():
    sys.path.insert(0, REF)
    from ghostmg import blfa as rb
    from ghostmg.rng import XorShift64Star as R

    for seed in (0, 1, 42, 2 ** 63):
        a, b = R(seed), XorShift64Star(seed)
        assert [a.next_u64() for _ in range(64)] == [b.next_u64() for _ in range(64)]
    rng = np.random.default_rng(0)
    for d in (1, 2, 3):
        for bc in ("dirichlet", "neumann"):
            for var in ("poly", "exp"):
                th = rng.uniform(0, 1.6, 200)
                want = [rb.dtau_opt(rb.BlfaQuery(bc=bc, d=d, theta=float(t), h=0.03125, variant=var)) for t in th]
                got_s = [blfa.dtau_opt(blfa.BlfaQuery(bc=bc, d=d, theta=float(t), h=0.03125, variant=var)) for t in th]
                got_b = blfa.dtau_opt_batch(np.full(200, bc == "dirichlet"), th, d, 0.03125, var)
                assert got_s == want
                assert np.array_equal(got_b, np.array(want))


def test_blfa_closed_forms():
    """dtau* = 2/(g0_max + g0_min) over the corner set; Neumann scales by h."""
    q = blfa.BlfaQuery(bc="dirichlet", d=2, theta=0.0, variant="exp")
    # EXP, theta = 0: g0 = 1 at every corner -> dtau = 1
    assert blfa.dtau_opt(q) == 1.0
    qn = blfa.BlfaQuery(bc="neumann", d=2, theta=0.5, h=0.1, variant="exp")
    ps = [blfa.symbol_p(a) for a in blfa.corner_points(2)]
    g = [p * math.exp(-p * 0.5) for p in ps]
    assert blfa.dtau_opt(qn) == 0.1 * (2.0 / (max(g) + min(g)))
    assert blfa.symbol_p((math.pi / 2,)) == math.log(2.0 + math.sqrt(3.0))
