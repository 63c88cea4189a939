"""ctypes binding of oracle/_build/libghostmg_oracle.so (test infrastructure).

Each wrapper restates one reference operation (see ghostmg_oracle.c for the
file:line each follows) on NumPy arrays.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libghostmg_oracle.so")
_lib = None

_d = ctypes.c_double
_i64 = ctypes.c_int64
_p = ctypes.c_void_p


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
                os.path.join(_HERE, "ghostmg_oracle.c")):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        sig = {
            "oracle_gs_sweep": (None, [ctypes.c_int, _i64, _p, _p, _p, _d, _d]),
            "oracle_ghost_sweep": (None, [ctypes.c_int, _i64, _p, _p, _p, _p, _p, _p]),
            "oracle_residual_internal": (_d, [ctypes.c_int, _i64, _p, _p, _p, _d, _d, _p]),
            "oracle_residual_ghost": (_d, [ctypes.c_int, _i64, _p, _p, _p, _p, _p]),
            "oracle_extrapolate": (None, [ctypes.c_int, _i64, ctypes.c_int, _p, _p, _p, _p, _p, _p, _p]),
            "oracle_band_bfs": (None, [ctypes.c_int, _i64, _i64, _p, _p, _p]),
            "oracle_band_transport": (None, [ctypes.c_int, _i64, _i64, _p, _p, _p, _p, _p]),
            "oracle_restrict_interior": (None, [ctypes.c_int, _i64, _p, _p, _p, _p]),
            "oracle_restrict_ghost": (None, [ctypes.c_int, _i64, _p, _p, _i64, _p, _p]),
            "oracle_interpolate_add": (None, [ctypes.c_int, _i64, _p, _p, _p]),
            "oracle_abs_max": (_d, [_p, _i64]),
            "oracle_np_sum": (_d, [_p, ctypes.c_int]),
            "oracle_ddot": (_d, [_p, _p, ctypes.c_int]),
            "oracle_sumsq": (_d, [_p, _i64]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a


def gs_sweep(plan, u, f):
    lib().oracle_gs_sweep(plan.d, plan.N, _ptr(plan.labels), _ptr(u), _ptr(f), plan.h2, plan.denom)


def ghost_sweep(plan, u, g, stencil=None):
    if plan.n_ghosts == 0:
        return
    st = _c(plan.stencil if stencil is None else stencil, np.int64)
    lib().oracle_ghost_sweep(plan.d, plan.n_ghosts, _ptr(plan.ghost_idx), _ptr(st),
                             _ptr(plan.ghost_w), _ptr(plan.ghost_dtau), _ptr(_c(g, np.float64)), _ptr(u))


def smooth(plan, u, f, g, count, stencil=None):
    st = _c(plan.stencil, np.int64) if stencil is None else stencil
    for _ in range(count):
        gs_sweep(plan, u, f)
        ghost_sweep(plan, u, g, st)


def residual_internal_full(plan, u, f):
    r = np.zeros(plan.n_nodes)
    m = lib().oracle_residual_internal(plan.d, plan.N, _ptr(plan.labels), _ptr(u), _ptr(f),
                                       plan.h2, plan.denom, _ptr(r))
    return r, m


def residual_ghost(plan, u, g, stencil=None):
    rg = np.zeros(plan.n_ghosts)
    if plan.n_ghosts == 0:
        return rg, 0.0
    st = _c(plan.stencil if stencil is None else stencil, np.int64)
    m = lib().oracle_residual_ghost(plan.d, plan.n_ghosts, _ptr(st), _ptr(plan.ghost_w),
                                    _ptr(_c(g, np.float64)), _ptr(u), _ptr(rg))
    return rg, m


def extrapolate(plan, values):
    """In place: fill the band of ``values`` (full grid array)."""
    if plan.n_band == 0:
        return values
    scratch = np.empty(plan.n_band)
    step = _c(plan.trans_step, np.int8)
    absn = _c(plan.trans_absn, np.float64)
    lib().oracle_extrapolate(plan.d, plan.N, len(plan.bfs_len), _ptr(_c(plan.bfs_len, np.int64)),
                             _ptr(plan.band_idx), _ptr(_c(plan.bfs_mask, np.uint8)), _ptr(step),
                             _ptr(absn), _ptr(values), _ptr(scratch))
    return values


def band_bfs(plan, values, idx, mask):
    """One BFS group of the band extension on the nodes ``idx`` (in place)."""
    idx = _c(idx, np.int64)
    if idx.size:
        lib().oracle_band_bfs(plan.d, plan.N, idx.size, _ptr(idx), _ptr(_c(mask, np.uint8)), _ptr(values))


def band_transport(plan, values, idx, step, absn):
    """One Jacobi transport step of the band extension on the nodes ``idx``."""
    idx = _c(idx, np.int64)
    if idx.size:
        scratch = np.empty(idx.size)
        lib().oracle_band_transport(plan.d, plan.N, idx.size, _ptr(idx), _ptr(_c(step, np.int8)),
                                    _ptr(_c(absn, np.float64)), _ptr(values), _ptr(scratch))


def restrict_interior(fine, coarse, r_fine):
    out = np.zeros(coarse.n_nodes)
    lib().oracle_restrict_interior(fine.d, fine.N, _ptr(fine.labels), _ptr(r_fine),
                                   _ptr(coarse.labels), _ptr(out))
    return out


def restrict_ghost(fine, coarse, r_ext):
    out = np.zeros(coarse.n_ghosts)
    if coarse.n_ghosts:
        lib().oracle_restrict_ghost(fine.d, fine.N, _ptr(fine.labels), _ptr(r_ext),
                                    coarse.n_ghosts, _ptr(coarse.ghost_idx), _ptr(out))
    return out


def interpolate_add(fine, u, e_coarse):
    lib().oracle_interpolate_add(fine.d, fine.N, _ptr(fine.labels), _ptr(u), _ptr(e_coarse))


def abs_max(u):
    return lib().oracle_abs_max(_ptr(u), u.size)


def np_sum(a):
    a = _c(a, np.float64)
    return lib().oracle_np_sum(_ptr(a), a.size)


def ddot(x, y):
    x = _c(x, np.float64)
    y = _c(y, np.float64)
    return lib().oracle_ddot(_ptr(x), _ptr(y), x.size)


def sumsq(a):
    a = _c(a, np.float64)
    return lib().oracle_sumsq(_ptr(a), a.size)
