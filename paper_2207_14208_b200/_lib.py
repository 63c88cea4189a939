"""ctypes binding of libghostmg_b200.so (include/ghostmg_b200.h).

The library is the product path: there is no Python or CPU fallback for any
cycle operation.  Importing works without a GPU (so the exported ABI can be
checked on CPU); creating a context without a CUDA device raises.
"""

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libghostmg_b200.so")
HEADER = os.path.join(HERE, "..", "include", "ghostmg_b200.h")

U, F, G, R_INT, R_EXT = 0, 1, 2, 3, 4
OP_GS_SWEEP, OP_GHOST_SWEEP, OP_SMOOTH, OP_RES_INT, OP_RES_GHOST = 0, 1, 2, 3, 4
OP_EXTEND_REXT, OP_EXTEND_U, OP_RESTRICT_INT, OP_RESTRICT_GHOST, OP_INTERP_ADD, OP_ZERO_U = 5, 6, 7, 8, 9, 10
OP_COARSE_SOLVE = 11
OP_RES_RESTRICT = 12
OP_BAND_BFS_REXT, OP_BAND_BFS_U, OP_BAND_STEP_REXT, OP_BAND_STEP_U, OP_CYCLE_TAIL = 13, 14, 15, 16, 17
KCLASS = {"gs_sweep": 0, "ghost_sweep": 1, "residual": 2, "band": 3, "restrict": 4,
          "interp": 5, "coarse": 6, "norm": 7}

_p = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_d = ctypes.c_double

COARSE_CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                             ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double))

SIGNATURES = {
    "gmg_version": (_i, []),
    "gmg_create": (_p, [_i, _i, _i]),
    "gmg_destroy": (None, [_p]),
    "gmg_last_error": (ctypes.c_char_p, [_p]),
    "gmg_set_stream": (_i, [_p, _p]),
    "gmg_set_level": (_i, [_p, _i, _i64, _d, _p, _i64, _p, _p, _p, _p, _p, _p, _i, _p, _p, _p, _p, _p]),
    "gmg_set_cycle": (_i, [_p, _i, _i, _i, _i, _i, _i]),
    "gmg_set_slab": (_i, [_p, _i, _i64, _i64]),
    "gmg_abs_max_planes": (_i, [_p, _i64, _i64, _p]),
    "gmg_initial_field": (_i, [_p, ctypes.c_uint64, _p, _i, _i64, _i64, _p, _p]),
    "gmg_set_coarse_callback": (_i, [_p, COARSE_CB, _p]),
    "gmg_set_coarse_inverse": (_i, [_p, _i64, _p, _i]),
    "gmg_set_coarse_nd": (_i, [_p, _i64, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p, _i]),
    "gmg_set_coarse_nd_coupling": (_i, [_p, _i64, _i64, _p, _p, _p]),
    "gmg_coarse_prog_begin": (_i, [_p, _i64, _p, _i64]),
    "gmg_coarse_prog_dense": (_i, [_p, _i64, _i64, _p, _i, _i64, _i64, _i64]),
    "gmg_coarse_prog_csr": (_i, [_p, _i64, _i64, _p, _p, _p, _i64, _i64, _i64]),
    "gmg_coarse_prog_end": (_i, [_p, _i64]),
    "gmg_set_vector": (_i, [_p, _i, _i, _p]),
    "gmg_get_vector": (_i, [_p, _i, _i, _p]),
    "gmg_device_pointer": (_p, [_p, _i, _i]),
    "gmg_vector_length": (_i64, [_p, _i, _i]),
    "gmg_apply": (_i, [_p, _i, _i, _i]),
    "gmg_cycle": (_i, [_p, _i]),
    "gmg_residual_norm": (_i, [_p, _i, _p]),
    "gmg_residual_norm_peak": (_i, [_p, _i, _p, _p]),
    "gmg_abs_max_scale": (_i, [_p, _d, _d, _p, _p]),
    "gmg_norm_begin": (_i, [_p]),
    "gmg_norm_end": (_i, [_p, _p]),
    "gmg_scale_u": (_i, [_p, _d]),
    "gmg_synchronize": (_i, [_p]),
    "gmg_launch_count": (_i64, [_p]),
    "gmg_debug_gs_trace": (_i64, [_p, _i, _p, _i64]),
    "gmg_debug_ghost_trace": (_i64, [_p, _i, _p, _i64]),
    "gmg_debug_gs_knobs": (_i, [_p, _p, _i]),
    "gmg_device_bytes": (_i64, [_p]),
    "gmg_profile": (_i, [_p, _i]),
    "gmg_profile_read": (_i, [_p, _i, _i, _p, _p]),
    "gmg_uniform_symmetric": (_i, [ctypes.c_uint64, _i64, _p]),
    "gmg_setup_classify_balls": (_i, [_i, _i, _i64, _p, _i, _i, _p, _p, _i, _p]),
    "gmg_setup_check_transfer": (_i, [_i, _i, _i64, _p, _i64, _p, _p]),
    "gmg_setup_last_error": (ctypes.c_char_p, []),
}

_lib = None


def load():
    """Load (building first if the sources are newer) the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    from . import _build
    path = os.environ.get("GMG_LIB_OVERRIDE")  # diagnostics: A/B builds (tools/build_alt.sh)
    if not path:
        path = LIB_PATH
        if _build.needs_build():
            _build.build()
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None and path != LIB_PATH:
            continue  # an older A/B build may lack newer diagnostics
        if fn is None:
            raise ImportError(f"{path} does not export {name}")
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None and a.size else None


class GmgError(RuntimeError):
    pass


class Context:
    """Owner of one gmg_ctx (device buffers of a whole hierarchy)."""

    def __init__(self, ndim, nlevels, device=0):
        self.lib = load()
        self.ctx = self.lib.gmg_create(device, ndim, nlevels)
        if not self.ctx:
            raise GmgError("gmg_create failed: no usable CUDA device "
                           "(the B200 path has no CPU fallback)")
        self.nlevels = nlevels
        self._keep = []

    def check(self, rc):
        if rc != 0:
            msg = self.lib.gmg_last_error(self.ctx)
            raise GmgError(msg.decode() if msg else f"gmg error {rc}")

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.gmg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- upload ---------------------------------------------------------
    def set_level(self, level, plan):
        c = np.ascontiguousarray
        self._lvl_arrays = arr = dict(
            labels=c(plan.labels, np.uint8), gi=c(plan.ghost_idx, np.int64),
            glow=c(plan.ghost_low, np.int64), gw=c(plan.ghost_w, np.float64),
            gdt=c(plan.ghost_dtau, np.float64), gpr=c(plan.ghost_promoted, np.uint8),
            gb=c(plan.ghost_batch, np.int32), bl=c(plan.bfs_len, np.int64),
            bi=c(plan.band_idx, np.int64), bm=c(plan.bfs_mask, np.uint8),
            ts=c(plan.trans_step, np.int8), ta=c(plan.trans_absn, np.float64))
        self.check(self.lib.gmg_set_level(
            self.ctx, level, plan.N, float(plan.reaction), ptr(arr["labels"]), plan.n_ghosts,
            ptr(arr["gi"]), ptr(arr["glow"]), ptr(arr["gw"]), ptr(arr["gdt"]), ptr(arr["gpr"]),
            ptr(arr["gb"]), len(arr["bl"]), ptr(arr["bl"]), ptr(arr["bi"]), ptr(arr["bm"]),
            ptr(arr["ts"]), ptr(arr["ta"])))
        del self._lvl_arrays

    def set_cycle(self, nu1, nu2, gamma, coarse_mode, coarse_sweeps, norm):
        self.check(self.lib.gmg_set_cycle(self.ctx, nu1, nu2, gamma, coarse_mode, coarse_sweeps, norm))

    def set_slab(self, level, lo, hi):
        """z-slab mode: this context updates planes [lo, hi) of `level` only.
        Returns the number of BFS groups of the level's band plan."""
        rc = self.lib.gmg_set_slab(self.ctx, level, lo, hi)
        if rc < 0:
            self.check(rc)
        return rc

    def initial_field(self, seed, n_nodes, elim_idx, elim_val, lane_len=64):
        """Seeded initial iterate generated on the device (reference
        solver.py:205-213) into U of the finest level."""
        from . import rng

        lanes = -(-int(n_nodes) // lane_len)
        K = max(1, (lanes - 1).bit_length())
        cols = [rng._power_columns(lane_len)]
        for _ in range(K - 1):
            cols.append(rng._compose(cols[-1], cols[-1]))
        jc = np.array(cols, dtype=np.uint64).reshape(-1)
        idx = np.ascontiguousarray(elim_idx, dtype=np.int64)
        val = np.ascontiguousarray(elim_val, dtype=np.float64)
        self.check(self.lib.gmg_initial_field(self.ctx, rng.seed_state(seed), ptr(jc), K, lane_len, len(idx),
                                              ptr(idx), ptr(val)))

    def abs_max_planes(self, lo, hi):
        peak = np.zeros(1)
        self.check(self.lib.gmg_abs_max_planes(self.ctx, lo, hi, ptr(peak)))
        return float(peak[0])

    def set_coarse_callback(self, fn):
        """fn(rhs ndarray) -> solution ndarray."""

        def trampoline(user, n, rhs, x):
            try:
                r = np.ctypeslib.as_array(rhs, shape=(n,)).copy()
                out = np.ctypeslib.as_array(x, shape=(n,))
                out[:] = fn(r)
                return 0
            except Exception:  # propagate as an error code
                import traceback
                traceback.print_exc()
                return 1

        cb = COARSE_CB(trampoline)
        self._keep.append(cb)
        self.check(self.lib.gmg_set_coarse_callback(self.ctx, cb, None))

    def set_coarse_inverse(self, n, ptr_value, on_device):
        self.check(self.lib.gmg_set_coarse_inverse(self.ctx, n, ptr_value, 1 if on_device else 0))

    def set_coarse_nd(self, n, na, nb, ns, perm, aai, bbi, g, w, si, on_device):
        """Nested-dissection coarse solve (pointers: device if on_device)."""
        perm = np.ascontiguousarray(perm, dtype=np.int32)
        self.check(self.lib.gmg_set_coarse_nd(self.ctx, n, na, nb, ns, ptr(perm), aai, bbi, g, w, si,
                                              1 if on_device else 0))

    def set_coarse_nd_coupling(self, ns, nab, rowptr, col, val):
        """Sparse separator coupling (host CSR) for the nested-dissection solve."""
        rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
        col = np.ascontiguousarray(col, dtype=np.int32)
        val = np.ascontiguousarray(val, dtype=np.float64)
        self.check(self.lib.gmg_set_coarse_nd_coupling(self.ctx, ns, nab, ptr(rowptr), ptr(col), ptr(val)))

    # -- coarse program (recursive nested dissection) ----------------------
    def coarse_prog_begin(self, n, perm, nwork):
        perm = np.ascontiguousarray(perm, dtype=np.int32)
        self.check(self.lib.gmg_coarse_prog_begin(self.ctx, n, ptr(perm), nwork))

    def coarse_prog_dense(self, m, k, dev_ptr, x_off, y_off, y0_off=-1):
        self.check(self.lib.gmg_coarse_prog_dense(self.ctx, m, k, dev_ptr, 1, x_off, y_off, y0_off))

    def coarse_prog_csr(self, C, x_off, y0_off, y_off):
        C = C.tocsr()
        C.sort_indices()
        rowptr = np.ascontiguousarray(C.indptr, dtype=np.int64)
        col = np.ascontiguousarray(C.indices, dtype=np.int32)
        val = np.ascontiguousarray(C.data, dtype=np.float64)
        self.check(self.lib.gmg_coarse_prog_csr(self.ctx, C.shape[0], C.shape[1], ptr(rowptr), ptr(col), ptr(val),
                                                x_off, y0_off, y_off))

    def coarse_prog_end(self, x_off):
        self.check(self.lib.gmg_coarse_prog_end(self.ctx, x_off))

    def set_stream(self, stream_handle):
        self.check(self.lib.gmg_set_stream(self.ctx, stream_handle))

    # -- vectors --------------------------------------------------------
    def vector_length(self, level, which):
        n = int(self.lib.gmg_vector_length(self.ctx, level, which))
        if n < 0:
            raise GmgError(f"no vector {which} on level {level}")
        return n

    def set_vector(self, level, which, host):
        host = np.ascontiguousarray(host, dtype=np.float64)
        n = self.vector_length(level, which)
        if host.ndim != 1 or host.size != n:
            raise ValueError(f"vector {which} of level {level} has {n} entries, got an array of shape {host.shape}")
        self.check(self.lib.gmg_set_vector(self.ctx, level, which, ptr(host)))

    def get_vector(self, level, which, n, out=None):
        if n != self.vector_length(level, which):
            raise ValueError(f"vector {which} of level {level} has {self.vector_length(level, which)} entries, not {n}")
        if out is None:
            out = np.empty(n, dtype=np.float64)
        elif out.shape != (n,) or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("out must be a contiguous float64 array of the vector's length")
        if n:
            self.check(self.lib.gmg_get_vector(self.ctx, level, which, ptr(out)))
        return out

    def device_pointer(self, level, which):
        return self.lib.gmg_device_pointer(self.ctx, level, which)

    def apply(self, level, op, count=1):
        self.check(self.lib.gmg_apply(self.ctx, level, op, count))

    def cycle(self, n=1):
        self.check(self.lib.gmg_cycle(self.ctx, n))

    def residual_parts(self, level=0):
        out = np.zeros(2)
        self.check(self.lib.gmg_residual_norm(self.ctx, level, ptr(out)))
        return float(out[0]), float(out[1])

    def residual_parts_peak(self, level=0):
        """(max|r_int|, max|r_g|, lower bound of max|u| or -1), one pass."""
        out = np.zeros(2)
        lb = np.zeros(1)
        self.check(self.lib.gmg_residual_norm_peak(self.ctx, level, ptr(out), ptr(lb)))
        return float(out[0]), float(out[1]), float(lb[0])

    def abs_max_scale(self, threshold=1e-250, factor=1e250):
        peak = np.zeros(1)
        scaled = np.zeros(1, dtype=np.int32)
        self.check(self.lib.gmg_abs_max_scale(self.ctx, threshold, factor, ptr(peak), ptr(scaled)))
        return float(peak[0]), bool(scaled[0])

    def norm_begin(self):
        self.check(self.lib.gmg_norm_begin(self.ctx))

    def norm_end(self):
        out = np.zeros(3)
        self.check(self.lib.gmg_norm_end(self.ctx, ptr(out)))
        return float(out[0]), float(out[1]), float(out[2])

    def scale_u(self, factor):
        self.check(self.lib.gmg_scale_u(self.ctx, factor))

    def synchronize(self):
        self.check(self.lib.gmg_synchronize(self.ctx))

    @property
    def launches(self):
        return int(self.lib.gmg_launch_count(self.ctx))

    def ghost_trace(self, level, nslots):
        """Ghost-sweep timeline of the last sweep on `level` (GMG_GS_TRACE=1)."""
        out = np.zeros((nslots, 3), dtype=np.int64)
        n = self.lib.gmg_debug_ghost_trace(self.ctx, level, out.ctypes.data, out.size)
        return out if n else None

    def gs_trace(self, level, ntasks):
        """GS task timeline of the last sweep on `level` (GMG_GS_TRACE=1)."""
        out = np.zeros((ntasks, 24), dtype=np.int64)
        n = self.lib.gmg_debug_gs_trace(self.ctx, level, out.ctypes.data, out.size)
        return out if n else None

    def gs_knobs(self, sleep_ns=None, variant=-1):
        """Diagnostics: GS loader/writer back-off (ns x4) and variant."""
        arr = None if sleep_ns is None else (ctypes.c_int * 4)(*sleep_ns)
        self.check(self.lib.gmg_debug_gs_knobs(self.ctx, arr, variant))

    @property
    def device_bytes(self):
        return int(self.lib.gmg_device_bytes(self.ctx))

    def profile(self, enable=True, classes=None):
        """Time kernel classes with CUDA events (all of them, or ``classes``)."""
        if not enable:
            mask = 0
        elif classes is None:
            mask = 0xFF
        else:
            mask = 0
            for c in classes:
                mask |= 1 << KCLASS.get(c, c)
        self.check(self.lib.gmg_profile(self.ctx, mask))

    def profile_read(self, kclass, level=-1):
        ms = np.zeros(1)
        cnt = np.zeros(1, dtype=np.int64)
        self.check(self.lib.gmg_profile_read(self.ctx, KCLASS.get(kclass, kclass), level, ptr(ms), ptr(cnt)))
        return float(ms[0]), int(cnt[0])


def uniform_symmetric_native(seed, n):
    out = np.empty(int(n), dtype=np.float64)
    if n:
        load().gmg_uniform_symmetric(int(seed) & ((1 << 64) - 1), int(n), ptr(out))
    return out


def setup_classify_balls(device, d, N, axis, kind, centers, radii, face_mask):
    """Labels of one level on the device (gmg_setup_classify_balls)."""
    lib = load()
    axis = np.ascontiguousarray(axis, dtype=np.float64)
    centers = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, d)
    radii = np.ascontiguousarray(radii, dtype=np.float64).reshape(-1)
    out = np.empty((N + 1) ** d, dtype=np.uint8)
    rc = lib.gmg_setup_classify_balls(device, d, N, ptr(axis), kind, len(radii), ptr(centers), ptr(radii), face_mask,
                                      ptr(out))
    if rc != 0:
        raise GmgError(lib.gmg_setup_last_error().decode())
    return out


def setup_check_transfer(device, d, Nf, lab_f, Nc, lab_c):
    """Bit mask of failed restriction-block checks (gmg_setup_check_transfer)."""
    lib = load()
    lab_f = np.ascontiguousarray(lab_f, dtype=np.uint8)
    lab_c = np.ascontiguousarray(lab_c, dtype=np.uint8)
    flags = np.zeros(1, dtype=np.int32)
    rc = lib.gmg_setup_check_transfer(device, d, Nf, ptr(lab_f), Nc, ptr(lab_c), ptr(flags))
    if rc != 0:
        raise GmgError(lib.gmg_setup_last_error().decode())
    return int(flags[0])
