// gs_stream.cu -- shared-memory-staged streaming lexicographic Gauss-Seidel
// sweep (sm_100a), the production kernel for levels with N >= 32.
//
// Same decomposition and dependency protocol as gs_sweep.cu (warp task =
// 32-column chunk x block of R rows x all planes; lane j one line behind
// lane j-1; progress words with release/acquire), but nothing on the
// per-step critical path touches global memory:
//
//  * every line's old u (plus the old right-halo column k0+32) is copied
//    into a 128-line shared ring 64 steps ahead with cp.async (LDGSTS), and
//    f + the line's "internal" bitmask 32 steps ahead into a 64-line ring;
//  * values produced by neighbour tasks (left halo column k0-1, and in 3-D
//    the row above the block) are fetched 32 steps ahead, after an
//    ld.acquire of the producer's progress word, with cp.async.cg (L2 only,
//    16-byte aligned superset) so no stale L1 line can be read;
//  * each step reads its stencil from shared memory (the ring pitch makes
//    the skewed diagonal access bank-conflict free), updates in place, and
//    the line that lane 31 just finished is written back to HBM as one
//    coalesced 256-byte row.
//
// Reference: gs_lex_sweep, /root/reference/pkg/src/ghostmg/smoothing.py:127-132.
#include <cstddef>

#include "gmg_kernels.cuh"

namespace gmg {

namespace {

constexpr int RLU = 128;  // u ring lines
constexpr int RLF = 64;   // f ring lines
constexpr int RP = 8;     // plane-row ring (3-D)
constexpr int PFU = 64;   // u prefetch distance (lines)
constexpr int PFF = 32;   // f / halo prefetch distance (lines)
// u ring row: [0] k0-2, [1] k0-1 (new left halo from chunk c-1), [2..33]
// columns k0..k0+31, [34] k0+32 (old right halo), [35] k0+33.  With the
// padded device layout every 16-byte chunk of that range is aligned, and the
// pitch of 36 doubles keeps the skewed diagonal access (lane j on row t-j)
// free of bank conflicts.
constexpr int UP = 36;

struct __align__(16) WarpRing {
  double u[RLU][UP];
  double f[RLF][32];
  double up[RP][32];  // row above the block (new values), 3-D
  double dn[RP][32];  // row below the block (old values), 3-D
  uint32_t mask[RLF];
};

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp16p(unsigned dst, const void* src, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q cp.async.ca.shared.global [%0], [%1], 16;\n}\n"
               ::"r"(dst), "l"(src), "r"((int)p));
}
__device__ __forceinline__ void cp16cgp(unsigned dst, const void* src, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q cp.async.cg.shared.global [%0], [%1], 16;\n}\n"
               ::"r"(dst), "l"(src), "r"((int)p));
}
__device__ __forceinline__ void cp4p(unsigned dst, const void* src, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q cp.async.ca.shared.global [%0], [%1], 4;\n}\n"
               ::"r"(dst), "l"(src), "r"((int)p));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Uniform line stream of a task: line L, row r, plane p, device position of
// (line, column k0) and index of the line's internal-bitmask word.
struct Stream {
  int L, r, p;
  int64_t off;
  int64_t mw;
  __device__ __forceinline__ void init(int L0, int R, int64_t pos0, int64_t s0, int64_t s1,
                                       int64_t mw0, int64_t mplane, int64_t mrow) {
    L = L0;
    p = L0 >= 0 ? L0 / R : -((-L0 + R - 1) / R);  // floor(L0 / R)
    r = L0 - p * R;
    off = pos0 + (int64_t)(p + 1) * s0 + (int64_t)r * s1;
    mw = mw0 + (int64_t)(p + 1) * mplane + (int64_t)r * mrow;
  }
  __device__ __forceinline__ void next(int R, int64_t s1, int64_t wrap, int64_t mrow, int64_t mwrap) {
    ++L;
    const bool w = ++r == R;
    r = w ? 0 : r;
    p += w;
    off += w ? wrap : s1;
    mw += w ? mwrap : mrow;
  }
};

}  // namespace

template <int DIM>
__global__ void __launch_bounds__(32) gs_stream_kernel(GsArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  WarpRing& S = reinterpret_cast<WarpRing*>(smem_raw)[threadIdx.x >> 5];
  const Geom g = a.g;
  const int N = (int)g.N;
  double* __restrict__ u = a.u;
  const double* __restrict__ f = a.f;
  const double h2 = g.h2, inv = g.inv;
  const unsigned sbase = smem_addr(&S);
  const unsigned sU16 = sbase + (unsigned)offsetof(WarpRing, u) + 16u + 16u * lane;  // row[2 + 2 lane]
  const unsigned sU0 = sbase + (unsigned)offsetof(WarpRing, u);
  const unsigned sF16 = sbase + (unsigned)offsetof(WarpRing, f) + 16u * lane;
  const unsigned sUP16 = sbase + (unsigned)offsetof(WarpRing, up) + 16u * lane;
  const unsigned sDN16 = sbase + (unsigned)offsetof(WarpRing, dn) + 16u * lane;
  const unsigned sM = sbase + (unsigned)offsetof(WarpRing, mask);
  const bool lane0 = lane == 0;
  const bool l16 = lane < 16;
  const bool l17 = lane < 17;

  for (;;) {
    int tid = 0;
    if (lane0) tid = atomicAdd(a.ticket, 1);
    tid = __shfl_sync(FULL, tid, 0);
    if (tid >= a.ntasks) return;
    const int2 tk = a.tasks[tid];
    const int c = tk.x, b = tk.y;
    const int k0 = 1 + 32 * c;
    const bool kval = k0 + lane <= N - 1;  // interior column
    const int R = DIM == 3 ? min(a.B1, N - 1 - b * a.B1) : 1;
    const int nLines = (N - 1) * R;
    const int uEnd = nLines + R;
    const int rowbase = DIM == 3 ? 1 + b * a.B1 : 0;
    const int64_t s0 = g.s0;
    const int64_t s1 = DIM == 3 ? g.s1 : g.s0;  // next row (3-D) / next line (2-D)
    const int64_t wrap = DIM == 3 ? g.s0 - (int64_t)(R - 1) * g.s1 : g.s0;
    const int64_t pos0 = (DIM == 3 ? (int64_t)rowbase * g.s1 : 0) + k0 + OFF;  // plane i0 = 0
    const int64_t mplane = DIM == 3 ? (int64_t)g.n * a.Cm : (int64_t)a.Cm;
    const int64_t mrow = DIM == 3 ? (int64_t)a.Cm : mplane;
    const int64_t mwrap = DIM == 3 ? mplane - (int64_t)(R - 1) * a.Cm : mplane;
    const int64_t mw0 = (DIM == 3 ? (int64_t)rowbase * a.Cm : 0) + c;  // mask word of plane i0 = 0
    int* myprog = a.progress + c * a.Bn + b;
    const int* lprog = c > 0 ? a.progress + (c - 1) * a.Bn + b : nullptr;
    const int* uprog = (DIM == 3 && b > 0) ? a.progress + c * a.Bn + (b - 1) : nullptr;
    int seenL = 0, seenU = 0;

    const int t0 = -(PFU + R);
    Stream pu, pf, pd;
    pu.init(t0 + PFU, R, pos0, s0, s1, mw0, mplane, mrow);
    pf.init(t0 + PFF, R, pos0, s0, s1, mw0, mplane, mrow);
    pd.init(t0 - 31, R, pos0, s0, s1, mw0, mplane, mrow);
    // this lane's compute line nl = t - lane: row within the plane and plane slot
    int cr, cp;
    {
      const int L0 = t0 - lane;
      cp = L0 >= 0 ? L0 / R : -((-L0 + R - 1) / R);
      cr = L0 - cp * R;
    }
    double prev = 0.0;
    const int last = nLines + 30;

    for (int t = t0; t <= last; ++t) {
      // ---------------- prefetch: one cp.async group per step -------------
      if (pu.L < uEnd) {
        const unsigned row = sU16 + (unsigned)(pu.L & (RLU - 1)) * (8u * UP);
        cp16p(row, u + pu.off + 2 * lane, l17);
      }
      pu.next(R, s1, wrap, mrow, mwrap);
      if (pf.L >= 0 && pf.L < nLines) {
        const unsigned sf = (unsigned)(pf.L & (RLF - 1));
        cp16p(sF16 + sf * 256u, f + pf.off + 2 * lane, l16);
        cp4p(sM + sf * 4u, a.imask + pf.mw, lane0);
        const bool plane_start = DIM == 3 && pf.r == 0;
        // producers' progress: every lane polls the same word (no divergence)
        if (lprog)
          while (seenL < pf.L + 1) seenL = ld_acquire(lprog);
        if (uprog && plane_start) {
          const int need = (pf.p + 1) * a.B1;
          while (seenU < need) seenU = ld_acquire(uprog);
        }
        cp16cgp(sU0 + (unsigned)(pf.L & (RLU - 1)) * (8u * UP), u + pf.off - 2, lane0);
        if (plane_start) {
          const unsigned sp = (unsigned)(pf.p & (RP - 1)) * 256u;
          cp16cgp(sUP16 + sp, u + pf.off - g.s1 + 2 * lane, l16);
          cp16p(sDN16 + sp, u + pf.off + (int64_t)R * g.s1 + 2 * lane, l16);
        }
      }
      pf.next(R, s1, wrap, mrow, mwrap);
      cp_commit();
      cp_wait<PFF>();
      __syncwarp();

      // ---------------- compute: lane j on line t - j (branch-free) --------
      {
        const int nl = t - lane;
        const bool valid = kval && nl >= 0 && nl < nLines;
        const int su = nl & (RLU - 1);
        const int sf = nl & (RLF - 1);
        const double* row = S.u[su];
        const double hf = h2 * S.f[sf][lane] + 0.0;  // (h2 f + 0) + S == h2 f + (S + 0)
        const double a0m = S.u[(nl - R) & (RLU - 1)][lane + 2];
        const double a0p = S.u[(nl + R) & (RLU - 1)][lane + 2];
        const double old = row[lane + 2];
        const double kp = row[lane + 3];
        const double km = row[lane + 1];  // new: lane j-1 wrote it last step (lane 0: halo)
        double s;
        if (DIM == 3) {
          const int sp = cp & (RP - 1);
          const double rm = cr > 0 ? prev : S.up[sp][lane];
          const double rp = cr < R - 1 ? S.u[(nl + 1) & (RLU - 1)][lane + 2] : S.dn[sp][lane];
          s = ((((a0m + a0p) + rm) + rp) + km) + kp;
        } else {
          s = ((a0m + a0p) + km) + kp;
        }
        const double val = (hf + s) * inv;
        const bool internal = (S.mask[sf] >> lane) & 1u;
        const double mine = (valid && internal) ? val : old;
        if (valid) S.u[su][lane + 2] = mine;
        prev = mine;
        const bool w = ++cr == R;
        cr = w ? 0 : cr;
        cp += w;
      }
      __syncwarp();

      // ---------------- write back the line lane 31 just finished ---------
      if (pd.L >= 0 && pd.L < nLines) {
        if (l16) {
          const double2 v = *reinterpret_cast<const double2*>(&S.u[pd.L & (RLU - 1)][2 + 2 * lane]);
          *reinterpret_cast<double2*>(u + pd.off + 2 * lane) = v;
        }
        if ((pd.L & 15) == 15 || pd.L == nLines - 1) {
          __syncwarp();
          if (lane0) st_release(myprog, pd.L + 1);
        }
      }
      pd.next(R, s1, wrap, mrow, mwrap);
    }
    cp_wait<0>();
    __syncwarp();
  }
}

size_t gs_stream_smem_per_warp() { return sizeof(WarpRing); }

void configure_gs_diag();
void configure_dense_gemv();

void configure_gs_kernels() {
  const int smem = (int)sizeof(WarpRing);  // one warp per CTA
  cudaFuncSetAttribute(gs_stream_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gs_stream_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  configure_gs_diag();
  configure_gs_chain();
  configure_dense_gemv();
}

void launch_gs_stream(const GsArgs& a, int grid, int warps_per_cta, cudaStream_t st) {
  const size_t smem = sizeof(WarpRing) * warps_per_cta;
  if (a.g.d == 3)
    gs_stream_kernel<3><<<grid, 32 * warps_per_cta, smem, st>>>(a);
  else
    gs_stream_kernel<2><<<grid, 32 * warps_per_cta, smem, st>>>(a);
}

}  // namespace gmg
