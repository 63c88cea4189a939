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
#include "gmg_kernels.cuh"

namespace gmg {

namespace {

constexpr int RLU = 128;  // u ring lines
constexpr int RLF = 64;   // f ring lines
constexpr int RP = 8;     // plane-row ring (3-D)
constexpr int PFU = 64;   // u prefetch distance (lines)
constexpr int PFF = 32;   // f / halo prefetch distance (lines)

struct __align__(16) WarpRing {
  double u[RLU][32];
  double f[RLF][32];
  double up[RP][34];  // row above the block (16-B aligned superset), new values
  double dn[RP][32];  // row below the block, old values
  double hr[RLU];     // old right halo k0+32
  double hl[RLF][2];  // new left halo k0-1 (16-B aligned pair)
  uint32_t mask[RLF];
};

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp16cg(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
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

// line L of a task -> (plane p, row r), for L >= -R (p = -1 is the boundary
// plane i0 = 0, p = P the boundary plane i0 = N).
struct LinePos {
  int p, r;
  __device__ void init(int L, int R) {
    p = L >= 0 ? L / R : -((-L + R - 1) / R);  // floor(L / R)
    r = L - p * R;
  }
  __device__ void next(int R) {
    if (++r == R) {
      r = 0;
      ++p;
    }
  }
};

}  // namespace

template <int DIM>
__global__ void __launch_bounds__(128, 1) gs_stream_kernel(GsArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  WarpRing& S = reinterpret_cast<WarpRing*>(smem_raw)[threadIdx.x >> 5];
  const Geom g = a.g;
  const int N = (int)g.N;
  double* __restrict__ u = a.u;
  const double* __restrict__ f = a.f;

  for (;;) {
    int tid = 0;
    if (lane == 0) tid = atomicAdd(a.ticket, 1);
    tid = __shfl_sync(FULL, tid, 0);
    if (tid >= a.ntasks) return;
    const int2 tk = a.tasks[tid];
    const int c = tk.x, b = tk.y;
    const int k0 = 1 + 32 * c;
    const int k = k0 + lane;
    const bool kval = k <= N - 1;
    const int R = DIM == 3 ? min(a.B1, N - 1 - b * a.B1) : 1;
    const int nLines = (N - 1) * R;
    const int uEnd = nLines + R;  // u lines run over [-R, nLines + R)
    const int rowbase = DIM == 3 ? 1 + b * a.B1 : 0;
    int* myprog = a.progress + c * a.Bn + b;
    const int* lprog = c > 0 ? a.progress + (c - 1) * a.Bn + b : nullptr;
    const int* uprog = (DIM == 3 && b > 0) ? a.progress + c * a.Bn + (b - 1) : nullptr;
    int seenL = 0, seenU = 0;

    auto line_node = [&](int p, int r) -> int64_t {
      if (DIM == 3) return (int64_t)(p + 1) * g.s0 + (int64_t)(rowbase + r) * g.s1 + k0;
      return (int64_t)(p + 1) * g.s0 + k0;
    };
    auto line_mask = [&](int p, int r) -> int64_t {
      if (DIM == 3) return ((int64_t)(p + 1) * g.n + rowbase + r) * a.C + c;
      return (int64_t)(p + 1) * a.C + c;
    };

    const int t0 = -(PFU + R);
    LinePos pu, pf, pc;   // prefetch-u, prefetch-f, compute (this lane's line)
    pu.init(t0 + PFU, R);
    pf.init(t0 + PFF, R);
    pc.init(t0 - lane, R);
    double mine = 0.0, prev = 0.0;
    const int last = nLines + 30;

    for (int t = t0; t <= last; ++t) {
      // ---------------- prefetch (one commit group per step) --------------
      const int Lu = t + PFU;
      if (Lu >= -R && Lu < uEnd) {
        const int64_t n0 = line_node(pu.p, pu.r);
        const int su = Lu & (RLU - 1);
        if (k0 + lane <= N) cp8(&S.u[su][lane], u + n0 + lane);
        if (lane == 0 && k0 + 32 <= N) cp8(&S.hr[su], u + n0 + 32);
      }
      const int Lf = t + PFF;
      if (Lf >= 0 && Lf < nLines) {
        const int64_t n0 = line_node(pf.p, pf.r);
        const int sf = Lf & (RLF - 1);
        if (k0 + lane <= N - 1) cp8(&S.f[sf][lane], f + n0 + lane);
        if (lane == 0) {
          cp4(&S.mask[sf], a.imask + line_mask(pf.p, pf.r));
          if (lprog)
            while (seenL < Lf + 1) seenL = ld_acquire(lprog);
          if (DIM == 3 && uprog && pf.r == 0) {
            const int need = (pf.p + 1) * a.B1;
            while (seenU < need) seenU = ld_acquire(uprog);
          }
        }
        __syncwarp();
        if (lane == 0) cp16cg(&S.hl[sf][0], u + ((n0 - 1) & ~(int64_t)1));
        if (DIM == 3 && pf.r == 0) {
          const int sp = pf.p & (RP - 1);
          const int64_t up0 = n0 - g.s1;  // row rowbase - 1, column k0
          const int64_t upa = up0 & ~(int64_t)1;
          if (lane < 17) cp16cg(&S.up[sp][2 * lane], u + upa + 2 * lane);
          const int64_t dn0 = n0 + (int64_t)R * g.s1;  // row rowbase + R
          if (k0 + lane <= N) cp8(&S.dn[sp][lane], u + dn0 + lane);
        }
      }
      cp_commit();
      pu.next(R);
      pf.next(R);
      cp_wait<PFF>();
      __syncwarp();

      // ---------------- compute: lane j on line t - j ----------------------
      const int nl = t - lane;
      const double left = __shfl_up_sync(FULL, mine, 1);
      if (nl >= 0 && nl < nLines && kval) {
        const int su = nl & (RLU - 1);
        const int sf = nl & (RLF - 1);
        const double old = S.u[su][lane];
        if ((S.mask[sf] >> lane) & 1u) {
          const double fv = S.f[sf][lane];
          const double a0m = S.u[(nl - R) & (RLU - 1)][lane];
          const double a0p = S.u[(nl + R) & (RLU - 1)][lane];
          double kp = lane < 31 ? S.u[su][lane + 1] : S.hr[su];
          double km = left;
          if (lane == 0) {
            const int64_t e = line_node(pc.p, pc.r) - 1;
            km = S.hl[sf][(int)(e & 1)];
          }
          double s;
          if (DIM == 3) {
            double rm, rp;
            const int sp = pc.p & (RP - 1);
            if (pc.r > 0) {
              rm = prev;
            } else {
              const int64_t up0 = line_node(pc.p, 0) - g.s1;
              rm = S.up[sp][(int)(up0 & 1) + lane];
            }
            rp = pc.r < R - 1 ? S.u[(nl + 1) & (RLU - 1)][lane] : S.dn[sp][lane];
            s = ((((a0m + a0p) + rm) + rp) + km) + kp;
          } else {
            s = ((a0m + a0p) + km) + kp;
          }
          s = s + 0.0;
          mine = (g.h2 * fv + s) * g.inv;
          S.u[su][lane] = mine;
        } else {
          mine = old;
        }
        prev = mine;
      }
      pc.next(R);
      __syncwarp();

      // ---------------- write back the line lane 31 finished --------------
      const int Ld = t - 31;
      if (Ld >= 0 && Ld < nLines) {
        LinePos pd;
        pd.init(Ld, R);
        const int64_t n0 = line_node(pd.p, pd.r);
        if (kval) u[n0 + lane] = S.u[Ld & (RLU - 1)][lane];
        if (((Ld & 7) == 7) || Ld == nLines - 1) {
          __syncwarp();
          if (lane == 0) st_release(myprog, Ld + 1);
        }
      }
    }
    cp_wait<0>();
    __syncwarp();
  }
}

size_t gs_stream_smem_per_warp() { return sizeof(WarpRing); }

void launch_gs_stream(const GsArgs& a, int grid, int warps_per_cta, cudaStream_t st) {
  const size_t smem = sizeof(WarpRing) * warps_per_cta;
  static bool configured[2] = {false, false};
  if (a.g.d == 3) {
    if (!configured[1]) {
      cudaFuncSetAttribute(gs_stream_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      configured[1] = true;
    }
    gs_stream_kernel<3><<<grid, 32 * warps_per_cta, smem, st>>>(a);
  } else {
    if (!configured[0]) {
      cudaFuncSetAttribute(gs_stream_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      configured[0] = true;
    }
    gs_stream_kernel<2><<<grid, 32 * warps_per_cta, smem, st>>>(a);
  }
}

}  // namespace gmg
