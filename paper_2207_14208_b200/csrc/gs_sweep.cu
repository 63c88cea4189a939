// gs_sweep.cu -- exact lexicographic Gauss-Seidel sweep over the internal
// nodes on sm_100a.
//
// Reference: gs_lex_sweep, /root/reference/pkg/src/ghostmg/smoothing.py:127-132
// (an anti-diagonal wavefront that equals the sequential lexicographic
// sweep value for value):  u_i <- (h^2 f_i + S_i) * (1/denom),
// S_i = ((((u[i-s0] + u[i+s0]) + u[i-s1]) + u[i+s1]) + u[i-s2]) + u[i+s2].
//
// Any update order that is a linear extension of "i before i + s_k" gives
// the lexicographic result.  The sweep is cut into warp tasks: a task owns
// a 32-wide chunk of the fastest axis (one column per lane) and, in 3-D, a
// block of B1 rows of axis 1, and walks every line (i0, i1) of its block in
// lexicographic order.  Lane j runs one line behind lane j-1 (a skew of one
// line per lane), so the value of (line, k-1) arrives from lane j-1 by a
// register shuffle one step after it was computed: the dependent chain per
// step is one shuffle plus the four ops (+u[k-1], +u[k+1], h^2 f +, *inv).
//
// Tasks depend on their left (chunk c-1) and upper (block b-1) neighbours;
// each publishes the number of completed lines in a progress word
// (st.release.gpu) and readers spin with ld.acquire.gpu.  Tasks are handed
// out through an atomic ticket in wavefront (c + b) order, so a task only
// ever waits on tasks already running: no co-residency requirement and no
// deadlock.  Values produced by other tasks are read with ld.global.cg (L2),
// never from a possibly stale L1 line.
#include "gmg_kernels.cuh"

namespace gmg {

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ double ld_l2(const double* p) { return __ldcg(p); }

template <int DIM>
__global__ void __launch_bounds__(128) gs_sweep_kernel(GsArgs a) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const Geom g = a.g;
  const int64_t N = g.N;
  double* __restrict__ u = a.u;
  const double* __restrict__ f = a.f;
  const uint8_t* __restrict__ labels = a.labels;

  for (;;) {
    int tid = 0;
    if (lane == 0) tid = atomicAdd(a.ticket, 1);
    tid = __shfl_sync(FULL, tid, 0);
    if (tid >= a.ntasks) return;
    const int2 tk = a.tasks[tid];
    const int c = tk.x, b = tk.y;
    const int64_t k = 1 + 32 * (int64_t)c + lane;
    const bool kval = k <= N - 1;
    const int R = DIM == 3 ? (int)min((int64_t)a.B1, N - 1 - (int64_t)b * a.B1) : 1;
    const int nLines = (int)(N - 1) * R;
    int* myprog = a.progress + c * a.Bn + b;
    const int* lprog = c > 0 ? a.progress + (c - 1) * a.Bn + b : nullptr;
    const int* uprog = (DIM == 3 && b > 0) ? a.progress + c * a.Bn + (b - 1) : nullptr;
    int seenL = 0, seenU = 0;  // lane 0's cache of the neighbours' progress
    double mine = 0.0, prev = 0.0;
    const int last = nLines + 30;
    for (int t = 0; t <= last; ++t) {
      const int nl = t - lane;
      const bool act = kval && nl >= 0 && nl < nLines;
      const double left = __shfl_up_sync(FULL, mine, 1);
      // dependencies of this step (warp-uniform wait by lane 0)
      int needL = 0, needU = 0;
      int p = 0, r = 0;
      if (nl >= 0 && nl < nLines) {
        p = nl / R;
        r = nl - p * R;
        if (lane == 0 && lprog) needL = nl + 1;
        if (DIM == 3 && uprog && r == 0) needU = (p + 1) * a.B1;
      }
      if (DIM == 3) needU = __reduce_max_sync(FULL, needU);
      if (lane == 0) {
        while (seenL < needL) seenL = ld_acquire(lprog);
        if (DIM == 3)
          while (seenU < needU) seenU = ld_acquire(uprog);
      }
      __syncwarp();
      if (act) {
        int64_t node;
        if (DIM == 3) {
          const int64_t i0 = p + 1, i1 = 1 + (int64_t)b * a.B1 + r;
          node = i0 * g.s0 + i1 * g.s1 + k + OFF;
        } else {
          node = (int64_t)(nl + 1) * g.s0 + k + OFF;
        }
        if (labels[node] == INTERNAL) {
          double s;
          const double fv = __ldg(f + node);
          if (DIM == 3) {
            const double a0m = u[node - g.s0];  // own task (previous plane) or boundary
            const double a0p = u[node + g.s0];
            const double a1m = r > 0 ? prev : ld_l2(u + node - g.s1);
            const double a1p = u[node + g.s1];
            const double a2m = lane > 0 ? left : ld_l2(u + node - 1);
            const double a2p = u[node + 1];
            s = ((((a0m + a0p) + a1m) + a1p) + a2m) + a2p;
          } else {
            const double a0m = nl > 0 ? prev : u[node - g.s0];
            const double a0p = u[node + g.s0];
            const double a1m = lane > 0 ? left : ld_l2(u + node - 1);
            const double a1p = u[node + 1];
            s = ((a0m + a0p) + a1m) + a1p;
          }
          s = s + 0.0;
          mine = (g.h2 * fv + s) * g.inv;
          u[node] = mine;
        } else {
          mine = u[node];
        }
        prev = mine;
      }
      if (t >= 31 && (((t - 31) & 7) == 7 || t == last)) {
        __syncwarp();
        if (lane == 0) st_release(myprog, t - 30);
      }
    }
  }
}

void launch_gs_sweep(const GsArgs& a, int grid, cudaStream_t st) {
  if (a.g.d == 3)
    gs_sweep_kernel<3><<<grid, 128, 0, st>>>(a);
  else
    gs_sweep_kernel<2><<<grid, 128, 0, st>>>(a);
}

}  // namespace gmg
