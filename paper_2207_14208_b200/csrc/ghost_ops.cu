// ghost_ops.cu -- ghost-row kernels on sm_100a: the batched lexicographic
// ghost relaxation, the ghost residual and the masked ghost restriction.
//
// Ghost data live in "slot" order: ghosts sorted by sweep batch (see
// transfer.ghost_dag_levels), lexicographic inside a batch.  Weights are
// stored [m][ng] so a warp reading one stencil entry for 32 ghosts is one
// coalesced load.
#include <algorithm>

#include "gmg_kernels.cuh"

namespace gmg {

template <int D>
__device__ __forceinline__ int64_t block_offset(const Geom& g, int j) {
  if constexpr (D == 3) {
    return (int64_t)(j / 9) * g.s0 + (int64_t)((j / 3) % 3) * g.s1 + (j % 3);
  } else {
    return (int64_t)(j / 3) * g.s0 + (j % 3);
  }
}

// One batch of the ghost sweep (reference smoothing.py:135-142):
// u_G += dtau * (g - ddot(w, u[block])).  No ghost of a batch reads another
// ghost of the same batch, so the batch is one parallel step.
template <int D>
__global__ void __launch_bounds__(256) ghost_batch_kernel(GhostArgs a, double* __restrict__ u,
                                                          int64_t lo, int64_t hi) {
  constexpr int M = D == 3 ? 27 : 9;
  const int64_t s = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= hi) return;
  const int64_t node = a.node[s];
  if (node < 0) return;
  const int64_t base = a.base[s];
  double x[M], y[M];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    x[j] = __ldg(a.w + (int64_t)j * a.ng + s);
    y[j] = u[base + block_offset<D>(a.g, j)];
  }
  const double dot = blas_ddot<M>(x, y);
  u[node] = u[node] + a.dtau[s] * (a.gval[s] - dot);
}

__device__ __forceinline__ int ld_acquire_i(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_i(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// The whole ghost sweep in one launch, ordered by the sweep DAG instead of
// batch barriers: warps claim 32-slot chunks in slot order (batch, lex); a
// ghost waits (acquire) on the done flags of exactly the earlier ghosts it
// reads or that read it, relaxes, stores, and releases its own flag.  Every
// dependency lies in an earlier batch, hence an earlier chunk already held by
// a running warp, so the sweep cannot deadlock, and each ghost sees the same
// values as in the reference's lexicographic loop.  flags[nslots] is the
// chunk cursor; all flags are zeroed before the launch.
template <int D>
__global__ void __launch_bounds__(256) ghost_persistent_kernel(GhostArgs a, double* __restrict__ u,
                                                               const int32_t* __restrict__ dep_off,
                                                               const int32_t* __restrict__ dep, int* flags) {
  constexpr int M = D == 3 ? 27 : 9;
  const int lane = threadIdx.x & 31;
  const int64_t nchunks = a.ng / 32;
  for (;;) {
    int chunk = 0;
    if (lane == 0) chunk = atomicAdd(&flags[a.ng], 1);
    chunk = __shfl_sync(0xffffffffu, chunk, 0);
    if (chunk >= nchunks) return;
    const int64_t s = (int64_t)chunk * 32 + lane;
    const int64_t node = a.node[s];
    if (node >= 0) {
      const int64_t base = a.base[s];
      double x[M], y[M];
#pragma unroll
      for (int j = 0; j < M; ++j) x[j] = __ldg(a.w + (int64_t)j * a.ng + s);
      const double gv = a.gval[s], dt = a.dtau[s];
      const int d1 = dep_off[s + 1];
      for (int k = dep_off[s]; k < d1; ++k) {
        const int* f = flags + dep[k];
        while (ld_acquire_i(f) == 0) {
        }
      }
#pragma unroll
      for (int j = 0; j < M; ++j) y[j] = __ldcg(u + base + block_offset<D>(a.g, j));
      const double dot = blas_ddot<M>(x, y);
      __stcg(u + node, __ldcg(u + node) + dt * (gv - dot));
      st_release_i(flags + s, 1);
    }
  }
}

void launch_ghost_persistent(const GhostArgs& a, double* u, const int32_t* dep_off, const int32_t* dep, int* flags,
                             int sms, cudaStream_t st) {
  const int64_t warps = a.ng / 32;
  int blocks = (int)std::min<int64_t>((warps + 7) / 8, (int64_t)sms * 8);
  if (blocks < 1) blocks = 1;
  if (a.g.d == 3)
    ghost_persistent_kernel<3><<<blocks, 256, 0, st>>>(a, u, dep_off, dep, flags);
  else
    ghost_persistent_kernel<2><<<blocks, 256, 0, st>>>(a, u, dep_off, dep, flags);
}


void launch_ghost_batch(const GhostArgs& a, double* u, int64_t lo, int64_t hi, cudaStream_t st) {
  if (hi <= lo) return;
  const int threads = 256;
  const int64_t blocks = (hi - lo + threads - 1) / threads;
  if (a.g.d == 3)
    ghost_batch_kernel<3><<<(unsigned)blocks, threads, 0, st>>>(a, u, lo, hi);
  else
    ghost_batch_kernel<2><<<(unsigned)blocks, threads, 0, st>>>(a, u, lo, hi);
}

__device__ __forceinline__ void block_max_commit(double v, unsigned long long* maxbits) {
  if (!maxbits) return;
  __shared__ double part[32];
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) part[w] = v;
  __syncthreads();
  if (w == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    double x = l < nw ? part[l] : 0.0;
    x = warp_max(x);
    if (l == 0) atomic_max_nonneg(maxbits, x);
  }
}

// Ghost residual (smoothing.py:120-124): r_g = g - pairwise(w * u[block]),
// scattered to r_ext at the ghost node; optional max |r_g|.
template <int D>
__global__ void __launch_bounds__(256) residual_ghost_kernel(GhostArgs a, const double* __restrict__ u,
                                                             double* __restrict__ r_ext,
                                                             unsigned long long* maxbits) {
  constexpr int M = D == 3 ? 27 : 9;
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double am = 0.0;
  if (s < a.ng && a.node[s] >= 0) {
    const int64_t base = a.base[s];
    double p[M];
#pragma unroll
    for (int j = 0; j < M; ++j) p[j] = __ldg(a.w + (int64_t)j * a.ng + s) * u[base + block_offset<D>(a.g, j)];
    const double r = a.gval[s] - np_sum<M>(p);
    r_ext[a.node[s]] = r;
    am = fabs(r);
  }
  block_max_commit(am, maxbits);
}

void launch_residual_ghost(const GhostArgs& a, const double* u, double* r_ext,
                           unsigned long long* maxbits, cudaStream_t st) {
  if (a.ng == 0) return;
  const int threads = 256;
  const int64_t blocks = (a.ng + threads - 1) / threads;
  if (a.g.d == 3)
    residual_ghost_kernel<3><<<(unsigned)blocks, threads, 0, st>>>(a, u, r_ext, maxbits);
  else
    residual_ghost_kernel<2><<<(unsigned)blocks, threads, 0, st>>>(a, u, r_ext, maxbits);
}

// Full-weighting row entry e of a 3^D block, ((1*a)*b)*c.
template <int D>
__device__ __forceinline__ double fw_entry(int e) {
  double v = 1.0;
  int o[3];
  int rem = e;
#pragma unroll
  for (int k = D - 1; k >= 0; --k) {
    o[k] = rem % 3;
    rem /= 3;
  }
#pragma unroll
  for (int k = 0; k < D; ++k) v = v * (o[k] == 1 ? 0.5 : 0.25);
  return v;
}

// GhostRestriction (transfer.py:96-121) for every coarse ghost slot:
// keep = in-box and (ghost or inactive) on the fine grid, w = FW*keep /
// pairwise(FW*keep), value = pairwise(w * r_ext[clamped block]); promoted
// coarse ghosts get 0 (solver.py:189).
template <int D>
__global__ void __launch_bounds__(256) restrict_ghost_kernel(Geom gf, const uint8_t* __restrict__ lab_f,
                                                             const double* __restrict__ r_ext,
                                                             GhostArgs c, double* __restrict__ gval_c) {
  constexpr int M = D == 3 ? 27 : 9;
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= c.ng) return;
  if (c.promoted[s] || c.node[s] < 0) {
    gval_c[s] = 0.0;
    return;
  }
  int64_t mc[3];
  pos_multi(c.g, c.node[s], mc);
  double w[M];
  int64_t blk[M];
#pragma unroll
  for (int e = 0; e < M; ++e) {
    int rem = e, o[3];
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
      o[k] = rem % 3;
      rem /= 3;
    }
    bool valid = true;
    int64_t mf[3];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      int64_t x = 2 * mc[k] + o[k] - 1;
      if (x < 0 || x > gf.N) valid = false;
      mf[k] = x < 0 ? 0 : (x > gf.N ? gf.N : x);
    }
    const int64_t flat = multi_pos(gf, mf);
    blk[e] = flat;
    const uint8_t L = lab_f[flat];
    const bool keep = valid && (L == GHOST || L == INACTIVE);
    w[e] = fw_entry<D>(e) * (keep ? 1.0 : 0.0);
  }
  const double sum = np_sum<M>(w);
  double p[M];
#pragma unroll
  for (int e = 0; e < M; ++e) p[e] = (w[e] / sum) * r_ext[blk[e]];
  gval_c[s] = np_sum<M>(p);
}

void launch_restrict_ghost(const Geom& gf, const uint8_t* lab_f, const double* r_ext,
                           const GhostArgs& coarse, double* gval_c, cudaStream_t st) {
  if (coarse.ng == 0) return;
  const int threads = 256;
  const int64_t blocks = (coarse.ng + threads - 1) / threads;
  if (gf.d == 3)
    restrict_ghost_kernel<3><<<(unsigned)blocks, threads, 0, st>>>(gf, lab_f, r_ext, coarse, gval_c);
  else
    restrict_ghost_kernel<2><<<(unsigned)blocks, threads, 0, st>>>(gf, lab_f, r_ext, coarse, gval_c);
}

}  // namespace gmg
