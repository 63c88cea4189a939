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
__device__ __forceinline__ void st_pair(double* p, double v);

template <int D>
__global__ void __launch_bounds__(256) ghost_batch_kernel(GhostArgs a, double* __restrict__ u,
                                                          int64_t lo, int64_t hi, double* pair) {
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
  const double nv = u[node] + a.dtau[s] * (a.gval[s] - dot);
  u[node] = nv;
  if (pair) st_pair(pair + 2 * s, nv);  // for DAG-ordered successors (ghost_persistent_kernel)
}

// (value, done tag) pairs: written with one 16-byte store, read with one
// 16-byte load through L2 -- the value travels with its flag, so neither side
// needs a memory barrier (gpu-scope release/acquire would drain the SM's
// memory pipeline / flush its L1 on every ghost).
__device__ __forceinline__ double2 ld_pair(const double* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_pair(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v), "d"(1.0) : "memory");
}
__device__ __forceinline__ double wait_pair(const double* p, int backoff) {
  double2 v = ld_pair(p);
  while (v.y == 0.0) {
    if (backoff) __nanosleep(backoff);
    v = ld_pair(p);
  }
  return v.x;
}

#ifndef GHOST_MINB
#define GHOST_MINB 2
#endif
// The whole ghost sweep in one launch, ordered by the sweep DAG instead of
// batch barriers: warps claim 32-slot chunks in slot order (batch, lex).  A
// ghost prefetches its weights and all 3^d stencil values, then takes the
// new value of every earlier ghost it reads (vmask, in stencil order) from
// that ghost's (value, tag) pair as soon as the tag is set, waits for the
// earlier ghosts that read its own old value, relaxes, and publishes its new
// value in u and in its pair.  Every dependency lies in an earlier batch,
// hence an earlier chunk already held by a running warp, so the sweep cannot
// deadlock, and each ghost sees the same values as in the reference's
// lexicographic loop.  Pairs and the chunk cursor are zeroed before the launch.
template <int D>
__global__ void __launch_bounds__(256, GHOST_MINB) ghost_persistent_kernel(GhostArgs a, double* __restrict__ u,
                                                               const int32_t* __restrict__ dep_off,
                                                               const int32_t* __restrict__ dep,
                                                               const uint32_t* __restrict__ vmask,
                                                               double* pair, int* cursor, int backoff,
                                                               long long* gtrace, bool defer) {
  constexpr int M = D == 3 ? 27 : 9;
  const int lane = threadIdx.x & 31;
  const int64_t nchunks = a.ng / 32;
  for (;;) {
    int chunk = 0;
    if (lane == 0) chunk = atomicAdd(cursor, 1);
    chunk = __shfl_sync(0xffffffffu, chunk, 0);
    if (chunk >= nchunks) return;
    const int64_t s = (int64_t)chunk * 32 + lane;
    const int64_t node = a.node[s];
    long long tg0 = 0, tg1 = 0;
    if (gtrace) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tg0));
    if (node >= 0) {
      const int64_t base = a.base[s];
      // the row weights go to shared memory by cp.async (in flight during the
      // wait, no registers held); the block values stay in registers
      extern __shared__ double wsm[];  // [M][blockDim.x]
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const unsigned dst = (unsigned)__cvta_generic_to_shared(&wsm[j * blockDim.x + threadIdx.x]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(a.w + (int64_t)j * a.ng + s)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      double y[M];
#pragma unroll
      for (int j = 0; j < M; ++j) y[j] = __ldcg(u + base + block_offset<D>(a.g, j));
      const double gv = a.gval[s], dt = a.dtau[s], uo = __ldcg(u + node);
      const uint32_t vm = vmask[s];
      const int k0 = dep_off[s];
      const int d1 = dep_off[s + 1];
      // all dependency pairs are (re)loaded together each round -- one L2
      // round trip per round -- until every tag is set
      {
        constexpr int WMAX = 8;  // wait-only dependencies polled together
        const int nv = __popc(vm);
        const int kw = k0 + nv, nw = min(d1 - kw, WMAX);
        for (;;) {
          double tg[M], wt[WMAX];
          int k = k0;
#pragma unroll
          for (int j = 0; j < M; ++j) {
            tg[j] = 1.0;
            if ((vm >> j) & 1u) {
              const double2 pv = ld_pair(pair + 2 * (int64_t)dep[k++]);
              y[j] = pv.x;
              tg[j] = pv.y;
            }
          }
#pragma unroll
          for (int q = 0; q < WMAX; ++q) wt[q] = q < nw ? ld_pair(pair + 2 * (int64_t)dep[kw + q]).y : 1.0;
          bool all = true;
#pragma unroll
          for (int j = 0; j < M; ++j) all = all && tg[j] != 0.0;
#pragma unroll
          for (int q = 0; q < WMAX; ++q) all = all && wt[q] != 0.0;
          if (all) break;
          if (backoff) __nanosleep(backoff);
        }
        for (int k = kw + WMAX; k < d1; ++k) wait_pair(pair + 2 * (int64_t)dep[k], backoff);
      }
      if (gtrace) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tg1));
      asm volatile("cp.async.wait_all;" ::: "memory");
      double x[M];
#pragma unroll
      for (int j = 0; j < M; ++j) x[j] = wsm[j * blockDim.x + threadIdx.x];
      const double dot = blas_ddot<M>(x, y);
      const double nv = uo + dt * (gv - dot);
      if (!defer) __stcg(u + node, nv);  // defer: u keeps the old value until the write-back
      st_pair(pair + 2 * s, nv);
    }
    if (gtrace) {
      long long tg2;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tg2));
      gtrace[3 * s] = tg0;
      gtrace[3 * s + 1] = tg1;
      gtrace[3 * s + 2] = tg2;
    }
  }
}

// Level-synchronous variant: one CTA per SM walks the sweep batches (DAG
// levels) in order; the CTAs split each batch's slots, then meet at a
// grid-wide counter (one polling thread per CTA, with back-off) before the
// next batch.  Values of earlier ghosts still come from their (value, tag)
// pairs -- the counter only throttles polling (its increments need no fence:
// a pair that is not visible yet is simply waited for).
template <int D>
__global__ void __launch_bounds__(1024) ghost_levels_kernel(GhostArgs a, double* __restrict__ u,
                                                            const int64_t* __restrict__ boff, int nbatch,
                                                            const int32_t* __restrict__ dep_off,
                                                            const int32_t* __restrict__ dep,
                                                            const uint32_t* __restrict__ vmask, double* pair,
                                                            int* counter) {
  constexpr int M = D == 3 ? 27 : 9;
  for (int b = 0; b < nbatch; ++b) {
    const int64_t lo = boff[b], hi = boff[b + 1];
    for (int64_t s = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < hi;
         s += (int64_t)gridDim.x * blockDim.x) {
      const int64_t node = a.node[s];
      if (node < 0) continue;
      const int64_t base = a.base[s];
      double x[M], y[M];
#pragma unroll
      for (int j = 0; j < M; ++j) {
        x[j] = __ldg(a.w + (int64_t)j * a.ng + s);
        y[j] = __ldcg(u + base + block_offset<D>(a.g, j));
      }
      const double gv = a.gval[s], dt = a.dtau[s], uo = __ldcg(u + node);
      const uint32_t vm = vmask[s];
      int k = dep_off[s];
#pragma unroll
      for (int j = 0; j < M; ++j)
        if ((vm >> j) & 1u) y[j] = wait_pair(pair + 2 * (int64_t)dep[k++], 0);
      const double dot = blas_ddot<M>(x, y);
      const double nv = uo + dt * (gv - dot);
      __stcg(u + node, nv);
      st_pair(pair + 2 * s, nv);
    }
    if (b + 1 == nbatch) break;
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd(counter, 1);
      const int target = (b + 1) * (int)gridDim.x;
      int v;
      for (;;) {
        asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        if (v >= target) break;
        __nanosleep(64);
      }
    }
    __syncthreads();
  }
}

void launch_ghost_levels(const GhostArgs& a, double* u, const int64_t* boff, int nbatch, const int32_t* dep_off,
                         const int32_t* dep, const uint32_t* vmask, double* pair, int* counter, int sms,
                         cudaStream_t st) {
  if (a.g.d == 3)
    ghost_levels_kernel<3><<<sms, 1024, 0, st>>>(a, u, boff, nbatch, dep_off, dep, vmask, pair, counter);
  else
    ghost_levels_kernel<2><<<sms, 1024, 0, st>>>(a, u, boff, nbatch, dep_off, dep, vmask, pair, counter);
}

void launch_ghost_persistent(const GhostArgs& a, double* u, const int32_t* dep_off, const int32_t* dep,
                             const uint32_t* vmask, double* pair, int* cursor, int sms, int blocks_per_sm,
                             int backoff, long long* gtrace, bool defer, cudaStream_t st) {
  const int64_t warps = a.ng / 32;
  int blocks = (int)std::min<int64_t>((warps + 7) / 8, (int64_t)sms * blocks_per_sm);
  if (blocks < 1) blocks = 1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ghost_persistent_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(27 * 256 * sizeof(double)));
    cudaFuncSetAttribute(ghost_persistent_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(9 * 256 * sizeof(double)));
    attr = true;
  }
  if (a.g.d == 3)
    ghost_persistent_kernel<3><<<blocks, 256, 27 * 256 * sizeof(double), st>>>(a, u, dep_off, dep, vmask, pair, cursor,
                                                                               backoff, gtrace, defer);
  else
    ghost_persistent_kernel<2><<<blocks, 256, 9 * 256 * sizeof(double), st>>>(a, u, dep_off, dep, vmask, pair, cursor,
                                                                              backoff, gtrace, defer);
}



// Write-back of a deferred sweep: u[ghost] = its new value from the pairs.
__global__ void ghost_writeback_kernel(GhostArgs a, const double* __restrict__ pair, double* __restrict__ u) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= a.ng) return;
  const int64_t node = a.node[s];
  if (node >= 0) u[node] = pair[2 * s];
}

void launch_ghost_writeback(const GhostArgs& a, const double* pair, double* u, cudaStream_t st) {
  if (a.ng > 0) ghost_writeback_kernel<<<(unsigned)((a.ng + 255) / 256), 256, 0, st>>>(a, pair, u);
}

void launch_ghost_batch(const GhostArgs& a, double* u, int64_t lo, int64_t hi, double* pair, cudaStream_t st) {
  if (hi <= lo) return;
  const int threads = 256;
  const int64_t blocks = (hi - lo + threads - 1) / threads;
  if (a.g.d == 3)
    ghost_batch_kernel<3><<<(unsigned)blocks, threads, 0, st>>>(a, u, lo, hi, pair);
  else
    ghost_batch_kernel<2><<<(unsigned)blocks, threads, 0, st>>>(a, u, lo, hi, pair);
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
    if (r_ext) r_ext[a.node[s]] = r;
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

// Same residual over the ghosts in lexicographic order (weights, bases and
// nodes stored in that order; the right-hand side stays in slot order).
template <int D>
__global__ void __launch_bounds__(256) residual_ghost_lex_kernel(GhostArgs a, const double* __restrict__ wl,
                                                                 const int64_t* __restrict__ basel,
                                                                 const int64_t* __restrict__ nodel,
                                                                 const int32_t* __restrict__ l2s, int64_t ng,
                                                                 const double* __restrict__ u,
                                                                 double* __restrict__ r_ext,
                                                                 unsigned long long* maxbits, int64_t i0, int64_t i1) {
  constexpr int M = D == 3 ? 27 : 9;
  const int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double am = 0.0;
  if (i < i1) {
    const int64_t base = basel[i];
    double p[M];
#pragma unroll
    for (int j = 0; j < M; ++j) p[j] = __ldg(wl + (int64_t)j * ng + i) * u[base + block_offset<D>(a.g, j)];
    const double r = a.gval[l2s[i]] - np_sum<M>(p);
    if (r_ext) r_ext[nodel[i]] = r;
    am = fabs(r);
  }
  block_max_commit(am, maxbits);
}

void launch_residual_ghost_lex(const GhostArgs& a, const double* wl, const int64_t* basel, const int64_t* nodel,
                               const int32_t* l2s, int64_t ng, const double* u, double* r_ext,
                               unsigned long long* maxbits, int64_t i0, int64_t i1, cudaStream_t st) {
  if (i1 <= i0) return;
  const int64_t blocks = (i1 - i0 + 255) / 256;
  if (a.g.d == 3)
    residual_ghost_lex_kernel<3><<<(unsigned)blocks, 256, 0, st>>>(a, wl, basel, nodel, l2s, ng, u, r_ext, maxbits, i0, i1);
  else
    residual_ghost_lex_kernel<2><<<(unsigned)blocks, 256, 0, st>>>(a, wl, basel, nodel, l2s, ng, u, r_ext, maxbits, i0, i1);
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
                                                             GhostArgs c, double* __restrict__ gval_c,
                                                             const int32_t* __restrict__ order, int64_t n) {
  // order: coarse ghosts visited in lexicographic order (slot = order[t]),
  // so neighbouring threads read neighbouring fine blocks; else slot order
  constexpr int M = D == 3 ? 27 : 9;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t s = order ? order[t] : t;
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
  // every w[e] is 0 or a power of two (products of 1/4, 1/2, 1/4), so
  // w[e] / sum == w[e] * (1 / sum) exactly: one division per ghost
  const double rs = 1.0 / sum;
  double p[M];
#pragma unroll
  for (int e = 0; e < M; ++e) p[e] = (w[e] * rs) * r_ext[blk[e]];
  gval_c[s] = np_sum<M>(p);
}

void launch_restrict_ghost(const Geom& gf, const uint8_t* lab_f, const double* r_ext,
                           const GhostArgs& coarse, double* gval_c, const int32_t* order, int64_t n_lex,
                           cudaStream_t st) {
  if (coarse.ng == 0) return;
  const int threads = 256;
  const int64_t n = order ? n_lex : coarse.ng;
  const int64_t blocks = (n + threads - 1) / threads;
  if (n == 0) return;
  if (gf.d == 3)
    restrict_ghost_kernel<3><<<(unsigned)blocks, threads, 0, st>>>(gf, lab_f, r_ext, coarse, gval_c, order, n);
  else
    restrict_ghost_kernel<2><<<(unsigned)blocks, threads, 0, st>>>(gf, lab_f, r_ext, coarse, gval_c, order, n);
}

}  // namespace gmg
