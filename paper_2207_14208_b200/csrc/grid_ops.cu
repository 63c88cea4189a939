// grid_ops.cu -- full-grid kernels on sm_100a: interior residual, interior
// restriction, d-linear interpolation + correction, band extrapolation,
// norms and the small gather/scatter helpers of the coarsest solve.
//
// All are HBM-streaming fp64 kernels (no tensor-core work on this path);
// the arithmetic order restates the reference op by op (file:line at each
// kernel).
#include "gmg_kernels.cuh"

namespace gmg {

namespace {

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

unsigned grid_for(int64_t n, int threads, int64_t cap = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace

// residual_internal (smoothing.py:111-118) into a full array:
// r = (f - (denom/h^2) u) + S/h^2 on internal nodes.
template <int D>
__global__ void __launch_bounds__(256) residual_interior_kernel(Geom g, const uint8_t* __restrict__ lab,
                                                                const double* __restrict__ u,
                                                                const double* __restrict__ f,
                                                                double* __restrict__ r,
                                                                unsigned long long* maxbits) {
  double am = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.nodes;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (lab[i] != INTERNAL) continue;
    double s;
    if (D == 3)
      s = ((((u[i - g.s0] + u[i + g.s0]) + u[i - g.s1]) + u[i + g.s1]) + u[i - 1]) + u[i + 1];
    else
      s = ((u[i - g.s0] + u[i + g.s0]) + u[i - 1]) + u[i + 1];
    s = s + 0.0;
    const double v = (f[i] - g.c * u[i]) + s / g.h2;
    r[i] = v;
    am = (__double_as_longlong(fabs(v)) > __double_as_longlong(am)) ? fabs(v) : am;
  }
  block_max_commit(am, maxbits);
}

void launch_residual_interior(const Geom& g, const uint8_t* labels, const double* u,
                              const double* f, double* r, unsigned long long* maxbits,
                              cudaStream_t st) {
  const unsigned blocks = grid_for(g.nodes, 256);
  if (g.d == 3)
    residual_interior_kernel<3><<<blocks, 256, 0, st>>>(g, labels, u, f, r, maxbits);
  else
    residual_interior_kernel<2><<<blocks, 256, 0, st>>>(g, labels, u, f, r, maxbits);
}

template <int D>
__device__ __forceinline__ double fw_w(int e) {
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

// InteriorRestriction.apply (transfer.py:64-93): coarse internal node at m
// takes pairwise(w * r[3^D fine block around 2m]); w = full weighting unless
// the block holds a ghost/inactive node, then 1/count on its internal nodes.
template <int D>
__global__ void __launch_bounds__(256) restrict_interior_kernel(Geom gf, const uint8_t* __restrict__ lab_f,
                                                                const double* __restrict__ r_f, Geom gc,
                                                                const uint8_t* __restrict__ lab_c,
                                                                double* __restrict__ f_c) {
  constexpr int M = D == 3 ? 27 : 9;
  for (int64_t ic = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ic < gc.nodes;
       ic += (int64_t)gridDim.x * blockDim.x) {
    if (lab_c[ic] != INTERNAL) continue;
    int64_t mc[3];
    pos_multi(gc, ic, mc);
#pragma unroll
    for (int k = 0; k < D; ++k) mc[k] *= 2;
    const int64_t center = multi_pos(gf, mc);
    int64_t blk[M];
    bool mixed = false;
    int cnt = 0;
    uint32_t internal_bits = 0;
#pragma unroll
    for (int e = 0; e < M; ++e) {
      int64_t off;
      if (D == 3)
        off = (int64_t)(e / 9 - 1) * gf.s0 + (int64_t)((e / 3) % 3 - 1) * gf.s1 + (e % 3 - 1);
      else
        off = (int64_t)(e / 3 - 1) * gf.s0 + (e % 3 - 1);
      blk[e] = center + off;
      const uint8_t L = lab_f[blk[e]];
      mixed |= (L == GHOST || L == INACTIVE);
      if (L == INTERNAL) {
        ++cnt;
        internal_bits |= 1u << e;
      }
    }
    double p[M];
    if (mixed) {
      const double dc = (double)cnt;
#pragma unroll
      for (int e = 0; e < M; ++e) p[e] = (((internal_bits >> e) & 1u) ? 1.0 : 0.0) / dc * r_f[blk[e]];
    } else {
#pragma unroll
      for (int e = 0; e < M; ++e) p[e] = fw_w<D>(e) * r_f[blk[e]];
    }
    f_c[ic] = np_sum<M>(p);
  }
}

void launch_restrict_interior(const Geom& gf, const uint8_t* lab_f, const double* r_f,
                              const Geom& gc, const uint8_t* lab_c, double* f_c,
                              cudaStream_t st) {
  const unsigned blocks = grid_for(gc.nodes, 256);
  if (gf.d == 3)
    restrict_interior_kernel<3><<<blocks, 256, 0, st>>>(gf, lab_f, r_f, gc, lab_c, f_c);
  else
    restrict_interior_kernel<2><<<blocks, 256, 0, st>>>(gf, lab_f, r_f, gc, lab_c, f_c);
}

// ErrorInterpolation + correction (transfer.py:124-151, solver.py:198):
// u += sum_c w_c e[src_c] on internal and ghost fine nodes; corner c of
// {0,1}^D in C order, w_c = prod_k (odd_k ? 1/2 : [c_k == 0]).
template <int D>
__global__ void __launch_bounds__(256) interp_add_kernel(Geom gf, const uint8_t* __restrict__ lab_f,
                                                         double* __restrict__ u, Geom gc,
                                                         const double* __restrict__ e) {
  constexpr int NC = 1 << D;
  const int64_t sc[3] = {gc.s0, gc.s1, gc.s2};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < gf.nodes;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t L = lab_f[i];
    if (L != INTERNAL && L != GHOST) continue;
    int64_t m[3], half[3];
    pos_multi(gf, i, m);
#pragma unroll
    for (int k = 0; k < D; ++k) half[k] = m[k] / 2;
    const int64_t cbase = multi_pos(gc, half);
    double p[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double w = 1.0;
      int64_t src = cbase;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const int off = (c >> (D - 1 - k)) & 1;
        const int odd = (int)(m[k] & 1);
        w = w * (odd ? 0.5 : (off == 0 ? 1.0 : 0.0));
        src += (odd ? off : 0) * sc[k];
      }
      p[c] = w * e[src];
    }
    u[i] = u[i] + np_sum<NC>(p);
  }
}

void launch_interp_add(const Geom& gf, const uint8_t* lab_f, double* u_f, const Geom& gc,
                       const double* e_c, cudaStream_t st) {
  const unsigned blocks = grid_for(gf.nodes, 256);
  if (gf.d == 3)
    interp_add_kernel<3><<<blocks, 256, 0, st>>>(gf, lab_f, u_f, gc, e_c);
  else
    interp_add_kernel<2><<<blocks, 256, 0, st>>>(gf, lab_f, u_f, gc, e_c);
}

// Band BFS group (transfer.py:245-246): x_i = (sum_k x[nbr_k] * mask_k) /
// popcount(mask).  Masked-out columns contribute +0 (the reference reads the
// still-unassigned band node itself, which holds +0 in every use).
template <int D>
__global__ void __launch_bounds__(256) band_bfs_kernel(BandArgs a, double* __restrict__ x, int64_t lo,
                                                       int64_t hi) {
  const int64_t q = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= hi) return;
  const int64_t i = a.idx[q];
  const unsigned mk = a.mask[q];
  const int64_t s[3] = {a.g.s0, a.g.s1, a.g.s2};
  double t[2 * D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const bool bit = (mk >> (2 * k + j)) & 1u;
      t[2 * k + j] = bit ? x[j ? i + s[k] : i - s[k]] * 1.0 : 0.0;
    }
  }
  x[i] = seq_sum<2 * D>(t) / (double)__popc(mk);
}

void launch_band_bfs(const BandArgs& a, double* x, int64_t lo, int64_t hi, cudaStream_t st) {
  if (hi <= lo) return;
  const unsigned blocks = (unsigned)((hi - lo + 255) / 256);
  if (a.g.d == 3)
    band_bfs_kernel<3><<<blocks, 256, 0, st>>>(a, x, lo, hi);
  else
    band_bfs_kernel<2><<<blocks, 256, 0, st>>>(a, x, lo, hi);
}

// One Jacobi transport step (transfer.py:249-251):
// v_i <- v_i - 0.5 * sum_k |n_k| (v_i - v[i - step_k s_k]).
template <int D>
__global__ void __launch_bounds__(256) band_step_kernel(BandArgs a, const double* __restrict__ x) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= a.nb) return;
  const int64_t i = a.idx[q];
  const int64_t s[3] = {a.g.s0, a.g.s1, a.g.s2};
  const double vi = x[i];
  double t[D];
#pragma unroll
  for (int k = 0; k < D; ++k) t[k] = a.absn[q * D + k] * (vi - x[i - (int64_t)a.step[q * D + k] * s[k]]);
  a.scratch[q] = vi - 0.5 * seq_sum<D>(t);
}

__global__ void band_commit_kernel(BandArgs a, double* __restrict__ x) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= a.nb) return;
  x[a.idx[q]] = a.scratch[q];
}

void launch_band_transport(const BandArgs& a, double* x, cudaStream_t st) {
  if (a.nb == 0) return;
  const unsigned blocks = (unsigned)((a.nb + 255) / 256);
  for (int it = 0; it < 6; ++it) {
    if (a.g.d == 3)
      band_step_kernel<3><<<blocks, 256, 0, st>>>(a, x);
    else
      band_step_kernel<2><<<blocks, 256, 0, st>>>(a, x);
    band_commit_kernel<<<blocks, 256, 0, st>>>(a, x);
  }
}

__global__ void abs_max_kernel(const double* __restrict__ u, int64_t n, unsigned long long* maxbits) {
  double am = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = fabs(u[i]);
    am = (__double_as_longlong(v) > __double_as_longlong(am)) ? v : am;
  }
  block_max_commit(am, maxbits);
}

void launch_abs_max(const double* u, int64_t n, unsigned long long* maxbits, cudaStream_t st) {
  abs_max_kernel<<<grid_for(n, 256), 256, 0, st>>>(u, n, maxbits);
}

__global__ void scale_kernel(double* __restrict__ u, int64_t n, double s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    u[i] = u[i] * s;
}

void launch_scale(double* u, int64_t n, double s, cudaStream_t st) {
  scale_kernel<<<grid_for(n, 256), 256, 0, st>>>(u, n, s);
}

// Coarsest solve right-hand side [f_c at internal nodes; g_c in lex order].
__global__ void gather_kernel(const int64_t* __restrict__ idx, int64_t n_int, const double* __restrict__ f,
                              const int32_t* __restrict__ ghost_slot, int64_t n_gh,
                              const double* __restrict__ gval, double* __restrict__ out) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < n_int)
    out[q] = f[idx[q]];
  else if (q < n_int + n_gh)
    out[q] = gval[ghost_slot[q - n_int]];
}

void launch_gather(const int64_t* idx, int64_t n_int, const double* f, const int32_t* ghost_slot,
                   int64_t n_gh, const double* gval, double* out, cudaStream_t st) {
  const int64_t n = n_int + n_gh;
  if (n == 0) return;
  gather_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(idx, n_int, f, ghost_slot, n_gh, gval, out);
}

__global__ void scatter_kernel(const int64_t* __restrict__ idx, int64_t n, const double* __restrict__ x,
                               double* __restrict__ e) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < n) e[idx[q]] = x[q];
}

void launch_scatter(const int64_t* idx, int64_t n, const double* x, double* e, cudaStream_t st) {
  if (n == 0) return;
  scatter_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(idx, n, x, e);
}

// dst[i] = src[perm[i]] (0 where perm[i] < 0)
__global__ void permute_kernel(const double* __restrict__ src, const int32_t* __restrict__ perm, int64_t n,
                               double* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = perm[i] >= 0 ? src[perm[i]] : 0.0;
}

void launch_permute(const double* src, const int32_t* perm, int64_t n, double* dst, cudaStream_t st) {
  if (n == 0) return;
  permute_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, perm, n, dst);
}

}  // namespace gmg
