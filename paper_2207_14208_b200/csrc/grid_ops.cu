// grid_ops.cu -- full-grid kernels on sm_100a: interior residual, interior
// restriction, d-linear interpolation + correction, band extrapolation,
// norms and the small gather/scatter helpers of the coarsest solve.
//
// All are HBM-streaming fp64 kernels (no tensor-core work on this path);
// the arithmetic order restates the reference op by op (file:line at each
// kernel).
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "gmg_kernels.cuh"

namespace cg = cooperative_groups;

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
                                                                unsigned long long* maxbits,
                                                                unsigned long long* peakbits) {
  double am = 0.0, pm = 0.0;  // pm: max |u| over the internal nodes (norm pass only, see launch_residual_interior)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.nodes;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (lab[i] != INTERNAL) continue;
    double s;
    if (D == 3)
      s = ((((u[i - g.s0] + u[i + g.s0]) + u[i - g.s1]) + u[i + g.s1]) + u[i - 1]) + u[i + 1];
    else
      s = ((u[i - g.s0] + u[i + g.s0]) + u[i - 1]) + u[i + 1];
    s = s + 0.0;
    const double uc = u[i];
    const double v = (f[i] - g.c * uc) + div_h2(g, s);
    if (r) r[i] = v;
    am = (__double_as_longlong(fabs(v)) > __double_as_longlong(am)) ? fabs(v) : am;
    pm = (__double_as_longlong(fabs(uc)) > __double_as_longlong(pm)) ? fabs(uc) : pm;
  }
  block_max_commit(am, maxbits);
  if (peakbits) {
    __syncthreads();
    block_max_commit(pm, peakbits);
  }
}

// 3-D plane-marching version (production): a CTA owns RM_TJ rows x RM_TK
// columns of every plane of its segment and walks the planes in order.  Each
// plane's u tile (+1 halo), f tile and labels arrive by cp.async in a ring
// of RM_S slots, RM_S - 1 planes ahead, so u is read from L2 about once
// (+ halo) instead of once per stencil neighbour.  Same arithmetic order as
// residual_interior_kernel.  r == nullptr: only the maximum (norm pass).
constexpr int RM_TK = 64, RM_UW = RM_TK + 4;  // u row: [pad, k0-1, k0 .. k0+63, k0+64, pad]
template <int RM_TJ, int RM_S>
struct __align__(16) ResMarchSmem {
  double u[RM_S][RM_TJ + 2][RM_UW];
  double f[RM_S][RM_TJ][RM_TK];
  uint8_t lab[RM_S][RM_TJ][RM_TK];
};

__device__ __forceinline__ void cpa16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cpa8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cpa4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <bool WRITE, int RM_TJ, int RM_S>
__global__ void __launch_bounds__(RM_TJ * 32) residual_march3_kernel(Geom g, const uint8_t* __restrict__ lab,
                                                                     const double* __restrict__ u,
                                                                     const double* __restrict__ f,
                                                                     double* __restrict__ r,
                                                                     unsigned long long* maxbits, int p_lo, int p_hi,
                                                                     unsigned long long* peakbits) {
  extern __shared__ __align__(16) unsigned char rm_raw[];
  ResMarchSmem<RM_TJ, RM_S>& S = *reinterpret_cast<ResMarchSmem<RM_TJ, RM_S>*>(rm_raw);
  const int N = (int)g.N;
  const int k0 = 1 + (int)blockIdx.x * RM_TK, j0 = 1 + (int)blockIdx.y * RM_TJ;
  // the internal planes [p_lo, p_hi] (1 .. N-1, or a z-slab of them) in gridDim.z segments
  const int per = (p_hi - p_lo + 1 + (int)gridDim.z - 1) / (int)gridDim.z;
  const int ib = p_lo + (int)blockIdx.z * per, ie = min(p_hi, ib + per - 1);
  if (ib > ie) return;
  const int tid = threadIdx.x;
  // Copy descriptors: each plane is the same set of RM_NCP copies (u rows with
  // halo, f and label rows) shifted by a plane stride, so every thread
  // resolves its (at most 3) copies once: shared address in slot 0, global
  // address in plane 0, size (0 = none).
  constexpr int UPR = RM_TK / 2 + 2, FPR = RM_TK / 2, LPR = RM_TK / 4;
  constexpr int NU = (RM_TJ + 2) * UPR, NF = RM_TJ * FPR, NL = RM_TJ * LPR, RM_NCP = NU + NF + NL;
  constexpr int NT = RM_TJ * 32, NQ = (RM_NCP + NT - 1) / NT;
  unsigned dsm[NQ], dss[NQ];
  const char* dg[NQ];
  int64_t dps[NQ];
  int dsz[NQ];
  const int64_t pstride = g.n * g.P;  // elements per plane
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int x = tid + q * NT;
    dsz[q] = 0;
    dsm[q] = dss[q] = 0;
    dg[q] = nullptr;
    dps[q] = 0;
    if (x < NU) {
      const int jr = x / UPR, c = x - jr * UPR, j = j0 - 1 + jr;
      int col = 0, kk = 0, sz = 0;
      if (c < RM_TK / 2) {
        col = 2 + 2 * c, kk = k0 + 2 * c, sz = k0 + 2 * c <= N - 1 ? 16 : 0;
      } else if (c == RM_TK / 2) {
        col = 1, kk = k0 - 1, sz = 8;
      } else {
        col = 2 + RM_TK, kk = k0 + RM_TK, sz = k0 + RM_TK <= N ? 8 : 0;
      }
      if (j > N) sz = 0;
      dsz[q] = sz;
      dsm[q] = (unsigned)__cvta_generic_to_shared(&S.u[0][jr][col]);
      dss[q] = (unsigned)sizeof(S.u[0]);
      dg[q] = reinterpret_cast<const char*>(u + (int64_t)j * g.P + OFF + kk);
      dps[q] = pstride * 8;
    } else if (x < NU + NF) {
      const int y = x - NU, jr = y / FPR, c = y - jr * FPR, j = j0 + jr;
      dsz[q] = (j <= N - 1 && k0 + 2 * c <= N - 1) ? 16 : 0;
      dsm[q] = (unsigned)__cvta_generic_to_shared(&S.f[0][jr][2 * c]);
      dss[q] = (unsigned)sizeof(S.f[0]);
      dg[q] = reinterpret_cast<const char*>(f + (int64_t)j * g.P + OFF + k0 + 2 * c);
      dps[q] = pstride * 8;
    } else if (x < RM_NCP) {
      const int y = x - NU - NF, jr = y / LPR, w = y - jr * LPR, j = j0 + jr;
      dsz[q] = (j <= N - 1 && k0 + 4 * w <= N - 1) ? 4 : 0;
      dsm[q] = (unsigned)__cvta_generic_to_shared(&S.lab[0][jr][4 * w]);
      dss[q] = (unsigned)sizeof(S.lab[0]);
      dg[q] = reinterpret_cast<const char*>(lab + (int64_t)j * g.P + OFF + k0 + 4 * w);
      dps[q] = pstride;
    }
  }
  // copy plane p into slot p mod RM_S
  auto fetch = [&](int p) {
    if (p <= N) {
      const unsigned sl = (unsigned)(p % RM_S);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const unsigned dst = dsm[q] + sl * dss[q];
        const char* src = dg[q] + (int64_t)p * dps[q];
        if (dsz[q] == 16)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        else if (dsz[q] == 8)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
        else if (dsz[q] == 4)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
      }
    }
    cpa_commit();
  };
  // prologue: planes ib-1 .. ib+RM_S-2
  for (int p = ib - 1; p <= ib + RM_S - 2; ++p) fetch(p);
  const int tj = tid >> 5, lane = tid & 31;
  const int j = j0 + tj;
  double am = 0.0, pm = 0.0;
  for (int i = ib; i <= ie; ++i) {
    cpa_wait<RM_S - 3>();  // planes <= i+1 have landed
    __syncthreads();
    const int sm = (i - 1) % RM_S, sc = i % RM_S, sp = (i + 1) % RM_S;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kk = lane + 32 * h, k = k0 + kk;
      if (j > N - 1 || k > N - 1) continue;
      if (S.lab[sc][tj][kk] != INTERNAL) continue;
      const double um = S.u[sm][tj + 1][kk + 2], up = S.u[sp][tj + 1][kk + 2];
      const double un = S.u[sc][tj][kk + 2], us = S.u[sc][tj + 2][kk + 2];
      const double uw = S.u[sc][tj + 1][kk + 1], ue = S.u[sc][tj + 1][kk + 3];
      const double uc = S.u[sc][tj + 1][kk + 2];
      double s = ((((um + up) + un) + us) + uw) + ue;
      s = s + 0.0;
      const double v = (S.f[sc][tj][kk] - g.c * uc) + div_h2(g, s);
      if (WRITE) r[((int64_t)i * g.n + j) * g.P + k + OFF] = v;
      am = (__double_as_longlong(fabs(v)) > __double_as_longlong(am)) ? fabs(v) : am;
      if (!WRITE) pm = (__double_as_longlong(fabs(uc)) > __double_as_longlong(pm)) ? fabs(uc) : pm;
    }
    __syncthreads();  // slot of plane i-1 is refilled next
    fetch(i + RM_S - 1);
  }
  cpa_wait<0>();
  block_max_commit(am, maxbits);
  if (!WRITE && peakbits) {
    __syncthreads();
    block_max_commit(pm, peakbits);
  }
}

static void launch_residual_march(const Geom& g, const uint8_t* labels, const double* u, const double* f, double* r,
                                  unsigned long long* maxbits, int p_lo, int p_hi, cudaStream_t st,
                                  unsigned long long* peakbits = nullptr);

void launch_residual_interior_planes(const Geom& g, const uint8_t* labels, const double* u, const double* f, double* r,
                                     unsigned long long* maxbits, int p_lo, int p_hi, cudaStream_t st) {
  if (p_hi >= p_lo) launch_residual_march(g, labels, u, f, r, maxbits, p_lo, p_hi, st);
}

void launch_residual_interior(const Geom& g, const uint8_t* labels, const double* u,
                              const double* f, double* r, unsigned long long* maxbits,
                              cudaStream_t st, unsigned long long* peakbits) {
  // peakbits (norm pass, r == nullptr): also max |u| over the internal nodes -- a lower bound of max |u| that
  // lets the caller skip the full-array pass of the renormalisation check (solver.py:241-245) when it is
  // already above the threshold
  if (g.d == 3)
    launch_residual_march(g, labels, u, f, r, maxbits, 1, (int)g.N - 1, st, peakbits);
  else
    residual_interior_kernel<2><<<grid_for(g.nodes, 256), 256, 0, st>>>(g, labels, u, f, r, maxbits, r ? nullptr : peakbits);
}

static void launch_residual_march(const Geom& g, const uint8_t* labels, const double* u, const double* f, double* r,
                                  unsigned long long* maxbits, int p_lo, int p_hi, cudaStream_t st,
                                  unsigned long long* peakbits) {
  {
    // 8-row x 64-column tiles; ring of 4 plane slots (5 CTAs per SM) on the
    // largest grids, 5 slots (4 CTAs per SM) below N = 512 (measured per level)
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(residual_march3_kernel<true, 8, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(ResMarchSmem<8, 5>));
      cudaFuncSetAttribute(residual_march3_kernel<false, 8, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(ResMarchSmem<8, 5>));
      cudaFuncSetAttribute(residual_march3_kernel<true, 8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(ResMarchSmem<8, 4>));
      cudaFuncSetAttribute(residual_march3_kernel<false, 8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(ResMarchSmem<8, 4>));
      attr = true;
    }
    const bool big = g.N >= 512;
    const int per_sm = big ? 5 : 4;
    const int64_t tk = (g.N - 1 + RM_TK - 1) / RM_TK, tj = (g.N - 1 + 8 - 1) / 8;
    const int64_t np = p_hi - p_lo + 1;
    // plane segments per tile: enough CTAs for ~7 waves of the resident slots as long as a segment keeps
    // >= 25 planes (its ring prologue costs about six planes' time), and never fewer than one wave
    // (512^3: 1 -> 10 segments, 679 -> 582 us; 256^3: 4 -> 10, 100 -> 95 us; smaller levels unchanged)
    const int64_t slots = 148 * per_sm, tiles = tk * tj;
    const int64_t one_wave = std::min<int64_t>(std::max<int64_t>(1, np / 4), slots / tiles);
    const int64_t waves7 = std::min<int64_t>(np / 25, (7 * slots + tiles - 1) / tiles);
    const int64_t segs = std::max<int64_t>(1, std::max(one_wave, waves7));
    dim3 grid((unsigned)tk, (unsigned)tj, (unsigned)segs);
    if (big) {
      if (r)
        residual_march3_kernel<true, 8, 4><<<grid, 256, sizeof(ResMarchSmem<8, 4>), st>>>(g, labels, u, f, r, maxbits, p_lo, p_hi, peakbits);
      else
        residual_march3_kernel<false, 8, 4><<<grid, 256, sizeof(ResMarchSmem<8, 4>), st>>>(g, labels, u, f, r, maxbits, p_lo, p_hi, peakbits);
    } else {
      if (r)
        residual_march3_kernel<true, 8, 5><<<grid, 256, sizeof(ResMarchSmem<8, 5>), st>>>(g, labels, u, f, r, maxbits, p_lo, p_hi, peakbits);
      else
        residual_march3_kernel<false, 8, 5><<<grid, 256, sizeof(ResMarchSmem<8, 5>), st>>>(g, labels, u, f, r, maxbits, p_lo, p_hi, peakbits);
    }
  }
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
// Row loop: a CTA takes coarse rows (grid-stride), its threads the columns
// of the row.  The fine-label pattern of every coarse node's 3^D block is
// precomputed once per hierarchy (restrict_mask_kernel): bit e = fine node e
// of the block is internal, bit 30 = the coarse node is internal, bit 31 =
// the block holds a ghost / inactive node ("mixed").  The 3^D residual
// loads do not depend on it, so they are all in flight together.
constexpr uint32_t RM_COARSE = 1u << 30, RM_MIXED = 1u << 31;

template <int D>
__device__ __forceinline__ int64_t block_off(const Geom& gf, int e) {
  if (D == 3) return (int64_t)(e / 9 - 1) * gf.s0 + (int64_t)((e / 3) % 3 - 1) * gf.s1 + (e % 3 - 1);
  return (int64_t)(e / 3 - 1) * gf.s0 + (e % 3 - 1);
}

template <int D>
__global__ void __launch_bounds__(256) restrict_mask_kernel(Geom gf, const uint8_t* __restrict__ lab_f, Geom gc,
                                                            const uint8_t* __restrict__ lab_c,
                                                            uint32_t* __restrict__ rmask) {
  constexpr int M = D == 3 ? 27 : 9;
  const int nc = (int)gc.n;
  const int64_t nrows = D == 3 ? (int64_t)nc * nc : nc;
  for (int64_t rr = blockIdx.x; rr < nrows; rr += gridDim.x) {
    const int I = D == 3 ? (int)(rr / nc) : 0;
    const int J = D == 3 ? (int)(rr % nc) : (int)rr;
    for (int K = threadIdx.x; K < nc; K += blockDim.x) {
      const int64_t ic = rr * gc.P + K + OFF;
      uint32_t m = 0;
      if (lab_c[ic] == INTERNAL) {
        const int64_t frow = D == 3 ? (int64_t)(2 * I) * gf.n + 2 * J : 2 * J;
        const int64_t center = frow * gf.P + 2 * K + OFF;
        m = RM_COARSE;
        for (int e = 0; e < M; ++e) {
          const uint8_t L = lab_f[center + block_off<D>(gf, e)];
          if (L == GHOST || L == INACTIVE) m |= RM_MIXED;
          if (L == INTERNAL) m |= 1u << e;
        }
      }
      rmask[ic] = m;
    }
  }
}

void launch_restrict_mask(const Geom& gf, const uint8_t* lab_f, const Geom& gc, const uint8_t* lab_c,
                          uint32_t* rmask, cudaStream_t st) {
  const int64_t nrows = gc.d == 3 ? gc.n * gc.n : gc.n;
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nrows, 148 * 8));
  if (gc.d == 3)
    restrict_mask_kernel<3><<<blocks, 256, 0, st>>>(gf, lab_f, gc, lab_c, rmask);
  else
    restrict_mask_kernel<2><<<blocks, 256, 0, st>>>(gf, lab_f, gc, lab_c, rmask);
}

template <int D>
__global__ void __launch_bounds__(256, 3) restrict_interior_kernel(Geom gf, const double* __restrict__ r_f, Geom gc,
                                                                const uint32_t* __restrict__ rmask,
                                                                double* __restrict__ f_c) {
  constexpr int M = D == 3 ? 27 : 9;
  const int nc = (int)gc.n;
  const int inner = nc - 2;  // rows/columns 1 .. N_c - 1 can hold internal nodes
  const int64_t nrows = D == 3 ? (int64_t)inner * inner : inner;
  for (int64_t rr = blockIdx.x; rr < nrows; rr += gridDim.x) {
    const int I = D == 3 ? (int)(rr / inner) + 1 : 0;
    const int J = D == 3 ? (int)(rr % inner) + 1 : (int)rr + 1;
    const int64_t crow = D == 3 ? (int64_t)I * nc + J : J;
    const int64_t frow = D == 3 ? (int64_t)(2 * I) * gf.n + 2 * J : 2 * J;
    for (int K = 1 + threadIdx.x; K <= nc - 2; K += blockDim.x) {
      const int64_t ic = crow * gc.P + K + OFF;
      const uint32_t m = rmask[ic];
      if (!(m & RM_COARSE)) continue;
      const double* rc = r_f + frow * gf.P + 2 * K + OFF;
      double p[M];
#pragma unroll
      for (int e = 0; e < M; ++e) p[e] = rc[block_off<D>(gf, e)];
      if (m & RM_MIXED) {
        const double dc = (double)__popc(m & ((1u << M) - 1u));
        const double w1 = 1.0 / dc;
#pragma unroll
        for (int e = 0; e < M; ++e) p[e] = (((m >> e) & 1u) ? w1 : 0.0) * p[e];  // == (bit ? 1 : 0) / dc * p
      } else {
#pragma unroll
        for (int e = 0; e < M; ++e) p[e] = fw_w<D>(e) * p[e];
      }
      f_c[ic] = np_sum<M>(p);
    }
  }
}

// Fused interior residual + interior restriction (3-D):
// residual_internal (smoothing.py:111-118) evaluated tile by tile and fed
// straight into InteriorRestriction.apply (transfer.py:88-93); the fine
// residual never goes to HBM (nothing else reads it).  A CTA owns FR_TKc x
// FR_TJc coarse nodes of every coarse plane of its segment and marches the
// fine planes 2Ib-1 .. 2Ie+1: u (+1 halo), f and labels of fine plane p
// arrive by cp.async in a ring of FR_S slots; the residual of each fine
// plane is kept in a 3-plane ring; after every odd fine plane 2I+1 the
// coarse plane I is restricted from that ring.  Non-internal fine nodes
// carry residual 0, as in the full residual array of the unfused path.
constexpr int FR_TJc = 4, FR_TKc = 32, FR_S = 6;
constexpr int FRJ = 2 * FR_TJc + 1, FRK = 2 * FR_TKc + 1;  // fine residual tile 9 x 65
constexpr int FRUJ = FRJ + 2, FRUW = 70, FRFW = 66, FRLW = 68;
struct __align__(16) FusedSmem {
  double u[FR_S][FRUJ][FRUW];  // column k0f-1+c at index c+1 (k0f at index 2: 16-byte aligned)
  double f[FR_S][FRJ][FRFW];   // column k0f+c at index c
  uint8_t lab[FR_S][FRJ][FRLW];
  double r[3][FRJ][FRFW];
};

__global__ void __launch_bounds__(256, 2) res_restrict3_kernel(Geom g, const uint8_t* __restrict__ lab,
                                                               const double* __restrict__ u,
                                                               const double* __restrict__ f, Geom gc,
                                                               const uint32_t* __restrict__ rmask,
                                                               double* __restrict__ f_c) {
  extern __shared__ __align__(16) unsigned char fr_raw[];
  FusedSmem& S = *reinterpret_cast<FusedSmem*>(fr_raw);
  const int N = (int)g.N, nc = (int)gc.n, innc = nc - 2;
  const int K0c = 1 + (int)blockIdx.x * FR_TKc, J0c = 1 + (int)blockIdx.y * FR_TJc;
  const int k0f = 2 * K0c - 1, j0f = 2 * J0c - 1;
  const int per = (innc + (int)gridDim.z - 1) / (int)gridDim.z;
  const int Ib = 1 + (int)blockIdx.z * per, Ie = min(innc, Ib + per - 1);
  if (Ib > Ie) return;
  const int tid = threadIdx.x;
  // copy descriptors (see residual_march3_kernel): u rows j0f-1 .. j0f+9 with
  // columns k0f-1 .. k0f+65, f / label rows j0f .. j0f+8 with columns k0f .. k0f+64
  constexpr int UPR = FR_TKc + 3, FPR = FR_TKc + 1, LPR = FR_TKc / 2 + 1;
  constexpr int NU = FRUJ * UPR, NF = FRJ * FPR, NL = FRJ * LPR, NCP = NU + NF + NL;
  constexpr int NQ = (NCP + 255) / 256;
  unsigned dsm[NQ], dss[NQ];
  const char* dg[NQ];
  int64_t dps[NQ];
  int dsz[NQ];
  const int64_t pstride = g.n * g.P;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int x = tid + q * 256;
    dsz[q] = 0;
    dsm[q] = dss[q] = 0;
    dg[q] = nullptr;
    dps[q] = 0;
    if (x < NU) {
      const int jr = x / UPR, c = x - jr * UPR, j = j0f - 1 + jr;
      int idx, k, sz;
      if (c < FR_TKc) {
        k = k0f + 2 * c, idx = 2 + 2 * c, sz = k + 1 <= N ? 16 : (k <= N ? 8 : 0);
      } else {
        const int e = c - FR_TKc;  // 0: k0f-1, 1: k0f+64, 2: k0f+65
        k = e == 0 ? k0f - 1 : k0f + 63 + e, idx = e == 0 ? 1 : 65 + e, sz = k <= N ? 8 : 0;
      }
      if (j > N) sz = 0;
      dsz[q] = sz;
      dsm[q] = (unsigned)__cvta_generic_to_shared(&S.u[0][jr][idx]);
      dss[q] = (unsigned)sizeof(S.u[0]);
      dg[q] = reinterpret_cast<const char*>(u + (int64_t)j * g.P + OFF + k);
      dps[q] = pstride * 8;
    } else if (x < NU + NF) {
      const int y = x - NU, jr = y / FPR, c = y - jr * FPR, j = j0f + jr;
      const int k = k0f + 2 * c;
      int sz = c < FR_TKc ? (k + 1 <= N ? 16 : (k <= N ? 8 : 0)) : (k <= N ? 8 : 0);
      if (j > N) sz = 0;
      dsz[q] = sz;
      dsm[q] = (unsigned)__cvta_generic_to_shared(&S.f[0][jr][2 * c]);
      dss[q] = (unsigned)sizeof(S.f[0]);
      dg[q] = reinterpret_cast<const char*>(f + (int64_t)j * g.P + OFF + k);
      dps[q] = pstride * 8;
    } else if (x < NCP) {
      const int y = x - NU - NF, jr = y / LPR, w = y - jr * LPR, j = j0f + jr;
      const int k = k0f + 4 * w;
      dsz[q] = (j <= N && k <= N) ? 4 : 0;  // the last word may run into the padding: in the row
      dsm[q] = (unsigned)__cvta_generic_to_shared(&S.lab[0][jr][4 * w]);
      dss[q] = (unsigned)sizeof(S.lab[0]);
      dg[q] = reinterpret_cast<const char*>(lab + (int64_t)j * g.P + OFF + k);
      dps[q] = pstride;
    }
  }
  auto fetch = [&](int p) {
    if (p <= N) {
      const unsigned sl = (unsigned)(p % FR_S);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const unsigned dst = dsm[q] + sl * dss[q];
        const char* src = dg[q] + (int64_t)p * dps[q];
        if (dsz[q] == 16)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        else if (dsz[q] == 8)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
        else if (dsz[q] == 4)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
      }
    }
    cpa_commit();
  };
  const int i0 = 2 * Ib - 1, i1 = 2 * Ie + 1;
  for (int p = i0 - 1; p <= i0 + FR_S - 2; ++p) fetch(p);
  // this thread's fine nodes of the residual tile (fixed across planes):
  // element offsets of u (centre), f / r, and the label byte; -1 = none
  constexpr int NR = (FRJ * FRK + 255) / 256;
  int ou[NR], of[NR], ol[NR];
  bool act[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    const int x = tid + 256 * q;
    const int jr = x / FRK, kc = x - jr * FRK;
    act[q] = x < FRJ * FRK;
    ou[q] = (jr + 1) * FRUW + kc + 2;
    of[q] = jr * FRFW + kc;
    ol[q] = jr * FRLW + kc;
    if (act[q] && !(j0f + jr <= N - 1 && k0f + kc <= N - 1)) ol[q] = -1;  // never internal
  }
  // this thread's coarse node (threads < 128)
  const int tk = tid % FR_TKc, tj = tid / FR_TKc;
  const int K = K0c + tk, J = J0c + tj;
  const bool cmine = tid < FR_TKc * FR_TJc && K <= nc - 2 && J <= nc - 2;
  const int rbase = 2 * tj * FRFW + 2 * tk;
  const double c = g.c;
  // restriction mask of the coarse plane restricted after the next odd fine
  // plane, loaded a residual phase ahead
  auto mask_of = [&](int I) -> uint32_t {
    return (cmine && I <= Ie) ? rmask[((int64_t)I * nc + J) * gc.P + K + OFF] : 0u;
  };
  uint32_t mnext = mask_of(Ib);
  for (int i = i0; i <= i1; ++i) {
    cpa_wait<FR_S - 3>();  // u planes <= i+1, f / labels of plane i have landed
    __syncthreads();
    // fine residual of plane i on the 9 x 65 tile (0 off the internal nodes)
    {
      const double* um_ = &S.u[(i - 1) % FR_S][0][0];
      const double* uc_ = &S.u[i % FR_S][0][0];
      const double* up_ = &S.u[(i + 1) % FR_S][0][0];
      const double* f_ = &S.f[i % FR_S][0][0];
      const uint8_t* l_ = &S.lab[i % FR_S][0][0];
      double* r_ = &S.r[i % 3][0][0];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        if (!act[q]) continue;
        double v = 0.0;
        if (ol[q] >= 0 && l_[ol[q]] == INTERNAL) {
          const int o = ou[q];
          double sum = ((((um_[o] + up_[o]) + uc_[o - FRUW]) + uc_[o + FRUW]) + uc_[o - 1]) + uc_[o + 1];
          sum = sum + 0.0;
          v = (f_[of[q]] - c * uc_[o]) + div_h2(g, sum);
        }
        r_[of[q]] = v;
      }
    }
    __syncthreads();
    fetch(i + FR_S - 1);  // into the slot of plane i-1, read for the last time above
    if ((i & 1) && i >= i0 + 2 && cmine) {
      // coarse plane I = (i-1)/2 from fine planes i-2, i-1, i
      const int I = (i - 1) >> 1;
      const int64_t ic = ((int64_t)I * nc + J) * gc.P + K + OFF;
      const uint32_t m = mnext;
      mnext = mask_of(I + 1);
      if (m & RM_COARSE) {
        const double* ra = &S.r[(i - 2) % 3][0][0] + rbase;
        const double* rb = &S.r[(i - 1) % 3][0][0] + rbase;
        const double* rc = &S.r[i % 3][0][0] + rbase;
        double p[27];
#pragma unroll
        for (int e = 0; e < 27; ++e) {
          const double* rp = e < 9 ? ra : (e < 18 ? rb : rc);
          p[e] = rp[((e / 3) % 3) * FRFW + e % 3];
        }
        if (m & RM_MIXED) {
          const double dc = (double)__popc(m & ((1u << 27) - 1u));
          const double w1 = 1.0 / dc;
#pragma unroll
          for (int e = 0; e < 27; ++e) p[e] = (((m >> e) & 1u) ? w1 : 0.0) * p[e];  // == (bit ? 1 : 0) / dc * p
        } else {
#pragma unroll
          for (int e = 0; e < 27; ++e) p[e] = fw_w<3>(e) * p[e];
        }
        f_c[ic] = np_sum<27>(p);
      }
    }
  }
  cpa_wait<0>();
}

void launch_res_restrict3(const Geom& gf, const uint8_t* labels, const double* u, const double* f, const Geom& gc,
                          const uint32_t* rmask, double* f_c, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(res_restrict3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FusedSmem));
    attr = true;
  }
  const int64_t innc = gc.n - 2;
  if (innc <= 0) return;
  const int64_t tx = (innc + FR_TKc - 1) / FR_TKc, ty = (innc + FR_TJc - 1) / FR_TJc;
  const int64_t slots = 148 * 2;
  const int64_t segs = std::max<int64_t>(1, std::min<int64_t>(innc / 4, (6 * slots + tx * ty - 1) / (tx * ty)));
  dim3 grid((unsigned)tx, (unsigned)ty, (unsigned)segs);
  res_restrict3_kernel<<<grid, 256, sizeof(FusedSmem), st>>>(gf, labels, u, f, gc, rmask, f_c);
}

void launch_restrict_interior(const Geom& gf, const double* r_f, const Geom& gc, const uint32_t* rmask,
                              double* f_c, cudaStream_t st) {
  const int64_t inner = gc.n - 2;
  const int64_t nrows = gf.d == 3 ? inner * inner : inner;
  // 64 CTAs per SM's worth of rows (512^3: 320 us at 148 * 8, 303 at * 32, 295 at * 64, 341 with one CTA per row)
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nrows, 148 * 64));
  if (gf.d == 3)
    restrict_interior_kernel<3><<<blocks, 256, 0, st>>>(gf, r_f, gc, rmask, f_c);
  else
    restrict_interior_kernel<2><<<blocks, 256, 0, st>>>(gf, r_f, gc, rmask, f_c);
}

// ErrorInterpolation + correction (transfer.py:124-151, solver.py:198):
// u += sum_c w_c e[src_c] on internal and ghost fine nodes; corner c of
// {0,1}^D in C order, w_c = prod_k (odd_k ? 1/2 : [c_k == 0]).
// A thread takes padded positions 4q .. 4q+3 of the fine array (fine columns
// 4q-3 .. 4q, one 32-byte-aligned group): u as two 16-byte loads, the labels
// as one 4-byte load, and per corner row only the three coarse columns
// 2q-2 .. 2q the four nodes share (12 coarse loads for 4 nodes instead of
// 16).  Zero-weight corners are still multiplied and summed, like the
// reference's dense 2^D product.
template <int D>
__global__ void __launch_bounds__(256, 4) interp_add4_kernel(Geom gf, const uint8_t* __restrict__ lab_f,
                                                          double* __restrict__ u, Geom gc,
                                                          const double* __restrict__ e) {
  constexpr int NC = 1 << D;
  constexpr int NR = D == 3 ? 4 : 2;
  const int nf = (int)gf.n;
  const int hq = (int)(gf.P >> 2);  // quads per row
  const int nq = (int)(gf.rows * hq);
  for (int q0 = blockIdx.x * blockDim.x + threadIdx.x; q0 < nq; q0 += gridDim.x * blockDim.x) {
    const int row = q0 / hq, m = q0 - row * hq;
    const int ii = D == 3 ? row / nf : 0;
    const int jj = D == 3 ? row - ii * nf : row;
    const double2 ua = reinterpret_cast<const double2*>(u)[2 * q0];
    const double2 ub = reinterpret_cast<const double2*>(u)[2 * q0 + 1];
    const uint32_t L4 = reinterpret_cast<const uint32_t*>(lab_f)[q0];
    const int oi = ii & 1, oj = jj & 1;
    const int hi = ii >> 1, hj = jj >> 1;
    const int c0 = max(2 * m - 2, 0) + (int)OFF, c1 = max(2 * m - 1, 0) + (int)OFF, c2 = 2 * m + (int)OFF;
    double e0[NR], e1[NR], e2[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int cc0 = D == 3 ? r >> 1 : 0, cc1 = r & 1;
      const int ri = hi + (oi ? cc0 : 0), rj = hj + (oj ? cc1 : 0);
      const double* er = e + (D == 3 ? ((int64_t)ri * gc.n + rj) * gc.P : (int64_t)rj * gc.P);
      e0[r] = er[c0];
      e1[r] = er[c1];
      e2[r] = er[c2];
    }
    double pa[NC], pb[NC], pc[NC], pd[NC];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int cc0 = D == 3 ? r >> 1 : 0, cc1 = r & 1;
      const double wi = oi ? 0.5 : (cc0 == 0 ? 1.0 : 0.0);
      const double wj = oj ? 0.5 : (cc1 == 0 ? 1.0 : 0.0);
      const double wr = D == 3 ? (1.0 * wi) * wj : 1.0 * wj;
      // k = 4m-3 (odd): columns 2m-2, 2m-1, weights 1/2, 1/2
      pa[2 * r] = (wr * 0.5) * e0[r];
      pa[2 * r + 1] = (wr * 0.5) * e1[r];
      // k = 4m-2 (even): column 2m-1, weights 1, 0
      pb[2 * r] = (wr * 1.0) * e1[r];
      pb[2 * r + 1] = (wr * 0.0) * e1[r];
      // k = 4m-1 (odd): columns 2m-1, 2m
      pc[2 * r] = (wr * 0.5) * e1[r];
      pc[2 * r + 1] = (wr * 0.5) * e2[r];
      // k = 4m (even): column 2m
      pd[2 * r] = (wr * 1.0) * e2[r];
      pd[2 * r + 1] = (wr * 0.0) * e2[r];
    }
    auto upd = [](uint8_t L) { return L == INTERNAL || L == GHOST; };
    const uint8_t la = L4 & 0xFF, lb = (L4 >> 8) & 0xFF, lc = (L4 >> 16) & 0xFF, ld = L4 >> 24;
    if (upd(la) || upd(lb)) {
      double2 o = ua;
      if (upd(la)) o.x = ua.x + np_sum<NC>(pa);
      if (upd(lb)) o.y = ua.y + np_sum<NC>(pb);
      reinterpret_cast<double2*>(u)[2 * q0] = o;
    }
    if (upd(lc) || upd(ld)) {
      double2 o = ub;
      if (upd(lc)) o.x = ub.x + np_sum<NC>(pc);
      if (upd(ld)) o.y = ub.y + np_sum<NC>(pd);
      reinterpret_cast<double2*>(u)[2 * q0 + 1] = o;
    }
  }
}

void launch_interp_add(const Geom& gf, const uint8_t* lab_f, double* u_f, const Geom& gc,
                       const double* e_c, cudaStream_t st) {
  const int64_t nq = gf.rows * (gf.P / 4);
  const unsigned blocks = grid_for(nq, 256, 148 * 8);  // 4 to 64 CTAs per SM's worth measured the same (497-503 us at 512^3)
  if (gf.d == 3)
    interp_add4_kernel<3><<<blocks, 256, 0, st>>>(gf, lab_f, u_f, gc, e_c);
  else
    interp_add4_kernel<2><<<blocks, 256, 0, st>>>(gf, lab_f, u_f, gc, e_c);
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

// Jacobi transport steps (transfer.py:249-251):
// v_i <- v_i - 0.5 * sum_k |n_k| (v_i - v[i - step_k s_k]).
// The six steps run on a compact vector: slots [0, nb) hold the band nodes,
// slots [nb, nb + nfix) the non-band upwind neighbours (constant during the
// transport), and nbr[q][k] is the slot of node q's upwind neighbour along
// axis k (q itself for step 0).  Gather once, ping-pong six times between
// two L2-resident copies, scatter once -- instead of six full passes over
// scattered grid positions.
__global__ void band_gather_kernel(BandArgs a, const double* __restrict__ x) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= a.nb + a.nfix) return;
  const double v = t < a.nb ? x[a.idx[t]] : x[a.fixpos[t - a.nb]];
  a.v0[t] = v;
  if (t >= a.nb) a.v1[t] = v;
}

template <int D>
__global__ void __launch_bounds__(256) band_iter_kernel(BandArgs a, const double* __restrict__ vin,
                                                        double* __restrict__ vout) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= a.nb) return;
  const double vi = vin[q];
  double t[D];
#pragma unroll
  for (int k = 0; k < D; ++k) t[k] = a.absn[q * D + k] * (vi - vin[a.nbr[q * D + k]]);
  vout[q] = vi - 0.5 * seq_sum<D>(t);
}

__global__ void band_scatter_kernel(BandArgs a, const double* __restrict__ v, double* __restrict__ x) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < a.nb) x[a.idx[q]] = v[q];
}

void launch_band_transport(const BandArgs& a, double* x, cudaStream_t st) {
  if (a.nb == 0) return;
  const unsigned blocks = (unsigned)((a.nb + 255) / 256);
  const unsigned gblocks = (unsigned)((a.nb + a.nfix + 255) / 256);
  band_gather_kernel<<<gblocks, 256, 0, st>>>(a, x);
  for (int it = 0; it < 6; ++it) {
    const double* vin = (it & 1) ? a.v1 : a.v0;
    double* vout = (it & 1) ? a.v0 : a.v1;
    if (a.g.d == 3)
      band_iter_kernel<3><<<blocks, 256, 0, st>>>(a, vin, vout);
    else
      band_iter_kernel<2><<<blocks, 256, 0, st>>>(a, vin, vout);
  }
  band_scatter_kernel<<<blocks, 256, 0, st>>>(a, a.v0, x);  // six steps: result back in v0
}

// One Jacobi transport step on the grid vector itself (z-slab mode: the slabs exchange a halo plane
// of x between steps): gather, one step v0 -> v1, scatter v1.
void launch_band_step(const BandArgs& a, double* x, cudaStream_t st) {
  if (a.nb == 0) return;
  const unsigned blocks = (unsigned)((a.nb + 255) / 256);
  const unsigned gblocks = (unsigned)((a.nb + a.nfix + 255) / 256);
  band_gather_kernel<<<gblocks, 256, 0, st>>>(a, x);
  if (a.g.d == 3)
    band_iter_kernel<3><<<blocks, 256, 0, st>>>(a, a.v0, a.v1);
  else
    band_iter_kernel<2><<<blocks, 256, 0, st>>>(a, a.v0, a.v1);
  band_scatter_kernel<<<blocks, 256, 0, st>>>(a, a.v1, x);
}

// The whole band extension of a small level in one cooperative launch: the
// BFS groups, the gather, the six Jacobi steps and the scatter as phases of a
// grid-stride loop separated by grid-wide barriers -- the same per-node
// arithmetic as band_bfs_kernel / band_*_kernel, without ~11 launches.
// SINGLE: one CTA (any block size), __syncthreads() for the phase barriers -- bands of a few thousand
// nodes, where eleven grid-wide barriers (~2.5 us each) are most of the cooperative launch's time.
template <int D, bool SINGLE>
__global__ void __launch_bounds__(SINGLE ? 1024 : 256) band_coop_kernel(BandArgs a, double* __restrict__ x, int64_t g1,
                                                                        int64_t g2, int64_t g3) {
  cg::grid_group grid = cg::this_grid();
  auto phase_sync = [&]() {
    if (SINGLE)
      __syncthreads();
    else
      grid.sync();
  };
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, ts = (int64_t)gridDim.x * blockDim.x;
  const int64_t s[3] = {a.g.s0, a.g.s1, a.g.s2};
  const int64_t goff[4] = {0, g1, g2, g3};
  for (int gi = 0; gi < 3; ++gi) {
    if (goff[gi + 1] <= goff[gi]) continue;
    for (int64_t q = goff[gi] + t0; q < goff[gi + 1]; q += ts) {
      const int64_t i = a.idx[q];
      const unsigned mk = a.mask[q];
      double t[2 * D];
#pragma unroll
      for (int k = 0; k < D; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const bool bit = (mk >> (2 * k + j)) & 1u;
          t[2 * k + j] = bit ? x[j ? i + s[k] : i - s[k]] * 1.0 : 0.0;
        }
      x[i] = seq_sum<2 * D>(t) / (double)__popc(mk);
    }
    phase_sync();
  }
  for (int64_t q = t0; q < a.nb + a.nfix; q += ts) {
    const double v = q < a.nb ? x[a.idx[q]] : x[a.fixpos[q - a.nb]];
    a.v0[q] = v;
    if (q >= a.nb) a.v1[q] = v;
  }
  phase_sync();
  for (int it = 0; it < 6; ++it) {
    const double* vin = (it & 1) ? a.v1 : a.v0;
    double* vout = (it & 1) ? a.v0 : a.v1;
    for (int64_t q = t0; q < a.nb; q += ts) {
      const double vi = vin[q];
      double t[D];
#pragma unroll
      for (int k = 0; k < D; ++k) t[k] = a.absn[q * D + k] * (vi - vin[a.nbr[q * D + k]]);
      vout[q] = vi - 0.5 * seq_sum<D>(t);
    }
    phase_sync();
  }
  for (int64_t q = t0; q < a.nb; q += ts) x[a.idx[q]] = a.v0[q];
}

// returns false when the cooperative launch is not possible (caller falls back)
bool launch_band_coop(const BandArgs& a, double* x, const int64_t* goff, int ngroups, cudaStream_t st) {
  if (ngroups > 3) return false;
  int64_t g[3] = {0, 0, 0};
  for (int k = 0; k < 3; ++k) g[k] = goff[std::min(k + 1, ngroups)];
  static int occ[2] = {0, 0};
  int& o = occ[a.g.d == 3 ? 1 : 0];
  if (o == 0) {
    if (a.g.d == 3)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, band_coop_kernel<3, false>, 256, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, band_coop_kernel<2, false>, 256, 0);
    if (o < 1) o = 1;
  }
  BandArgs aa = a;
  if (a.nb + a.nfix <= 12288) {  // small band: one CTA, block barriers
    if (a.g.d == 3)
      band_coop_kernel<3, true><<<1, 1024, 0, st>>>(aa, x, g[0], g[1], g[2]);
    else
      band_coop_kernel<2, true><<<1, 1024, 0, st>>>(aa, x, g[0], g[1], g[2]);
    return true;
  }
  const int64_t want = (a.nb + a.nfix + 255) / 256;
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, 148 * (int64_t)std::min(o, 2)));
  void* args[] = {&aa, &x, &g[0], &g[1], &g[2]};
  cudaError_t e = a.g.d == 3 ? cudaLaunchCooperativeKernel((void*)band_coop_kernel<3, false>, blocks, 256, args, 0, st)
                             : cudaLaunchCooperativeKernel((void*)band_coop_kernel<2, false>, blocks, 256, args, 0, st);
  return e == cudaSuccess;
}

// Seeded initial field (reference solver.py:205-213, rng.py:14-56): value i of the xorshift64* stream
// on flat node i, 0 on inactive nodes.  The stream is cut into lanes of `len` values; thread l jumps
// to its lane's start state with the GF(2) powers of the state update (cols[b] = the 64 column images
// of step^(len * 2^b)), then steps through its lane.  Bit for bit the sequential stream.
__global__ void __launch_bounds__(128) initial_field_kernel(Geom g, const uint8_t* __restrict__ lab, double* __restrict__ u,
                                                            uint64_t state, const uint64_t* __restrict__ cols, int K,
                                                            int64_t len, int64_t nflat) {
  const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t i = l * len;
  if (i >= nflat) return;
  uint64_t s = state;
  for (int b = 0; b < K; ++b)
    if ((l >> b) & 1) {
      uint64_t o = 0;
      const uint64_t* c = cols + 64 * b;
      for (int k = 0; k < 64; ++k) o ^= ((s >> k) & 1ull) ? __ldg(c + k) : 0ull;
      s = o;
    }
  const int64_t end = min(nflat, i + len);
  int64_t row = i / g.n, col = i - row * g.n;
  for (; i < end; ++i) {
    s ^= s >> 12;
    s ^= s << 25;
    s ^= s >> 27;
    const uint64_t v = s * 2685821657736338717ull;
    const int64_t pos = row * g.P + col + OFF;
    u[pos] = lab[pos] == INACTIVE ? 0.0 : 2.0 * ((double)(v >> 11) * 0x1.0p-53) - 1.0;
    if (++col == g.n) {
      col = 0;
      ++row;
    }
  }
}

void launch_initial_field(const Geom& g, const uint8_t* labels, double* u, uint64_t state, const uint64_t* cols, int K,
                          int64_t len, cudaStream_t st) {
  const int64_t nflat = g.rows * g.n;
  const int64_t lanes = (nflat + len - 1) / len;
  initial_field_kernel<<<(unsigned)((lanes + 127) / 128), 128, 0, st>>>(g, labels, u, state, cols, K, len, nflat);
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

// NumPy pairwise sum of squares (the reference's (r**2).sum(), solver.py:138;
// SURVEY Appendix A.3) over a compacted vector, evaluated as its own tree:
// leaves of <= 128 consecutive elements (8 strided accumulators, fixed
// combine; < 8 elements: a left-to-right chain from -0), then every internal
// node = left + right, one launch per tree height.  The leaf segments and
// node list come from the host (the tree depends only on the length).
// leaf over the internal nodes of grid positions [start, end) in order
__global__ void l2_leaf_scan_kernel(const uint8_t* __restrict__ lab, const double* __restrict__ r,
                                    const int64_t* __restrict__ start, const int64_t* __restrict__ end,
                                    const int32_t* __restrict__ len, int64_t nleaves, double* __restrict__ vals) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nleaves) return;
  const int n = len[t];
  double acc[8];
  double res = -0.0;
  int i = 0;
  const int body = n - (n % 8);
  for (int64_t p = start[t]; p < end[t]; ++p) {
    if (lab[p] != INTERNAL) continue;
    const double v = r[p];
    const double sq = v * v;
    if (n < 8) {
      res = res + sq;
    } else if (i < 8) {
      acc[i] = sq;
    } else if (i < body) {
      acc[i & 7] = acc[i & 7] + sq;
    } else {
      if (i == body) res = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
      res = res + sq;
    }
    ++i;
  }
  if (n >= 8 && body == n) res = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  vals[t] = res;
}

// leaf over entries [off, off+len) of the lexicographic ghost list (value x[pos[slot[i]]])
__global__ void l2_leaf_list_kernel(const double* __restrict__ x, const int64_t* __restrict__ pos,
                                    const int32_t* __restrict__ slot, const int64_t* __restrict__ off,
                                    const int32_t* __restrict__ len, int64_t nleaves, double* __restrict__ vals) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nleaves) return;
  const int n = len[t];
  const int64_t o = off[t];
  double res = -0.0;
  if (n < 8) {
    for (int i = 0; i < n; ++i) {
      const double v = x[pos[slot[o + i]]];
      res = res + v * v;
    }
  } else {
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double v = x[pos[slot[o + j]]];
      acc[j] = v * v;
    }
    const int body = n - (n % 8);
    for (int i = 8; i < body; i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double v = x[pos[slot[o + i + j]]];
        acc[j] = acc[j] + v * v;
      }
    res = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    for (int i = body; i < n; ++i) {
      const double v = x[pos[slot[o + i]]];
      res = res + v * v;
    }
  }
  vals[t] = res;
}

// internal nodes of one tree height: vals[dst[k]] = vals[a[k]] + vals[b[k]]
__global__ void l2_combine_kernel(double* __restrict__ vals, const int32_t* __restrict__ a,
                                  const int32_t* __restrict__ b, const int32_t* __restrict__ dst, int64_t n) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) vals[dst[k]] = vals[a[k]] + vals[b[k]];
}

void launch_l2_leaves_scan(const uint8_t* lab, const double* r, const int64_t* start, const int64_t* end,
                           const int32_t* len, int64_t nleaves, double* vals, cudaStream_t st) {
  if (nleaves > 0)
    l2_leaf_scan_kernel<<<(unsigned)((nleaves + 127) / 128), 128, 0, st>>>(lab, r, start, end, len, nleaves, vals);
}

void launch_l2_leaves_list(const double* x, const int64_t* pos, const int32_t* slot, const int64_t* off,
                           const int32_t* len, int64_t nleaves, double* vals, cudaStream_t st) {
  if (nleaves > 0)
    l2_leaf_list_kernel<<<(unsigned)((nleaves + 127) / 128), 128, 0, st>>>(x, pos, slot, off, len, nleaves, vals);
}

void launch_l2_combine(double* vals, const int32_t* a, const int32_t* b, const int32_t* dst, int64_t n,
                       cudaStream_t st) {
  if (n > 0) l2_combine_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(vals, a, b, dst, n);
}

// Host-layout <-> padded device layout: row r of length n sits at
// r * n in the contiguous (host) array and at r * P + OFF on the device.
// The host copy is one contiguous DMA into a staging buffer; these kernels
// re-pitch on the device (a 2-D memcpy with 4 KB rows runs far below the
// PCIe / C2C rate).
template <bool TO_PADDED>
__global__ void __launch_bounds__(256) repitch_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                                      int64_t rows, int64_t n, int64_t P) {
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const double* s = TO_PADDED ? src + r * n : src + r * P + OFF;
    double* d = TO_PADDED ? dst + r * P + OFF : dst + r * n;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) d[k] = s[k];
  }
}

void launch_repitch(const double* src, double* dst, int64_t rows, int64_t n, int64_t P, bool to_padded,
                    cudaStream_t st) {
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(rows, 148 * 16));
  if (to_padded)
    repitch_kernel<true><<<blocks, 256, 0, st>>>(src, dst, rows, n, P);
  else
    repitch_kernel<false><<<blocks, 256, 0, st>>>(src, dst, rows, n, P);
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
