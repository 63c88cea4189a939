// gs_small.cu -- lexicographic Gauss-Seidel sweep of a small level by ONE CTA:
// hyperplane wavefront i0 + i1 (+ i2) = s, one barrier per hyperplane.
//
// Reference: gs_lex_sweep, /root/reference/pkg/src/ghostmg/smoothing.py:127-132.
// The nodes of a hyperplane do not depend on one another and every node's
// "earlier" neighbours lie on the previous hyperplane, so sweeping the
// hyperplanes in order reproduces the sequential lexicographic sweep value
// for value.  Levels with N <= 32 (3-D) / N < 64 (2-D) have at most ~1000
// nodes per hyperplane and fewer than 100 of them: a multi-CTA pipeline with
// flags through L2 (gs_stream.cu, gs_sweep.cu) spends 100-240 us per sweep on
// hand-offs there, one CTA with __syncthreads() a few tens.
//
// Arithmetic per node as in gs_sweep.cu (bitwise the oracle's):
// S = ((((u[i-s0] + u[i+s0]) + u[i-s1]) + u[i+s1]) + u[i-s2]) + u[i+s2],
// u_i = (h^2 f_i + (S + 0)) * (1 / denom).
#include "gmg_kernels.cuh"

namespace gmg {

template <int DIM>
__global__ void __launch_bounds__(1024) gs_small_kernel(Geom g, const uint8_t* __restrict__ labels, double* u,
                                                       const double* __restrict__ f) {
  const int M = (int)g.N - 1;
  const int per = DIM == 3 ? M * M : M;
  for (int s = DIM; s <= DIM * M; ++s) {
    for (int q = threadIdx.x; q < per; q += blockDim.x) {
      int i0, i1 = 0, k;
      if (DIM == 3) {
        i0 = q / M + 1;
        i1 = q - (i0 - 1) * M + 1;
        k = s - i0 - i1;
      } else {
        i0 = q + 1;
        k = s - i0;
      }
      if (k < 1 || k > M) continue;
      const int64_t node = DIM == 3 ? (int64_t)i0 * g.s0 + (int64_t)i1 * g.s1 + k + OFF : (int64_t)i0 * g.s0 + k + OFF;
      if (labels[node] != INTERNAL) continue;
      double sum;
      if (DIM == 3)
        sum = ((((u[node - g.s0] + u[node + g.s0]) + u[node - g.s1]) + u[node + g.s1]) + u[node - 1]) + u[node + 1];
      else
        sum = ((u[node - g.s0] + u[node + g.s0]) + u[node - 1]) + u[node + 1];
      sum = sum + 0.0;
      u[node] = (g.h2 * f[node] + sum) * g.inv;
    }
    __syncthreads();
  }
}

void launch_gs_small(const Geom& g, const uint8_t* labels, double* u, const double* f, cudaStream_t st) {
  if (g.d == 3)
    gs_small_kernel<3><<<1, 1024, 0, st>>>(g, labels, u, f);
  else
    gs_small_kernel<2><<<1, 1024, 0, st>>>(g, labels, u, f);
}

}  // namespace gmg
