// coarse_dense.cu -- device coarsest-level solve x = A^{-1} rhs (sm_100a).
//
// Optional replacement for the reference's host SuperLU solve
// (/root/reference/pkg/src/ghostmg/solver.py:146-166): the coarsest operator
// (a few 10^4 unknowns for the pore-space hierarchy) is inverted once at
// setup and every cycle applies the dense inverse with an HBM-streaming
// GEMV.  Deterministic: the column range is cut into fixed chunks, each
// (row, chunk) partial is a fixed warp-shuffle tree, and the chunk partials
// are added in chunk order.  Not bitwise equal to SuperLU (the reference's
// own solve is only reproducible by calling SuperLU), so it is an opt-in
// mode; tests bound its effect on residual histories.
#include <algorithm>

#include "gmg_kernels.cuh"

namespace gmg {

constexpr int GEMV_CHUNK = 8192;  // columns per chunk (64 KB of rhs in shared memory)
constexpr int GEMV_ROWS = 64;     // rows per CTA

__global__ void __launch_bounds__(256) gemv_partial_kernel(const double* __restrict__ A, const double* __restrict__ x,
                                                           int64_t n, double* __restrict__ part) {
  extern __shared__ double xs[];
  const int ch = blockIdx.y;
  const int64_t c0 = (int64_t)ch * GEMV_CHUNK;
  const int len = (int)min((int64_t)GEMV_CHUNK, n - c0);
  for (int i = threadIdx.x; i < len; i += blockDim.x) xs[i] = x[c0 + i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * GEMV_ROWS;
  for (int rr = warp; rr < GEMV_ROWS; rr += 8) {
    const int64_t row = r0 + rr;
    if (row >= n) break;
    const double* a = A + row * n + c0;
    double s0 = 0.0, s1 = 0.0;
    int j = lane;
    for (; j + 32 < len; j += 64) {
      s0 = __fma_rn(__ldcs(a + j), xs[j], s0);
      s1 = __fma_rn(__ldcs(a + j + 32), xs[j + 32], s1);
    }
    if (j < len) s0 = __fma_rn(__ldcs(a + j), xs[j], s0);
    double s = s0 + s1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) part[(int64_t)ch * n + row] = s;
  }
}

__global__ void gemv_reduce_kernel(const double* __restrict__ part, int64_t n, int nch, double* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = part[i];
  for (int c = 1; c < nch; ++c) s += part[(int64_t)c * n + i];
  y[i] = s;
}

__global__ void gemv_rect_partial_kernel(const double* __restrict__ A, const double* __restrict__ x, int64_t m,
                                         int64_t k, int chunk, double* __restrict__ part);

void configure_dense_gemv() {
  cudaFuncSetAttribute(gemv_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(GEMV_CHUNK * sizeof(double)));
  cudaFuncSetAttribute(gemv_rect_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(GEMV_CHUNK * sizeof(double)));
}

int gemv_chunks(int64_t n) { return (int)((n + GEMV_CHUNK - 1) / GEMV_CHUNK); }

void launch_dense_gemv(const double* A, const double* x, int64_t n, double* part, double* y, cudaStream_t st) {
  const int nch = gemv_chunks(n);
  dim3 grid((unsigned)((n + GEMV_ROWS - 1) / GEMV_ROWS), (unsigned)nch);
  gemv_partial_kernel<<<grid, 256, GEMV_CHUNK * sizeof(double), st>>>(A, x, n, part);
  gemv_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, n, nch, y);
}

// Rectangular variant for the nested-dissection coarse solve: y = M x or
// y = y0 - M x with M row-major m x k; the k range is cut into `chunk`
// columns (<= GEMV_CHUNK) so short-and-wide blocks still fill the GPU.
__global__ void __launch_bounds__(256) gemv_rect_partial_kernel(const double* __restrict__ A,
                                                                const double* __restrict__ x, int64_t m,
                                                                int64_t k, int chunk, double* __restrict__ part) {
  extern __shared__ double xs[];
  const int ch = blockIdx.y;
  const int64_t c0 = (int64_t)ch * chunk;
  const int len = (int)min((int64_t)chunk, k - c0);
  for (int i = threadIdx.x; i < len; i += blockDim.x) xs[i] = x[c0 + i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * GEMV_ROWS;
  for (int rr = warp; rr < GEMV_ROWS; rr += 8) {
    const int64_t row = r0 + rr;
    if (row >= m) break;
    const double* a = A + row * k + c0;
    // four independent accumulators (4 loads per lane in flight), fixed order
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int j = lane;
    for (; j + 96 < len; j += 128) {
      const double a0 = __ldcs(a + j), a1 = __ldcs(a + j + 32), a2 = __ldcs(a + j + 64), a3 = __ldcs(a + j + 96);
      s0 = __fma_rn(a0, xs[j], s0);
      s1 = __fma_rn(a1, xs[j + 32], s1);
      s2 = __fma_rn(a2, xs[j + 64], s2);
      s3 = __fma_rn(a3, xs[j + 96], s3);
    }
    for (; j < len; j += 32) s0 = __fma_rn(__ldcs(a + j), xs[j], s0);
    double s = (s0 + s1) + (s2 + s3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) part[(int64_t)ch * m + row] = s;
  }
}

__global__ void gemv_rect_reduce_kernel(const double* __restrict__ part, int64_t m, int nch,
                                        const double* __restrict__ y0, double* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s = part[i];
  for (int c = 1; c < nch; ++c) s += part[(int64_t)c * m + i];
  y[i] = y0 ? y0[i] - s : s;
}

// t[i] = y0[i] - sum_k val[k] * x[col[k]] over row i of a CSR matrix (one
// warp per row, fixed shuffle tree): the separator coupling A_S,AB applied to
// the half solves, instead of the dense G = A_S,AB blkdiag(AAi, BBi).
__global__ void csr_residual_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                    const double* __restrict__ val, const double* __restrict__ x,
                                    const double* __restrict__ y0, int64_t m, double* __restrict__ t) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  double s = 0.0;
  for (int64_t k = rowptr[row] + lane; k < rowptr[row + 1]; k += 32) s = __fma_rn(val[k], x[col[k]], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) t[row] = y0[row] - s;
}

void launch_csr_residual(const int64_t* rowptr, const int32_t* col, const double* val, const double* x,
                         const double* y0, int64_t m, double* t, cudaStream_t st) {
  if (m > 0) csr_residual_kernel<<<(unsigned)((m * 32 + 255) / 256), 256, 0, st>>>(rowptr, col, val, x, y0, m, t);
}

int gemv_rect_chunk(int64_t m, int64_t k) {
  // enough (row block, chunk) CTAs for ~4 per SM
  const int64_t rb = (m + GEMV_ROWS - 1) / GEMV_ROWS;
  int64_t want = (148 * 4 + rb - 1) / rb;
  int64_t chunk = (k + want - 1) / want;
  chunk = ((chunk + 255) / 256) * 256;
  return (int)std::max<int64_t>(256, std::min<int64_t>(chunk, GEMV_CHUNK));
}

int64_t gemv_rect_part_size(int64_t m, int64_t k) {
  const int chunk = gemv_rect_chunk(m, k);
  return ((k + chunk - 1) / chunk) * m;
}

void launch_gemv_rect(const double* A, const double* x, int64_t m, int64_t k, double* part, const double* y0,
                      double* y, cudaStream_t st) {
  if (m <= 0) return;
  const int chunk = gemv_rect_chunk(m, k);
  const int nch = (int)((k + chunk - 1) / chunk);
  dim3 grid((unsigned)((m + GEMV_ROWS - 1) / GEMV_ROWS), (unsigned)nch);
  gemv_rect_partial_kernel<<<grid, 256, chunk * sizeof(double), st>>>(A, x, m, k, chunk, part);
  gemv_rect_reduce_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(part, m, nch, y0, y);
}

}  // namespace gmg
