// gmg_common.cuh -- shared device helpers for the ghost-point multigrid
// kernels (sm_100a).
//
// Every kernel reproduces the floating-point evaluation order of the
// reference package (/root/reference/pkg/src/ghostmg) as NumPy/OpenBLAS
// execute it.  The library is compiled with
// --fmad=false so that a*b+c is never contracted; the only FMAs are the
// explicit __fma_rn calls that restate OpenBLAS ddot.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gmg {

enum Label : uint8_t { INTERNAL = 0, GHOST = 1, INACTIVE = 2, ELIMINATED = 3, PAD = 4 };

// Left-to-right sum of n < 8 terms, then + 0.0: NumPy's add.reduce over a
// short axis (an all-zero result comes out as +0).
template <int N>
__device__ __forceinline__ double seq_sum(const double (&a)[N]) {
  double s = a[0];
#pragma unroll
  for (int i = 1; i < N; ++i) s = s + a[i];
  return s + 0.0;
}

// NumPy pairwise_sum for 8 <= N <= 128: eight strided partial sums, a
// fixed tree, then the tail left to right; + 0.0 from the reduction.
template <int N>
__device__ __forceinline__ double np_sum(const double (&a)[N]) {
  if constexpr (N < 8) {
    return seq_sum<N>(a);
  } else {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    constexpr int body = N - (N % 8);
#pragma unroll
    for (int i = 8; i < body; i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = r[j] + a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
#pragma unroll
    for (int i = body; i < N; ++i) res = res + a[i];
    return res + 0.0;
  }
}

// OpenBLAS 0.3.30 ddot on the SkylakeX core (the reference's
// `co[t] @ u[st[t]]`, smoothing.py:142): n < 16 is an FMA chain from 0;
// n = 27 runs four mul+add lanes over i < 16, combines (L0+L2)+(L1+L3) and
// finishes with an FMA chain over i >= 16.
template <int N>
__device__ __forceinline__ double blas_ddot(const double (&x)[N], const double (&y)[N]) {
  if constexpr (N < 16) {
    double d = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) d = __fma_rn(x[i], y[i], d);
    return d;
  } else {
    double L[4] = {0.0, 0.0, 0.0, 0.0};
    constexpr int body = N & ~15;
#pragma unroll
    for (int i = 0; i < body; i += 4)
#pragma unroll
      for (int l = 0; l < 4; ++l) L[l] = L[l] + __dmul_rn(x[i + l], y[i + l]);
    double d = (L[0] + L[2]) + (L[1] + L[3]);
#pragma unroll
    for (int i = body; i < N; ++i) d = __fma_rn(x[i], y[i], d);
    return d;
  }
}

// max-reduction of non-negative doubles (and NaN, whose bit pattern orders
// above +inf) through their uint64 images.
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* slot, double v) {
  unsigned long long bits = __double_as_longlong(v);
  atomicMax(slot, bits);
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double w = __shfl_xor_sync(0xffffffffu, v, o);
    // NaN-propagating max on non-negative values: compare bit patterns
    v = (__double_as_longlong(w) > __double_as_longlong(v)) ? w : v;
  }
  return v;
}

// Device grid layout: rows along the fastest axis are padded to a pitch P
// (multiple of 4 doubles, >= N + 4) and node k of a row sits at column
// k + OFF with OFF = 3, so column k0 = 1 + 32c of every row is 32-byte
// aligned.  pos(i0, i1, k) = (i0 * n + i1) * P + k + OFF in 3-D,
// i0 * P + k + OFF in 2-D.  Padding columns carry label PAD and value 0.
constexpr int64_t OFF = 3;

struct Geom {
  int d;               // 2 or 3
  int64_t N;           // cells per axis
  int64_t n;           // N + 1 nodes per axis
  int64_t P;           // row pitch (doubles)
  int64_t rows;        // n^2 (3-D) or n (2-D)
  int64_t s0, s1, s2;  // position strides of axes 0, 1, 2 (the fastest axis has stride 1)
  int64_t nodes;       // allocated positions = rows * P
  double h2, denom, inv, c;  // h^2, 2d + reaction h^2, 1/denom, denom/h^2
  double rh2;                // 1/h^2; exact stand-in for "/ h2" when h2 is a power of two
  int h2pow2;                // h2 is a power of two (then x / h2 == x * rh2 bit for bit)
};

// x / h^2 as the reference computes it; a multiply when that is exact
__device__ __forceinline__ double div_h2(const Geom& g, double x) { return g.h2pow2 ? x * g.rh2 : x / g.h2; }

// position -> multi-index (m[d-1] is the fastest axis); returns false on padding
__device__ __forceinline__ bool pos_multi(const Geom& g, int64_t pos, int64_t* m) {
  const int64_t row = pos / g.P;
  const int64_t k = pos - row * g.P - OFF;
  if (g.d == 3) {
    m[0] = row / g.n;
    m[1] = row - m[0] * g.n;
    m[2] = k;
  } else {
    m[0] = row;
    m[1] = k;
  }
  return k >= 0 && k <= g.N;
}

__device__ __forceinline__ int64_t multi_pos(const Geom& g, const int64_t* m) {
  if (g.d == 3) return (m[0] * g.n + m[1]) * g.P + m[2] + OFF;
  return m[0] * g.P + m[1] + OFF;
}

}  // namespace gmg
