// Dependent-chain latency probes (clock64), one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b;
  __shared__ double sm[64];
  sm[threadIdx.x] = a;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x + y; x = x + y; x = x + y; x = x + y; }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) { x = x * y; x = x * y; x = x * y; x = x * y; }
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, y, a); x = fma(x, y, a); x = fma(x, y, a); x = fma(x, y, a); }
  long long t3 = clock64();
  double z = x;
  for (int i = 0; i < n; ++i) { z = __shfl_up_sync(0xffffffff, z, 1) + y; }
  long long t4 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < n; ++i) { double v = sm[idx]; idx = (int)v & 31; idx += threadIdx.x & 1; }
  long long t5 = clock64();
  float fx = (float)a, fy = (float)b;
  for (int i = 0; i < n; ++i) { fx = fx + fy; fx = fx + fy; fx = fx + fy; fx = fx + fy; }
  long long t6 = clock64();
  out[threadIdx.x] = x + z + idx + fx;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 512); cudaMallocManaged(&c, 64);
  int n = 4096;
  k<<<1, 32>>>(o, c, 1.0000001, 1e-9, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.0000001, 1e-9, n); cudaDeviceSynchronize();
  printf("DADD %.2f  DMUL %.2f  DFMA %.2f  SHFL+DADD %.2f  LDS.64+cvt %.2f  FADD %.2f cycles\n",
         c[0] / (4.0 * n), c[1] / (4.0 * n), c[2] / (4.0 * n), c[3] / (1.0 * n), c[4] / (1.0 * n), c[5] / (4.0 * n));
  return 0;
}
