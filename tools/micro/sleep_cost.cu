// Micro-benchmark: actual duration of __nanosleep(n) and of an L2 poll
// (ld.relaxed.gpu) from one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kern(long long* out, int* flag) {
  long long t0 = clock64();
  for (int i = 0; i < 100; ++i) __nanosleep(20);
  long long t1 = clock64();
  for (int i = 0; i < 100; ++i) __nanosleep(200);
  long long t2 = clock64();
  int acc = 0;
  for (int i = 0; i < 100; ++i) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag + acc * 0) : "memory");
    acc += v;
  }
  long long t3 = clock64();
  for (int i = 0; i < 100; ++i) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag + acc * 0) : "memory");
    acc += v;
  }
  long long t4 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = acc; }
}
int main() {
  long long* d; int* f; cudaMalloc(&d, 64); cudaMalloc(&f, 64); cudaMemset(f, 0, 64);
  long long h[5];
  for (int r = 0; r < 2; ++r) {
    kern<<<1, 32>>>(d, f);
    cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
    printf("nanosleep(20): %.0f cyc, nanosleep(200): %.0f cyc, ld.relaxed.gpu poll: %.0f cyc, ld.acquire.gpu: %.0f cyc\n",
           h[0] / 100.0, h[1] / 100.0, h[2] / 100.0, h[3] / 100.0);
  }
  return 0;
}
