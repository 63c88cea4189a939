// Micro-benchmark: cost of mbarrier try_wait / test_wait on an already
// completed phase, and of an ld.acquire.cta / plain ld.shared poll.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void kern(long long* out, int reps) {
  __shared__ unsigned long long bar;
  __shared__ int flag;
  const unsigned b = sa(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(1) : "memory");
    flag = 5;
  }
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
  __syncthreads();
  unsigned ok = 0, acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(b), "r"(0) : "memory");
    acc += ok;
  }
  long long t1 = clock64();
  for (int i = 0; i < reps; ++i) {
    asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(b), "r"(0) : "memory");
    acc += ok;
  }
  long long t2 = clock64();
  for (int i = 0; i < reps; ++i) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(sa(&flag)) : "memory");
    acc += v;
  }
  long long t3 = clock64();
  for (int i = 0; i < reps; ++i) {
    int v;
    asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"(sa(&flag)) : "memory");
    acc += v;
  }
  long long t4 = clock64();
  for (int i = 0; i < reps; ++i) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(sa(&flag)), "r"(i) : "memory");
  }
  long long t5 = clock64();
  // dependent chain: next barrier address depends on the previous result
  unsigned bb = b;
  for (int i = 0; i < reps; ++i) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(bb), "r"(0) : "memory");
    bb = b + (ok - 1) * 8;
  }
  long long t6 = clock64();
  int fv = 0;
  unsigned fa = sa(&flag);
  for (int i = 0; i < reps; ++i) {
    int v;
    asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"(fa) : "memory");
    fa = sa(&flag) + (v == -12345 ? 4 : 0);
    fv += v;
  }
  long long t7 = clock64();
  if (threadIdx.x == 0) {
    out[6] = t6 - t5; out[7] = t7 - t6 + (bb == 0) + (fv == 1);
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; out[5] = acc;
  }
}
int main() {
  long long* d; cudaMalloc(&d, 64); long long h[8];
  const int reps = 10000;
  for (int r = 0; r < 2; ++r) {
    kern<<<1, 32>>>(d, reps);
    printf("launch: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("dependent try_wait %.1f, dependent ld.volatile %.1f\n", (double)h[6] / reps, (double)h[7] / reps);
    printf("try_wait %.1f  test_wait %.1f  ld.acquire.cta %.1f  ld.volatile %.1f  st.release.cta %.1f cycles\n",
           (double)h[0] / reps, (double)h[1] / reps, (double)h[2] / reps, (double)h[3] / reps, (double)h[4] / reps);
  }
  return 0;
}
