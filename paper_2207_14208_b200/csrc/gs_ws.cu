// gs_ws.cu -- warp-specialised lexicographic Gauss-Seidel sweep (sm_100a):
// the production GS kernel for levels with N >= 64.
//
// Same decomposition, line skew and inter-task progress protocol as
// gs_stream.cu (a task = 32-column chunk c x block b of R = 16 rows x all
// planes; lane j of the compute warp one line behind lane j-1), but each CTA
// runs one task with two warps:
//
//  * warp 1 (producer) moves the task's lines into shared rings with TMA
//    tensor copies, 8 lines per instruction -- u columns k0-2..k0+33 (the
//    new left halo from chunk c-1, the task's 32 columns and the old right
//    halo), f columns k0..k0+31 and the 8 internal-bitmask words -- plus,
//    at each plane start, the new row above / old row below the block with
//    1-D bulk copies.  It polls the neighbour tasks' progress words first
//    (ld.acquire.gpu), prefetches 64 lines ahead into L2
//    (cp.async.bulk.prefetch.tensor), writes every finished line back with a
//    TMA bulk store and publishes the task's progress (st.release.gpu after
//    the stores completed);
//  * warp 0 (consumer) waits on one mbarrier per 8 lines and otherwise only
//    runs the dependent Gauss-Seidel chain from shared memory.
//
// In 3-D every block has R = 16 rows; the last block's 16th row is the
// boundary row N (no internal node), so every batch of 8 lines is 8
// consecutive rows of the device layout, i.e. one TMA box.
//
// Reference: gs_lex_sweep, /root/reference/pkg/src/ghostmg/smoothing.py:127-132.
#include <cstddef>

#include "gmg_kernels.cuh"

namespace gmg {

namespace {

constexpr int RU = 96;        // u ring lines
constexpr int RF = 80;        // f / mask ring lines
constexpr int G = 8;          // lines per batch (TMA box height)
constexpr int NB = 12;        // mbarriers (>= RU / G)
constexpr int RPW = 8;        // plane-row slots (3-D)
constexpr int L2AHEAD = 64;   // L2 prefetch distance (lines)
constexpr int UPITCH = 36;    // u row: [k0-2, k0-1 | k0..k0+31 | k0+32, k0+33]
constexpr unsigned BATCH_BYTES = G * (UPITCH * 8 + 32 * 8 + 16);

struct __align__(128) WsSmem {
  double u[RU][UPITCH];   // pitch 36: lane j on row t-j -> bank pair (c - 35 j) mod 16, conflict free
  double f[RF][32];       // pitch 32: (c - 31 j) mod 16, conflict free
  uint32_t mask[RF][4];   // 16-B chunk of the line's bitmask words, word c & 3
  double up[RPW][32];     // row above the block (new values), 3-D
  double dn[RPW][32];     // row below the block (old values), 3-D
  unsigned long long full[NB];
  int cons_step;          // consumer: last completed step
  int task;               // ticket broadcast
};

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load_2d(unsigned dst, const void* map, int x, int y, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const void* map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, unsigned src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(sa(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(sa(p)), "r"(v) : "memory");
}
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int floordiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

}  // namespace

template <int DIM>
__global__ void __launch_bounds__(64, 1) gs_ws_kernel(GsArgs a, const __grid_constant__ WsMaps maps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  WsSmem& S = *reinterpret_cast<WsSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const Geom g = a.g;
  const int N = (int)g.N;
  double* __restrict__ u = a.u;
  constexpr int R = DIM == 3 ? 16 : 1;

  for (;;) {
    if (threadIdx.x == 32) {
      S.task = atomicAdd(a.ticket, 1);
      for (int i = 0; i < NB; ++i) mbar_init(sa(&S.full[i]), 1);
      S.cons_step = -1;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      fence_async_shared();
    }
    __syncthreads();
    const int tid = S.task;
    if (tid >= a.ntasks) return;
    const int2 tk = a.tasks[tid];
    const int c = tk.x, b = tk.y;
    const int k0 = 1 + 32 * c;
    // 2-D runs one dummy line (row N, no internal node) so line counts are multiples of 8
    const int nLines = DIM == 3 ? (N - 1) * R : N;
    const int uEnd = nLines + R;  // u lines run over [-R, nLines + R)
    const int rowbase = DIM == 3 ? 1 + b * 16 : 0;
    // tensor row of line L (plane p = floor(L / R), row r): (p + 1) * n + rowbase + r in 3-D,
    // L + 1 in 2-D; a batch of 8 lines starting at L0 = 8 q - R never crosses a plane.
    auto trow = [&](int L) -> int {
      if (DIM == 3) {
        const int p = floordiv(L, R);
        return (int)((p + 1) * g.n) + rowbase + (L - p * R);
      }
      return L + 1;
    };
    const int last = nLines + 30;  // last consumer step
    long long* const tr = a.trace ? a.trace + (int64_t)tid * 24 : nullptr;

    if (warp == 1) {
      // =============================== producer ===========================
      if (lane == 0) {
        int* myprog = a.progress + c * a.Bn + b;
        const int* lprog = c > 0 ? a.progress + (c - 1) * a.Bn + b : nullptr;
        const int* uprog = (DIM == 3 && b > 0) ? a.progress + c * a.Bn + (b - 1) : nullptr;
        int seenL = 0, seenU = 0;
        const int nbatches = (uEnd + R + G - 1) / G;  // Lr = L + R over [0, uEnd + R)
        const int nwb = nLines / G;           // write-back batches (nLines multiple of G)
        const int ux = k0 + (int)OFF - 2, fx = k0 + (int)OFF, mx = c & ~3;
        int q = 0, w = 0, published = 0, l2q = L2AHEAD / G;
        long long waitL = 0, waitU = 0, idle = 0;
        while (q < nbatches || published < nLines) {
          const int cs = ld_acquire_cta(&S.cons_step);
          bool did = false;
          // ---- write back finished batches (line L done at step L + 31)
          while (w < nwb && cs >= w * G + G - 1 + 31) {
            for (int i = 0; i < G; ++i) {
              const int L = w * G + i;
              const int64_t row = trow(L);
              bulk_store(u + row * g.P + fx, sa(&S.u[(L + R) % RU][2]), 256u);
            }
            bulk_commit();
            ++w;
            did = true;
          }
          // ---- publish progress; the newest 2 store groups may be in flight
          if (w == nwb && published < nLines) {
            bulk_wait<0>();
            fence_async_global();
            st_release(myprog, nLines);
            published = nLines;
          } else if (w >= 3 && (w - 2) * G >= published + 16) {
            bulk_wait<2>();
            fence_async_global();
            st_release(myprog, (w - 2) * G);
            published = (w - 2) * G;
          }
          // ---- load the next batch once its ring slots are free
          if (q < nbatches) {
            const int L0 = q * G - R;
            // u slots last used by lines L0-RU.., f slots by L0-RF..
            const int lastU = L0 - RU + G - 1, lastF = L0 - RF + G - 1;
            bool ok = cs >= lastU + R + 31 && cs >= lastF + 31;
            if (ok && lastU >= 0) {
              const int need_w = min(lastU, nLines - 1) / G + 1;
              ok = w >= need_w;
              if (ok) {
                if (need_w <= w - 2)
                  bulk_wait_read<2>();
                else
                  bulk_wait_read<0>();
              }
            }
            if (ok) {
              const int lastreal = min(L0 + G, nLines) - 1;
              if (lprog && lastreal >= 0 && seenL < lastreal + 1) {
                const long long c0 = tr ? clock64() : 0;
                while (seenL < lastreal + 1) seenL = ld_acquire(lprog);
                if (tr) waitL += clock64() - c0;
              }
              const bool pstart = DIM == 3 && L0 >= 0 && L0 < nLines && (L0 % R) == 0;
              if (uprog && pstart) {
                const int need = (L0 / R + 1) * 16;
                const long long c0 = tr ? clock64() : 0;
                while (seenU < need) seenU = ld_acquire(uprog);
                if (tr) waitU += clock64() - c0;
              }
              fence_async_global();
              const unsigned bar = sa(&S.full[q % NB]);
              mbar_expect_tx(bar, BATCH_BYTES + (pstart ? 512u : 0u));
              const int y = trow(L0);
              const int su = (L0 + R) % RU, sf = (L0 + R) % RF;
              tma_load_2d(sa(&S.u[su][0]), &maps.u, ux, y, bar);
              tma_load_2d(sa(&S.f[sf][0]), &maps.f, fx, y, bar);
              tma_load_2d(sa(&S.mask[sf][0]), &maps.m, mx, y, bar);
              if (pstart) {
                const int sp = (L0 / R) & (RPW - 1);
                const int64_t up_row = y - 1;
                const int64_t dn_row = y + min(R, N - rowbase);  // row rowbase + R, clamped to N
                bulk_load(sa(&S.up[sp][0]), u + up_row * g.P + fx, 256u, bar);
                bulk_load(sa(&S.dn[sp][0]), u + dn_row * g.P + fx, 256u, bar);
              }
              // L2 prefetch L2AHEAD lines ahead
              for (; l2q < min(q + 1 + L2AHEAD / G, nbatches); ++l2q) {
                const int yl = trow(l2q * G - R);
                tma_prefetch_2d(&maps.u, ux, yl);
                tma_prefetch_2d(&maps.f, fx, yl);
              }
              ++q;
              did = true;
            }
          }
          if (!did) {
            ++idle;
            __nanosleep(32);
          }
        }
        bulk_wait<0>();
        if (tr) {
          tr[5] = waitL;
          tr[6] = waitU;
          tr[7] = idle;
        }
      }
      __syncwarp();
    } else {
      // =============================== consumer ===========================
      // Software-pipelined: everything step t+1 needs except u[k-1] (written
      // by lane j-1 during step t) is loaded and partially summed at the end
      // of step t, so the loop-carried chain is only
      // ld.shared u[k-1] -> +, +, + -> * -> select -> st.shared.
      const double h2 = g.h2, inv = g.inv;
      const bool kval = k0 + lane <= N - 1;
      const int mword = c & 3;
      int ready = 0;
      long long cwait = 0;
      const long long cstart = clock64();
      if (tr && lane == 0) {
        tr[0] = gtimer();
        unsigned sm;
        asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
        tr[2] = sm;
      }
      auto wait_lines = [&](int t) {
        // lines up to t + R must be resident: batch of Lr = t + 2R
        while (ready * G <= min(t + 2 * R, uEnd + R - 1)) {
          const unsigned bar = sa(&S.full[ready % NB]);
          const unsigned par = (unsigned)((ready / NB) & 1);
          if (!mbar_try_wait(bar, par)) {
            const long long c0 = tr ? clock64() : 0;
            while (!mbar_try_wait(bar, par)) {
            }
            if (tr) cwait += clock64() - c0;
          }
          ++ready;
        }
      };
      int cr, cpl;  // row / plane of this lane's line t - lane
      {
        const int L0 = -lane;
        cpl = floordiv(L0, R);
        cr = L0 - cpl * R;
      }
      int su = ((R - lane) % RU + RU) % RU;  // u slot of line t - lane at t = 0
      int sf = ((R - lane) % RF + RF) % RF;
      // staged operands of the coming step
      double p4, kp, hf, old;
      bool upd;
      auto stage = [&](int t, double prevv) {
        const int nl = t - lane;
        int sm = su - R;
        sm += sm < 0 ? RU : 0;
        int sp = su + R;
        sp -= sp >= RU ? RU : 0;
        int s1 = su + 1;
        s1 -= s1 >= RU ? RU : 0;
        const double a0m = S.u[sm][lane + 2];
        const double a0p = S.u[sp][lane + 2];
        old = S.u[su][lane + 2];
        kp = S.u[su][lane + 3];
        hf = h2 * S.f[sf][lane] + 0.0;  // (h2 f + 0) + S == h2 f + (S + 0)
        const bool internal = (S.mask[sf][mword] >> lane) & 1u;
        upd = kval && nl >= 0 && nl < nLines && internal;
        if (DIM == 3) {
          const int pw = cpl & (RPW - 1);
          const double upv = S.up[pw][lane];
          const double dnv = S.dn[pw][lane];
          const double nxt = S.u[s1][lane + 2];
          const double rm = cr > 0 ? prevv : upv;
          const double rp = cr < R - 1 ? nxt : dnv;
          p4 = ((a0m + a0p) + rm) + rp;
        } else {
          p4 = a0m + a0p;
        }
      };
      wait_lines(0);
      stage(0, 0.0);
      for (int t = 0; t <= last; ++t) {
        const double km = S.u[su][lane + 1];  // new: lane j-1 wrote it at step t-1 (lane 0: halo)
        const double val = (hf + ((p4 + km) + kp)) * inv;
        const double mine = upd ? val : old;
        const int nl = t - lane;
        if (kval && nl >= 0 && nl < nLines) S.u[su][lane + 2] = mine;
        // advance to step t + 1 and stage it (reads nothing lane j-1 writes now)
        if (DIM == 3) {
          const bool wrp = ++cr == R;
          cr = wrp ? 0 : cr;
          cpl += wrp;
        }
        su = su + 1 == RU ? 0 : su + 1;
        sf = sf + 1 == RF ? 0 : sf + 1;
        if (t < last) {
          wait_lines(t + 1);
          stage(t + 1, mine);
        }
        if ((t & (G - 1)) == G - 1 || t == last) {
          fence_async_shared();  // results visible to the TMA stores
          __syncwarp();
          if (lane == 0) st_release_cta(&S.cons_step, t);
        }
        __syncwarp();
      }
      if (tr && lane == 0) {
        tr[1] = gtimer();
        tr[3] = cwait;
        tr[4] = clock64() - cstart;
      }
    }
    __syncthreads();
  }
}

size_t gs_ws_smem() { return sizeof(WsSmem); }

void configure_gs_ws() {
  const int smem = (int)sizeof(WsSmem);
  cudaFuncSetAttribute(gs_ws_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gs_ws_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

void launch_gs_ws(const GsArgs& a, const WsMaps& maps, int grid, cudaStream_t st) {
  const size_t smem = sizeof(WsSmem);
  const int k = a.g.d == 3 ? 1 : 0;
  if (k)
    gs_ws_kernel<3><<<grid, 64, smem, st>>>(a, maps);
  else
    gs_ws_kernel<2><<<grid, 64, smem, st>>>(a, maps);
}

}  // namespace gmg
