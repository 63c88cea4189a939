// gs_rows.cu -- lexicographic Gauss-Seidel sweep with one grid row per warp
// (sm_100a): the 3-D GS kernel for levels with N >= 64.
//
// Reference: gs_lex_sweep, /root/reference/pkg/src/ghostmg/smoothing.py:127-132
// (u_i <- (h^2 f_i + sum of the 2d neighbours) / (2d + h^2 c) over internal
// nodes in lexicographic order, newest values where already updated).
//
// Order.  Node (p, r, k) needs the NEW values of (p-1, r, k), (p, r-1, k),
// (p, r, k-1) and the OLD values of (p+1, r, k), (p, r+1, k), (p, r, k+1);
// any schedule that respects those six relations reproduces the sequential
// sweep value for value.
//
// Tasks.  A task is a 32-column chunk c (columns k0 = 1+32c .. k0+31) x a
// block b of RR rows (rowbase = 1 + RR b ..) x the planes [P0, P1] that hold
// internal nodes of the task (planes outside that range are unchanged).
// Compute warp w owns row rowbase + w and lane j column k0 + j; at step t it
// relaxes plane p = P0 + t - w - j.  Then every NEW operand was produced one
// step earlier -- the row above by warp w-1, the left neighbour by lane j-1,
// the plane below by the lane itself -- and every OLD operand is produced one
// step later, so one CTA barrier per step orders the whole task, which runs
// (P1 - P0) + RR + 31 steps (a one-warp-per-task wavefront runs ~RR times
// that).
//
// Data.  Each plane of a task is a shared-memory slot filled by TMA (u rows
// rowbase-1 .. rowbase+RR over positions 32c .. 32c+39, f, the internal-node
// mask words) into a ring of NSLOT slots; the warps update u in place in
// the slot, a writer warp copies finished planes back to HBM.  Lane j at
// plane p_j = p_0 - j touches slot p_j mod NSLOT at column 4+j: slots are
// 3072 B = 24 x 128 B apart, so the 32 lanes hit 32 distinct bank pairs.
//
// Neighbour tasks.  The row above the block (task (c, b-1)) and the column
// left of the chunk (task (c-1, b)) arrive as per-node cells (value, tag):
// the upstream task's warp RR-1 / lane 31 store each final value of its last
// row / column with one 16-byte store as soon as it is computed, and cell
// loader warps here poll them per lane (L2), put them into the slots and
// raise per-lane ready counters.  The hand-off therefore lags by RR steps
// (rows) / 32 steps (columns) plus an L2 round trip, not by a whole task.
// Tags carry a per-level sweep sequence number (advanced by the last CTA of
// each sweep), so cells never need clearing.  Tasks are claimed by ticket
// in an order that puts every task after its two upstream tasks, so the
// sweep cannot deadlock for any grid size; planes without internal nodes are
// forwarded to the downstream cells at task start.
//
// Arithmetic per node is the reference's: ((h^2 f + 0) + ((((pb + pa) + ra)
// + rb) + lf) + rt)) * (1 / denom) with pb, pa, ra, rb, lf, rt the plane
// below / above, row above / below, left / right values (smoothing.py:132,
// neighbour order operators.py:145-147), bitwise equal to gs_macro.cu and the
// oracle.
#include <cstddef>

#include "gmg_kernels.cuh"
#include "gs_ptx.cuh"

namespace gmg {

namespace {

constexpr int RR = GS_ROWS;                   // grid rows per task = compute warps
constexpr int NSLOT = 64;                     // plane slots in the ring
constexpr int UROWB = 40 * 8;                 // u tile row: positions 32c .. 32c+39 (k0-4 .. k0+35)
constexpr int U_BYTES = (RR + 2) * UROWB;     // rows rowbase-1 .. rowbase+RR
constexpr int F_OFF = (U_BYTES + 127) / 128 * 128;
constexpr int F_BYTES = RR * 256;             // rows rowbase .. rowbase+RR-1, columns k0 .. k0+31
constexpr int M_OFF = F_OFF + F_BYTES;
constexpr int M_BYTES = RR * 16;              // mask words c&~3 .. c|3 of the RR rows
constexpr int SLOT = (M_OFF + M_BYTES + 255) / 256 * 256;
constexpr int NWARPS = RR + 4;                // compute, TMA loader, writer, row cells, column cells
constexpr int BIG = 1 << 30;
static_assert(SLOT % 256 == 0 && F_OFF % 128 == 0 && M_OFF % 128 == 0, "slot layout");

struct __align__(128) RwCtl {
  unsigned long long bar[NSLOT];
  int task;
  int lready;     // planes < lready (from P0-1 on) have landed
  int cstep;      // compute steps < cstep are complete
  int wfree;      // slots of planes < wfree may be refilled
  int bready[32]; // per column: planes < bready[j] have the row above in their slot
  int cready[RR]; // per row: planes < cready[w] have the left column in their slot
};
constexpr size_t RW_SMEM = (size_t)NSLOT * SLOT + sizeof(RwCtl);
static_assert(RW_SMEM <= 227 * 1024, "one CTA per SM");

__device__ __forceinline__ void cell_put(double2* p, double v, double tag) {
  asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v), "d"(tag) : "memory");
}
__device__ __forceinline__ double2 cell_get(const double2* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(32 * RR) : "memory"); }

}  // namespace

__global__ void __launch_bounds__(32 * NWARPS, 1) gs_rows_kernel(GsRowArgs a, const __grid_constant__ RowMaps maps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  RwCtl& S = *reinterpret_cast<RwCtl*>(smem_raw + (size_t)NSLOT * SLOT);
  const unsigned ring = sa(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const Geom g = a.g;
  const int N = (int)g.N;
  const int n = N + 1;
  // this sweep's cell tags: (sequence + 1) * 4096 + plane (the sequence
  // advances only after every CTA of this launch has read it)
  const double tagbase = 4096.0 * (double)(*(volatile int*)a.ctl + 1);
  auto slot = [&](int p) -> unsigned { return ring + (unsigned)(p % NSLOT) * SLOT; };

  for (;;) {
    if (threadIdx.x == 0) {
      S.task = atomicAdd(a.ctl + 2, 1);
      for (int i = 0; i < NSLOT; ++i) mbar_init(sa(&S.bar[i]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int tid = S.task;
    if (tid >= a.ntasks) break;
    const int2 tk = a.tasks[tid];
    const int c = tk.x, b = tk.y;
    const int cb = c * a.Bn + b;
    const int k0 = 1 + 32 * c;
    const int rowbase = 1 + RR * b;
    const int Rb = min(RR, N - 1 - RR * b);
    const int2 pr = a.prange[cb];
    const int P0 = pr.x, P1 = pr.y;  // P0 > P1: no internal node in the task
    const int T = P1 >= P0 ? (P1 - P0) + RR + 31 : 0;
    double2* const bout = b + 1 < a.Bn ? a.bcell + (size_t)cb * n * 32 : nullptr;
    double2* const cout_ = c + 1 < a.C ? a.ccell + (size_t)cb * n * RR : nullptr;
    const double2* const bin = b > 0 ? a.bcell + (size_t)(cb - 1) * n * 32 : nullptr;
    const double2* const cin = c > 0 ? a.ccell + (size_t)(cb - a.Bn) * n * RR : nullptr;
    if (threadIdx.x == 0) {
      S.lready = P0 - 1;
      S.cstep = 0;
      S.wfree = P0 - 1;
    }
    if (threadIdx.x < 32) S.bready[threadIdx.x] = bin ? P0 : BIG;
    if (threadIdx.x < RR) S.cready[threadIdx.x] = cin ? P0 : BIG;
    __syncthreads();

    if (warp < RR) {
      // ============================ compute ==============================
      const int w = warp, j = lane;
      if (T > 0) {
        const unsigned own = (unsigned)(w + 1) * UROWB + (unsigned)(4 + j) * 8u;
        const unsigned fcol = F_OFF + (unsigned)w * 256u + (unsigned)j * 8u;
        const unsigned mcol = M_OFF + (unsigned)w * 16u + (unsigned)(c & 3) * 4u;
        while (ld_flag(&S.lready) <= P0) __nanosleep(32);
        double prev = lds(slot(P0 - 1) + own);  // plane below of the first plane (never changes)
        double oo = lds(slot(P0) + own);        // old value of the current plane
        uint32_t mw = 0;
        const bool rowok = w < Rb;
        const bool wantB = w == 0 && bin, wantC = j == 0 && cin;
        int lr = P0 + 1, br = wantB ? P0 : BIG, cr = wantC ? P0 : BIG;
        const double h2 = g.h2, inv = g.inv;
        for (int t = 0; t < T; ++t) {
          const int p = P0 + t - w - j;
          const bool act = rowok && p >= P0 && p <= P1;
          mw = __shfl_up_sync(0xffffffffu, mw, 1);  // lane j-1's word of the previous step = this plane's
          double pa = 0.0, rb = 0.0, rt = 0.0, fv = 0.0;
          unsigned sp = 0;
          if (act) {
            if (p + 1 >= lr) {
              lr = ld_flag(&S.lready);
              while (p + 1 >= lr) lr = ld_flag(&S.lready);
            }
            if (p >= br) {
              br = ld_flag(&S.bready[j]);
              while (p >= br) br = ld_flag(&S.bready[j]);
            }
            if (p >= cr) {
              cr = ld_flag(&S.cready[w]);
              while (p >= cr) cr = ld_flag(&S.cready[w]);
            }
            sp = slot(p);
            pa = lds(slot(p + 1) + own);
            rb = lds(sp + own + UROWB);
            rt = lds(sp + own + 8);
            fv = lds(sp + fcol);
            if (j == 0) mw = lds32(sp + mcol);
          }
          bar_compute();  // step t-1's new values (row above, left) are in the slots
          if (act) {
            const double ra = lds(sp + own - UROWB);
            const double lf = lds(sp + own - 8);
            double s = prev + pa;
            s = s + ra;
            s = s + rb;
            s = s + lf;
            s = s + rt;
            const double hf = h2 * fv + 0.0;  // (h2 f + 0) + S == h2 f + (S + 0)
            const double v = (hf + s) * inv;
            const bool in = (mw >> j) & 1u;
            const double m = in ? v : oo;
            if (in) sts(sp + own, m);
            prev = m;
            oo = pa;
            if (bout && w == RR - 1) cell_put(bout + (size_t)p * 32 + j, m, tagbase + (double)p);
            if (cout_ && j == 31) cell_put(cout_ + (size_t)p * RR + w, m, tagbase + (double)p);
          }
          if (threadIdx.x == 0) st_flag(&S.cstep, t);  // every warp has finished step t-1
        }
        bar_compute();
        if (threadIdx.x == 0) st_flag(&S.cstep, T);
      }
    } else if (warp == RR) {
      // ============================ TMA loader ===========================
      // Planes P0-1 .. P1+1 into slot p mod NSLOT once the slot's previous
      // plane is written out; lready counts the landed planes in order.
      if (T > 0 && lane == 0) {
        int q = P0 - 1, qa = P0 - 1, wf = P0 - 1;
        const int qend = P1 + 1;
        while (qa <= qend) {
          bool did = false;
          while (q <= qend) {
            if (q - NSLOT >= wf) {
              wf = ld_flag(&S.wfree);
              if (q - NSLOT >= wf) break;
            }
            const unsigned bar = sa(&S.bar[q % NSLOT]);
            const unsigned dst = slot(q);
            mbar_expect_tx(bar, (unsigned)(U_BYTES + F_BYTES + M_BYTES));
            tma_load_3d(dst, &maps.u, 32 * c, rowbase - 1, q, bar);
            tma_load_3d(dst + F_OFF, &maps.f, 32 * c + 4, rowbase, q, bar);
            tma_load_2d(dst + M_OFF, &maps.m, c & ~3, q * n + rowbase, bar);
            ++q;
            did = true;
          }
          if (qa < q && mbar_test(sa(&S.bar[qa % NSLOT]), (unsigned)(((qa - (P0 - 1)) / NSLOT) & 1))) {
            ++qa;
            st_flag(&S.lready, qa);
            did = true;
          }
          if (!did) __nanosleep(20);
        }
      }
    } else if (warp == RR + 1) {
      // ============================ writer ===============================
      // First the cells of planes without internal nodes (old values, which
      // no one changes), then every finished plane back to HBM.
      const double* u = a.u;
      for (int p = 1; p <= N - 1; ++p) {
        if (p >= P0 && p <= P1) continue;
        const int64_t row = (int64_t)p * n + rowbase;
        if (bout) cell_put(bout + (size_t)p * 32 + lane, __ldcg(u + (row + RR - 1) * g.P + k0 + OFF + lane), tagbase + p);
        if (cout_ && lane < Rb)
          cell_put(cout_ + (size_t)p * RR + lane, __ldcg(u + (row + lane) * g.P + k0 + OFF + 31), tagbase + p);
      }
      if (T > 0) {
        double* const uo = a.u;
        int cs = 0;
        while ((cs = ld_flag(&S.cstep)) < 1) __nanosleep(64);
        if (lane == 0) st_flag(&S.wfree, P0);  // plane P0-1 was read at the compute warps' start
        for (int q = P0; q <= P1; ++q) {
          const int need = (q - P0) + RR + 31;  // plane q is final once step need-1 is done
          while (cs < need) {
            __nanosleep(64);
            cs = ld_flag(&S.cstep);
          }
          const unsigned sq = slot(q) + (unsigned)(4 + lane) * 8u;
          for (int w = 0; w < Rb; ++w) {
            const double v = lds(sq + (unsigned)(w + 1) * UROWB);
            uo[((int64_t)q * n + rowbase + w) * g.P + k0 + OFF + lane] = v;
          }
          __syncwarp();
          if (lane == 0) st_flag(&S.wfree, q + 1);
        }
      }
    } else if (warp == RR + 2) {
      // ============================ row cells ============================
      // Lane j: the row above the block, column k0+j, plane by plane, from
      // task (c, b-1)'s cells (four planes polled per L2 round trip).
      if (T > 0 && bin) {
        int p = P0, lr = P0 - 1;
        while (p <= P1) {
          double2 v[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) v[k] = p + k <= P1 ? cell_get(bin + (size_t)(p + k) * 32 + lane) : make_double2(0.0, -1.0);
          int adv = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (adv == k && v[k].y == tagbase + (double)(p + k)) {
              while (lr <= p + k) lr = ld_flag(&S.lready);  // the slot must hold its plane first
              sts(slot(p + k) + (unsigned)(4 + lane) * 8u, v[k].x);
              adv = k + 1;
            }
          }
          if (adv) {
            p += adv;
            st_flag(&S.bready[lane], p);
          } else {
            __nanosleep(32);
          }
        }
      }
    } else {
      // ============================ column cells =========================
      // Lane w < Rb: column k0-1 of row rowbase+w from task (c-1, b).
      if (T > 0 && cin && lane < Rb) {
        int p = P0, lr = P0 - 1;
        while (p <= P1) {
          double2 v[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) v[k] = p + k <= P1 ? cell_get(cin + (size_t)(p + k) * RR + lane) : make_double2(0.0, -1.0);
          int adv = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (adv == k && v[k].y == tagbase + (double)(p + k)) {
              while (lr <= p + k) lr = ld_flag(&S.lready);
              sts(slot(p + k) + (unsigned)(lane + 1) * UROWB + 3u * 8u, v[k].x);
              adv = k + 1;
            }
          }
          if (adv) {
            p += adv;
            st_flag(&S.cready[lane], p);
          } else {
            __nanosleep(32);
          }
        }
      }
    }
    __syncthreads();
  }
  // the last CTA to finish advances the sweep sequence and resets the ticket
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.ctl + 1, 1) == (int)gridDim.x - 1) {
      a.ctl[1] = 0;
      a.ctl[2] = 0;
      __threadfence();
      atomicAdd(a.ctl, 1);
    }
  }
}

size_t gs_rows_smem() { return RW_SMEM; }
int gs_rows_rows() { return RR; }

void configure_gs_rows() {
  cudaFuncSetAttribute(gs_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RW_SMEM);
}

void launch_gs_rows(const GsRowArgs& a, const RowMaps& maps, int grid, cudaStream_t st) {
  gs_rows_kernel<<<grid, 32 * NWARPS, RW_SMEM, st>>>(a, maps);
}

}  // namespace gmg
