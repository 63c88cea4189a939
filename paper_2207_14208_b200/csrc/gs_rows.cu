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
// Data.  Groups of G planes of a task are filled by three TMA boxes (u rows
// rowbase-1 .. rowbase+RR over positions 32c .. 32c+39, f, the internal-node
// mask words) into a ring of NG group slots (NG * G = 64 planes); the warps
// update u in place in the ring, a writer warp copies finished planes back
// to HBM.  Lane j at plane p_j = p_0 - j touches its plane's u tile at column
// 4+j: plane tiles start at multiples of 128 B, so the 32 lanes hit 32
// distinct bank pairs.
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
constexpr int G = 4;                          // planes per TMA group
constexpr int NG = 16;                        // group slots in the ring
constexpr int NSLOT = G * NG;                 // planes in the ring
constexpr int UROWB = 40 * 8;                 // u tile row: positions 32c .. 32c+39 (k0-4 .. k0+35)
constexpr int U_BYTES = (RR + 2) * UROWB;     // rows rowbase-1 .. rowbase+RR of one plane
constexpr int F_BYTES = RR * 256;             // rows rowbase .. rowbase+RR-1, columns k0 .. k0+31
constexpr int M_BYTES = RR * 16;              // mask words c&~3 .. c|3 of the RR rows
constexpr int F_OFF = G * U_BYTES;
constexpr int M_OFF = F_OFF + G * F_BYTES;
constexpr int GSLOT = M_OFF + G * M_BYTES;
constexpr int NWARPS = RR + 4;                // compute, TMA loader, writer, row cells, column cells
constexpr int BIG = 1 << 30;
constexpr int KB = 4;                         // compute steps per readiness check
constexpr int CW = 16;                        // cell planes polled per L2 round trip
constexpr int PBIAS = 4 * NSLOT;              // plane bias: planes >= -PBIAS map to ring positions
static_assert(U_BYTES % 128 == 0 && F_BYTES % 128 == 0 && M_OFF % 128 == 0 && GSLOT % 128 == 0, "ring layout");

struct __align__(128) RwCtl {
  unsigned long long bar[NG];
  int task;
  int lready;     // planes < lready (from P0-1 on) have landed
  int cstep;      // compute steps < cstep are complete
  int wfree;      // ring space of planes < wfree may be refilled
  int bready[32]; // per column: planes < bready[j] have the row above in the ring
  int cready[RR]; // per row: planes < cready[w] have the left column in the ring
};
constexpr size_t RW_SMEM = (size_t)NG * GSLOT + sizeof(RwCtl);
static_assert(RW_SMEM <= 227 * 1024, "one CTA per SM");

__device__ __forceinline__ void cell_put(double2* p, double v, double tag) {
  asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v), "d"(tag) : "memory");
}
__device__ __forceinline__ double2 cell_get(const double2* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void hint_put(long long* p, long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ long long hint_get(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(32 * RR) : "memory"); }

// shared-memory addresses of plane p's tiles in the ring
struct Ring {
  unsigned base;
  __device__ unsigned group(int p) const { return base + (unsigned)(((p + PBIAS) / G) % NG) * GSLOT; }
  __device__ unsigned u(int p) const { return group(p) + (unsigned)((p + PBIAS) % G) * U_BYTES; }
};

}  // namespace

__global__ void __launch_bounds__(32 * NWARPS, 1) gs_rows_kernel(GsRowArgs a, const __grid_constant__ RowMaps maps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  RwCtl& S = *reinterpret_cast<RwCtl*>(smem_raw + (size_t)NG * GSLOT);
  const Ring ring{sa(smem_raw)};
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const Geom g = a.g;
  const int N = (int)g.N;
  const int n = N + 1;
  // this sweep's cell tags: (sequence + 1) * 4096 + plane (the sequence
  // advances only after every CTA of this launch has read it)
  const int seq = *(volatile int*)a.ctl + 1;
  const double tagbase = 4096.0 * (double)seq;
  const long long hseq = (long long)seq << 32;  // progress hints of this sweep: hseq | plane

  for (;;) {
    if (threadIdx.x == 0) {
      S.task = atomicAdd(a.ctl + 2, 1);
      for (int i = 0; i < NG; ++i) mbar_init(sa(&S.bar[i]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int tid = S.task;
    if (tid >= a.ntasks) break;
    // diagnostics (GMG_GS_TRACE=1): [0] claim, [1] done, [2] SM, [3] compute start (globaltimer ns);
    // with -DGS_ROWS_TRACE=1 also [4] compute cycles, [5] waiting for slots, [6] for cells, [7] at the step barrier
    long long* const tr = a.trace ? a.trace + (int64_t)tid * 16 : nullptr;
    if (tr && threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tr[0] = gtimer();
      tr[2] = smid;
    }
    const int2 tk = a.tasks[tid];
    const int c = tk.x, b = tk.y;
    const int cb = c * a.Bn + b;
    const int k0 = 1 + 32 * c;
    const int rowbase = 1 + RR * b;
    const int Rb = min(RR, N - 1 - RR * b);
    const int2 pr = a.prange[cb];
    const int P0 = pr.x, P1 = pr.y;  // P0 > P1: no internal node in the task
    const int T = P1 >= P0 ? (P1 - P0) + RR + 31 : 0;
#if GS_ROWS_EXP >= 2  // timing experiments (wrong results): 2 no cell waits, 3 no cells at all
    double2* const bout = GS_ROWS_EXP == 2 && b + 1 < a.Bn ? a.bcell + (size_t)cb * n * 32 : nullptr;
    double2* const cout_ = GS_ROWS_EXP == 2 && c + 1 < a.C ? a.ccell + (size_t)cb * n * RR : nullptr;
    const double2* const bin = nullptr;
    const double2* const cin = nullptr;
#else
    double2* const bout = b + 1 < a.Bn ? a.bcell + (size_t)cb * n * 32 : nullptr;
    double2* const cout_ = c + 1 < a.C ? a.ccell + (size_t)cb * n * RR : nullptr;
    const double2* const bin = b > 0 ? a.bcell + (size_t)(cb - 1) * n * 32 : nullptr;
    const double2* const cin = c > 0 ? a.ccell + (size_t)(cb - a.Bn) * n * RR : nullptr;
#endif
    long long* const hint_out = (bout || cout_) ? a.hint + (size_t)cb * 16 : nullptr;
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
      // Steps run in blocks of KB: the planes / cells a lane needs during a
      // block are checked once at its start, and every lane executes the same
      // straight-line step (ring loads are always in bounds; stores are
      // predicated on the lane's plane being in [P0, P1]).
      const int w = warp, j = lane;
      if (T > 0) {
        const unsigned own = (unsigned)(w + 1) * UROWB + (unsigned)(4 + j) * 8u;
        const unsigned fcol = (unsigned)w * 256u + (unsigned)j * 8u;
        const unsigned mcol = (unsigned)w * 16u + (unsigned)(c & 3) * 4u;
        const unsigned rend = ring.base + (unsigned)(NG * GSLOT);
        while (ld_flag(&S.lready) <= P0) {
        }
        if (tr && threadIdx.x == 0) tr[3] = gtimer();
#if GS_ROWS_TRACE
        long long c_slot = 0, c_cell = 0, c_bar = 0;
        const long long c_start = clock64();
#endif
        double prev = lds(ring.u(P0 - 1) + own);  // plane below of the first plane (never changes)
        double oo = lds(ring.u(P0) + own);        // old value of the current plane
        uint32_t mw = 0;
        const bool rowok = w < Rb;
        const bool wantB = w == 0 && bin, wantC = j == 0 && cin;
        const bool putB = bout && w == RR - 1, putC = cout_ && j == 31 && rowok;
        const double h2 = g.h2, inv = g.inv;
        int p = P0 - w - j;  // this lane's plane at step 0
        // this plane's group slot and position in it
        unsigned gs = ring.group(p);
        int kin = (p + PBIAS) % G;
        double2* bput = putB ? bout + (ptrdiff_t)p * 32 + j : nullptr;
        double2* cput = putC ? cout_ + (ptrdiff_t)p * RR + w : nullptr;
        double tag = tagbase + (double)p;
        for (int t0 = 0; t0 < T; t0 += KB) {
          {  // readiness of the block's planes (this lane's planes p .. p + KB - 1)
#if GS_ROWS_TRACE
            const long long c0 = clock64();
            if (tr && tid < 8 && threadIdx.x == 0 && t0 / KB < 256) {
              long long* st = a.trace + (int64_t)a.ntasks * 16 + (int64_t)tid * 1024 + (t0 / KB) * 4;
              st[0] = c0;
              st[1] = ld_flag(&S.lready);
              st[2] = ld_flag(&S.wfree);
              st[3] = p;
            }
#endif
            const int lo = max(p, P0), hi = min(p + KB - 1, P1);
            if (rowok && lo <= hi) {
              while (ld_flag(&S.lready) <= hi + 1) {
              }
#if GS_ROWS_TRACE
              c_slot += clock64() - c0;
              const long long c1 = clock64();
#endif
              if (wantB)
                while (ld_flag(&S.bready[j]) <= hi) {
                }
              if (wantC)
                while (ld_flag(&S.cready[w]) <= hi) {
                }
#if GS_ROWS_TRACE
              c_cell += clock64() - c1;
#endif
            }
          }
#pragma unroll
          for (int k = 0; k < KB; ++k) {
            const bool act = rowok && p >= P0 && p <= P1;
            // plane p+1: next position in the group, or the next group slot
            const bool wrap = kin == G - 1;
            const unsigned gs1 = wrap ? (gs + GSLOT == rend ? ring.base : gs + GSLOT) : gs;
            const int kin1 = wrap ? 0 : kin + 1;
            const unsigned su = gs + (unsigned)kin * U_BYTES;
            const unsigned su1 = gs1 + (unsigned)kin1 * U_BYTES;
            mw = __shfl_up_sync(0xffffffffu, mw, 1);  // lane j-1's word of the previous step = this plane's
            const double pa = lds(su1 + own);
            const double rb = lds(su + own + UROWB);
            const double rt = lds(su + own + 8);
            const double fv = lds(gs + F_OFF + (unsigned)kin * F_BYTES + fcol);
            if (j == 0) mw = lds32(gs + M_OFF + (unsigned)kin * M_BYTES + mcol);
#if GS_ROWS_TRACE
            const long long cb0 = clock64();
#endif
            bar_compute();  // the previous step's new values (row above, left) are in the ring
#if GS_ROWS_TRACE
            c_bar += clock64() - cb0;
#endif
            const double ra = lds(su + own - UROWB);
            const double lf = lds(su + own - 8);
            double sum = prev + pa;
            sum = sum + ra;
            sum = sum + rb;
            sum = sum + lf;
            sum = sum + rt;
            const double hf = h2 * fv + 0.0;  // (h2 f + 0) + S == h2 f + (S + 0)
            const double v = (hf + sum) * inv;
            const bool in = act && ((mw >> j) & 1u);
            const double m = in ? v : oo;
            if (in) sts(su + own, m);
            if (act) {
              prev = m;
              oo = pa;
              if (putB) cell_put(bput, m, tag);
              if (putC) cell_put(cput, m, tag);
            }
            if (threadIdx.x == 0 && k == 0) {
              st_flag(&S.cstep, t0);  // every warp has finished step t0-1
              // progress hint for the downstream tasks: planes < P0 + t0 - w - j of lane (w, j) are done
              // (their cells' tags still decide; the hint only says which cells are worth reading)
              if (hint_out) hint_put(hint_out, hseq | (long long)(P0 + t0));
            }
            ++p;
            gs = gs1;
            kin = kin1;
            tag += 1.0;
            bput += 32;
            cput += RR;
          }
        }
        bar_compute();
        if (threadIdx.x == 0) {
          st_flag(&S.cstep, BIG);
          if (hint_out) hint_put(hint_out, hseq | (long long)BIG);
        }
#if GS_ROWS_TRACE
        if (tr && threadIdx.x == 0) {
          tr[4] = clock64() - c_start;
          tr[5] = c_slot;
          tr[6] = c_cell;
          tr[7] = c_bar;
        }
#endif
      }
    } else if (warp == RR) {
      // ============================ TMA loader ===========================
      // Groups of G planes (from the one holding P0-1 to the one holding
      // P1+1) into group slot (group mod NG) once every plane of its previous
      // group is written out; lready counts the landed planes in order.
      if (T > 0 && lane == 0) {
        const int glo = (P0 - 1) / G, ghi = (P1 + 1) / G;
        int gq = glo, ga = glo, wf = P0 - 1;
#if GS_ROWS_TRACE
        long long t_issue = 0, t_land = 0, c_ring = 0, n_lat = 0, s_lat = 0;
        long long issued_at[NG];
#endif
        while (ga <= ghi) {
          bool did = false;
          while (gq <= ghi) {
            const int need = (gq - NG + 1) * G;  // planes < need must be free
            if (need > wf) {
              wf = ld_flag(&S.wfree);
              if (need > wf) {
#if GS_ROWS_TRACE
                if (ga == gq) c_ring += 1;
#endif
                break;
              }
            }
#if GS_ROWS_TRACE
            issued_at[gq % NG] = clock64();
#endif
            const unsigned bar = sa(&S.bar[gq % NG]);
            const unsigned dst = ring.base + (unsigned)(gq % NG) * GSLOT;
#if GS_ROWS_EXP == 1  // timing experiment: no loads (wrong results)
            mbar_arrive(bar);
            (void)dst;
#else
            mbar_expect_tx(bar, (unsigned)GSLOT);
            tma_load_3d(dst, &maps.u, 32 * c, rowbase - 1, gq * G, bar);
            tma_load_3d(dst + F_OFF, &maps.f, 32 * c + 4, rowbase, gq * G, bar);
            tma_load_3d(dst + M_OFF, &maps.m, c & ~3, rowbase, gq * G, bar);
#endif
            ++gq;
            did = true;
          }
          const int ga0 = ga;
          while (ga < gq && mbar_test(sa(&S.bar[ga % NG]), (unsigned)(((ga - glo) / NG) & 1))) {
#if GS_ROWS_TRACE
            s_lat += clock64() - issued_at[ga % NG];
            ++n_lat;
#endif
            ++ga;
          }
          if (ga != ga0) {
            st_flag(&S.lready, ga * G);
            did = true;
          }
          (void)did;  // no back-off: a sleeping warp wakes up microseconds late
        }
#if GS_ROWS_TRACE
        if (tr) {
          tr[8] = c_ring;
          tr[10] = n_lat ? s_lat / n_lat : 0;  // mean cycles from issue to observed landing
        }
        (void)t_issue;
        (void)t_land;
#endif
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
        while ((cs = ld_flag(&S.cstep)) < 1) {
        }
        if (lane == 0) st_flag(&S.wfree, P0);  // plane P0-1 was read at the compute warps' start
        for (int q = P0; q <= P1; ++q) {
          const int need = (q - P0) + RR + 31;  // plane q is final once step need-1 is done
          while (cs < need) cs = ld_flag(&S.cstep);  // spin: __nanosleep wakes up ~2 us late
          const unsigned sq = ring.u(q) + (unsigned)(4 + lane) * 8u;
          double v[RR];
#pragma unroll
          for (int w = 0; w < RR; ++w) v[w] = lds(sq + (unsigned)(w + 1) * UROWB);
          double* const dst = uo + ((int64_t)q * n + rowbase) * g.P + k0 + OFF + lane;
#pragma unroll
          for (int w = 0; w < RR; ++w)
            if (w < Rb) dst[(int64_t)w * g.P] = v[w];
          __syncwarp();
          if (lane == 0) st_flag(&S.wfree, q + 1);
        }
      }
    } else if (warp == RR + 2) {
      // ============================ row cells ============================
      // Lane j: the row above the block, column k0+j, plane by plane, from
      // task (c, b-1)'s cells: CW planes polled per L2 round trip, so the
      // hand-off keeps pace with an upstream task up to CW planes per trip.
      if (T > 0 && bin) {
        const int2 pu = a.prange[cb - 1];
        const long long* const hin = a.hint + (size_t)(cb - 1) * 16;
        int p = P0;
        while (p <= P1) {
          // cells worth reading: the upstream's planes outside its computed range (forwarded at its
          // start) and those its progress hint covers for this lane
          const long long h = hint_get(hin);
          const int X = (h >> 32) == (hseq >> 32) ? (int)(h & 0xffffffffll) : pu.x;
          const int lim = X - (RR - 1) - lane;
          const int top = min(P1, ld_flag(&S.lready) - 1);  // only planes the ring already holds
          double2 v[CW];
#pragma unroll
          for (int k = 0; k < CW; ++k) {
            const int q = p + k;
            v[k] = q <= top && (q < pu.x || q > pu.y || q < lim) ? cell_get(bin + (size_t)q * 32 + lane)
                                                                 : make_double2(0.0, -1.0);
          }
          int adv = 0;
#pragma unroll
          for (int k = 0; k < CW; ++k) {
            if (adv == k && v[k].y == tagbase + (double)(p + k)) {
              sts(ring.u(p + k) + (unsigned)(4 + lane) * 8u, v[k].x);
              adv = k + 1;
            }
          }
          if (adv) {
            p += adv;
            st_flag(&S.bready[lane], p);
          }
        }
      }
    } else {
      // ============================ column cells =========================
      // Lane w < Rb: column k0-1 of row rowbase+w from task (c-1, b).
      if (T > 0 && cin && lane < Rb) {
        const int2 pu = a.prange[cb - a.Bn];
        const long long* const hin = a.hint + (size_t)(cb - a.Bn) * 16;
        int p = P0;
        while (p <= P1) {
          const long long h = hint_get(hin);
          const int X = (h >> 32) == (hseq >> 32) ? (int)(h & 0xffffffffll) : pu.x;
          const int lim = X - 31 - lane;
          const int top = min(P1, ld_flag(&S.lready) - 1);  // only planes the ring already holds
          double2 v[CW];
#pragma unroll
          for (int k = 0; k < CW; ++k) {
            const int q = p + k;
            v[k] = q <= top && (q < pu.x || q > pu.y || q < lim) ? cell_get(cin + (size_t)q * RR + lane)
                                                                 : make_double2(0.0, -1.0);
          }
          int adv = 0;
#pragma unroll
          for (int k = 0; k < CW; ++k) {
            if (adv == k && v[k].y == tagbase + (double)(p + k)) {
              sts(ring.u(p + k) + (unsigned)(lane + 1) * UROWB + 3u * 8u, v[k].x);
              adv = k + 1;
            }
          }
          if (adv) {
            p += adv;
            st_flag(&S.cready[lane], p);
          }
        }
      }
    }
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[1] = gtimer();
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
int gs_rows_group() { return G; }

void configure_gs_rows() {
  cudaFuncSetAttribute(gs_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RW_SMEM);
}

void launch_gs_rows(const GsRowArgs& a, const RowMaps& maps, int grid, cudaStream_t st) {
  gs_rows_kernel<<<grid, 32 * NWARPS, RW_SMEM, st>>>(a, maps);
}

}  // namespace gmg
