// gs_diag.cu -- lexicographic Gauss-Seidel sweep on a lane-diagonal ring
// (sm_100a): the production GS kernel for levels with N >= 64.
//
// Reference: gs_lex_sweep, /root/reference/pkg/src/ghostmg/smoothing.py:127-132
// (u_i <- (h^2 f_i + sum of the 2d neighbours) / (2d + h^2 c) over internal
// nodes in lexicographic order, newest values where already updated).
//
// Decomposition.  A task is a 32-column chunk c (columns k0 = 1+32c ..
// k0+31) x a block b of RB = 14 rows x all planes.  Its work is a sequence
// of "lines" (one row of the chunk): per plane PL = 16 pseudo-lines -- the
// row above the block (new values, read only), the RB rows, the row below
// (old values, read only) and padding.  Lane j of the compute warp handles
// column k0+j and runs one line behind lane j-1, so at step t lane j
// relaxes line t-j: its left neighbour (lane j-1, same line) was finished at
// step t-1, its upper neighbour is lane j's own previous result, the plane
// below is lane j's result from PL steps ago.
//
// Diagonal ring.  Cell (line L, column slot ci) of a line (ci = 0 .. 33 <->
// columns k0-1 .. k0+32) lives in ring row (L + ci - 1) mod RU.  Every
// operand of step t is then in ring row t + const, identical for all lanes:
// the compute warp addresses shared memory with per-batch base registers
// plus compile-time offsets and issues ~20 instructions per step.
//
// Warps of a CTA (one task at a time):
//  * warp 0 compute: 8-step batches, operands for step t+1 loaded while the
//    dependent chain of step t runs; only ld.shared(left neighbour) ->
//    4 dadd/dmul -> select -> st.shared is loop-carried through memory;
//  * warp 1 bulk loader: cp.async (8 B, L1-allocating: these values are not
//    modified by anyone before this task reads them) of the task's own
//    columns + right halo, 16+ lines ahead, and of f / internal-node masks;
//    completion signalled on mbarriers; L2 prefetch further ahead (TMA);
//  * warp 2 halo loader: the new values produced by neighbour tasks -- left
//    halo column k0-1 (task c-1) and the row above the block (task b-1) --
//    after polling their progress words (ld.acquire.gpu), read through L2;
//  * warp 3 writer: copies finished lines out of the diagonal ring, stores
//    them coalesced and publishes the task's progress (st.release.gpu).
// Tasks are claimed by ticket in wavefront order, so every task waited on is
// already running: the sweep cannot deadlock for any grid size.
#include <cstddef>

#include "gmg_kernels.cuh"
#include "gs_ptx.cuh"

namespace gmg {

namespace {

constexpr int PL = 16;   // pseudo-lines per plane (3-D)
constexpr int RB = 14;   // grid rows per block (3-D)
constexpr int UW = 36;   // ring row pitch (doubles): [pad, ci 0 .. 33, pad]
constexpr int RU = 104;  // u ring rows
constexpr int RFL = 80;  // f / mask ring lines (+ 8 mirrored rows)
constexpr int NUB = 16, NFB = 16;  // mbarrier rings
constexpr int HDEPTH = 8;                  // halo batches in flight
#ifndef GS_PFD
#define GS_PFD 4
#endif
constexpr int PFD = GS_PFD;                // L2 prefetch distance (batches)

struct __align__(128) DgSmem {
  double u[RU][UW];    // cell (L, ci) at [(L + ci - 1) mod RU][ci + 1]
  double f[RFL + 8][32];   // line L at slot L mod RFL; slots 0..7 mirrored at RFL..RFL+7
  uint32_t m[RFL + 8][4];  // internal-node bitmask words c&~3 .. c|3 of line L (same slots)
  double st[8][32];        // writer staging: finished lines, contiguous for TMA stores
  int flag[2][4];          // writer: progress value, stored with a 16-B TMA store
  unsigned long long ubar[NUB];
  unsigned long long fbar[NFB];
  int uready; // u loader: u batches landed
  int fready; // f loader: f / mask batches landed
  int hready; // halo loader: halo batches stored
  int cons;   // compute warp: last completed step
  int wdone;  // writer: lines copied out of the ring
  int task;
};
static_assert(sizeof(DgSmem) <= 56 * 1024, "four CTAs per SM (228 KB incl. 1 KB reserved each)");

__device__ uint32_t g_zero_words[4];  // zero mask word for non-computed lines
// Line geometry of one task.
struct Lines {
  int d, N, rowbase, Rb, nLines;
  int64_t n;
  // kind of pseudo-line L: 0 up halo, 1 computed row, 2 down halo, 3 padding;
  // sets the tensor row (plane * n + row, or row in 2-D).
  __device__ __forceinline__ int kind(int L, int64_t& trow) const {
    if (d == 3) {
      const int p = floordiv(L, PL) + 1;  // plane 0 .. N
      const int r = L - (p - 1) * PL;
      trow = (int64_t)p * n + rowbase - 1 + r;
      if (r == 0) return 0;
      if (r <= Rb) return (p >= 1 && p <= N - 1) ? 1 : 2;
      return r == Rb + 1 ? 2 : 3;
    }
    trow = L;
    if (L == 0) return 2;  // boundary row 0: plain old values
    if (L < N) return 1;
    return L == N ? 2 : 3;
  }
};

// Tensor row of the first line of the 8-line batch starting at L0 (8-aligned;
// in 3-D a batch never leaves its plane) and the range [ilo, ihi] of lines in it
// that are loaded (computed rows + down halo) or, with computed_only, computed.
__device__ __forceinline__ int64_t batch_rows(const Lines& ln, const Geom& g, int L0, bool computed_only,
                                              int& ilo, int& ihi) {
  if (ln.d == 3) {
    const int p = (L0 >> 4) + 1;  // floor(L0 / PL) + 1, PL = 16
    const int r0 = L0 - (p - 1) * PL;
    const int top = computed_only ? ln.Rb : ln.Rb + 1;
    ilo = max(0, 1 - r0);
    ihi = min(7, top - r0);
    if (computed_only && (p < 1 || p > ln.N - 1)) ihi = -1;
    return (int64_t)p * g.n + ln.rowbase - 1 + r0;
  }
  ilo = computed_only ? max(0, 1 - L0) : 0;
  ihi = min(7, (computed_only ? ln.N - 1 : ln.N) - L0);
  return L0;
}

}  // namespace

template <int D>
__global__ void __launch_bounds__(160, 4) gs_diag_kernel(GsArgs a, const __grid_constant__ WsMaps maps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  DgSmem& S = *reinterpret_cast<DgSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const Geom g = a.g;
  const int N = (int)g.N;
  constexpr int pl = D == 3 ? PL : 0;

  for (;;) {
    if (threadIdx.x == 0) {
      S.task = atomicAdd(a.ticket, 1);
      for (int i = 0; i < NUB; ++i) mbar_init(sa(&S.ubar[i]), 32);
      for (int i = 0; i < NFB; ++i) mbar_init(sa(&S.fbar[i]), 1);
      S.uready = 0;
      S.fready = 0;
      S.hready = 0;
      S.cons = -1;
      S.wdone = 0;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int tid = S.task;
    if (tid >= a.ntasks) return;
    const int2 tk = a.tasks[tid];
    const int c = tk.x, b = tk.y;
    if (a.empty && a.empty[tid]) {
      // no internal node in this chunk x block: nothing changes, neighbours
      // read its columns / rows as they are
      if (threadIdx.x == 0) {
        const int nl = D == 3 ? (N - 1) * PL : ((N + 1 + 7) & ~7);
        st_relaxed(a.progress + a.pstride * (c * a.Bn + b), nl);
      }
      __syncthreads();
      continue;
    }
    const int k0 = 1 + 32 * c;
    Lines ln;
    ln.d = D;
    ln.N = N;
    ln.n = g.n;
    if (D == 3) {
      ln.rowbase = 1 + RB * b;
      ln.Rb = min(RB, N - 1 - RB * b);
      ln.nLines = (N - 1) * PL;
    } else {
      ln.rowbase = 0;
      ln.Rb = N - 1;
      ln.nLines = (N + 1 + 7) & ~7;
    }
    const int nLines = ln.nLines;
    const int NUq = (nLines + 2 * pl) / 8;  // u lines [-pl, nLines + pl)
    const int NFq = (nLines + 72) / 8;      // f / mask lines [-32, nLines + 40)
    const int NHq = nLines / 8;             // halo batches, lines [0, nLines)
    const int NCq = (nLines + 38) / 8;      // compute batches: steps [0, nLines + 31)
    const int col0 = k0 + (int)OFF;         // padded position of column k0
    // line L is dead (no cell read again) once step L + DEADLAG is done: last
    // read is as the plane below of line L + PL by lane 31 (3-D), or as the left
    // neighbour of lane 31 (2-D)
    constexpr int DEADLAG = D == 3 ? PL + 31 : 32;
    long long* const tr = a.trace ? a.trace + (int64_t)tid * 24 : nullptr;

    if (warp == 0) {
      // ============================ compute ==============================
      const double h2 = g.h2, inv = g.inv;
      const unsigned ub = sa(&S.u[0][0]), fb = sa(&S.f[0][0]), mb = sa(&S.m[0]);
      constexpr unsigned RBY = UW * 8;  // ring row bytes
      const unsigned lu = (unsigned)(lane + 2) * 8u;  // ci = lane + 1 -> index lane + 2
      const uint32_t mybit = 1u << lane;
      const unsigned mword = (unsigned)(c & 3) * 4u;
      long long cwU = 0, cwF = 0, cwH = 0;
      const long long cstart = clock64();
      if (tr && lane == 0) {
        tr[0] = gtimer();
        unsigned sm;
        unsigned wid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
        asm volatile("mov.u32 %0, %warpid;" : "=r"(wid));
        tr[2] = sm | ((long long)wid << 16);
      }
      // the loaders publish plain counters (S.uready, S.fready, S.hready):
      // one shared load each per batch
      auto wait_batch = [&](int k) {
        const long long c0 = tr ? clock64() : 0;
        const int cu = min(k + 2 + 2 * pl / 8, NUq), cf = min(k + 6, NFq);
        const bool nap = true;
        while (ld_flag(&S.uready) < cu) {
          if (nap) __nanosleep(20);
        }
        while (ld_flag(&S.fready) < cf) {
          if (nap) __nanosleep(20);
        }
        const long long c1 = tr ? clock64() : 0;
        const int ch = min(k + 1, NHq);
        while (ld_flag(&S.hready) < ch) {
          if (nap) __nanosleep(20);
        }
        if (tr) {
          cwU += c1 - c0;
          cwH += clock64() - c1;
          if (lane == 0 && k == 64) tr[6] = gtimer();  // compute warp: halo batch 64 available
        }
      };
      // staged operands of the coming step
      double s1, nx, kp, hf;
      uint32_t mw;
      double old = 0.0, rm = 0.0;
      // ring rows of batch k: r0 = 8k mod RU (RU, PL multiples of 8: no wrap inside a batch)
      int r0 = 0;
      int f0 = lane == 0 ? 0 : RFL - lane;  // f slot of line 8k - lane (mirrored: no wrap in a batch)
      auto urow = [&](int r) -> unsigned { return ub + (unsigned)r * RBY + lu; };
      auto rmod = [&](int r) -> int { return r < 0 ? r + RU : (r >= RU ? r - RU : r); };
      // operands of step t (rows relative to t) given the row of t, its f row
      auto stage = [&](int rt, int fs) {
        const unsigned nt = urow(rmod(rt + 1));
        nx = lds(nt);
        kp = lds(nt + 8);
        if (D == 3) {
          const double mn = lds(urow(rmod(rt - PL)));
          const double pv = lds(urow(rmod(rt + PL)));
          s1 = mn + pv;
        }
        const unsigned fa = fb + (unsigned)fs * 256u + (unsigned)lane * 8u;
        hf = h2 * lds(fa) + 0.0;  // (h2 f + 0) + S == h2 f + (S + 0)
        mw = lds32(mb + (unsigned)fs * 16u + mword);
      };
      wait_batch(0);
      stage(0, f0);
      old = lds(urow(0));
      for (int k = 0; k < NCq; ++k) {
        if (k > 0) wait_batch(k);
        const unsigned cb = urow(r0);                       // row of step 8k
        const unsigned kb0 = urow(rmod(r0 - 1)) - 8u;       // km of step 8k (row 8k-1, ci = lane)
        const int r8 = rmod(r0 + 8);
        const unsigned nb = urow(r8);                       // row of step 8k + 8
        unsigned mnb = 0, plb = 0, mn8 = 0, pl8 = 0;
        if (D == 3) {
          mnb = urow(rmod(r0 - PL));
          plb = urow(rmod(r0 + PL));
          mn8 = urow(rmod(r8 - PL));
          pl8 = urow(rmod(r8 + PL));
        }
        const int f8 = f0 + 8 >= RFL ? f0 + 8 - RFL : f0 + 8;
        const unsigned fcb = fb + (unsigned)f0 * 256u + (unsigned)lane * 8u;
        const unsigned mcb = mb + (unsigned)f0 * 16u + mword;
        const unsigned f8b = fb + (unsigned)f8 * 256u + (unsigned)lane * 8u;
        const unsigned m8b = mb + (unsigned)f8 * 16u + mword;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          // ---- operands of this step staged last step: s1, nx, kp, hf, mw
          const double c_s1 = s1, c_nx = nx, c_kp = kp, c_hf = hf;
          const uint32_t c_mw = mw;
          // ---- stage step i+1 (rows i+1 / i+2 of this batch, or the next batch)
          {
            const unsigned n1 = i < 6 ? cb + (unsigned)(i + 2) * RBY : (i == 6 ? nb : nb + RBY);
            nx = lds(n1);
            kp = lds(n1 + 8);
            if (D == 3) {
              const double mn = lds(i < 7 ? mnb + (unsigned)(i + 1) * RBY : mn8);
              const double pv = lds(i < 7 ? plb + (unsigned)(i + 1) * RBY : pl8);
              s1 = mn + pv;
            }
            const unsigned fa = i < 7 ? fcb + (unsigned)(i + 1) * 256u : f8b;
            const unsigned ma = i < 7 ? mcb + (unsigned)(i + 1) * 16u : m8b;
            hf = h2 * lds(fa) + 0.0;
            mw = lds32(ma);
          }
          // ---- the dependent chain of step 8k + i
          const double km = lds(i == 0 ? kb0 : cb + (unsigned)(i - 1) * RBY - 8u);
          double sacc = D == 3 ? (c_s1 + rm) + c_nx : rm + c_nx;
          sacc = (sacc + km) + c_kp;
          const double val = (c_hf + sacc) * inv;
          const double mine = (c_mw & mybit) ? val : old;
          sts(cb + (unsigned)i * RBY, mine);
          __syncwarp();  // lane j+1 reads it next step
          rm = mine;
          old = c_nx;
        }
        r0 = r8;
        f0 = f8;
        __syncwarp();
        if (lane == 0) st_flag(&S.cons, 8 * k + 7);
        if (tr && lane == 0 && k == 68) tr[17] = gtimer();  // compute: line 519 finished by lane 31
        if (tr && lane == 0 && (k == 64 || k == 512)) tr[k == 64 ? 5 : 7] = gtimer();
      }
      if (tr && lane == 0) {
        tr[1] = gtimer();
        tr[3] = cwU + cwF + cwH;
        tr[4] = clock64() - cstart;
        tr[8] = cwU + cwF;  // u + f waits (tr[3] - tr[8]: halo waits)
        (void)cwH;
      }
    } else if (warp == 1) {
      // ============================ u loader =============================
      // cp.async (8 B per lane, L1-allocating: these values -- own columns,
      // boundary planes, the row below the block -- are not modified by anyone
      // before this task reads them) of 8 lines per batch into the diagonal
      // ring; completion arrives on the batch's mbarrier and is republished
      // as the plain counter S.uready.  The right-halo column (ci = 33) comes
      // with the halo loader.
      long long tU = 0, bidle = 0, leadU = 0;
      constexpr unsigned RBY = UW * 8;
      const unsigned ubase = sa(&S.u[0][lane + 2]);
      // batch q covers lines 8q - pl ..; in 3-D batch parity = half of a plane
      // (pseudo-lines 0-7 / 8-15), loaded lines: computed rows + the row below
      int ilo0, ihi0, ilo1, ihi1;
      if (D == 3) {
        ilo0 = 1;
        ihi0 = min(7, ln.Rb + 1);
        ilo1 = 0;
        ihi1 = ln.Rb + 1 - 8;  // may be < 0
      } else {
        ilo0 = ilo1 = 0;
        ihi0 = ihi1 = 7;
      }
      // global row of the first line of batch q: advanced incrementally
      int64_t brow = D == 3 ? (int64_t)ln.rowbase - 1 : 0;  // plane 0, pseudo-line 0
      int64_t prow = brow;                                  // prefetch cursor (batch pfU)
      auto advance = [&](int64_t& row, int q) {              // row of batch q -> q + 1
        if (D == 3)
          row += (q & 1) ? g.n - 8 : 8;
        else
          row += 8;
      };
      const int pl_lane = lane >> 2, pl_part = lane & 3;  // prefetch: 4 lanes per line
      auto prefetch = [&](int64_t row) {
        const double* b0 = a.u + (row + pl_lane) * g.P + ((col0 - 1) & ~3) + 4 * pl_part;
        prefetch_l2(b0);
        prefetch_l2(b0 + 16);
        if (pl_part < 2) prefetch_l2(b0 + 32);
      };
      int qU = 0, pfU = 0, aU = 0;
      for (; pfU < min(PFD, NUq); ++pfU) {
        prefetch(prow);
        advance(prow, pfU);
      }
      int su = umod(-pl + lane, RU);  // ring row of (line 8 qU - pl, ci = lane + 1)
      while (qU < NUq || aU < NUq) {
        // republish completed batches
        while (aU < qU && mbar_test(sa(&S.ubar[aU % NUB]), (unsigned)((aU / NUB) & 1))) ++aU;
        if (lane == 0) st_flag(&S.uready, aU);
        const int cs = ld_flag(&S.cons);
        const int lo = 8 * qU - pl;
        // a cell of line L replaces the same cell of line L - RU: that line must be dead
        const int old = lo + 7 - RU;
        bool ok = qU < NUq && cs >= old + DEADLAG;
        if (ok && old >= 0) ok = ld_flag(&S.wdone) >= min(old + 1, nLines);
        if (!ok) {
          ++bidle;
          __nanosleep(a.sleep_ns[0]);
          continue;
        }
        const long long c0 = tr ? clock64() : 0;
        leadU += (lo + 25) - 8 - cs;
        const int ilo = (D == 3 && (qU & 1)) ? ilo1 : ilo0;
        const int ihi = D == 3 ? ((qU & 1) ? ihi1 : ihi0) : min(ihi0, N - lo);  // 2-D: rows <= N
        const double* src = a.u + (brow + ilo) * g.P + col0 + lane;
        int s = su + ilo;
        s -= s >= RU ? RU : 0;
        for (int i = ilo; i <= ihi; ++i) {
          cp_async8(ubase + (unsigned)s * RBY, src);
          src += g.P;
          s = s + 1 == RU ? 0 : s + 1;
        }
        cp_async_arrive(sa(&S.ubar[qU % NUB]));
        advance(brow, qU);
        ++qU;
        su += 8;
        su -= su >= RU ? RU : 0;
        if (pfU < NUq) {
          prefetch(prow);
          advance(prow, pfU);
          ++pfU;
        }
        if (tr) tU += clock64() - c0;
      }
      if (tr && lane == 0) {
        tr[10] = bidle;
        (void)leadU;
        (void)tU;
      }
    } else if (warp == 4) {
      // ============================ f loader =============================
      // f / mask batches: TMA 2-D tiles into the linear f ring (slot 0's batch
      // also into the mirror rows); lines outside the task load zero masks via
      // out-of-bounds fill.  Completion is republished as S.fready.
      const CUtensorMap* mmap = D == 3 ? &maps.m2 : &maps.m;
      long long tF = 0, leadF = 0;
      int qF = 0, pfF = 0, aF = 0;
      while (qF < NFq || aF < NFq) {
        while (aF < qF && mbar_test(sa(&S.fbar[aF % NFB]), (unsigned)((aF / NFB) & 1))) ++aF;
        if (lane == 0) st_flag(&S.fready, aF);
        const int cs = ld_flag(&S.cons);
        // slot of line L held line L - RFL, read by lane 31 up to step L - RFL + 31
        if (!(qF < NFq && cs >= 8 * qF - 32 + 7 - RFL + 30)) {
          __nanosleep(a.sleep_ns[1]);
          continue;
        }
        const int lo = 8 * qF - 32;
        if (lane == 0) {
          const long long c0 = tr ? clock64() : 0;
          leadF += (lo - 9) - cs;
          const unsigned bar = sa(&S.fbar[qF % NFB]);
          const int fs = umod(lo, RFL);
          const int copies = fs == 0 ? 2 : 1;
          const bool inside = lo >= 0 && lo < nLines;
          mbar_expect_tx(bar, (unsigned)copies * ((inside ? 2048u : 0u) + 128u));
          const int mrow = D == 3 ? (((lo >> 4) * a.Bn + b) * PL + (lo & (PL - 1))) : lo;
          int ilo, ihi;
          const int64_t frow = inside ? batch_rows(ln, g, lo, false, ilo, ihi) : 0;
          for (int cp = 0; cp < copies; ++cp) {
            const int slot = fs + cp * RFL;
            if (inside) tma_load_2d(sa(&S.f[slot][0]), &maps.f, col0, (int)frow, bar);
            tma_load_2d(sa(&S.m[slot][0]), mmap, c & ~3, inside ? mrow : -8, bar);
          }
          if (tr) tF += clock64() - c0;
        }
        for (; pfF < min(qF + PFD + 1, NFq); ++pfF) {
          const int L = 8 * pfF - 32;
          if (L >= 0 && L < nLines) {  // the 8 sectors of each of the 8 lines
            int plo, phi;
            const double* b0 = a.f + batch_rows(ln, g, L, false, plo, phi) * g.P + col0;
            prefetch_l2(b0 + (lane >> 3) * g.P + 4 * (lane & 7));
            prefetch_l2(b0 + (4 + (lane >> 3)) * g.P + 4 * (lane & 7));
          }
        }
        ++qF;
      }
      if (tr && lane == 0) {
        (void)tF;
        (void)leadF;
      }
    } else if (warp == 2) {
      if (!a.halo_multi) {
        // ============================ halo loader ==========================
        // Per 8-line batch h: left halo (column k0-1, new values of task c-1),
        // right halo (column k0+32, old) and, once per plane, the row above the
        // block (new values of task b-1).  Two batches in flight: the loads of
        // batch h+1 are issued before batch h's values are stored, so one L2
        // latency is overlapped with the next poll.
        const int* lprog = c > 0 ? a.progress + a.pstride * ((c - 1) * a.Bn + b) : nullptr;
        const int* uprog = (D == 3 && b > 0) ? a.progress + a.pstride * (c * a.Bn + (b - 1)) : nullptr;
        int seenL = 0, seenU = 0;
        auto up_line = [&](int h) -> int {  // up-halo pseudo-line loaded with batch h, or -1
          if (D != 3) return -1;
          if (h == 0) return 0;
          const int L = 8 * h + 8;
          return (L % PL == 0 && L < nLines) ? L : -1;
        };
        // may batch h be issued?  poll: refresh the neighbours' progress (L2 round trip)
        auto ready = [&](int h, bool poll) -> bool {
          const int Lu = up_line(h);
          const int old = max(Lu, 8 * h + 7) - RU;  // ring predecessors must be dead
          const int cs = ld_flag(&S.cons);
          if (cs < old + DEADLAG) return false;
          if (old >= 0 && ld_flag(&S.wdone) < min(old + 1, nLines)) return false;
          const int needL = min(8 * h + 8, nLines), needU = Lu >= 0 ? Lu + PL : 0;
          if (lprog && seenL < needL && poll) {
            seenL = ld_relaxed(lprog);
            if (tr && lane == 0 && seenL >= 8 * 65 && !tr[12]) tr[12] = gtimer();
          }
          if (lprog && seenL < needL) return false;
          if (uprog && seenU < needU && poll) seenU = ld_relaxed(uprog);
          return !(uprog && seenU < needU);
        };
        auto issue = [&](int h, double& hv, double& uw) {
          if (tr && lane == 0 && h == 64) tr[14] = gtimer();
          hv = uw = 0.0;
          if (lane < 16) {  // lanes 0-7: left halo (new), 8-15: right halo (old) of line 8h + (lane & 7)
            const int L = 8 * h + (lane & 7);
            int64_t trow;
            if (ln.kind(L, trow) == 1) hv = __ldcg(a.u + trow * g.P + col0 + (lane < 8 ? -1 : 32));
          }
          const int Lu = up_line(h);
          if (Lu >= 0) {
            int64_t trow;
            ln.kind(Lu, trow);
            uw = __ldcg(a.u + trow * g.P + col0 + lane);
          }
        };
        auto store = [&](int h, double hv, double uw) {
          if (tr && lane == 0 && h == 64) tr[9] = gtimer();
          if (lane < 8) {
            S.u[umod(8 * h + lane - 1, RU)][1] = hv;  // ci = 0 of line 8h + lane
          } else if (lane < 16) {
            S.u[umod(8 * h + lane - 8 + 32, RU)][34] = hv;  // ci = 33 of line 8h + lane - 8
          }
          const int Lu = up_line(h);
          if (Lu >= 0) S.u[umod(Lu + lane, RU)][lane + 2] = uw;
          __syncwarp();
          if (lane == 0) st_flag(&S.hready, h + 1);
          if (tr && lane == 0 && h == 64) tr[15] = gtimer();
        };
        int hs = 0, hi = 0;  // next batch to store / to issue
        double hvA = 0.0, uwA = 0.0, hvB = 0.0, uwB = 0.0;
        while (hs < NHq) {
          if (hi == hs) {  // slot A empty: block until batch hs may be issued
            while (!ready(hs, true)) __nanosleep(a.sleep_ns[2]);
            issue(hs, hvA, uwA);
            ++hi;
          }
          // the progress poll for batch hs+1 is in flight while batch hs is stored
          // (its result is consumed afterwards; the shared-memory flags carry no
          // fence, so nothing waits for the outstanding load)
          const bool want = hi == hs + 1 && hi < NHq;
          int pL = seenL, pU = seenU;
          if (want) {
            if (lprog && seenL < min(8 * hi + 8, nLines)) pL = ld_relaxed(lprog);
            const int Lu = up_line(hi);
            if (uprog && Lu >= 0 && seenU < Lu + PL) pU = ld_relaxed(uprog);
          }
          store(hs, hvA, uwA);
          seenL = max(seenL, pL);
          seenU = max(seenU, pU);
          if (want && ready(hi, false)) {
            issue(hi, hvB, uwB);
            ++hi;
          }
          ++hs;
          hvA = hvB;
          uwA = uwB;
        }
      } else {
        // ============================ halo loader ==========================
        // Per 8-line batch h: left halo (column k0-1, new values of task c-1),
        // right halo (column k0+32, old) and, once per plane, the row above the
        // block (new values of task b-1).  Each iteration issues one progress
        // poll (its result is consumed at the end of the iteration) and, in the
        // same L2 round trip, the loads of every batch already known to be
        // ready -- up to four batches, one line per lane -- so the loader keeps
        // pace with the compute warp however far the neighbours' publications
        // are behind, instead of paying one round trip per batch.
        const int* lprog = c > 0 ? a.progress + a.pstride * ((c - 1) * a.Bn + b) : nullptr;
        const int* uprog = (D == 3 && b > 0) ? a.progress + a.pstride * (c * a.Bn + (b - 1)) : nullptr;
        int seenL = lprog ? 0 : (1 << 30), seenU = uprog ? 0 : (1 << 30);
        auto up_line = [&](int h) -> int {  // up-halo pseudo-line loaded with batch h, or -1
          if (D != 3) return -1;
          if (h == 0) return 0;
          const int L = 8 * h + 8;
          return (L % PL == 0 && L < nLines) ? L : -1;
        };
        // ring cells of batch h dead, neighbours' lines published?
        auto ready = [&](int h, int cs, int wd) -> bool {
          const int Lu = up_line(h);
          const int old = max(Lu, 8 * h + 7) - RU;  // ring predecessors must be dead
          if (cs < old + DEADLAG) return false;
          if (old >= 0 && wd < min(old + 1, nLines)) return false;
          if (seenL < min(8 * h + 8, nLines)) return false;
          return !(Lu >= 0 && seenU < Lu + PL);
        };
        // In flight: loads of batches [hs, hi) (registers), stored next iteration
        // while the following progress poll is outstanding.
        int hs = 0, hi = 0;
        double hv = 0.0, rv = 0.0;
        bool hl = false;
        int Lup[3] = {-1, -1, -1};
        double uw[3] = {0.0, 0.0, 0.0};
        while (hs < NHq) {
          // 1. poll the neighbours (consumed after the pending batches are stored)
          // (only while the neighbours' known progress limits the next batches)
          int pL = seenL, pU = seenU;
          const int hn = min(hi + 2, NHq);
          if (seenL < min(8 * hn, nLines)) pL = ld_relaxed(lprog);
          if (seenU < min(8 * hn + PL, nLines)) pU = ld_relaxed(uprog);
          // 2. store the batches loaded last iteration
          if (hi > hs) {
            const int L = 8 * hs + lane;
            if (L < 8 * hi) {
              S.u[umod(L - 1, RU)][1] = hl ? hv : 0.0;    // ci = 0 of line L
              S.u[umod(L + 32, RU)][34] = hl ? rv : 0.0;  // ci = 33 of line L
            }
  #pragma unroll
            for (int q = 0; q < 3; ++q)
              if (Lup[q] >= 0) S.u[umod(Lup[q] + lane, RU)][lane + 2] = uw[q];
            __syncwarp();
            if (lane == 0) st_flag(&S.hready, hi);
            if (tr && lane == 0 && hs <= 64 && 64 < hi) tr[15] = gtimer();
            hs = hi;
          }
          // 3. consume the poll, then issue the loads of every ready batch (<= 4)
          seenL = max(seenL, pL);
          seenU = max(seenU, pU);
          if (tr && lane == 0 && seenL >= 8 * 65 && !tr[12]) tr[12] = gtimer();
          const int cs = ld_flag(&S.cons), wd = ld_flag(&S.wdone);
          int he = hs;
          while (he < NHq && he < hs + 4 && ready(he, cs, wd)) ++he;
          if (he > hs) {
            if (tr && lane == 0 && hs <= 64 && 64 < he) tr[14] = gtimer();
            const int L = 8 * hs + lane;  // lane l: left / right halo of line 8 hs + l
            hv = rv = 0.0;
            hl = false;
            if (L < 8 * he) {
              int64_t trow;
              if (ln.kind(L, trow) == 1) {
                const double* row = a.u + trow * g.P + col0;
                hv = __ldcg(row - 1);
                rv = __ldcg(row + 32);
                hl = true;
              }
            }
            // up lines of batches [hs, he): at most three (batch 0 and odd batches)
            int nu = 0;
            Lup[0] = Lup[1] = Lup[2] = -1;
            for (int h = hs; h < he; ++h) {
              const int Lu = up_line(h);
              if (Lu >= 0) {
                if (nu == 0) Lup[0] = Lu;
                else if (nu == 1) Lup[1] = Lu;
                else Lup[2] = Lu;
                ++nu;
              }
            }
  #pragma unroll
            for (int q = 0; q < 3; ++q) {
              if (Lup[q] >= 0) {
                int64_t trow;
                ln.kind(Lup[q], trow);
                uw[q] = __ldcg(a.u + trow * g.P + col0 + lane);
              }
            }
            hi = he;
          } else if (a.sleep_ns[2] > 0) {
            __nanosleep(a.sleep_ns[2]);
          }
        }
      }
    } else if (warp == 3) {
      // ============================ writer ===============================
      // Finished lines go out with TMA tile stores from a staging copy; the
      // progress word is itself written by a 16-B bulk store issued only after
      // the data group has completed (wait_group), so publishing needs no
      // memory barrier and overlaps the next batch.
      int* myprog = a.progress + a.pstride * (c * a.Bn + b);
      const int NWq = nLines / 8;
      long long idle = 0, wpub = 0;
      int w = 0;
      while (w < NWq) {
        const int cs = ld_flag(&S.cons);
        bool did = false;
        if (w < NWq && cs >= 8 * w + 7 + 31) {
          if (tr && lane == 0 && w == 64) tr[16] = gtimer();  // writer: batch 64 ready
          if (lane == 0) bulk_wait_read<0>();  // staging free
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) S.st[i][lane] = S.u[umod(8 * w + i + lane, RU)][lane + 2];
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            st_flag(&S.wdone, 8 * w + 8);
            // one TMA tile store: 3-D rows r = 1..7 or 8..14 of the block's pseudo-lines
            // (rows past row N are clipped; a ragged block's row N gets its own old value);
            // 2-D rows 8w..8w+7 (boundary rows keep their values)
            if (D == 3) {
              const int p = ((8 * w) >> 4) + 1, r0 = (8 * w) & (PL - 1);
              tma_store_3d(&maps.ust, col0, ln.rowbase - 1 + (r0 == 0 ? 1 : r0), p, sa(&S.st[r0 == 0 ? 1 : 0][0]));
            } else {
              tma_store_2d(&maps.ust, col0, 8 * w, sa(&S.st[0][0]));
            }
            bulk_commit();
            const long long c0 = tr ? clock64() : 0;
            bulk_wait<0>();  // this batch's lines are in L2
            if (tr) wpub += clock64() - c0;
            if (tr && w == 64) tr[11] = gtimer();
            st_relaxed(myprog, 8 * w + 8);
          }
          __syncwarp();
          ++w;
          did = true;
        }
        if (!did) {
          ++idle;
          __nanosleep(a.sleep_ns[3]);
        }
      }
      if (lane == 0) {
        bulk_wait<0>();
        st_relaxed(myprog, nLines);
      }
      if (tr && lane == 0) tr[13] = wpub;
      (void)idle;
    }
    __syncthreads();
  }
}

size_t gs_diag_smem() { return sizeof(DgSmem); }

void configure_gs_diag() {
  const int smem = (int)sizeof(DgSmem);
  cudaFuncSetAttribute(gs_diag_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gs_diag_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

void launch_gs_diag(const GsArgs& a, const WsMaps& maps, int grid, cudaStream_t st) {
  const size_t smem = sizeof(DgSmem);
  if (a.g.d == 3)
    gs_diag_kernel<3><<<grid, 160, smem, st>>>(a, maps);
  else
    gs_diag_kernel<2><<<grid, 160, smem, st>>>(a, maps);
}

}  // namespace gmg
