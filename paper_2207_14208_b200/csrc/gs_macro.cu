// gs_macro.cu -- lexicographic Gauss-Seidel sweep with two independent line
// chains per lane (sm_100a): the 3-D GS kernel for levels with N >= 64.
//
// Reference: gs_lex_sweep, /root/reference/pkg/src/ghostmg/smoothing.py:127-132
// (u_i <- (h^2 f_i + sum of the 2d neighbours) / (2d + h^2 c) over internal
// nodes in lexicographic order, newest values where already updated).
//
// Same tasks (32-column chunk c x block b of 14 rows x all planes), warp roles
// (compute, u loader, halo loader, writer, f/mask loader) and progress-word
// protocol as gs_diag.cu, but a lane relaxes two nodes per step.  Within a
// column, node (p, r) depends only on (p, r-1) and (p-1, r), so the upper half
// of plane k+1 (pseudo-rows 0-7: the row above the block and rows 1-7) and the
// lower half of plane k (rows 8-14 and the row below) are independent.
// Macro-line m = 8k + i is the pair
//     slot A: plane k+1, pseudo-row i        slot B: plane k, pseudo-row 8+i
// and lane j relaxes macro-line t-j at step t (k = 0 .. N-1: A covers planes
// 1..N, B planes 0..N-1; boundary planes are masked).  Every neighbour keeps a
// fixed macro offset -- row above m-1 (A's previous result; for B at i = 0 the
// A result of the previous step), row below m+1 (slot B when A is at i = 7),
// plane below m-8, plane above m+8 -- so the lane-diagonal ring of gs_diag.cu
// carries over with two slots per ring row, and the two dependent chains of a
// step overlap: a step costs about what a one-line step costs while the task
// takes half as many steps.  The summation order per node is the reference's
// (bitwise equal to gs_diag.cu and to the oracle).
#include <cstddef>

#include "gmg_kernels.cuh"
#include "gs_ptx.cuh"

namespace gmg {

namespace {

constexpr int MRB = 14;  // grid rows per block
constexpr int MW = 34;   // ring slot pitch (doubles): ci 0 .. 33 <-> columns k0-1 .. k0+32
constexpr int MRU = 72;  // ring rows (macro-lines)
constexpr int MRF = 56;  // f / mask ring macro-lines
constexpr int MNUB = 16, MNFB = 16;
constexpr int MPFD = 4;            // L2 prefetch distance (batches)
constexpr int MDEAD = 8 + 31;      // macro-line m is dead once step m + MDEAD is done
constexpr unsigned SLOTB = MW * 8;       // byte offset of slot B in a ring row
constexpr unsigned MRBY = 2 * MW * 8;    // ring row bytes
constexpr unsigned FSB = MRF * 256u;     // byte offset of slot B's f ring
constexpr unsigned MSB = MRF * 16u;      // byte offset of slot B's mask ring

// Row-above hand-off between blocks b and b+1 (a.edge): lane j of the upper
// task stores (value, 1) for its column of row 14 of plane p as soon as it has
// relaxed it; lane j of the lower task's halo loader polls that one cell, puts
// the value into its ring and clears the cell (every cell is produced and
// consumed exactly once per sweep, so the buffer is all-zero between sweeps).
// The lower task then lags the upper one by 14 steps + an L2 round trip instead
// of waiting for the upper task's writer batch (46 steps + the progress word).
__device__ __forceinline__ void edge_put(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v), "d"(1.0) : "memory");
}
__device__ __forceinline__ double2 edge_get(const double* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void edge_clear(double* p) {
  asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %1};" ::"l"(p), "d"(0.0) : "memory");
}

struct __align__(128) MgSmem {
  double st[2][8][32];        // writer staging (TMA store sources)
  double f[2][MRF][32];       // slot s, macro-line m at [s][m mod MRF]
  double u[MRU][2][MW];       // cell (m, s, ci) at [(m + ci - 1) mod MRU][s][ci]
  uint32_t m[2][MRF][4];      // internal-node mask words c&~3 .. c|3 (same slots as f)
  unsigned long long ubar[MNUB];
  unsigned long long fbar[MNFB];
  int uready, fready, hready, cons, wdone, task;
  int aready[32];  // per column: row-above batches stored by the halo loader (edge mode)
};
static_assert(sizeof(MgSmem) <= 75 * 1024, "three CTAs per SM (228 KB incl. 1 KB reserved each)");

}  // namespace

template <bool EDGE>
__global__ void __launch_bounds__(EDGE ? 192 : 160, 3) gs_macro_kernel(GsArgs a, const __grid_constant__ WsMaps maps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  MgSmem& S = *reinterpret_cast<MgSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const Geom g = a.g;
  const int N = (int)g.N;
  const int nM = 8 * N;  // macro-lines of a task

  for (;;) {
    if (threadIdx.x == 0) {
      S.task = atomicAdd(a.ticket, 1);
      for (int i = 0; i < MNUB; ++i) mbar_init(sa(&S.ubar[i]), 32);
      for (int i = 0; i < MNFB; ++i) mbar_init(sa(&S.fbar[i]), 1);
      S.uready = 0;
      S.fready = 0;
      S.hready = 0;
      S.cons = -1;
      S.wdone = 0;
      for (int i = 0; i < 32; ++i) S.aready[i] = 0;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int tid = S.task;
    if (tid >= a.ntasks) return;
    // diagnostics (GMG_GS_TRACE=1): [0] claim, [1] done, [2] SM, [4] compute-warp cycles
    long long* const tr = a.trace ? a.trace + (int64_t)tid * 24 : nullptr;
    if (tr && threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tr[0] = gtimer();
      tr[2] = smid;
    }
    const int2 tk = a.tasks[tid];
    const int c = tk.x, b = tk.y;
    // this task's row-14 cells for block b+1, and block b-1's cells for this one
    double* const eout = (EDGE && b + 1 < a.Bn && !a.empty_cb[c * a.Bn + b + 1]) ? a.edge + (int64_t)(c * a.Bn + b) * (N + 1) * 64 : nullptr;
    double* const ein = (EDGE && b > 0) ? a.edge + (int64_t)(c * a.Bn + b - 1) * (N + 1) * 64 : nullptr;
    if (a.empty && a.empty[tid]) {
      if (eout) {  // no internal node: row 14 keeps its old values
        const int64_t r14 = 1 + MRB * b + 13, cc = 1 + 32 * c + (int)OFF;
        for (int t = threadIdx.x; t < (N - 1) * 32; t += blockDim.x) {
          const int pl = 1 + (t >> 5), j = t & 31;
          edge_put(eout + ((int64_t)pl * 32 + j) * 2, __ldcg(a.u + ((int64_t)pl * g.n + r14) * g.P + cc + j));
        }
      }
      if (threadIdx.x == 0) st_relaxed(a.progress + a.pstride * (c * a.Bn + b), nM);
      if (tr && threadIdx.x == 0) tr[1] = gtimer();
      __syncthreads();
      continue;
    }
    const int k0 = 1 + 32 * c;
    const int rowbase = 1 + MRB * b;          // grid row of pseudo-row 1
    const int Rb = min(MRB, N - 1 - MRB * b);  // computed rows of the block
    const int col0 = k0 + (int)OFF;
    const int NUq = N + 2;          // u batches q: macro-lines [8q - 8, 8q)  (A plane q, B plane q-1)
    const int NFq = (nM + 72) / 8;  // f batches: macro-lines [-32, nM + 40)
    const int NHq = N;              // halo batches = macro batches
    const int NCq = (nM + 38) / 8;  // compute batches: steps [0, nM + 31)

    if (warp == 0) {
      // ============================ compute ==============================
      const double h2 = g.h2, inv = g.inv;
      const unsigned ub = sa(&S.u[0][0][0]), fb = sa(&S.f[0][0][0]), mb = sa(&S.m[0][0][0]);
      const unsigned lu = (unsigned)(lane + 1) * 8u;  // ci = lane + 1
      const uint32_t mybit = 1u << lane;
      const unsigned mword = (unsigned)(c & 3) * 4u;
      auto wait_batch = [&](int k) {
        const int cu = min(k + 3, NUq), cf = min(k + 5, NFq), ch = min(k + 1, NHq);
        while (ld_flag(&S.uready) < cu) __nanosleep(20);
        while (ld_flag(&S.fready) < cf) __nanosleep(20);
        while (ld_flag(&S.hready) < ch) __nanosleep(20);
        if (EDGE) {  // lane j stages the row above of batch k - j/8 during this batch
          const int need = min(k - (lane >> 3) + 1, NHq);
          while (!__all_sync(0xffffffffu, ld_flag(&S.aready[lane]) >= need)) __nanosleep(20);
        }
      };
      auto urow = [&](int r) -> unsigned { return ub + (unsigned)r * MRBY + lu; };
      auto rmod = [&](int r) -> int { return r < 0 ? r + MRU : (r >= MRU ? r - MRU : r); };
      auto fslot = [&](int s) -> int { return s >= MRF ? s - MRF : s; };
      double s1A, s1B, nxA, nxB, kpA, kpB, hfA, hfB, oA, oB;
      uint32_t mwA, mwB;
      // operands of a step: own cell row, row below (m+1) row, plane below / above rows, f slot
      auto stage = [&](unsigned own, unsigned nxr, unsigned mnr, unsigned pvr, int fs, bool a7) {
        nxA = lds(nxr + (a7 ? SLOTB : 0u));  // A at i = 7: the row below is B's first row
        kpA = lds(nxr + 8);
        nxB = lds(nxr + SLOTB);
        kpB = lds(nxr + SLOTB + 8);
        s1A = lds(mnr) + lds(pvr);
        s1B = lds(mnr + SLOTB) + lds(pvr + SLOTB);
        oA = lds(own);
        oB = lds(own + SLOTB);
        const unsigned fa = fb + (unsigned)fs * 256u + (unsigned)lane * 8u;
        hfA = h2 * lds(fa) + 0.0;  // (h2 f + 0) + S == h2 f + (S + 0)
        hfB = h2 * lds(fa + FSB) + 0.0;
        const unsigned ma = mb + (unsigned)fs * 16u + mword;
        mwA = lds32(ma);
        mwB = lds32(ma + MSB);
      };
      double mA = 0.0, mB = 0.0;  // this lane's results of the previous step
      int r0 = 0;                                // ring row of step 8k
      int f0 = lane == 0 ? 0 : MRF - lane;       // f slot of macro-line 8k - lane
      const long long c0 = clock64();
      wait_batch(0);
      stage(urow(0), urow(1), urow(MRU - 8), urow(8), f0, ((0 - lane) & 7) == 7);
      for (int k = 0; k < NCq; ++k) {
        const unsigned cb = urow(r0);                  // row of step 8k
        const unsigned kb0 = urow(rmod(r0 - 1)) - 8u;  // left neighbour of step 8k
        const int r8 = rmod(r0 + 8);
        const unsigned nb = urow(r8);
        const unsigned mnb = urow(rmod(r0 - 8));
        const unsigned p16 = urow(rmod(r0 + 16));
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double c_s1A = s1A, c_s1B = s1B, c_nxA = nxA, c_nxB = nxB, c_kpA = kpA, c_kpB = kpB;
          const double c_hfA = hfA, c_hfB = hfB, c_oA = oA, c_oB = oB;
          const uint32_t c_mwA = mwA, c_mwB = mwB;
          const bool first = ((i - lane) & 7) == 0;  // this lane's macro-line has i = 0
          if (i == 7 && k + 1 < NCq) {
            wait_batch(k + 1);
            if (tr && lane == 0 && (k + 1 == 64 || k + 1 == 512)) tr[k + 1 == 64 ? 8 : 11] = gtimer();
          }
          {  // stage step 8k + i + 1
            const unsigned own1 = i < 7 ? cb + (unsigned)(i + 1) * MRBY : nb;
            const unsigned nx1 = i < 6 ? cb + (unsigned)(i + 2) * MRBY : (i == 6 ? nb : nb + MRBY);
            const unsigned mn1 = i < 7 ? mnb + (unsigned)(i + 1) * MRBY : cb;
            const unsigned pv1 = i < 7 ? nb + (unsigned)(i + 1) * MRBY : p16;
            stage(own1, nx1, mn1, pv1, fslot(f0 + i + 1), ((i + 1 - lane) & 7) == 7);
          }
          // ---- the two dependent chains of step 8k + i
          const unsigned km = i == 0 ? kb0 : cb + (unsigned)(i - 1) * MRBY - 8u;
          const double lA = lds(km), lB = lds(km + SLOTB);
          const double rB = first ? mA : mB;
          double sA = (c_s1A + mA) + c_nxA;
          double sB = (c_s1B + rB) + c_nxB;
          sA = (sA + lA) + c_kpA;
          sB = (sB + lB) + c_kpB;
          const double vA = (c_hfA + sA) * inv;
          const double vB = (c_hfB + sB) * inv;
          mA = (c_mwA & mybit) ? vA : c_oA;
          mB = (c_mwB & mybit) ? vB : c_oB;
          if (EDGE && eout && ((i - lane) & 7) == 6) {  // this lane's B line is row 14 of plane (8k + i - lane) / 8
            const int mline = 8 * k + i - lane;
            const int pl = mline >> 3;
            if (mline >= 0 && pl >= 1 && pl <= N - 1) edge_put(eout + ((int64_t)pl * 32 + lane) * 2, mB);
          }
          if (8 * k + i - lane < nM + 8) {  // cells past the last loaded line may alias unwritten lines
            sts(cb + (unsigned)i * MRBY, mA);
            sts(cb + (unsigned)i * MRBY + SLOTB, mB);
          }
          __syncwarp();  // lane j+1 reads them next step
        }
        r0 = r8;
        f0 = fslot(f0 + 8);
        __syncwarp();
        if (lane == 0) st_flag(&S.cons, 8 * k + 7);
        if (tr && lane == 0 && k == 68) tr[10] = gtimer();
      }
      if (tr && lane == 0) tr[4] = clock64() - c0;
    } else if (warp == 1) {
      // ============================ u loader =============================
      // cp.async of the task's own columns (old values: computed rows and the
      // row below, both slots) 8 macro-lines per batch into the ring.
      const unsigned ubase = sa(&S.u[0][0][lane + 1]);
      auto rows_of = [&](int q, int s, int& ilo, int& ihi) -> int64_t {
        const int plane = s == 0 ? q : q - 1;
        if (s == 0) {
          ilo = 1;
          ihi = min(7, Rb + 1);
        } else {
          ilo = 0;
          ihi = Rb + 1 - 8;
        }
        if (plane < 0 || plane > N) ihi = -1;
        return (int64_t)plane * g.n + rowbase - 1 + 8 * s;  // grid row of in-batch index 0
      };
      auto prefetch = [&](int q) {
        const int li = lane >> 1, s = li >> 3, i = li & 7;
        const int plane = s == 0 ? q : q - 1;
        const int r = rowbase - 1 + 8 * s + i;
        if (plane < 0 || plane > N || r > N) return;
        const double* b0 = a.u + ((int64_t)plane * g.n + r) * g.P + ((col0 - 1) & ~15) + 16 * (lane & 1);
        prefetch_l2(b0);
        prefetch_l2(b0 + 32);
      };
      int qU = 0, pfU = 0, aU = 0;
      for (; pfU < min(MPFD, NUq); ++pfU) prefetch(pfU);
      int su = umod(-8 + lane, MRU);  // ring row of (macro-line 8 qU - 8, ci = lane + 1)
      while (qU < NUq || aU < NUq) {
        while (aU < qU && mbar_test(sa(&S.ubar[aU % MNUB]), (unsigned)((aU / MNUB) & 1))) ++aU;
        if (lane == 0) st_flag(&S.uready, aU);
        const int cs = ld_flag(&S.cons);
        const int lo = 8 * qU - 8;
        const int old = lo + 7 - MRU;  // ring predecessors must be dead and written out
        bool ok = qU < NUq && cs >= old + MDEAD;
        if (ok && old >= 0) ok = ld_flag(&S.wdone) >= min(old + 1, nM);
        if (!ok) {
          __nanosleep(a.sleep_ns[0]);
          continue;
        }
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          int ilo, ihi;
          const int64_t r0 = rows_of(qU, s, ilo, ihi);
          const double* src = a.u + (r0 + ilo) * g.P + col0 + lane;
          int rr = su + ilo;
          rr -= rr >= MRU ? MRU : 0;
          for (int i = ilo; i <= ihi; ++i) {
            cp_async8(ubase + (unsigned)rr * MRBY + (unsigned)s * SLOTB, src);
            src += g.P;
            rr = rr + 1 == MRU ? 0 : rr + 1;
          }
        }
        cp_async_arrive(sa(&S.ubar[qU % MNUB]));
        ++qU;
        su += 8;
        su -= su >= MRU ? MRU : 0;
        if (pfU < NUq) prefetch(pfU++);
      }
    } else if (warp == 4) {
      // ============================ f loader =============================
      // f / mask batches: per slot one TMA 2-D tile (8 rows of one plane);
      // lines outside the task get zero masks via out-of-bounds fill.
      int qF = 0, pfF = 0, aF = 0;
      while (qF < NFq || aF < NFq) {
        while (aF < qF && mbar_test(sa(&S.fbar[aF % MNFB]), (unsigned)((aF / MNFB) & 1))) ++aF;
        if (lane == 0) st_flag(&S.fready, aF);
        const int cs = ld_flag(&S.cons);
        const int lo = 8 * qF - 32;
        // the slot of line L held line L - MRF, staged by lane 31 at step L - MRF + 30
        if (!(qF < NFq && cs >= lo + 7 - MRF + 30)) {
          __nanosleep(a.sleep_ns[1]);
          continue;
        }
        if (lane == 0) {
          const unsigned bar = sa(&S.fbar[qF % MNFB]);
          const int fs = umod(lo, MRF);
          const int k = lo >> 3;
          const bool inA = lo >= 0 && lo < nM && k <= N - 2;  // A: plane k+1 in 1 .. N-1
          const bool inB = lo >= 0 && lo < nM && k >= 1;      // B: plane k in 1 .. N-1
          mbar_expect_tx(bar, (inA ? 2048u : 0u) + (inB ? 2048u : 0u) + 256u);
          if (inA) tma_load_2d(sa(&S.f[0][fs][0]), &maps.f, col0, (int)((int64_t)(k + 1) * g.n + rowbase - 1), bar);
          if (inB) tma_load_2d(sa(&S.f[1][fs][0]), &maps.f, col0, (int)((int64_t)k * g.n + rowbase + 7), bar);
          tma_load_2d(sa(&S.m[0][fs][0]), &maps.m2, c & ~3, inA ? (k * a.Bn + b) * 16 : -8, bar);
          tma_load_2d(sa(&S.m[1][fs][0]), &maps.m2, c & ~3, inB ? ((k - 1) * a.Bn + b) * 16 + 8 : -8, bar);
        }
        for (; pfF < min(qF + MPFD + 1, NFq); ++pfF) {
          const int L = 8 * pfF - 32;
          if (L < 0 || L >= nM) continue;
          const int k = L >> 3, li = lane >> 1, s = li >> 3, i = li & 7;
          const int plane = s == 0 ? k + 1 : k;
          const int r = rowbase - 1 + 8 * s + i;
          if (plane >= 1 && plane <= N - 1 && r <= N)
            prefetch_l2(a.f + ((int64_t)plane * g.n + r) * g.P + col0 + 16 * (lane & 1));
        }
        ++qF;
      }
    } else if (warp == 2) {
      // ============================ halo loader ==========================
      // Per macro batch h: left halo (column k0-1, new values of task c-1) and
      // right halo (column k0+32, old) of its 16 lines, and the row above the
      // block for slot A's i = 0 line (plane h+1, new values of task b-1, whose
      // row 14 of plane h+1 is in its macro batch h+1).  Two batches in
      // flight, as in gs_diag.cu.
      const int* lprog = c > 0 ? a.progress + a.pstride * ((c - 1) * a.Bn + b) : nullptr;
      const int* uprog = (b > 0 && !EDGE) ? a.progress + a.pstride * (c * a.Bn + (b - 1)) : nullptr;
      int seenL = 0, seenU = 0;
      const int hsl = (lane >> 3) & 1, hil = lane & 7;  // lane's halo line: slot, in-batch index
      const bool right = lane >= 16;
      auto ready = [&](int h, bool poll) -> bool {
        const int old = 8 * h + 7 - MRU;
        const int cs = ld_flag(&S.cons);
        if (cs < old + MDEAD) return false;
        if (old >= 0 && ld_flag(&S.wdone) < min(old + 1, nM)) return false;
        const int needL = min(8 * h + 8, nM), needU = min(8 * h + 16, nM);
        if (lprog && seenL < needL && poll) seenL = ld_relaxed(lprog);
        if (lprog && seenL < needL) return false;
        if (uprog && seenU < needU && poll) seenU = ld_relaxed(uprog);
        return !(uprog && seenU < needU);
      };
      auto issue = [&](int h, double& hv, double& uw) {
        if (tr && h == 64 && lane == 0) tr[6] = gtimer();
        hv = uw = 0.0;
        const int plane = hsl == 0 ? h + 1 : h;
        const int r = 8 * hsl + hil;
        if (plane >= 1 && plane <= N - 1 && r >= 1 && r <= Rb)
          hv = __ldcg(a.u + ((int64_t)plane * g.n + rowbase - 1 + r) * g.P + col0 + (right ? 32 : -1));
        if (!EDGE && h + 1 <= N - 1) uw = __ldcg(a.u + ((int64_t)(h + 1) * g.n + rowbase - 1) * g.P + col0 + lane);
      };
      auto store = [&](int h, double hv, double uw) {
        const int m = 8 * h + hil;
        if (!right)
          S.u[umod(m - 1, MRU)][hsl][0] = hv;  // ci = 0
        else
          S.u[umod(m + 32, MRU)][hsl][33] = hv;  // ci = 33
        if (!EDGE && h + 1 <= N - 1) S.u[umod(8 * h + lane, MRU)][0][lane + 1] = uw;  // (8h, A, ci = lane + 1)
        __syncwarp();
        if (lane == 0) st_flag(&S.hready, h + 1);
        if (tr && h == 64 && lane == 0) tr[7] = gtimer();
      };
      int hs = 0, hi = 0;  // next batch to store / to issue
      double hvA = 0.0, uwA = 0.0, hvB = 0.0, uwB = 0.0;
      while (hs < NHq) {
        if (hi == hs) {
          while (!ready(hs, true)) __nanosleep(a.sleep_ns[2]);
          issue(hs, hvA, uwA);
          ++hi;
        }
        // the progress poll for batch hs+1 is in flight while batch hs is stored
        const bool want = hi == hs + 1 && hi < NHq;
        int pL = seenL, pU = seenU;
        if (want) {
          if (lprog && seenL < min(8 * hi + 8, nM)) pL = ld_relaxed(lprog);
          if (uprog && seenU < min(8 * hi + 16, nM)) pU = ld_relaxed(uprog);
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
    } else if (warp == 3) {
      // ============================ writer ===============================
      // Macro batch w is final once lane 31 finished it (step 8w + 38): both
      // slots go out with one TMA tile store each (A: plane w+1 rows 1-7, B:
      // plane w rows 8-14; rows past row N are clipped, boundary planes are
      // skipped), then the progress word.
      int* myprog = a.progress + a.pstride * (c * a.Bn + b);
      int w = 0;
      while (w < N) {
        const int cs = ld_flag(&S.cons);
        if (cs < 8 * w + 7 + 31) {
          __nanosleep(a.sleep_ns[3]);
          continue;
        }
        if (tr && w == 64 && lane == 0) tr[9] = gtimer();
        if (lane == 0) bulk_wait_read<0>();  // staging free
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = umod(8 * w + i + lane, MRU);
          S.st[0][i][lane] = S.u[rr][0][lane + 1];
          S.st[1][i][lane] = S.u[rr][1][lane + 1];
        }
        fence_async_shared();
        __syncwarp();
        if (lane == 0) {
          st_flag(&S.wdone, 8 * w + 8);
          bool any = false;
          if (w + 1 <= N - 1) {
            tma_store_3d(&maps.ust, col0, rowbase, w + 1, sa(&S.st[0][1][0]));
            any = true;
          }
          if (w >= 1 && Rb >= 8) {
            tma_store_3d(&maps.ust, col0, rowbase + 7, w, sa(&S.st[1][0][0]));
            any = true;
          }
          if (any) {
            bulk_commit();
            bulk_wait<0>();  // this batch's lines are in L2
          }
          st_relaxed(myprog, 8 * w + 8);
          if (tr && (w == 64 || w == 65)) tr[w == 64 ? 5 : 12] = gtimer();
        }
        __syncwarp();
        ++w;
      }
      if (lane == 0) bulk_wait<0>();
      if (tr && lane == 0) tr[1] = gtimer();
    } else if (EDGE && warp == 5) {
      // ============================ row-above loader (edge mode) ========
      // Lane j moves the row-above cell of column j for batch ha into ring
      // cell (8ha, A, ci = j + 1) once block b-1 has relaxed it (or, for the
      // first block, from the boundary row), then clears the cell.
      // Up to four batches are polled per L2 round trip (independent loads in
      // flight), so a lane delivers several batches per round trip once the
      // upper block is ahead.
      int ha = 0;
      auto ring_free = [&](int h) -> bool {
        const int old = 8 * h + 7 - MRU;
        if (ld_flag(&S.cons) < old + MDEAD) return false;
        return !(old >= 0 && ld_flag(&S.wdone) < min(old + 1, nM));
      };
      while (ha < NHq) {
        int nb = 0;
        while (nb < 4 && ha + nb < NHq && ring_free(ha + nb)) ++nb;
        if (nb == 0) {
          __nanosleep(a.sleep_ns[2]);
          continue;
        }
        double2 pv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          pv[q] = make_double2(0.0, 1.0);
          if (q < nb && ha + q + 1 <= N - 1) {
            if (ein)
              pv[q] = edge_get(ein + ((int64_t)(ha + q + 1) * 32 + lane) * 2);
            else
              pv[q].x = __ldcg(a.u + ((int64_t)(ha + q + 1) * g.n + rowbase - 1) * g.P + col0 + lane);
          }
        }
        const int h0 = ha;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (q >= nb || ha != h0 + q || pv[q].y == 0.0) continue;
          if (ha + 1 <= N - 1) {
            if (ein) edge_clear(ein + ((int64_t)(ha + 1) * 32 + lane) * 2);
            S.u[umod(8 * ha + lane, MRU)][0][lane + 1] = pv[q].x;  // (8ha, A, ci = lane + 1)
          }
          ++ha;
        }
        if (ha != h0)
          st_flag(&S.aready[lane], ha);
        else
          __nanosleep(a.sleep_ns[2]);
      }
    }
    __syncthreads();
  }
}

size_t gs_macro_smem() { return sizeof(MgSmem); }

void configure_gs_macro() {
  cudaFuncSetAttribute(gs_macro_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(MgSmem));
  cudaFuncSetAttribute(gs_macro_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(MgSmem));
}

int gs_macro_ctas_per_sm() {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gs_macro_kernel<false>, 160, sizeof(MgSmem)) != cudaSuccess) return 1;
  return n > 0 ? n : 1;
}

void launch_gs_macro(const GsArgs& a, const WsMaps& maps, int grid, cudaStream_t st) {
  if (a.edge)
    gs_macro_kernel<true><<<grid, 192, sizeof(MgSmem), st>>>(a, maps);
  else
    gs_macro_kernel<false><<<grid, 160, sizeof(MgSmem), st>>>(a, maps);
}

}  // namespace gmg
