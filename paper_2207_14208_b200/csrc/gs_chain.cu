// gs_chain.cu -- lexicographic Gauss-Seidel sweep, register chains (sm_100a):
// the 3-D GS kernel for levels with N >= 64.
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
// Tasks.  A task is a 16-column chunk c (columns k0 = 1+16c .. k0+15) x a
// block b of 8 rows (rowbase = 1 + 8b ..) x the planes [P0, P1] that hold
// internal nodes of the task.  One CTA of five warps runs a task.  Two
// compute warps: warp A owns columns k0 .. k0+7, warp B columns k0+8 ..
// k0+15 and runs SHB = 8 steps behind A; lane (g, j) of a warp owns its
// column j and the two rows ("chains") rowbase + 2g + i, i = 0, 1, and chain
// i relaxes plane p = P0 + t - j - 2g - i (- SHB for B) at step t.  Then
// every NEW operand of a node was produced one step earlier and is still in a
// register -- the plane below by the chain itself, the row above by the
// lane's chain 0 (for chain 0: row group g-1's chain 1, one shuffle), the left
// neighbour by lane j-1 (one shuffle; B's lane 0 reads A's column 7 from the
// ring) -- and every OLD operand is read before the step that overwrites it.
// The loop-carried dependency of a step is a shuffle and seven fp64
// operations; there is no barrier inside a task.  A task runs
// (P1 - P0) + 23 steps.
//
// Data.  A loader warp (one lane) fills groups of G planes of the task with
// two TMA boxes (u rows rowbase-1 .. rowbase+8 over columns k0-2 .. k0+17 -- a
// box starts on a 16-byte boundary -- and f) into a ring of NS plane slots;
// the compute warps update u in place in the ring, a writer warp copies
// finished planes back to HBM and pushes the last row / column to the
// downstream tasks.  Which nodes are internal comes from a plane-transposed
// bit mask (word (p >> 5, r, k), bit p & 31) that each lane reads from global
// memory once per 32 steps and chain, all lanes at the same steps.
//
// Neighbour tasks.  The row above the block (task (c, b-1)) and the column
// left of the chunk (task (c-1, b)) arrive as per-node cells (value, tag):
// the upstream writer stores each final value of its last row / column with
// one 16-byte store, and the cells warp here polls them per lane (L2), puts
// them into the ring's halo row / column and raises per-column / per-row
// ready counters.  The hand-off lags by 7 steps (rows) / 15 steps (columns)
// plus the writer's lag and an L2 round trip.  Tags carry a per-level sweep
// sequence number (advanced by the last CTA of each sweep), so cells never
// need clearing.  Tasks are claimed by ticket in an order that puts every
// task after its two upstream tasks, so the sweep cannot deadlock for any
// grid size; planes without internal nodes are forwarded to the downstream
// cells in batches before and after the task's own planes.
//
// Arithmetic per node is the reference's: ((h^2 f + 0) + ((((pb + pa) + ra)
// + rb) + lf) + rt)) * (1 / denom) with pb, pa, ra, rb, lf, rt the plane
// below / above, row above / below, left / right values (smoothing.py:132,
// neighbour order operators.py:145-147), bitwise equal to the oracle.
#include <cstddef>

#include "gmg_kernels.cuh"
#include "gs_ptx.cuh"

namespace gmg {

namespace {

#ifndef GS_CHAIN_EXP
#define GS_CHAIN_EXP 0
#endif
#ifndef GS_CHAIN_XP
#define GS_CHAIN_XP 0  // step timing experiments (wrong results): 1 no fp64 chain, 2 no mask logic, 4 no shuffles, 8 no stores
#endif
#ifndef GS_CHAIN_TRACE
#define GS_CHAIN_TRACE 0
#endif
constexpr int CW = GS_CHAIN_COLS;             // columns per task = lanes per half-warp
constexpr int CH = 2;                         // chains (rows) per lane
constexpr int RR = GS_CHAIN_ROWS;             // rows per task
static_assert(CW == 16 && RR == 4 * CH, "lane layout: two warps of 8 columns, four row groups of two rows each");
#ifndef GS_CHAIN_SHB
#define GS_CHAIN_SHB 8
#endif
constexpr int SHB = GS_CHAIN_SHB;             // steps warp B runs behind warp A (>= 7 + KB - 1)
#ifndef GS_CHAIN_CP
#define GS_CHAIN_CP 4  // 512^3: 1.70 ms at 4, 1.76 at 8, 2.05 at 2 (with KB = 2)
#endif
// Back-off (ns) of the warps that spin on shared-memory flags -- compute warps waiting for planes /
// cells, the loader waiting for ring space, the writer waiting for steps.  Four of a CTA's five warps
// spin most of the time and share the SM's four schedulers with the cells warps, whose poll loop is on
// the critical path of every hand-off.
#ifndef GS_CHAIN_NAP_C
#define GS_CHAIN_NAP_C 0
#endif
#ifndef GS_CHAIN_NAP_L
#define GS_CHAIN_NAP_L 0
#endif
#ifndef GS_CHAIN_NAP_W
#define GS_CHAIN_NAP_W 0
#endif
#ifndef GS_CHAIN_ADAPT
#define GS_CHAIN_ADAPT 0
#endif
#ifndef GS_CHAIN_G
#define GS_CHAIN_G 2
#endif
#ifndef GS_CHAIN_NS
#define GS_CHAIN_NS 42
#endif
constexpr int G = GS_CHAIN_G;                 // planes per TMA group
constexpr int NS = GS_CHAIN_NS;               // plane slots in the ring
constexpr int NG = NS / G;
static_assert(NS % G == 0 && G % 2 == 0, "groups tile the ring; group starts 128-byte aligned");
constexpr int UCOLS = CW + 4;                 // u tile: columns k0-2 .. k0+17
constexpr int UROWB = UCOLS * 8;              // 160 B
constexpr int UPL = (RR + 2) * UROWB;         // rows rowbase-1 .. rowbase+8 of one plane: 1600 B
constexpr int FPL = RR * CW * 8;              // 1024 B
constexpr int F_OFF = NS * UPL;
constexpr int RING = NS * (UPL + FPL);
constexpr int SKEW = (CW / 2 - 1) + (RR - 1) + SHB;  // steps between the first and the last lane/chain on a plane
constexpr int NWARPS = 5;                     // compute A, compute B, TMA loader, writer, cells
constexpr int BIG = 1 << 30;
#ifndef GS_CHAIN_KB
#define GS_CHAIN_KB 2  // 512^3: 1.70 ms at (KB, SHB) = (2, 8), 1.73 at (4, 10) and (1, 7)
#endif
constexpr int KB = GS_CHAIN_KB;                         // compute steps per readiness check
#ifndef GS_CHAIN_PFD
#define GS_CHAIN_PFD -1000  // off: measured no gain at 512^3, and the early prefetches doubled the DRAM reads
#endif
constexpr int PFD = GS_CHAIN_PFD;             // L2 prefetch distance beyond the ring, in groups
constexpr int CP = GS_CHAIN_CP;                        // cell planes polled per L2 round trip
constexpr int PBIAS = 4 * NS;                 // planes >= -PBIAS map to ring positions
static_assert((G * UPL) % 128 == 0 && (G * FPL) % 128 == 0 && F_OFF % 128 == 0 && RING % 128 == 0, "ring layout");

struct __align__(128) ChCtl {
  unsigned long long bar[NG];
  int task;
  int lready;      // planes < lready (from P0-1 on) have landed
  int cstep[2];    // steps < cstep[w] of compute warp w are complete
  int wfree;       // ring space of planes < wfree may be refilled
  int bready[CW];  // per column: planes < bready[j] have the row above in the ring
  int cready[RR];  // per row: planes < cready[I] have the left column in the ring
};
constexpr size_t CH_SMEM = (size_t)RING + sizeof(ChCtl);
#ifndef GS_CHAIN_ONE_CTA
static_assert(2 * (CH_SMEM + 1024) <= 228 * 1024, "two CTAs per SM");
#endif

// Cells are self-validating 16-byte words (value, tag), written and read with single 128-bit accesses
// that bypass L1 (.cg: L2 is the point of coherence); no ordering between cells is needed, so weak
// accesses do (GS_CHAIN_STRONG=1: relaxed.gpu accesses, for A/B timing).
#ifndef GS_CHAIN_STRONG
#define GS_CHAIN_STRONG 0
#endif
__device__ __forceinline__ void cell_put(double2* p, double v, double tag) {
#if GS_CHAIN_STRONG
  asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v), "d"(tag) : "memory");
#else
  asm volatile("st.global.cg.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v), "d"(tag) : "memory");
#endif
}
__device__ __forceinline__ double2 cell_get(const double2* p) {
  double2 v;
#if GS_CHAIN_STRONG
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
#else
  asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
#endif
  return v;
}
__device__ __forceinline__ uint32_t ldg_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Ring accesses are volatile: every one of them follows (loads) or precedes (stores) a volatile
// flag access of the same thread that orders it against another warp or the TMA unit, and ptxas
// keeps volatile accesses in program order (it hoists weak ld.shared above a spin loop on a flag).
#ifndef GS_CHAIN_VLD
#define GS_CHAIN_VLD 0
#endif
#if GS_CHAIN_VLD
#define GS_CHAIN_LD "ld.volatile.shared.f64"
#else
// weak loads whose ADDRESS depends on the flag value that made them safe (dep0 below): ptxas cannot
// issue them before that flag load has returned, and does not have to keep them in program order
#define GS_CHAIN_LD "ld.shared.f64"
#endif
__device__ __forceinline__ double ldr(unsigned a) {
  double v;
  asm volatile(GS_CHAIN_LD " %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
// 0, computed from a flag value (always < 2^31) so that addresses derived from it depend on the flag load
__device__ __forceinline__ unsigned dep0(int flag) {
  unsigned z;
  asm volatile("and.b32 %0, %1, 0x80000000;" : "=r"(z) : "r"(flag));
  return z;
}
__device__ __forceinline__ void str(unsigned a, double v) {
  asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
// predicated forms (no divergent branch in the step)
__device__ __forceinline__ void ldr_if(double& v, unsigned a, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q " GS_CHAIN_LD " %0, [%1];\n}\n"
               : "+d"(v)
               : "r"(a), "r"((unsigned)p)
               : "memory");
}
__device__ __forceinline__ void str_if(unsigned a, double v, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.volatile.shared.f64 [%0], %1;\n}\n" ::"r"(a), "d"(v),
               "r"((unsigned)p)
               : "memory");
}
__device__ __forceinline__ void cell_put_if(double2* ptr, double v, double tag, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n @q st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};\n}\n" ::"l"(ptr),
               "d"(v), "d"(tag), "r"((unsigned)p)
               : "memory");
}
__device__ __forceinline__ void st_flag_if(int* f, int v, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.volatile.shared.b32 [%0], %1;\n}\n" ::"r"(sa(f)), "r"(v),
               "r"((unsigned)p)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const void* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map), "r"(x), "r"(y), "r"(z)
               : "memory");
}
__device__ __forceinline__ void stg_if(double* ptr, double v, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.global.f64 [%0], %1;\n}\n" ::"l"(ptr), "d"(v), "r"((unsigned)p)
               : "memory");
}
// bits of mask word w (planes 32 w .. 32 w + 31) that lie in the planes [P0, P1]: the chains carry a
// node along unchanged wherever its bit is clear, which is how planes outside the task's range -- also
// those of another z-slab, which do hold internal nodes -- stay untouched
__device__ __forceinline__ uint32_t wclip(int w, int P0, int P1) {
  const int lo = max(P0 - 32 * w, 0), hi = min(P1 - 32 * w, 31);
  return lo > 31 || hi < 0 ? 0u : ((0xffffffffu >> (31 - hi)) & (0xffffffffu << lo));
}
__device__ __forceinline__ unsigned slot_of(int p) { return (unsigned)((p + PBIAS) % NS); }

}  // namespace

__global__ void __launch_bounds__(32 * NWARPS, 2) gs_chain_kernel(GsChainArgs a, const __grid_constant__ ChainMaps maps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ChCtl& S = *reinterpret_cast<ChCtl*>(smem_raw + (size_t)RING);
  const unsigned ubase = sa(smem_raw);
  const unsigned fbase = ubase + F_OFF;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const Geom g = a.g;
  const int N = (int)g.N;
  const int n = N + 1;
  // this sweep's cell tags: (sequence + 1) * 4096 + plane (the sequence
  // advances only after every CTA of this launch has read it)
  const int seq = *(volatile int*)a.ctl + 1;
  const long long hseq = (long long)seq << 32;  // cell tags of this sweep: hseq | plane
  // roles of the CTA's five warps: 0, 1 compute (columns 0-7 / 8-15), 2 TMA loader, 3 writer, 4 cells
  const int role = warp;

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
    // with -DGS_CHAIN_TRACE=1 also [4] compute cycles, [5] waiting for slots, [6] for cells
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
    const int k0 = 1 + CW * c;
    const int rowbase = 1 + RR * b;
    const int Rb = min(RR, N - 1 - RR * b);
    const int2 pr = a.prange[cb];
    const int P0 = pr.x, P1 = pr.y;  // P0 > P1: no internal node in the task
    const int T = P1 >= P0 ? (P1 - P0) + SKEW + 1 : 0;
#if GS_CHAIN_EXP & 6  // timing experiments (wrong results), bit mask: 1 no loads, 2 no cell waits, 4 no cells at all
    double2* const bout = (GS_CHAIN_EXP & 6) == 2 && b + 1 < a.Bn ? a.bcell + (size_t)cb * a.cplanes * CW : nullptr;
    double2* const cout_ = (GS_CHAIN_EXP & 6) == 2 && c + 1 < a.C ? a.ccell + (size_t)cb * a.cplanes * RR : nullptr;
    const double2* const bin = nullptr;
    const double2* const cin = nullptr;
#else
    double2* const bout = b + 1 < a.Bn ? a.bcell + (size_t)cb * a.cplanes * CW : nullptr;
    double2* const cout_ = c + 1 < a.C ? a.ccell + (size_t)cb * a.cplanes * RR : nullptr;
    const double2* const bin = b > 0 ? a.bcell + (size_t)(cb - 1) * a.cplanes * CW : nullptr;
    const double2* const cin = c > 0 ? a.ccell + (size_t)(cb - a.Bn) * a.cplanes * RR : nullptr;
#endif
    if (threadIdx.x == 0) {
      S.lready = P0 - 1;
      S.cstep[0] = 0;
      S.cstep[1] = 0;
      S.wfree = P0 - 1;
    }
    if (threadIdx.x < CW) S.bready[threadIdx.x] = bin ? P0 : BIG;
    if (threadIdx.x < RR) S.cready[threadIdx.x] = cin ? P0 : BIG;
    __syncthreads();

    if (role < 2) {
      // ============================ compute ==============================
      // Two warps: warp A (role 0) owns columns k0 .. k0+7 of the task, warp B
      // (role 1) columns k0+8 .. k0+15 and runs SHB steps behind, taking A's
      // column 7 from the ring.  Lane (g, j) of a warp owns its column j and
      // the rows 2g, 2g+1.  Steps run in blocks of KB: the planes / cells /
      // (for B) steps of A that a lane needs during a block are checked once at
      // its start (one warp-uniform loop), and every lane executes the same
      // straight-line step.  A chain needs no "active" predicate: outside
      // [P0, P1] and on rows / columns outside the grid's interior its mask
      // bits are zero, so it only carries the old values along (m = old, no
      // store), which also primes prev / old for plane P0.
      const int wB = role;
      const int SH = wB ? SHB : 0;
      const int Tw = T > 0 ? (P1 - P0) + (CW / 2 - 1) + (RR - 1) + SH + 1 : 0;
      if (T > 0) {
        const int g4 = lane >> 3, j = lane & 7;
        const int col = (CW / 2) * wB + j;
        const unsigned uend = ubase + (unsigned)(NS * UPL);
        const unsigned fend = fbase + (unsigned)(NS * FPL);
        // internal-node bits of each chain's line along the planes: three words A, B, C cover the
        // planes [32 wbw, 32 wbw + 96) that the lanes touch during 32 steps, D is in flight for the next
        // 32; all lanes rotate at the same steps (a load into a register that another lane reads one
        // step later would stall the whole warp on the scoreboard)
        uint32_t mA[CH], mB[CH], mC[CH], mD[CH];
        const uint32_t* mp[CH];
        int wbw = floordiv(P0 - SKEW - SH, 32);
        const int wmax = N >> 5;
        const size_t wstride = (size_t)n * g.P;
#pragma unroll
        for (int i = 0; i < CH; ++i) {
          const int row = min(rowbase + CH * g4 + i, N);
          mp[i] = a.pmask + (size_t)row * g.P + (k0 + col + OFF);
          mA[i] = wbw >= 0 ? ldg_u32(mp[i] + (size_t)wbw * wstride) & wclip(wbw, P0, P1) : 0u;
          mB[i] = wbw + 1 >= 0 && wbw + 1 <= wmax ? ldg_u32(mp[i] + (size_t)(wbw + 1) * wstride) & wclip(wbw + 1, P0, P1) : 0u;
          mC[i] = wbw + 2 >= 0 && wbw + 2 <= wmax ? ldg_u32(mp[i] + (size_t)(wbw + 2) * wstride) & wclip(wbw + 2, P0, P1) : 0u;
          mD[i] = wbw + 3 >= 0 && wbw + 3 <= wmax ? ldg_u32(mp[i] + (size_t)(wbw + 3) * wstride) & wclip(wbw + 3, P0, P1) : 0u;
        }
        int fl0;
        do {
          fl0 = ld_flag(&S.lready);
        } while (!__all_sync(0xffffffffu, fl0 > P0));
        const unsigned z0 = dep0(fl0);
        if (tr && threadIdx.x == 0) tr[3] = gtimer();
#if GS_CHAIN_TRACE
        long long c_wait = 0;
        const long long c_start = clock64();
#endif
        const double h2 = g.h2, inv = g.inv;
        const bool jfirst = j == 0, g0 = g4 == 0;
        const bool wantB = g0 && bin, wantC = jfirst && cin && !wB;
        // flags this lane polls: the row-above cells of its column (row group 0), the left-column cells
        // of its two rows (lane 0 of each row group of warp A); lanes that need none poll lready again
        const int* const fB = wantB ? &S.bready[col] : &S.lready;
        const int* fC[CH];
#pragma unroll
        for (int i = 0; i < CH; ++i) fC[i] = wantC && CH * g4 + i < Rb ? &S.cready[CH * g4 + i] : &S.lready;
        // Ring addresses.  ub[i] / fb[i]: chain i's current plane, at row rowbase + 2g, column k0 + col
        // (chain i's own node is i rows further: an immediate offset); chain 1 is one plane behind
        // chain 0, so the addresses move down the chains and only the leading plane's is computed.
        const int ps = P0 - j - CH * g4 - SH;  // plane of chain 0 at step 0
        const unsigned lane_u = (unsigned)(1 + CH * g4) * UROWB + (unsigned)(2 + col) * 8u + z0;
        const unsigned lane_f = (unsigned)(CH * g4) * (CW * 8) + (unsigned)col * 8u + z0;
        unsigned ub[CH], fb[CH];
        double prev[CH], oo[CH];
#pragma unroll
        for (int i = 0; i < CH; ++i) {
          ub[i] = ubase + slot_of(ps - i) * UPL + lane_u;
          fb[i] = fbase + slot_of(ps - i) * FPL + lane_f;
          // values of the plane below the chain's first plane and of that plane (planes <= P0 have landed;
          // further down the ring holds garbage that never reaches an internal node)
          prev[i] = ldr(ubase + slot_of(ps - i - 1) * UPL + lane_u + (unsigned)i * UROWB);
          oo[i] = ldr(ub[i] + (unsigned)i * UROWB);
        }
        unsigned un = ubase + slot_of(ps + 1) * UPL + lane_u;  // plane above chain 0's
        int p = ps;                 // chain i of this lane is at plane p - i
        int pw = ps - 32 * wbw;     // ... at bit pw - i of the mask window
        for (int t0 = 0; t0 < Tw; t0 += KB) {
          if (t0 > 0 && (t0 & 31) == 0) {  // next 32 planes of the masks (uniform over the warp)
            ++wbw;
            pw -= 32;
#pragma unroll
            for (int i = 0; i < CH; ++i) {
              mA[i] = mB[i];
              mB[i] = mC[i];
              mC[i] = mD[i];
              mD[i] = wbw + 3 >= 0 && wbw + 3 <= wmax ? ldg_u32(mp[i] + (size_t)(wbw + 3) * wstride) & wclip(wbw + 3, P0, P1) : 0u;
            }
          }
          {  // readiness of the block's planes (chain 0 leads: planes p .. p + KB - 1, chain 1 lags one)
#if GS_CHAIN_TRACE
            const long long c0 = clock64();
#endif
            const int lo = max(p - (CH - 1), P0), hi = min(p + KB - 1, P1);
            const bool need = lo <= hi;
            int fl;
            for (;;) {
              const int a1 = ld_flag(&S.lready);
              const int b1 = ld_flag(fB);
              // warp B reads warp A's column 7 (new) SHB - 7 steps after A wrote it and overwrites the old
              // values A's column 7 reads as right neighbours SHB - 7 steps after A read them: A must have
              // finished the first step of this block
              const int s1 = ld_flag(&S.cstep[0]);
              bool ok = a1 > hi + 1 && (!wantB || b1 > hi);
              fl = a1 | b1 | s1;
#pragma unroll
              for (int i = 0; i < CH; ++i) {
                const int c1 = ld_flag(fC[i]);
                const int hc = min(p - i + KB - 1, P1);
                ok = ok && (fC[i] == &S.lready || hc < P0 || c1 > hc);
                fl |= c1;
              }
              if (__all_sync(0xffffffffu, (ok || !need) && (!wB || s1 > t0))) break;
              if (GS_CHAIN_NAP_C) __nanosleep(GS_CHAIN_NAP_C);
            }
#if GS_CHAIN_TRACE
            c_wait += clock64() - c0;
#endif
            // the block's ring loads depend on the flags just read (BIG and plane numbers are < 2^31)
            const unsigned z = dep0(fl);
#pragma unroll
            for (int i = 0; i < CH; ++i) {
              ub[i] += z;
              fb[i] += z;
            }
            un += z;
          }
#pragma unroll
          for (int k = 0; k < KB; ++k) {
            double pa[CH], fv[CH], lf[CH], rt[CH];
            pa[0] = ldr(un);
#pragma unroll
            for (int i = 1; i < CH; ++i) pa[i] = ldr(ub[i - 1] + (unsigned)i * UROWB);  // plane p - i + 1
#pragma unroll
            for (int i = 0; i < CH; ++i) {
              fv[i] = ldr(fb[i] + (unsigned)i * (CW * 8));
              rt[i] = ldr(ub[i] + (unsigned)i * UROWB + 8u);  // old right neighbour (B's column 0 / the halo column)
            }
            double rbl = ldr(ub[CH - 1] + (unsigned)CH * UROWB);  // old row below the lane's last row
#pragma unroll
            for (int i = 0; i < CH; ++i) {
#if GS_CHAIN_XP & 4
              lf[i] = prev[i];
#else
              lf[i] = __shfl_up_sync(0xffffffffu, prev[i], 1);
#endif
              // lane 0 of a row group: the column to the left from the ring (halo column: cells; B: A's column 7)
              ldr_if(lf[i], ub[i] + (unsigned)i * UROWB - 8u, jfirst);
            }
#if GS_CHAIN_XP & 4
            double ra0 = prev[CH - 1];
#else
            double ra0 = __shfl_up_sync(0xffffffffu, prev[CH - 1], 8);  // row group g - 1's last row
#endif
            ldr_if(ra0, ub[0] - UROWB, g0);  // row group 0: the halo row (cells)
            // the chains op by op (independent dependency chains side by side); chain i reads chain
            // i-1's value of the previous step, so every prev[] is read before any is replaced
            double sum[CH], hf[CH], m[CH];
            bool in[CH];
#pragma unroll
            for (int i = 0; i < CH; ++i) sum[i] = prev[i] + pa[i];
#pragma unroll
            for (int i = 0; i < CH; ++i) sum[i] = sum[i] + (i == 0 ? ra0 : prev[i - 1]);
#pragma unroll
            for (int i = 0; i < CH; ++i) sum[i] = sum[i] + (i == CH - 1 ? rbl : pa[i + 1]);
#pragma unroll
            for (int i = 0; i < CH; ++i) sum[i] = sum[i] + lf[i];
#pragma unroll
            for (int i = 0; i < CH; ++i) sum[i] = sum[i] + rt[i];
#pragma unroll
            for (int i = 0; i < CH; ++i) hf[i] = h2 * fv[i] + 0.0;  // (h2 f + 0) + S == h2 f + (S + 0)
#pragma unroll
            for (int i = 0; i < CH; ++i) {
              const double v = (hf[i] + sum[i]) * inv;
              const int idx = pw - i;  // in [0, 96)
              const uint32_t mw = idx < 32 ? mA[i] : (idx < 64 ? mB[i] : mC[i]);
              in[i] = (mw >> (idx & 31)) & 1u;
              m[i] = in[i] ? v : oo[i];
            }
#pragma unroll
            for (int i = 0; i < CH; ++i) {
              str_if(ub[i] + (unsigned)i * UROWB, m[i], in[i]);
              prev[i] = m[i];
              oo[i] = pa[i];
            }
            st_flag_if(&S.cstep[wB], t0 + k + 1, lane == 0);  // steps <= t0 + k are complete (stores above included)
            // next plane: the addresses move down the chains
#pragma unroll
            for (int i = CH - 1; i > 0; --i) {
              ub[i] = ub[i - 1];
              fb[i] = fb[i - 1];
            }
            ub[0] = un;
            un = un + UPL >= uend ? un + UPL - NS * UPL : un + UPL;
            fb[0] = fb[0] + FPL >= fend ? fb[0] + FPL - NS * FPL : fb[0] + FPL;
            ++p;
            ++pw;
          }
        }
        __syncwarp();
        if (lane == 0) st_flag(&S.cstep[wB], BIG);
#if GS_CHAIN_TRACE
        if (tr && threadIdx.x == 0) {
          tr[4] = clock64() - c_start;
          tr[5] = c_wait;
        }
#endif
      }
    } else if (role == 2) {
      // ============================ TMA loader ===========================
      // Groups of G planes (from the one holding P0-1 to the one holding
      // P1+1) into group slot (group mod NG) once every plane of its previous
      // occupant is written out; lready counts the landed planes in order.
      if (T > 0 && lane == 0) {
        const int glo = floordiv(P0 - 1, G), ghi = floordiv(P1 + 1, G);
        int gq = glo, ga = glo, wf = P0 - 1;
        // L2 prefetch of the groups PFD ahead of the ring: the ring's own depth (about 12 planes beyond
        // the 30 the lanes and the writer still hold) covers an L2 hit's latency, not a DRAM access's
        int gp = glo;
#if GS_CHAIN_TRACE
        long long l_ring = 0, l_land = 0, l_t = clock64();
#endif
        while (ga <= ghi) {
#if GS_CHAIN_TRACE
          {  // attribute the time since the last look to what the loader was blocked on
            const long long now = clock64();
            if (gq <= ghi && (gq - NG + 1) * G > wf) l_ring += now - l_t; else l_land += now - l_t;
            l_t = now;
          }
#endif
          for (const int gpe = min(ghi, gq + NG + PFD); gp <= gpe; ++gp) {
            if (gp < glo + NG) continue;  // the first ring fill is loaded directly
            tma_prefetch_3d(&maps.u, CW * c + 2, rowbase - 1, gp * G);
            tma_prefetch_3d(&maps.f, CW * c + 4, rowbase, gp * G);
          }
          while (gq <= ghi) {
            const int need = (gq - NG + 1) * G;  // planes < need must be free
            if (need > wf) {
              wf = ld_flag(&S.wfree);
              if (need > wf) break;
            }
            const int gs = umod(gq, NG);
            const unsigned bar = sa(&S.bar[gs]);
#if GS_CHAIN_EXP & 1  // timing experiment: no loads (wrong results)
            mbar_arrive(bar);
#else
            mbar_expect_tx(bar, (unsigned)(G * (UPL + FPL)));
            tma_load_3d(ubase + (unsigned)gs * (G * UPL), &maps.u, CW * c + 2, rowbase - 1, gq * G, bar);
            tma_load_3d(fbase + (unsigned)gs * (G * FPL), &maps.f, CW * c + 4, rowbase, gq * G, bar);
#endif
            ++gq;
          }
          const int ga0 = ga;
          while (ga < gq && mbar_test(sa(&S.bar[umod(ga, NG)]), (unsigned)(((ga - glo) / NG) & 1))) ++ga;
          if (ga != ga0)
            st_flag(&S.lready, ga * G);
          else if (GS_CHAIN_NAP_L)
            __nanosleep(GS_CHAIN_NAP_L);
        }
#if GS_CHAIN_TRACE
        if (tr) {
          tr[8] = l_ring;
          tr[9] = l_land;
        }
#endif
      }
    } else if (role == 3) {
      // ============================ writer ===============================
      // The downstream tasks take a cell for every plane of THEIR range.  For the planes outside this
      // task's range the values are the old ones, which no one changes: those below P0 are forwarded
      // first (the consumers need them first), those above P1 after the last plane is written.  Eight
      // planes per batch so that the loads overlap (the domain of a sparse level set leaves most
      // planes of most tasks to this loop).
      const double* u = a.u;
      const int h = lane >> 4, j = lane & 15;
      // this lane's consumer: (c, b+1) for the row cells (lanes 0..15), (c+1, b) for the column cells
      const bool fw_on = h == 0 ? bout != nullptr : (cout_ != nullptr && j < Rb);
      const int2 prd = !fw_on ? make_int2(1, 0) : a.prange[h == 0 ? cb + 1 : cb + a.Bn];
      const double* const fsrc = h == 0 ? u + ((int64_t)rowbase + RR - 1) * g.P + k0 + OFF + j
                                        : u + ((int64_t)rowbase + j) * g.P + k0 + OFF + CW - 1;
      double2* const fdst = h == 0 ? bout + j : cout_ + j;
      const int fstride = h == 0 ? CW : RR;
      const int64_t fplane = (int64_t)n * g.P;
      auto forward = [&](int lo, int hi) {
        for (int p0 = lo; p0 <= hi; p0 += 8) {
          double v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = p0 + k <= hi ? __ldcg(fsrc + (int64_t)(p0 + k) * fplane) : 0.0;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (p0 + k <= hi)
              cell_put(fdst + (size_t)(p0 + k) * fstride, v[k], __longlong_as_double(hseq | (long long)(p0 + k)));
        }
      };
      if (fw_on) forward(prd.x, T > 0 ? min(prd.y, P0 - 1) : prd.y);
      __syncwarp();
      if (T > 0) {
        // Every step: the cells of the values that just became final (row rowbase+7 of column k0+j
        // after step (q - P0) + j + 7, column k0+15 of row rowbase+I after step (q - P0) + 15 + I), read
        // from the ring; then every plane all lanes are done with goes back to HBM -- lane 0 issues one
        // 128-byte bulk copy per row (shared -> global, no registers) -- and frees its slot once the
        // copies have read it.
        const bool isB = lane < CW;
        const int q_ = isB ? lane : lane - CW;  // column j / row I
        const bool pushes = isB ? bout != nullptr : (cout_ != nullptr && q_ < RR && q_ < Rb);
        // the compute warp that produces the lane's cells, and the step after which they are final
        const int cw_ = isB ? (q_ >= CW / 2 ? 1 : 0) : 1;
        const int lagp = isB ? (q_ & (CW / 2 - 1)) + (RR - 1) + (cw_ ? SHB : 0) : (CW / 2 - 1) + q_ + SHB;
        const unsigned srco = isB ? (unsigned)RR * UROWB + (unsigned)(2 + q_) * 8u : (unsigned)(1 + q_) * UROWB + (unsigned)(CW + 1) * 8u;
        const int cstride = isB ? CW : RR;
        const unsigned uend = ubase + (unsigned)(NS * UPL);
        int cs = 0, csw = 0;
        while ((cs = ld_flag(&S.cstep[0])) < 1) {
        }
        // (plane P0-1 is read by every chain on its way to P0: its slot is freed with plane P0's)
        // cell source / destination of plane qc, write-back source / destination of plane qw
        int qc = P0, qw = P0;
        unsigned csrc = ubase + slot_of(P0) * UPL + srco;
        double2* cdst = pushes ? (isB ? bout : cout_) + (size_t)P0 * cstride + q_ : nullptr;
        // write-back: lane (h, j) copies rows rowbase + h, + 2, + 4, + 6 of column k0 + j
        const int h = lane >> 4, j = lane & 15;
        unsigned wsrc = ubase + slot_of(P0) * UPL + (unsigned)(1 + h) * UROWB + (unsigned)(2 + j) * 8u;
        const size_t wplane = (size_t)n * g.P, wrow = (size_t)g.P;
        double* wd[RR / 2];
        bool wok[RR / 2];
#pragma unroll
        for (int w = 0; w < RR / 2; ++w) {
          wd[w] = a.u + ((int64_t)P0 * n + rowbase + 2 * w + h) * g.P + k0 + OFF + j;
          wok[w] = 2 * w + h < Rb && k0 + j <= N;
        }
        long long ctag = hseq | (long long)P0;
#if GS_CHAIN_TRACE
        long long w_wait = 0, w_busy = 0, w_t = clock64();
#endif
        while (qw <= P1) {
          {
            const int ca = ld_flag(&S.cstep[0]);
            csw = ld_flag(&S.cstep[1]);  // warp B finishes every plane last
            cs = cw_ ? csw : ca;
          }
#if GS_CHAIN_TRACE
          {
            const long long now = clock64();
            if (csw >= (qw - P0) + SKEW + 1) w_busy += now - w_t; else w_wait += now - w_t;
            w_t = now;
          }
#endif
          const unsigned z = dep0(cs | csw);
          if (pushes)
            while (qc <= P1 && cs > (qc - P0) + lagp) {
              cell_put(cdst, ldr(csrc + z), __longlong_as_double(ctag));
#if GS_CHAIN_TRACE
              if (a.trace && lane == 0) a.trace[(size_t)a.ntasks * 16 + ((size_t)cb * 2 + 0) * a.cplanes + qc] = gtimer();
#endif
              ++qc;
              ++ctag;
              cdst += cstride;
              csrc = csrc + UPL >= uend ? csrc + UPL - NS * UPL : csrc + UPL;
            }
          __syncwarp();
          const int qw0 = qw;
          while (qw <= P1 && csw >= (qw - P0) + SKEW + 1) {  // plane qw is final once warp B's step SKEW is done
            double v[RR / 2];
#pragma unroll
            for (int w = 0; w < RR / 2; ++w) v[w] = ldr(wsrc + z + (unsigned)(2 * w) * UROWB);
#pragma unroll
            for (int w = 0; w < RR / 2; ++w) {
              stg_if(wd[w], v[w], wok[w]);
              wd[w] += wplane;
            }
            (void)wrow;
            ++qw;
            wsrc = wsrc + UPL >= uend ? wsrc + UPL - NS * UPL : wsrc + UPL;
          }
          if (qw != qw0) {
            __syncwarp();  // every lane's ring reads of the planes < qw are done
            st_flag_if(&S.wfree, qw, lane == 0);
          } else if (GS_CHAIN_NAP_W) {
            __nanosleep(GS_CHAIN_NAP_W);
          }
        }
#if GS_CHAIN_TRACE
        if (tr && lane == 0) {
          tr[6] = w_wait;
          tr[7] = w_busy;
        }
#endif
        if (fw_on) forward(max(prd.x, P1 + 1), prd.y);
      }
    } else {
      // ============================ cells ================================
      // Lanes 0..15: the row above the block, column k0+j, from task (c, b-1)'s
      // cells; lanes 16..23: column k0-1 of row rowbase+I from task (c-1, b).
      // CP planes polled per L2 round trip, so the hand-off keeps pace with an
      // upstream task up to CP planes per trip.
      const bool isB = lane < CW;
      const int q_ = isB ? lane : lane - CW;  // column j / row I
      const double2* const src = isB ? bin : cin;
      const bool on = T > 0 && src && (isB || (q_ < RR && q_ < Rb));
      if (on) {
        const int stride = isB ? CW : RR;
        const unsigned dsto = isB ? (unsigned)(2 + q_) * 8u : (unsigned)(1 + q_) * UROWB + 8u;
        int* const ready = isB ? &S.bready[q_] : &S.cready[q_];
        int p = P0;
#if GS_CHAIN_TRACE
        long long rtt_sum = 0, rtt_n = 0, it_n = 0, it_hit = 0;
#endif
#if GS_CHAIN_ADAPT
        int want = 1;  // cells per poll: 1 while the upstream has nothing new, doubling up to CP while it is ahead
#else
        constexpr int want = CP;
#endif
        while (p <= P1) {
          // the next CP cells of this lane, whether or not the upstream task has produced them yet (their
          // tags decide); only planes the ring already holds.  One poll in flight per lane: a second
          // one half a round trip later was measured slower (1.80 vs 1.70 ms at 512^3; the extra L2
          // traffic lengthens every round trip), as were CP = 8 and 16.
          const int top = min(P1, ld_flag(&S.lready) - 1);
          double2 v[CP];
#if GS_CHAIN_TRACE
          const long long tq0 = clock64();
#endif
#pragma unroll
          for (int k = 0; k < CP; ++k) {
            const int q = p + k;
            v[k] = q <= top && k < want ? cell_get(src + (size_t)q * stride + q_) : make_double2(0.0, -1.0);
          }
#if GS_CHAIN_TRACE
          if (p <= top) {  // cycles until the poll's last cell is back (the compare below needs it)
            long long tq1;  // read the clock only once both the first and the last cell have arrived
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(tq1) : "l"(__double_as_longlong(v[CP - 1].y)), "l"(__double_as_longlong(v[0].y)) : "memory");
            rtt_sum += tq1 - tq0;
            ++rtt_n;
          }
          ++it_n;
#endif
          int adv = 0;
#pragma unroll
          for (int k = 0; k < CP; ++k) {
            if (adv == k && __double_as_longlong(v[k].y) == (hseq | (long long)(p + k))) {
              str(ubase + slot_of(p + k) * UPL + dsto, v[k].x);
#if GS_CHAIN_TRACE
              if (a.trace && lane == 0) a.trace[(size_t)a.ntasks * 16 + ((size_t)cb * 2 + 1) * a.cplanes + p + k] = gtimer();
#endif
              adv = k + 1;
            }
          }
          if (adv) {
            p += adv;
            st_flag(ready, p);
#if GS_CHAIN_TRACE
            ++it_hit;
#endif
          }
          else if (p <= top && a.poll_nap > 0) {
            // nothing new from the upstream task: when more tasks than CTA slots share the L2 (512^3 and up)
            // a pause before the next poll takes 2-3 % off the sweep; on the hop-bound smaller levels it
            // only adds latency (128^3: 157 -> 179 us with 1 us), so the host sets it per level
            __nanosleep(a.poll_nap);
          }
#if GS_CHAIN_ADAPT
          want = adv == want ? min(2 * want, CP) : 1;
#endif
        }
#if GS_CHAIN_TRACE
        if (tr && lane == 0) {
          tr[10] = rtt_sum;
          tr[11] = rtt_n;
          tr[12] = it_n;
          tr[13] = it_hit;
        }
#endif
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

// plane-transposed internal-node mask: word ((pw * n + r) * P + pos), bit b <=> node (32 pw + b, r, pos) internal
__global__ void chain_pmask_kernel(Geom g, const uint8_t* __restrict__ labels, uint32_t* __restrict__ pm, int64_t total) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int64_t plane = g.n * g.P;
  const int64_t pw = idx / plane, rem = idx - pw * plane;
  uint32_t w = 0;
  for (int bbit = 0; bbit < 32; ++bbit) {
    const int64_t p = 32 * pw + bbit;
    if (p < g.n && labels[p * plane + rem] == INTERNAL) w |= 1u << bbit;
  }
  pm[idx] = w;
}

size_t gs_chain_smem() { return CH_SMEM; }
int gs_chain_group() { return G; }

void configure_gs_chain() {
  cudaFuncSetAttribute(gs_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CH_SMEM);
  cudaFuncSetAttribute(gs_chain_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

void launch_gs_chain(const GsChainArgs& a, const ChainMaps& maps, int grid, cudaStream_t st) {
  gs_chain_kernel<<<grid, 32 * NWARPS, CH_SMEM, st>>>(a, maps);
}

void launch_chain_pmask(const Geom& g, const uint8_t* labels, uint32_t* pm, cudaStream_t st) {
  const int64_t total = ((g.n + 31) / 32) * g.n * g.P;
  chain_pmask_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(g, labels, pm, total);
}

}  // namespace gmg
