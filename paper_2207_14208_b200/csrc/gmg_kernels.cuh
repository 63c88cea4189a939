// gmg_kernels.cuh -- kernel argument blocks and launch entry points.
#pragma once

#include <cuda.h>

#include "gmg_common.cuh"

namespace gmg {

struct GsArgs {
  Geom g;
  const uint8_t* labels;
  double* u;
  const double* f;
  const int2* tasks;  // (chunk c, block b) in wavefront order
  const uint8_t* empty;  // gs_diag: task without internal nodes (published as done at once), or null
  int ntasks;
  int* ticket;
  int* progress;      // completed lines per task, at progress[pstride * (c * Bn + b)]
  int pstride;        // ints between two tasks' progress words (4 or 32: one 128-byte line each)
  double* edge;       // gs_macro: per-cell hand-off of each block's last row, (value, tag) pairs
                      // [task c * Bn + b][plane 0..N][32 columns]; all tags zero between sweeps, or null
  const uint8_t* empty_cb;  // task (c * Bn + b) has no internal node
  int B1, Bn, C;
  const uint32_t* imask;  // per (line, chunk) bitmask of internal nodes, row stride Cm
  int Cm;                 // C rounded up to a multiple of 4
  long long* trace;       // diagnostics: [ntasks][16] timeline per task, or null
  int sleep_ns[4];        // back-off of the u / f / halo loaders and the writer when idle
  int halo_multi;         // gs_diag: halo loader issues up to 4 ready batches per poll (levels with
                          // at most ~1 task per SM; the 2-batch loader is faster when 4 share an SM)
};

// Ghost rows of one level, stored in sweep-slot order (batch, then lex).
struct GhostArgs {
  Geom g;
  int64_t ng;            // slots (ghosts padded per batch); node < 0 marks an empty slot
  const int64_t* node;   // ghost node
  const int64_t* base;   // flat index of the 3^d block's low corner
  const double* w;       // [m][ng] row weights, m = 3^d
  const double* dtau;
  const double* gval;    // right-hand side per slot
  const uint8_t* promoted;
};

struct BandArgs {
  Geom g;
  int64_t nb;
  const int64_t* idx;     // band nodes, BFS groups concatenated
  const uint8_t* mask;    // BFS assigned-neighbour bits
  const int8_t* step;     // [nb][d] upwind step
  const double* absn;     // [nb][d]
  double* scratch;        // [nb]
  // compact transport: slots [0, nb) band nodes, [nb, nb + nfix) fixed upwind neighbours
  int64_t nfix;
  const int64_t* fixpos;  // [nfix] positions of the fixed neighbours
  const int32_t* nbr;     // [nb][d] slot of the upwind neighbour along each axis
  double *v0, *v1;        // [nb + nfix] ping-pong values
};

// gs_chain.cu (3-D production kernel): one warp per task of GS_CHAIN_COLS columns x GS_CHAIN_ROWS rows,
// register chains, per-node cells between tasks
#define GS_CHAIN_COLS 16
#define GS_CHAIN_ROWS 8
struct GsChainArgs {
  Geom g;
  double* u;
  const int2* tasks;      // (chunk c, block b), every task after (c-1, b) and (c, b-1)
  const int2* prange;     // per task c * Bn + b: first / last plane with an internal node (first > last: none)
  const uint32_t* pmask;  // plane-transposed internal-node bits: word ((p >> 5) * n + r) * P + pos, bit p & 31
  int ntasks, C, Bn;
  int cplanes;            // planes per task in the cell arrays (N + 1 + 32: the chains run past the last plane)
  int* ctl;               // [0] sweep sequence, [1] finished CTAs, [2] ticket (zero between sweeps)
  double2* bcell;         // [c * Bn + b][cplanes][GS_CHAIN_COLS]: (value, tag) of the block's last row, per plane
  double2* ccell;         // [c * Bn + b][cplanes][GS_CHAIN_ROWS]: (value, tag) of the chunk's last column
  long long* trace;       // diagnostics: [ntasks][16] per task (ticket order), or null
  int poll_nap;           // ns the cells warp pauses after a poll that brought nothing (0: none)
};
struct ChainMaps {  // boxes of gs_chain_group() planes
  CUtensorMap u;    // (P, n, n) doubles, box (GS_CHAIN_COLS + 4) x (GS_CHAIN_ROWS + 2) x G
  CUtensorMap f;    // (P, n, n) doubles, box GS_CHAIN_COLS x GS_CHAIN_ROWS x G
};
void launch_gs_chain(const GsChainArgs& a, const ChainMaps& maps, int grid, cudaStream_t st);
void launch_chain_pmask(const Geom& g, const uint8_t* labels, uint32_t* pm, cudaStream_t st);
size_t gs_chain_smem();
int gs_chain_group();
void configure_gs_chain();

void launch_gs_small(const Geom& g, const uint8_t* labels, double* u, const double* f, cudaStream_t st);
void launch_gs_sweep(const GsArgs& a, int grid, cudaStream_t st);
void launch_gs_stream(const GsArgs& a, int grid, int warps_per_cta, cudaStream_t st);
size_t gs_stream_smem_per_warp();
// TMA tensor maps of one level for the warp-specialised GS kernel
struct WsMaps {
  CUtensorMap u, f, m;
  CUtensorMap m2;  // 3-D: internal-node masks per (plane, block, pseudo-line), zero on halo lines
  CUtensorMap ust; // u as (plane, row, col) with 7-row boxes (3-D) / (row, col) 8-row boxes (2-D), TMA stores
};
void launch_gs_diag(const GsArgs& a, const WsMaps& maps, int grid, cudaStream_t st);
size_t gs_diag_smem();
void configure_gs_kernels();  // set max dynamic shared memory of the GS / GEMV kernels

void launch_ghost_batch(const GhostArgs& a, double* u, int64_t lo, int64_t hi, double* pair, cudaStream_t st);
void launch_ghost_levels(const GhostArgs& a, double* u, const int64_t* boff, int nbatch, const int32_t* dep_off,
                         const int32_t* dep, const uint32_t* vmask, double* pair, int* counter, int sms,
                         cudaStream_t st);
void launch_ghost_persistent(const GhostArgs& a, double* u, const int32_t* dep_off, const int32_t* dep,
                             const uint32_t* vmask, double* pair, int* cursor, int sms, int blocks_per_sm,
                             int backoff, long long* gtrace, bool defer, cudaStream_t st);
void launch_ghost_writeback(const GhostArgs& a, const double* pair, double* u, cudaStream_t st);
void launch_residual_ghost(const GhostArgs& a, const double* u, double* r_ext,
                           unsigned long long* maxbits, cudaStream_t st);
void launch_residual_ghost_lex(const GhostArgs& a, const double* wl, const int64_t* basel, const int64_t* nodel,
                               const int32_t* l2s, int64_t ng, const double* u, double* r_ext,
                               unsigned long long* maxbits, int64_t i0, int64_t i1, cudaStream_t st);
void launch_residual_interior(const Geom& g, const uint8_t* labels, const double* u,
                              const double* f, double* r, unsigned long long* maxbits,
                              cudaStream_t st, unsigned long long* peakbits = nullptr);
// the same over the internal planes [p_lo, p_hi] only (3-D, z-slab mode)
void launch_residual_interior_planes(const Geom& g, const uint8_t* labels, const double* u, const double* f, double* r,
                                     unsigned long long* maxbits, int p_lo, int p_hi, cudaStream_t st);
void launch_band_step(const BandArgs& a, double* x, cudaStream_t st);
void launch_band_bfs(const BandArgs& a, double* x, int64_t lo, int64_t hi, cudaStream_t st);
void launch_band_transport(const BandArgs& a, double* x, cudaStream_t st);
bool launch_band_coop(const BandArgs& a, double* x, const int64_t* goff, int ngroups, cudaStream_t st);
void launch_restrict_interior(const Geom& gf, const double* r_f, const Geom& gc, const uint32_t* rmask,
                              double* f_c, cudaStream_t st);
void launch_res_restrict3(const Geom& gf, const uint8_t* labels, const double* u, const double* f, const Geom& gc,
                          const uint32_t* rmask, double* f_c, cudaStream_t st);
void launch_restrict_mask(const Geom& gf, const uint8_t* lab_f, const Geom& gc, const uint8_t* lab_c,
                          uint32_t* rmask, cudaStream_t st);
void launch_restrict_ghost(const Geom& gf, const uint8_t* lab_f, const double* r_ext,
                           const GhostArgs& coarse, double* gval_c, const int32_t* order, int64_t n_lex,
                           cudaStream_t st);
void launch_interp_add(const Geom& gf, const uint8_t* lab_f, double* u_f, const Geom& gc,
                       const double* e_c, cudaStream_t st);
void launch_initial_field(const Geom& g, const uint8_t* labels, double* u, uint64_t state, const uint64_t* cols, int K,
                          int64_t len, cudaStream_t st);
void launch_abs_max(const double* u, int64_t n, unsigned long long* maxbits, cudaStream_t st);
void launch_scale(double* u, int64_t n, double s, cudaStream_t st);
void launch_gather(const int64_t* idx, int64_t n_int, const double* f, const int32_t* ghost_slot,
                   int64_t n_gh, const double* gval, double* out, cudaStream_t st);
void launch_scatter(const int64_t* idx, int64_t n, const double* x, double* e, cudaStream_t st);
void launch_dense_gemv(const double* A, const double* x, int64_t n, double* part, double* y, cudaStream_t st);
int gemv_chunks(int64_t n);
void launch_gemv_rect(const double* A, const double* x, int64_t m, int64_t k, double* part, const double* y0,
                      double* y, cudaStream_t st);
int64_t gemv_rect_part_size(int64_t m, int64_t k);
void launch_csr_residual(const int64_t* rowptr, const int32_t* col, const double* val, const double* x,
                         const double* y0, int64_t m, double* t, cudaStream_t st);
void launch_repitch(const double* src, double* dst, int64_t rows, int64_t n, int64_t P, bool to_padded,
                    cudaStream_t st);
void launch_l2_leaves_scan(const uint8_t* lab, const double* r, const int64_t* start, const int64_t* end,
                           const int32_t* len, int64_t nleaves, double* vals, cudaStream_t st);
void launch_l2_leaves_list(const double* x, const int64_t* pos, const int32_t* slot, const int64_t* off,
                           const int32_t* len, int64_t nleaves, double* vals, cudaStream_t st);
void launch_l2_combine(double* vals, const int32_t* a, const int32_t* b, const int32_t* dst, int64_t n,
                       cudaStream_t st);
void launch_permute(const double* src, const int32_t* perm, int64_t n, double* dst,
                    cudaStream_t st);

}  // namespace gmg
