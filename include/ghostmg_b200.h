/*
 * ghostmg_b200.h -- C ABI of the B200-native ghost-point multigrid V-cycle.
 *
 * The reference (arXiv 2207.14208 artifact `ghostmg`, pure Python) has no
 * FFI; its drop-in seam is the Python solver object.  Each entry point
 * below replaces one piece of that object, cited as
 *   ref: /root/reference/pkg/src/ghostmg/<file>:<lines>
 * The Python host layer (paper_2207_14208_b200/solver.py) binds these with
 * ctypes and keeps the reference's build_solver / solve / measure_rho API.
 *
 * Conventions: plain pointers and sizes only; host arrays are read/written
 * synchronously unless stated; device memory is owned by the context.
 * Every int-returning call returns 0 on success and a negative code on
 * failure, with a message in gmg_last_error().  Grid arrays are flat
 * C-order (N+1)^d float64 like the reference (geometry.py:91-111); ghost
 * vectors follow the ascending ghost order (geometry.py:416).
 */
#ifndef GHOSTMG_B200_H
#define GHOSTMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gmg_ctx gmg_ctx;

/* Coarsest-level direct solve supplied by the host (the reference's SciPy
 * SuperLU object, ref solver.py:146-166): solve A x = rhs for the active
 * unknowns (internal then ghost).  Return 0 on success. */
typedef int (*gmg_coarse_cb)(void *user, int64_t n, const double *rhs, double *x);

/* vector selectors for gmg_set_vector / gmg_get_vector / gmg_device_pointer */
enum gmg_vector {
  GMG_U = 0,      /* iterate / coarse error, full grid                      */
  GMG_F = 1,      /* interior right-hand side, full grid                    */
  GMG_G = 2,      /* ghost-row right-hand side, ascending ghost order       */
  GMG_R_INT = 3,  /* interior residual scratch, full grid                   */
  GMG_R_EXT = 4   /* ghost residual + band extension scratch, full grid     */
};

/* single-operation hooks for gmg_apply (parity tests, profiling) */
enum gmg_op {
  GMG_OP_GS_SWEEP = 0,       /* ref smoothing.py:127-132 gs_lex_sweep        */
  GMG_OP_GHOST_SWEEP = 1,    /* ref smoothing.py:135-142 ghost_relax_sweep   */
  GMG_OP_SMOOTH = 2,         /* ref smoothing.py:145-149 smooth(count)       */
  GMG_OP_RES_INT = 3,        /* ref smoothing.py:111-118 -> GMG_R_INT        */
  GMG_OP_RES_GHOST = 4,      /* ref smoothing.py:120-124 -> GMG_R_EXT ghosts */
  GMG_OP_EXTEND_REXT = 5,    /* ref transfer.py:241-252 on GMG_R_EXT         */
  GMG_OP_EXTEND_U = 6,       /* ref transfer.py:241-252 on GMG_U             */
  GMG_OP_RESTRICT_INT = 7,   /* ref transfer.py:88-93  R_INT(l) -> F(l+1)    */
  GMG_OP_RESTRICT_GHOST = 8, /* ref transfer.py:116-121 R_EXT(l) -> G(l+1)   */
  GMG_OP_INTERP_ADD = 9,     /* ref transfer.py:149-151 + solver.py:198      */
  GMG_OP_ZERO_U = 10,
  GMG_OP_COARSE_SOLVE = 11,  /* ref solver.py:157-166 on the coarsest level */
  GMG_OP_RES_RESTRICT = 12,  /* 3-D: smoothing.py:111-118 fused into transfer.py:88-93,
                                U, F(l) -> F(l+1) without materialising R_INT */
  /* z-slab schedule (paper_2207_14208_b200/slabs.py): the band extension of
     transfer.py:241-252 phase by phase, so the slabs can exchange a halo plane
     between phases, and the tail of a cycle on an agglomerated level */
  GMG_OP_BAND_BFS_REXT = 13, /* BFS group `count` of the extension of GMG_R_EXT  */
  GMG_OP_BAND_BFS_U = 14,    /* ... of GMG_U                                      */
  GMG_OP_BAND_STEP_REXT = 15,/* one Jacobi transport step on GMG_R_EXT            */
  GMG_OP_BAND_STEP_U = 16,   /* ... on GMG_U                                      */
  GMG_OP_CYCLE_TAIL = 17     /* ref solver.py:190-197 from level l down: U(l) = 0, gamma cycles
                                (or the coarsest solve) with F(l), G(l), then the band
                                extension of U(l)                                 */
};

/* z-slab mode: this context updates only the planes
 * [lo, hi) (reference axis 0, geometry.py:108-111) of level `level`: the GS
 * and ghost sweeps (smoothing.py:127-142), both residuals and the norms
 * (smoothing.py:111-124, solver.py:135-142) touch only nodes / ghosts of those
 * planes; the other operations still run on the whole level, which is
 * harmless because the slab schedule refreshes the neighbour planes they read.
 * Only 3-D levels with N >= 64 can be split; lo = 0, hi = N + 1 restores the
 * whole level.  Returns the number of BFS groups of the level's band plan. */
int gmg_set_slab(gmg_ctx* ctx, int level, int64_t lo, int64_t hi);

/* max |u| over the planes [lo, hi) of the finest level (the slab's part of the
 * renormalisation guard, reference solver.py:239-243). */
int gmg_abs_max_planes(gmg_ctx* ctx, int64_t lo, int64_t hi, double* peak);

/* The seeded initial iterate on the device (reference solver.py:205-213:
 * uniform(-1, 1) from XorShift64Star(seed), rng.py:14-56, prescribed values on
 * eliminated nodes, 0 on inactive ones) written straight into GMG_U of the
 * finest level.  `state` is the seeded generator state, `jump_cols` holds K
 * sets of 64 column images: set b is the GF(2) matrix of `lane_len * 2^b`
 * generator steps (K * 64 words; K must cover the number of lanes).  The
 * eliminated nodes come as (flat index, value) pairs.  Bit for bit the
 * sequential stream of the reference. */
int gmg_initial_field(gmg_ctx* ctx, uint64_t state, const uint64_t* jump_cols, int K, int64_t lane_len,
                      int64_t n_elim, const int64_t* elim_idx, const double* elim_val);

/* ---- setup on the device -------------------------
 * Node labels of one level for the ball family of level sets (reference
 * classify, geometry.py:374-416: sign of phi, box faces, internal neighbours):
 * kind 0 = pore space, domain outside n_balls balls (phi = max_k (r_k - |x - c_k|)),
 * kind 1 = signed sphere (phi = |x - c| - R).  `axis` holds the N + 1 node
 * coordinates of one axis, `face_mask` bit 2*axis + side the eliminated faces,
 * `labels_out` the flat C-order (N+1)^d labels (0 internal, 1 ghost, 2
 * inactive, 3 eliminated), bit for bit the host classification before the
 * promotion closure (which, like the ghost geometry, runs on the host). */
int gmg_setup_classify_balls(int device, int d, int64_t N, const double* axis, int kind, int n_balls,
                             const double* centers, const double* radii, int face_mask, uint8_t* labels_out);
/* What the reference's restriction constructors raise (transfer.py:64-114),
 * checked for every coarse node: flags 1 interior block leaves the box, 2 mixed
 * block without an internal node, 4 coarse ghost without an in-box ghost /
 * inactive fine node, 8 / 16 block centre with the wrong fine label. */
int gmg_setup_check_transfer(int device, int d, int64_t Nf, const uint8_t* lab_f, int64_t Nc, const uint8_t* lab_c,
                             int* flags_out);
const char* gmg_setup_last_error(void);

/* Library version (major*10000 + minor*100 + patch). */
int gmg_version(void);

/* Create a context for `nlevels` grid levels of dimension `ndim` (2 or 3)
 * on CUDA device `device`.  Replaces MultigridSolver.__init__'s per-level
 * plan construction (ref solver.py:103-127).  NULL on failure. */
gmg_ctx *gmg_create(int device, int ndim, int nlevels);
void gmg_destroy(gmg_ctx *ctx);
const char *gmg_last_error(const gmg_ctx *ctx);

/* Launch on a caller-owned cudaStream_t (e.g. torch's current stream);
 * NULL restores the context's own stream. */
int gmg_set_stream(gmg_ctx *ctx, void *cuda_stream);

/* Upload one level: labels (ref geometry.py:374-431), ghost rows
 * (ref operators.py:73-96, smoothing.py:50-77, 80-109: block low corner,
 * 3^d weights, dtau, promotion flag), the order-equivalent ghost sweep
 * batches, and the band plan (ref transfer.py:154-239: BFS group lengths,
 * band nodes, neighbour masks, upwind steps, |n|). */
int gmg_set_level(gmg_ctx *ctx, int level, int64_t N, double reaction,
                  const uint8_t *labels, int64_t n_ghost, const int64_t *ghost_idx,
                  const int64_t *ghost_low, const double *ghost_w,
                  const double *ghost_dtau, const uint8_t *ghost_promoted,
                  const int32_t *ghost_batch, int n_groups, const int64_t *bfs_len,
                  const int64_t *band_idx, const uint8_t *bfs_mask,
                  const int8_t *trans_step, const double *trans_absn);

/* Cycle parameters (ref smoothing.py:30-47 SmootherConfig, solver.py:49-69
 * CycleConfig): nu1, nu2, gamma (1 = V, 2 = W), coarse_mode (0 = host
 * callback direct solve, 1 = `coarse_sweeps` smoothing sweeps, 2 = device
 * dense inverse set by gmg_set_coarse_inverse), norm (0 = inf, 1 = l2). */
int gmg_set_cycle(gmg_ctx *ctx, int nu1, int nu2, int gamma, int coarse_mode,
                  int coarse_sweeps, int norm);
int gmg_set_coarse_callback(gmg_ctx *ctx, gmg_coarse_cb cb, void *user);
/* Dense inverse (row-major n x n, n = internal + ghost unknowns of the
 * coarsest level, ordered like gmg_coarse_cb's rhs) for coarse_mode 2; the
 * pointer is host memory or (on_device != 0) device memory, copied. */
int gmg_set_coarse_inverse(gmg_ctx *ctx, int64_t n, const double *inv, int on_device);
/* The same coarse_mode-2 solve by one level of nested dissection (takes
 * precedence over the dense inverse): the n unknowns permuted to [A | B | S]
 * (perm[i] = index in gmg_coarse_cb's rhs order of permuted unknown i; A and B
 * decoupled, S their separator), row-major blocks AAi (na x na) = A_AA^-1,
 * BBi (nb x nb) = A_BB^-1, G (ns x (na+nb)) = [A_SA AAi, A_SB BBi],
 * W ((na+nb) x ns) = [AAi A_AS; BBi A_BS], Si (ns x ns) = the inverse Schur
 * complement.  Host or (on_device != 0) device pointers, copied.
 * Replaces the reference's splu solve (solver.py:146-166) like the inverse. */
int gmg_set_coarse_nd(gmg_ctx *ctx, int64_t n, int64_t na, int64_t nb, int64_t ns, const int32_t *perm,
                      const double *aai, const double *bbi, const double *g, const double *w,
                      const double *si, int on_device);
/* Optional: the separator rows' coupling [A_SA A_SB] as host CSR (ns rows,
 * columns in the permuted [A | B] order); the reduced right-hand side is then
 * b_S - C [AAi b_A; BBi b_B] with a sparse product instead of the dense G. */
int gmg_set_coarse_nd_coupling(gmg_ctx *ctx, int64_t ns, int64_t nab, const int64_t *rowptr,
                               const int32_t *col, const double *val);
/* General form of the coarse_mode-2 solve (takes precedence over both of the
 * above): a program of dense / sparse products on a workspace of nwork
 * doubles.  begin: perm[i] = rhs-order index of workspace entry i (the
 * permuted rhs lands in [0, n)); dense: y = M x, or y = y0 - M x when
 * y0_off >= 0 (M row-major m x k, host or device memory, copied); csr:
 * y = y0 - C x (host CSR, m rows, columns < k); end: the solution (permuted
 * order) is at [x_off, x_off + n).  Used for recursive nested dissection. */
int gmg_coarse_prog_begin(gmg_ctx *ctx, int64_t n, const int32_t *perm, int64_t nwork);
int gmg_coarse_prog_dense(gmg_ctx *ctx, int64_t m, int64_t k, const double *M, int on_device,
                          int64_t x_off, int64_t y_off, int64_t y0_off);
int gmg_coarse_prog_csr(gmg_ctx *ctx, int64_t m, int64_t k, const int64_t *rowptr, const int32_t *col,
                        const double *val, int64_t x_off, int64_t y0_off, int64_t y_off);
int gmg_coarse_prog_end(gmg_ctx *ctx, int64_t x_off);

/* Host <-> device copies of a level vector (see enum gmg_vector).  The host
 * array must hold exactly gmg_vector_length(ctx, level, which) doubles
 * (the reference raises IndexError on a wrongly sized u; the Python binding
 * checks the length before every copy). */
int64_t gmg_vector_length(const gmg_ctx *ctx, int level, int which);
int gmg_set_vector(gmg_ctx *ctx, int level, int which, const double *host);
int gmg_get_vector(gmg_ctx *ctx, int level, int which, double *host);
/* Device address of a level vector (valid for the context's lifetime).  Grids
 * are stored padded (row pitch roundup(N+4,4), column offset 3); GMG_G is
 * stored in sweep-slot order (batches padded to 32 slots), not ghost order. */
void *gmg_device_pointer(gmg_ctx *ctx, int level, int which);

/* Run one operation on a level (see enum gmg_op). */
int gmg_apply(gmg_ctx *ctx, int level, int op, int count);

/* Run `ncycles` cycles on level 0 in place (ref solver.py:170-203
 * _cycle/run_cycle).  Asynchronous on the context stream except for the
 * host coarse callback, which synchronizes.  Without a host callback the
 * whole cycle is captured once into a CUDA graph and replayed. */
int gmg_cycle(gmg_ctx *ctx, int ncycles);

/* Residual norms of a level (ref solver.py:135-142): out[0] = max |r_int|,
 * out[1] = max |r_ghost| (norm = inf), or out[0] = sum r_int^2 and
 * out[1] = sum r_ghost^2 in NumPy's pairwise order (norm = l2).
 * Synchronizes. */
int gmg_residual_norm(gmg_ctx *ctx, int level, double *out);

/* The same, and *peak_lb = max |u| over the level's internal nodes, taken in
 * the same pass (the values are loaded for the residual anyway): a lower bound
 * of the max |u| that the renormalisation guard of the solve loop tests
 * (ref solver.py:239-243, `0 < peak < RENORM_THRESHOLD`), so a caller that
 * finds it >= the threshold knows the guard's outcome without
 * gmg_abs_max_scale's pass over the full array.  -1 when it was not computed
 * (l2 norm, z-slab mode); 0 on a level without internal nodes.  Synchronizes. */
int gmg_residual_norm_peak(gmg_ctx *ctx, int level, double *out, double *peak_lb);

/* peak = max |u| on level 0; if 0 < peak < threshold, u *= factor and
 * *scaled = 1 (ref solver.py:239-243).  Synchronizes. */
int gmg_abs_max_scale(gmg_ctx *ctx, double threshold, double factor, double *peak,
                      int *scaled);

int gmg_synchronize(gmg_ctx *ctx);

/* Kernels launched by this context so far. */
int64_t gmg_launch_count(const gmg_ctx *ctx);
/* Batched solves (many contexts, one stream each; inf norm): norm_begin
 * enqueues residual_norm's two maxima (ref solver.py:135-142) and max|u|
 * (the renormalisation guard, solver.py:239-243) of the finest level with an
 * asynchronous copy; norm_end waits for this context's stream and returns
 * {max|r_int|, max|r_g|, max|u|}; scale_u multiplies the finest u. */
int gmg_norm_begin(gmg_ctx *ctx);
int gmg_norm_end(gmg_ctx *ctx, double *out3);
int gmg_scale_u(gmg_ctx *ctx, double factor);

/* Diagnostics: with GMG_GS_TRACE=1 in the environment the Gauss-Seidel
 * kernel records 16 int64 per task (start/end globaltimer ns, SM id, compute
 * warp cycles waiting for data / in total, loader waits and idle polls, see
 * tools/gs_trace.py).  Copies up to `cap` values of the last sweep on
 * `level`; returns the count (0 if not traced). */
int64_t gmg_debug_gs_trace(gmg_ctx *ctx, int level, long long *host, int64_t cap);
/* Diagnostics: ghost-sweep timeline (GMG_GS_TRACE=1), 3 int64 per sweep slot
 * (claimed, dependencies met, stored; globaltimer ns) of the last sweep. */
int64_t gmg_debug_ghost_trace(gmg_ctx *ctx, int level, long long *host, int64_t cap);
/* Diagnostics: GS loader / writer back-off (4 values, ns; NULL keeps them)
 * and implementation variant (< 0 keeps it) for the following sweeps. */
int gmg_debug_gs_knobs(gmg_ctx *ctx, const int *sleep_ns, int variant);
/* Device bytes held by the context. */
int64_t gmg_device_bytes(const gmg_ctx *ctx);

/* Per-kernel-class CUDA-event timing on the launch stream (0 gs sweep,
 * 1 ghost sweep, 2 residuals, 3 band, 4 restriction, 5 interpolation,
 * 6 coarse solve, 7 norms).  gmg_profile(ctx, mask) clears the
 * accumulators and times the classes whose bit is set in mask (0 stops);
 * inside a captured cycle graph the event pairs become graph nodes.
 * gmg_profile_read synchronizes and returns the summed milliseconds and the
 * number of timed regions of that class on `level` (-1: all levels). */
int gmg_profile(gmg_ctx *ctx, int mask);
int gmg_profile_read(gmg_ctx *ctx, int kclass, int level, double *total_ms, int64_t *count);

/* Host helper: n draws of the reference's xorshift64* stream from (-1, 1)
 * (ref rng.py:14-56 uniform_symmetric), written to out. */
int gmg_uniform_symmetric(uint64_t seed, int64_t n, double *out);

#ifdef __cplusplus
}
#endif

#endif /* GHOSTMG_B200_H */
