/*
 * ghostmg_oracle.c -- CPU restatement of the ghost-point multigrid V-cycle
 * operators, used ONLY as the parity checker (tests/, __graft_entry__.smoke)
 * and as the CPU baseline in bench.py.  Never linked into the product.
 *
 * Each routine restates one per-cycle operation of the reference package
 * (/root/reference/pkg/src/ghostmg) on flat C-order float64 arrays of the
 * (N+1)^d grid, with the exact floating-point evaluation order the
 * reference obtains from NumPy / OpenBLAS in the build container
 * (SURVEY.md Appendix A):
 *
 *   - sums of < 8 terms: left to right, then + 0.0 (NumPy's add.reduce
 *     turns an all-zero -0 result into +0);
 *   - sums of >= 8 terms: NumPy's pairwise scheme (8 strided partial sums,
 *     tree combine, sequential tail), then + 0.0;
 *   - the ghost-row dot `co[t] @ u[st[t]]` is OpenBLAS 0.3.30 ddot on the
 *     SkylakeX core: n < 16 an FMA chain from 0; n = 27 four mul+add lanes
 *     over i < 16 combined (L0+L2)+(L1+L3), then an FMA tail;
 *   - no FMA contraction anywhere else (built with -ffp-contract=off).
 *
 * Pinned by tests/test_oracle_golden.py against vectors produced by the
 * reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define INTERNAL 0
#define GHOST 1
#define INACTIVE 2
#define ELIMINATED 3

static double seq_sum(const double *a, int n) {
  double s = a[0];
  for (int i = 1; i < n; ++i) s = s + a[i];
  return s + 0.0;
}

/* NumPy pairwise_sum for n >= 8 (and the short-case fallback). */
static double np_sum(const double *a, int n) {
  if (n < 8) return seq_sum(a, n);
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = r[j] + a[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res = res + a[i];
  return res + 0.0;
}

/* OpenBLAS ddot (SkylakeX kernel) as probed in the build container. */
static double blas_ddot(const double *x, const double *y, int n) {
  if (n < 16) {
    double d = 0.0;
    for (int i = 0; i < n; ++i) d = fma(x[i], y[i], d);
    return d;
  }
  double L[4] = {0.0, 0.0, 0.0, 0.0};
  int i = 0;
  for (; i + 4 <= (n & ~15); i += 4)
    for (int l = 0; l < 4; ++l) L[l] = L[l] + x[i + l] * y[i + l];
  double d = (L[0] + L[2]) + (L[1] + L[3]);
  for (; i < n; ++i) d = fma(x[i], y[i], d);
  return d;
}

static void strides64(int d, int64_t n, int64_t *s) {
  int64_t v = 1;
  for (int k = d - 1; k >= 0; --k) { s[k] = v; v *= n; }
}

static void unflatten(int d, int64_t n, int64_t flat, int64_t *m) {
  for (int k = d - 1; k >= 0; --k) { m[k] = flat % n; flat /= n; }
}

/* ---- smoother ---------------------------------------------------------
 * gs_lex_sweep: reference smoothing.py:127-132 (wavefront == lex order);
 * u_i <- (h2*f_i + sum[i-s0, i+s0, i-s1, i+s1, i-s2, i+s2]) * (1/denom). */
void oracle_gs_sweep(int d, int64_t N, const uint8_t *labels, double *u,
                     const double *f, double h2, double denom) {
  int64_t n = N + 1, s[3], total = 1;
  strides64(d, n, s);
  for (int k = 0; k < d; ++k) total *= n;
  const double inv = 1.0 / denom;
  double t[6];
  for (int64_t i = 0; i < total; ++i) {
    if (labels[i] != INTERNAL) continue;
    for (int k = 0; k < d; ++k) { t[2 * k] = u[i - s[k]]; t[2 * k + 1] = u[i + s[k]]; }
    u[i] = (h2 * f[i] + seq_sum(t, 2 * d)) * inv;
  }
}

/* ghost_relax_sweep: reference smoothing.py:135-142, lexicographic ghost
 * order, freshest values: u_G += dtau * (g - co . u[st]). */
void oracle_ghost_sweep(int d, int64_t ng, const int64_t *ghost_idx,
                        const int64_t *stencil, const double *coeffs,
                        const double *dtau, const double *g, double *u) {
  int m = d == 1 ? 3 : d == 2 ? 9 : 27;
  double y[27];
  for (int64_t t = 0; t < ng; ++t) {
    const int64_t *st = stencil + t * m;
    for (int j = 0; j < m; ++j) y[j] = u[st[j]];
    double dot = blas_ddot(coeffs + t * m, y, m);
    u[ghost_idx[t]] = u[ghost_idx[t]] + dtau[t] * (g[t] - dot);
  }
}

/* residual_internal (smoothing.py:111-118) written into a full array:
 * r_i = (f_i - (denom/h2)*u_i) + S_i/h2 on internal nodes; untouched
 * elsewhere.  Returns max |r_i|. */
double oracle_residual_internal(int d, int64_t N, const uint8_t *labels,
                                const double *u, const double *f, double h2,
                                double denom, double *r) {
  int64_t n = N + 1, s[3], total = 1;
  strides64(d, n, s);
  for (int k = 0; k < d; ++k) total *= n;
  const double c = denom / h2;
  double t[6], m = 0.0;
  for (int64_t i = 0; i < total; ++i) {
    if (labels[i] != INTERNAL) continue;
    for (int k = 0; k < d; ++k) { t[2 * k] = u[i - s[k]]; t[2 * k + 1] = u[i + s[k]]; }
    double v = (f[i] - c * u[i]) + seq_sum(t, 2 * d) / h2;
    r[i] = v;
    if (fabs(v) > m) m = fabs(v);
  }
  return m;
}

/* residual_ghost (smoothing.py:120-124): r_g = g - pairwise(w * u[st]).
 * Output aligned with the ghost list.  Returns max |r_g|. */
double oracle_residual_ghost(int d, int64_t ng, const int64_t *stencil,
                             const double *coeffs, const double *g,
                             const double *u, double *rg) {
  int m = d == 1 ? 3 : d == 2 ? 9 : 27;
  double p[27], mx = 0.0;
  for (int64_t t = 0; t < ng; ++t) {
    for (int j = 0; j < m; ++j) p[j] = coeffs[t * m + j] * u[stencil[t * m + j]];
    double v = g[t] - np_sum(p, m);
    rg[t] = v;
    if (fabs(v) > mx) mx = fabs(v);
  }
  return mx;
}

/* ---- band extrapolation (transfer.py:241-252), in place on `out` ------
 * BFS groups: out_i = (sum_k out[nbr_k] * mask_k) / popcount(mask), the
 * masked-out columns pointing at i itself; then 6 Jacobi transport steps
 * v_i <- v_i - 0.5 * sum_k |n_k| (v_i - v[i - step_k * s_k]). */
void oracle_extrapolate(int d, int64_t N, int ngroups, const int64_t *group_len,
                        const int64_t *band_idx, const uint8_t *bfs_mask,
                        const int8_t *step, const double *absn, double *out,
                        double *scratch) {
  int64_t n = N + 1, s[3];
  strides64(d, n, s);
  int64_t off = 0, nb = 0;
  double t[6];
  for (int gi = 0; gi < ngroups; ++gi) nb += group_len[gi];
  for (int gi = 0; gi < ngroups; ++gi) {
    for (int64_t q = off; q < off + group_len[gi]; ++q) {
      int64_t i = band_idx[q];
      uint8_t mk = bfs_mask[q];
      int cnt = 0;
      for (int k = 0; k < d; ++k)
        for (int j = 0; j < 2; ++j) {
          int bit = (mk >> (2 * k + j)) & 1;
          int64_t nbr = bit ? (j ? i + s[k] : i - s[k]) : i;
          t[2 * k + j] = out[nbr] * (bit ? 1.0 : 0.0);
          cnt += bit;
        }
      out[i] = seq_sum(t, 2 * d) / (double)cnt;
    }
    off += group_len[gi];
  }
  if (nb == 0) return;
  for (int it = 0; it < 6; ++it) {
    for (int64_t q = 0; q < nb; ++q) {
      int64_t i = band_idx[q];
      double vi = out[i];
      for (int k = 0; k < d; ++k) {
        int64_t nbr = i - (int64_t)step[q * d + k] * s[k];
        t[k] = absn[q * d + k] * (vi - out[nbr]);
      }
      scratch[q] = vi - 0.5 * seq_sum(t, d);
    }
    for (int64_t q = 0; q < nb; ++q) out[band_idx[q]] = scratch[q];
  }
}

/* The two phases of oracle_extrapolate on a subset of the band, for the
 * z-slab schedule tests (tests/test_slabs.py): one BFS group over the nodes
 * idx[0..m) (same arithmetic as above), and one Jacobi transport step over
 * them (all reads before any write, like the reference's vectorised step). */
void oracle_band_bfs(int d, int64_t N, int64_t m, const int64_t *idx, const uint8_t *mask, double *out) {
  int64_t n = N + 1, s[3];
  strides64(d, n, s);
  double t[6];
  for (int64_t q = 0; q < m; ++q) {
    int64_t i = idx[q];
    uint8_t mk = mask[q];
    int cnt = 0;
    for (int k = 0; k < d; ++k)
      for (int j = 0; j < 2; ++j) {
        int bit = (mk >> (2 * k + j)) & 1;
        int64_t nbr = bit ? (j ? i + s[k] : i - s[k]) : i;
        t[2 * k + j] = out[nbr] * (bit ? 1.0 : 0.0);
        cnt += bit;
      }
    out[i] = seq_sum(t, 2 * d) / (double)cnt;
  }
}

void oracle_band_transport(int d, int64_t N, int64_t m, const int64_t *idx, const int8_t *step,
                           const double *absn, double *out, double *scratch) {
  int64_t n = N + 1, s[3];
  strides64(d, n, s);
  double t[3];
  for (int64_t q = 0; q < m; ++q) {
    int64_t i = idx[q];
    double vi = out[i];
    for (int k = 0; k < d; ++k) {
      int64_t nbr = i - (int64_t)step[q * d + k] * s[k];
      t[k] = absn[q * d + k] * (vi - out[nbr]);
    }
    scratch[q] = vi - 0.5 * seq_sum(t, d);
  }
  for (int64_t q = 0; q < m; ++q) out[idx[q]] = scratch[q];
}

/* ---- restrictions ------------------------------------------------------
 * InteriorRestriction.apply (transfer.py:64-93): per coarse internal node,
 * pairwise(w * r[3^d fine block around 2m]) with w = full weighting, or
 * 1/count on the block's internal nodes when it holds a ghost/inactive
 * node.  Writes coarse f (full coarse array, untouched elsewhere). */
void oracle_restrict_interior(int d, int64_t Nf, const uint8_t *lab_f,
                              const double *r_f, const uint8_t *lab_c,
                              double *f_c) {
  int64_t nf = Nf + 1, nc = Nf / 2 + 1, sf[3], sc[3], totc = 1;
  strides64(d, nf, sf);
  strides64(d, nc, sc);
  for (int k = 0; k < d; ++k) totc *= nc;
  int m = d == 1 ? 3 : d == 2 ? 9 : 27;
  double fw[27], w[27], p[27];
  int64_t blk[27];
  for (int e = 0; e < m; ++e) {
    double v = 1.0;
    int rem = e;
    int o[3];
    for (int k = d - 1; k >= 0; --k) { o[k] = rem % 3; rem /= 3; }
    for (int k = 0; k < d; ++k) v = v * (o[k] == 1 ? 0.5 : 0.25);
    fw[e] = v;
  }
  int64_t mc[3];
  for (int64_t ic = 0; ic < totc; ++ic) {
    if (lab_c[ic] != INTERNAL) continue;
    unflatten(d, nc, ic, mc);
    int mixed = 0, cnt = 0;
    for (int e = 0; e < m; ++e) {
      int rem = e;
      int64_t flat = 0;
      int o[3];
      for (int k = d - 1; k >= 0; --k) { o[k] = rem % 3; rem /= 3; }
      for (int k = 0; k < d; ++k) flat += (2 * mc[k] + o[k] - 1) * sf[k];
      blk[e] = flat;
      uint8_t L = lab_f[flat];
      if (L == GHOST || L == INACTIVE) mixed = 1;
      if (L == INTERNAL) cnt++;
    }
    for (int e = 0; e < m; ++e)
      w[e] = mixed ? (lab_f[blk[e]] == INTERNAL ? 1.0 : 0.0) / (double)cnt : fw[e];
    for (int e = 0; e < m; ++e) p[e] = w[e] * r_f[blk[e]];
    f_c[ic] = np_sum(p, m);
  }
}

/* GhostRestriction (transfer.py:96-121): per coarse ghost (list order),
 * w = FW * keep / pairwise(FW * keep), keep = in-box and ghost/inactive;
 * value = pairwise(w * r_ext[clamped block]). */
void oracle_restrict_ghost(int d, int64_t Nf, const uint8_t *lab_f,
                           const double *r_ext, int64_t ngc,
                           const int64_t *ghost_c, double *g_c) {
  int64_t nf = Nf + 1, nc = Nf / 2 + 1, sf[3];
  strides64(d, nf, sf);
  int m = d == 1 ? 3 : d == 2 ? 9 : 27;
  double fw[27], w[27], p[27];
  int64_t blk[27];
  for (int e = 0; e < m; ++e) {
    double v = 1.0;
    int rem = e, o[3];
    for (int k = d - 1; k >= 0; --k) { o[k] = rem % 3; rem /= 3; }
    for (int k = 0; k < d; ++k) v = v * (o[k] == 1 ? 0.5 : 0.25);
    fw[e] = v;
  }
  int64_t mc[3];
  for (int64_t q = 0; q < ngc; ++q) {
    unflatten(d, nc, ghost_c[q], mc);
    for (int e = 0; e < m; ++e) {
      int rem = e, o[3], valid = 1;
      int64_t flat = 0;
      for (int k = d - 1; k >= 0; --k) { o[k] = rem % 3; rem /= 3; }
      for (int k = 0; k < d; ++k) {
        int64_t x = 2 * mc[k] + o[k] - 1;
        if (x < 0 || x > Nf) valid = 0;
        x = x < 0 ? 0 : x > Nf ? Nf : x;
        flat += x * sf[k];
      }
      blk[e] = flat;
      uint8_t L = lab_f[flat];
      int keep = valid && (L == GHOST || L == INACTIVE);
      w[e] = fw[e] * (keep ? 1.0 : 0.0);
    }
    double sum = np_sum(w, m);
    for (int e = 0; e < m; ++e) p[e] = (w[e] / sum) * r_ext[blk[e]];
    g_c[q] = np_sum(p, m);
  }
}

/* ErrorInterpolation + correction (transfer.py:124-151, solver.py:198):
 * every fine internal or ghost node gets u += sum_c w_c e[src_c], corners
 * c in {0,1}^d (C order), w_c = prod_k (odd_k ? 1/2 : [c_k == 0]). */
void oracle_interpolate_add(int d, int64_t Nf, const uint8_t *lab_f, double *u_f,
                            const double *e_c) {
  int64_t nf = Nf + 1, nc = Nf / 2 + 1, sc[3], totf = 1, m[3];
  strides64(d, nc, sc);
  for (int k = 0; k < d; ++k) totf *= nf;
  int nco = 1 << d;
  double p[8];
  for (int64_t i = 0; i < totf; ++i) {
    uint8_t L = lab_f[i];
    if (L != INTERNAL && L != GHOST) continue;
    unflatten(d, nf, i, m);
    for (int c = 0; c < nco; ++c) {
      double w = 1.0;
      int64_t src = 0;
      for (int k = 0; k < d; ++k) {
        int off = (c >> (d - 1 - k)) & 1;
        int odd = (int)(m[k] & 1);
        w = w * (odd ? 0.5 : (off == 0 ? 1.0 : 0.0));
        src += (m[k] / 2 + (odd ? off : 0)) * sc[k];
      }
      p[c] = w * e_c[src];
    }
    u_f[i] = u_f[i] + np_sum(p, nco);
  }
}

double oracle_abs_max(const double *u, int64_t n) {
  double m = 0.0;
  for (int64_t i = 0; i < n; ++i)
    if (fabs(u[i]) > m) m = fabs(u[i]);
  return m;
}

/* Exposed for the pinning tests. */
double oracle_np_sum(const double *a, int n) { return np_sum(a, n); }
double oracle_ddot(const double *x, const double *y, int n) { return blas_ddot(x, y, n); }

/* (r**2).sum() over a 1-D array: NumPy's recursive pairwise sum with
 * 128-element leaves (loops_utils.h.src), added to the reduction's 0. */
static double np_pairwise_sq(const double *a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res = res + a[i] * a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j] * a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = r[j] + a[i + j] * a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res = res + a[i] * a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sq(a, n2) + np_pairwise_sq(a + n2, n - n2);
}

double oracle_sumsq(const double *a, int64_t n) { return 0.0 + np_pairwise_sq(a, n); }
