// setup_ops.cu -- per-level setup work that is pure per-node label logic, on
// the device: node classification for the ball
// family of level sets and the restriction-block checks.
//
// Reference: classify, /root/reference/pkg/src/ghostmg/geometry.py:374-446
// (labels from the sign of phi, the box faces and the internal neighbours);
// InteriorRestriction / GhostRestriction constructors,
// /root/reference/pkg/src/ghostmg/transfer.py:64-114 (what they raise).
// The ghost geometry (projection, normals, theta, stencils) stays on the host
// for the whole ghost batch (geometry.py:266-276, 433-446).
//
// The sign of phi restates the host level sets bit for bit (levelsets.py):
// |x - c| = sqrt(((dx*dx + dy*dy) + dz*dz) + 0.0) with dx = axis[i] - c (the
// library is compiled with --fmad=false; sqrt and the sums are IEEE).
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ghostmg_b200.h"
#include "gmg_common.cuh"

namespace {

using gmg::ELIMINATED;
using gmg::GHOST;
using gmg::INACTIVE;
using gmg::INTERNAL;

std::string g_setup_err;

// phi < 0 per node.  kind 0: pore space, domain = outside every ball (phi = max_k (r_k - |x - c_k|));
// kind 1: signed sphere, domain = inside the ball (phi = |x - c| - R).
template <int D>
__global__ void __launch_bounds__(256) sign_balls_kernel(int64_t N, const double* __restrict__ axis, int kind, int nb,
                                                         const double* __restrict__ cen, const double* __restrict__ rad,
                                                         uint8_t* __restrict__ neg, int64_t total) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int64_t n = N + 1;
  int64_t m[3] = {0, 0, 0};
  int64_t rem = idx;
  for (int k = D - 1; k >= 0; --k) {
    m[k] = rem % n;
    rem /= n;
  }
  double x[3];
  for (int k = 0; k < D; ++k) x[k] = axis[m[k]];
  bool out;
  if (kind == 0) {
    bool nonneg = false;
    for (int b = 0; b < nb; ++b) {
      double sq = 0.0;
      for (int k = 0; k < D; ++k) {
        const double t = x[k] - cen[b * D + k];
        sq = k == 0 ? t * t : sq + t * t;
      }
      nonneg = nonneg || (rad[b] - sqrt(sq + 0.0) >= 0.0);
    }
    out = !nonneg;
  } else {
    double sq = 0.0;
    for (int k = 0; k < D; ++k) {
      const double t = x[k] - cen[k];
      sq = k == 0 ? t * t : sq + t * t;
    }
    out = sqrt(sq + 0.0) - rad[0] < 0.0;
  }
  neg[idx] = out ? 1 : 0;
}

// labels from the sign, the box faces and the internal neighbours (geometry.py:385-416)
template <int D>
__global__ void __launch_bounds__(256) labels_kernel(int64_t N, const uint8_t* __restrict__ neg, int face_mask,
                                                     uint8_t* __restrict__ lab, int64_t total) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int64_t n = N + 1;
  int64_t m[3] = {0, 0, 0}, st[3] = {0, 0, 0};
  int64_t rem = idx, s = 1;
  for (int k = D - 1; k >= 0; --k) {
    m[k] = rem % n;
    rem /= n;
    st[k] = s;
    s *= n;
  }
  auto eliminated = [&](const int64_t* q, int64_t flat) {
    bool on_box = false, forced = false;
    for (int k = 0; k < D; ++k) {
      if (q[k] == 0) {
        on_box = true;
        forced = forced || ((face_mask >> (2 * k)) & 1);
      }
      if (q[k] == N) {
        on_box = true;
        forced = forced || ((face_mask >> (2 * k + 1)) & 1);
      }
    }
    return forced || (on_box && neg[flat]);
  };
  const bool elim = eliminated(m, idx);
  const bool internal = neg[idx] && !elim;
  bool near = false;
  for (int k = 0; k < D; ++k)
    for (int sg = -1; sg <= 1; sg += 2) {
      const int64_t v = m[k] + sg;
      if (v < 0 || v > N) continue;
      int64_t q[3] = {m[0], m[1], m[2]};
      q[k] = v;
      const int64_t f = idx + sg * st[k];
      near = near || (neg[f] && !eliminated(q, f));
    }
  lab[idx] = internal ? INTERNAL : (elim ? ELIMINATED : (near ? GHOST : INACTIVE));
}

// restriction-block checks (transfer.py:64-114); flags: 1 interior block leaves the box, 2 mixed block
// without an internal node, 4 coarse ghost without an in-box ghost / inactive node, 8 / 16 block centre of
// a coarse internal / ghost node with the wrong fine label
template <int D>
__global__ void __launch_bounds__(256) check_transfer_kernel(int64_t Nf, const uint8_t* __restrict__ lf, int64_t Nc,
                                                             const uint8_t* __restrict__ lc, int* __restrict__ flags,
                                                             int64_t total) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const uint8_t c = lc[idx];
  if (c != INTERNAL && c != GHOST) return;
  const int64_t nc = Nc + 1, nf = Nf + 1;
  int64_t m[3] = {0, 0, 0};
  int64_t rem = idx;
  for (int k = D - 1; k >= 0; --k) {
    m[k] = rem % nc;
    rem /= nc;
  }
  bool all_valid = true, any_int = false, any_go = false, any_keep = false;
  constexpr int M = D == 3 ? 27 : 9;
  for (int e = 0; e < M; ++e) {
    int o[3] = {0, 0, 0};
    int r = e;
    for (int k = D - 1; k >= 0; --k) {
      o[k] = r % 3 - 1;
      r /= 3;
    }
    bool valid = true;
    int64_t flat = 0;
    for (int k = 0; k < D; ++k) {
      int64_t v = 2 * m[k] + o[k];
      if (v < 0 || v > Nf) valid = false;
      v = v < 0 ? 0 : (v > Nf ? Nf : v);
      flat = flat * nf + v;
    }
    const uint8_t l = lf[flat];
    all_valid = all_valid && valid;
    any_int = any_int || l == INTERNAL;
    const bool go = l == GHOST || l == INACTIVE;
    any_go = any_go || go;
    any_keep = any_keep || (valid && go);
  }
  int64_t cf = 0;
  for (int k = 0; k < D; ++k) cf = cf * nf + 2 * m[k];
  const uint8_t lcen = lf[cf];
  int f = 0;
  if (c == INTERNAL) {
    if (!all_valid) f |= 1;
    if (any_go && !any_int) f |= 2;
    if (lcen != INTERNAL) f |= 8;
  } else {
    if (!any_keep) f |= 4;
    if (lcen != GHOST && lcen != INACTIVE) f |= 16;
  }
  if (f) atomicOr(flags, f);
}

int setup_fail(const std::string& m) {
  g_setup_err = m;
  return -1;
}

#define SETUP_CHECK(call)                                                               \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      for (void* p_ : bufs)                                                             \
        if (p_) cudaFree(p_);                                                           \
      return setup_fail(std::string(#call) + ": " + cudaGetErrorString(e_));            \
    }                                                                                   \
  } while (0)

int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

}  // namespace

extern "C" {

const char* gmg_setup_last_error(void) { return g_setup_err.c_str(); }

int gmg_setup_classify_balls(int device, int d, int64_t N, const double* axis, int kind, int n_balls,
                             const double* centers, const double* radii, int face_mask, uint8_t* labels_out) {
  if ((d != 2 && d != 3) || N < 2 || n_balls < 1 || (kind != 0 && kind != 1)) return setup_fail("bad arguments");
  std::vector<void*> bufs;
  SETUP_CHECK(cudaSetDevice(device));
  const int64_t total = ipow(N + 1, d);
  double *dax = nullptr, *dc = nullptr, *dr = nullptr;
  uint8_t *dneg = nullptr, *dlab = nullptr;
  SETUP_CHECK(cudaMalloc(&dax, sizeof(double) * (N + 1)));
  bufs.push_back(dax);
  SETUP_CHECK(cudaMalloc(&dc, sizeof(double) * n_balls * d));
  bufs.push_back(dc);
  SETUP_CHECK(cudaMalloc(&dr, sizeof(double) * n_balls));
  bufs.push_back(dr);
  SETUP_CHECK(cudaMalloc(&dneg, total));
  bufs.push_back(dneg);
  SETUP_CHECK(cudaMalloc(&dlab, total));
  bufs.push_back(dlab);
  SETUP_CHECK(cudaMemcpy(dax, axis, sizeof(double) * (N + 1), cudaMemcpyHostToDevice));
  SETUP_CHECK(cudaMemcpy(dc, centers, sizeof(double) * n_balls * d, cudaMemcpyHostToDevice));
  SETUP_CHECK(cudaMemcpy(dr, radii, sizeof(double) * n_balls, cudaMemcpyHostToDevice));
  const unsigned blocks = (unsigned)((total + 255) / 256);
  if (d == 3) {
    sign_balls_kernel<3><<<blocks, 256>>>(N, dax, kind, n_balls, dc, dr, dneg, total);
    labels_kernel<3><<<blocks, 256>>>(N, dneg, face_mask, dlab, total);
  } else {
    sign_balls_kernel<2><<<blocks, 256>>>(N, dax, kind, n_balls, dc, dr, dneg, total);
    labels_kernel<2><<<blocks, 256>>>(N, dneg, face_mask, dlab, total);
  }
  SETUP_CHECK(cudaGetLastError());
  SETUP_CHECK(cudaMemcpy(labels_out, dlab, total, cudaMemcpyDeviceToHost));
  for (void* p : bufs) cudaFree(p);
  return 0;
}

int gmg_setup_check_transfer(int device, int d, int64_t Nf, const uint8_t* lab_f, int64_t Nc, const uint8_t* lab_c,
                             int* flags_out) {
  if ((d != 2 && d != 3) || Nf != 2 * Nc) return setup_fail("bad arguments");
  std::vector<void*> bufs;
  SETUP_CHECK(cudaSetDevice(device));
  const int64_t tf = ipow(Nf + 1, d), tc = ipow(Nc + 1, d);
  uint8_t *df = nullptr, *dcl = nullptr;
  int* dfl = nullptr;
  SETUP_CHECK(cudaMalloc(&df, tf));
  bufs.push_back(df);
  SETUP_CHECK(cudaMalloc(&dcl, tc));
  bufs.push_back(dcl);
  SETUP_CHECK(cudaMalloc(&dfl, sizeof(int)));
  bufs.push_back(dfl);
  SETUP_CHECK(cudaMemcpy(df, lab_f, tf, cudaMemcpyHostToDevice));
  SETUP_CHECK(cudaMemcpy(dcl, lab_c, tc, cudaMemcpyHostToDevice));
  SETUP_CHECK(cudaMemset(dfl, 0, sizeof(int)));
  const unsigned blocks = (unsigned)((tc + 255) / 256);
  if (d == 3)
    check_transfer_kernel<3><<<blocks, 256>>>(Nf, df, Nc, dcl, dfl, tc);
  else
    check_transfer_kernel<2><<<blocks, 256>>>(Nf, df, Nc, dcl, dfl, tc);
  SETUP_CHECK(cudaGetLastError());
  SETUP_CHECK(cudaMemcpy(flags_out, dfl, sizeof(int), cudaMemcpyDeviceToHost));
  for (void* p : bufs) cudaFree(p);
  return 0;
}

}  // extern "C"
