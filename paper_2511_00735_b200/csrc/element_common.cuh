// Shared by the element kernels (element.cu, element_v5.cu): kernel
// arguments, the recovery copy-out and the boundary Schur / ItI epilogue.
#pragma once

#include "device.cuh"
#include "linalg.cuh"
#include "internal.hpp"

namespace hpsb {

constexpr int kThreads = 256;

struct ElemArgs {
  int ne, order, m, ni, nb;
  double eta;
  const double* mass;   // [np]
  const double* diff;   // [np*np] col-major, scaled by 2/h
  const double* stiff;  // [np*np] col-major
  const double* coeff;  // [ne][np*np]
  const double2* source;  // [ne][ni] or null
  double2* T;
  double2* H;
  int* status;
  double* ws;        // per-slot workspace
  size_t ws_stride;  // doubles per slot
  const int* elist;  // optional element list (fallback re-run)
  int nlist;
  const int* nlist_dev;  // list length on the device (overrides nlist)
  int npad, nbc;     // v2: padded interior size (multiple of 16), padded rhs count
  double* Y;         // [e][nb+2][ni]: L_ii^{-1} [L_iG | re b~ | im b~] kept for recovery
};

// Keep Y = L_ii^{-1} [L_iG | b~] (ld ldy in the workspace) for the solution
// recovery u_i = Y_b - Y_G u_G (problems.cpp:60-92 / element.cpp:176-188).
static __device__ __forceinline__ void keep_interior(const ElemArgs& a, int e, const double* Y, int ldy) {
  const int ni = a.ni, cols = a.nb + 2;
  double* dst = a.Y + static_cast<size_t>(e) * ni * cols;
  for (int idx = threadIdx.x; idx < ni * cols; idx += blockDim.x) {
    const int q = idx % ni, c = idx / ni;
    dst[idx] = Y[q + static_cast<size_t>(c) * ldy];
  }
}

// Boundary Schur complement and ItI map from the interior solve
// Y = L_ii^{-1} [L_iG | b~] (ld ldy, interior order q = (i-1) m + (j-1)):
//   S = L_GG - L_Gi Y,  f = L_Gi y_b,  T = I - 2 i eta S^{-1},  H = 2 i eta S^{-1} f.
// L_Gi / L_GG are the impedance rows I_in = deriv + i eta trace
// (element.cpp:92-125, :137-139); L_Gi has N-1 entries per row.
static __device__ bool iti_epilogue(const ElemArgs& a, int e, const double* Y, int ldy, double2* S,
                             double2* f, int* perm, double* red_v, int* red_i,
                             const double* diff_s = nullptr) {
  const int tid = threadIdx.x, m = a.m, nb = a.nb, np = a.order + 1, N = a.order;
  auto D = [&](int r, int c) { return diff_s ? diff_s[r + c * np] : __ldg(a.diff + r + c * np); };
  auto lgi = [&](int b, int k, int& q) {  // entry of row b at interior node k of its line
    const int side = b / m, t = b % m + 1;
    switch (side) {
      case 0: q = (k - 1) * m + (t - 1); return -D(0, k);
      case 1: q = (k - 1) * m + (t - 1); return D(N, k);
      case 2: q = (t - 1) * m + (k - 1); return -D(0, k);
      default: q = (t - 1) * m + (k - 1); return D(N, k);
    }
  };
  for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
    const int b = idx % nb, c = idx / nb;
    const int side = b / m, t = b % m + 1;
    double acc = 0.0;
    for (int k = 1; k <= m; ++k) {
      int q;
      const double d = lgi(b, k, q);
      acc += d * Y[q + static_cast<size_t>(c) * ldy];
    }
    // L_GG: derivative entries on the two boundary nodes of the same line
    const int cs = c / m, ct = c % m + 1;
    double lgg = 0.0;
    if (ct == t) {
      if (side <= 1 && cs <= 1)
        lgg = (side == 0 ? -1.0 : 1.0) * D(side == 0 ? 0 : N, cs == 0 ? 0 : N);
      else if (side >= 2 && cs >= 2)
        lgg = (side == 2 ? -1.0 : 1.0) * D(side == 2 ? 0 : N, cs == 2 ? 0 : N);
    }
    double2 sv = make_double2(lgg - acc, 0.0);
    if (b == c) sv.y += a.eta;
    S[idx] = sv;
  }
  double2 fv = make_double2(0.0, 0.0);
  if (tid < nb && a.source)
    for (int k = 1; k <= m; ++k) {
      int q;
      const double d = lgi(tid, k, q);
      fv.x += d * Y[q + static_cast<size_t>(nb) * ldy];
      fv.y += d * Y[q + static_cast<size_t>(nb + 1) * ldy];
    }
  __syncthreads();
  const bool ok = gj_inverse_cta(S, nb, perm, red_v, red_i);
  if (tid < nb) f[tid] = fv;
  __syncthreads();
  const double te = 2.0 * a.eta;
  double2* Te = a.T + static_cast<size_t>(e) * nb * nb;
  for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
    const double2 s = S[idx];
    const int b = idx % nb, c = idx / nb;
    Te[idx] = make_double2((b == c ? 1.0 : 0.0) + te * s.y, -te * s.x);
  }
  if (tid < nb) {
    double2 acc = make_double2(0.0, 0.0);
    if (a.source)
      for (int c = 0; c < nb; ++c) acc = cfma(S[tid + c * nb], f[c], acc);
    a.H[static_cast<size_t>(e) * nb + tid] = make_double2(-te * acc.y, te * acc.x);
  }
  __syncthreads();
  return ok;
}

// v5 (batched blocked Cholesky over element chunks, element_v5.cu); returns
// false when no v5 configuration applies.
bool element_v5_build(Context* ctx, const ElemArgs& a, int nwork);

}  // namespace hpsb
