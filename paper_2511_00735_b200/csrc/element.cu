#include <mutex>
// K1 element_iti: batched local impedance-to-impedance build.
//
// Replaces ElementOperators (proj/src/element.cpp:127-160) + source_to_outgoing
// (:167-174), batched over the mesh as build_elements (proj/src/mesh.cpp:36-109).
// Instead of the reference's complex LU of the full corner-free operator L
// (t x t), the kernel uses the identity
//     T = I - 2 i eta (L^{-1})_GG,   (L^{-1})_GG = S^{-1},
//     S = L_GG - L_Gi L_ii^{-1} L_iG,
//     H = -2 i eta (L^{-1}[0; b~])_G = 2 i eta S^{-1} L_Gi L_ii^{-1} b~,
// where L_ii = Kx(x)My + Mx(x)Ky - diag(c) Mx(x)My on the interior nodes is
// real symmetric positive definite for the configs (Appendix B.2).  Per
// element: real Cholesky of L_ii (ni = (N-1)^2), two triangular solves with
// nb + 2 right-hand sides (nb = 4(N-1)), the sparse boundary rows, and a
// complex nb x nb Gauss-Jordan inverse.
//
// Data layout: coeff[e][(N+1)^2] real c = kappa^2 (1 - b); source[e][ni]
// complex samples of s; T[e] nb x nb complex column-major in the boundary
// order left|right|bottom|top; H[e] nb complex.
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"
#include "linalg.cuh"
#include "internal.hpp"
#include "element_common.cuh"

namespace hpsb {

namespace {

// v1 / fallback: unblocked right-looking Cholesky (pivoted LU when L_ii is
// indefinite) on the element's workspace.  Processes a.elist when given.
__global__ void __launch_bounds__(kThreads) element_kernel(ElemArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int m = a.m, ni = a.ni, nb = a.nb, np = a.order + 1, N = a.order;
  const int ncol = nb + 2;
  double2* S = reinterpret_cast<double2*>(smem_raw);       // nb*nb
  double2* f = S + nb * nb;                                // nb
  double* colk = reinterpret_cast<double*>(f + nb);        // ni
  double* mass = colk + ni;                                // np
  int* perm = reinterpret_cast<int*>(mass + np);           // nb
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_fail;

  double* Lii = a.ws + blockIdx.x * a.ws_stride;  // ni*ni
  double* Y = Lii + static_cast<size_t>(ni) * ni;   // ni*ncol

  for (int i = tid; i < np; i += blockDim.x) mass[i] = a.mass[i];
  auto K = [&](int r, int c) { return __ldg(a.stiff + r + c * np); };
  const int count = a.elist ? (a.nlist_dev ? *a.nlist_dev : a.nlist) : a.ne;

  for (int ii = blockIdx.x; ii < count; ii += gridDim.x) {
    const int e = a.elist ? a.elist[ii] : ii;
    __syncthreads();
    if (tid == 0) s_fail = 0;
    const double* ce = a.coeff + static_cast<size_t>(e) * np * np;
    // 1. interior block L_ii (element.cpp:57-90 restricted to interior nodes)
    auto assemble_lii = [&]() {
      for (int idx = tid; idx < ni * ni; idx += blockDim.x) {
        const int r = idx % ni, c = idx / ni;
        const int i = r / m + 1, j = r % m + 1, k = c / m + 1, l = c % m + 1;
        double v = 0.0;
        if (j == l) v += K(i, k) * mass[j];
        if (i == k) v += mass[i] * K(j, l);
        if (r == c) v -= __ldg(ce + i * np + j) * mass[i] * mass[j];
        Lii[idx] = v;
      }
    };
    assemble_lii();
    // 2. right-hand sides [L_iG | re b~ | im b~]
    for (int idx = tid; idx < ni * ncol; idx += blockDim.x) {
      const int q = idx % ni, b = idx / ni;
      const int i = q / m + 1, j = q % m + 1;
      double v = 0.0;
      if (b < nb) {
        const int side = b / m, t = b % m + 1;
        switch (side) {
          case 0: v = (j == t) ? K(i, 0) * mass[j] : 0.0; break;
          case 1: v = (j == t) ? K(i, N) * mass[j] : 0.0; break;
          case 2: v = (i == t) ? mass[i] * K(j, 0) : 0.0; break;
          default: v = (i == t) ? mass[i] * K(j, N) : 0.0; break;
        }
      } else if (a.source) {
        const double2 s = a.source[static_cast<size_t>(e) * ni + q];
        const double w = mass[i] * mass[j];
        v = (b == nb) ? s.x * w : s.y * w;
      }
      Y[idx] = v;
    }
    __syncthreads();
    // 3. Cholesky L_ii = R R^T (lower, in place), right-looking
    for (int k = 0; k < ni; ++k) {
      if (tid == 0) {
        const double d = Lii[k + k * ni];
        if (!(d > 0.0)) s_fail = 1;
        Lii[k + k * ni] = sqrt(fmax(d, 1e-300));
      }
      __syncthreads();
      const double inv = 1.0 / Lii[k + k * ni];
      for (int i = k + 1 + tid; i < ni; i += blockDim.x) {
        const double v = Lii[i + k * ni] * inv;
        Lii[i + k * ni] = v;
        colk[i] = v;
      }
      __syncthreads();
      const int rem = ni - k - 1;
      for (int idx = tid; idx < rem * rem; idx += blockDim.x) {
        const int i = k + 1 + idx % rem, j = k + 1 + idx / rem;
        if (j <= i) Lii[i + j * ni] -= colk[i] * colk[j];
      }
      __syncthreads();
      if (s_fail) break;  // indefinite: fall back to pivoted LU below
    }
    __syncthreads();
    if (s_fail) {
      // Pivoted-LU fallback for an indefinite L_ii (c h^2 above the first
      // Dirichlet eigenvalue): P L_ii = L U with
      // partial pivoting, the row swaps applied to the right-hand sides.
      assemble_lii();
      __syncthreads();
      if (tid == 0) s_fail = 0;
      for (int k = 0; k < ni; ++k) {
        double best = -1.0;
        int bi = k;
        for (int i = k + tid; i < ni; i += blockDim.x) {
          const double v = fabs(Lii[i + k * ni]);
          if (v > best) best = v, bi = i;
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > best || (ov == best && oi < bi)) best = ov, bi = oi;
        }
        if ((tid & 31) == 0) red_v[tid >> 5] = best, red_i[tid >> 5] = bi;
        __syncthreads();
        if (tid == 0) {
          double b = -1.0;
          int p = k;
          for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            if (red_v[w] > b || (red_v[w] == b && red_i[w] < p)) b = red_v[w], p = red_i[w];
          perm[0] = p;
          if (!(b > 0.0)) s_fail = 2;
        }
        __syncthreads();
        const int p = perm[0];
        if (p != k) {
          for (int j = tid; j < ni; j += blockDim.x) {
            const double t = Lii[k + j * ni];
            Lii[k + j * ni] = Lii[p + j * ni];
            Lii[p + j * ni] = t;
          }
          for (int c = tid; c < ncol; c += blockDim.x) {
            const double t = Y[k + c * ni];
            Y[k + c * ni] = Y[p + c * ni];
            Y[p + c * ni] = t;
          }
        }
        __syncthreads();
        const double piv = Lii[k + k * ni];
        const double inv = piv != 0.0 ? 1.0 / piv : 0.0;
        for (int i = k + 1 + tid; i < ni; i += blockDim.x) {
          const double v = Lii[i + k * ni] * inv;
          Lii[i + k * ni] = v;
          colk[i] = v;
        }
        __syncthreads();
        const int rem = ni - k - 1;
        for (int idx = tid; idx < rem * rem; idx += blockDim.x) {
          const int i = k + 1 + idx % rem, j = k + 1 + idx / rem;
          Lii[i + j * ni] -= colk[i] * Lii[k + j * ni];
        }
        __syncthreads();
      }
      for (int k = 0; k < ni; ++k) {  // unit-lower forward substitution
        const int rem = ni - k - 1;
        for (int idx = tid; idx < rem * ncol; idx += blockDim.x) {
          const int i = k + 1 + idx % rem, c = idx / rem;
          Y[i + c * ni] -= Lii[i + k * ni] * Y[k + c * ni];
        }
        __syncthreads();
      }
      for (int k = ni - 1; k >= 0; --k) {  // upper back substitution
        const double d = Lii[k + k * ni];
        const double inv = d != 0.0 ? 1.0 / d : 0.0;
        for (int c = tid; c < ncol; c += blockDim.x) Y[k + c * ni] *= inv;
        __syncthreads();
        for (int idx = tid; idx < k * ncol; idx += blockDim.x) {
          const int i = idx % k, c = idx / k;
          Y[i + c * ni] -= Lii[i + k * ni] * Y[k + c * ni];
        }
        __syncthreads();
      }
    } else {
    // 4. solve R R^T Y = B
    for (int k = 0; k < ni; ++k) {
      const double inv = 1.0 / Lii[k + k * ni];
      for (int c = tid; c < ncol; c += blockDim.x) Y[k + c * ni] *= inv;
      __syncthreads();
      const int rem = ni - k - 1;
      for (int idx = tid; idx < rem * ncol; idx += blockDim.x) {
        const int i = k + 1 + idx % rem, c = idx / rem;
        Y[i + c * ni] -= Lii[i + k * ni] * Y[k + c * ni];
      }
      __syncthreads();
    }
    for (int k = ni - 1; k >= 0; --k) {
      const double inv = 1.0 / Lii[k + k * ni];
      for (int c = tid; c < ncol; c += blockDim.x) Y[k + c * ni] *= inv;
      __syncthreads();
      for (int idx = tid; idx < k * ncol; idx += blockDim.x) {
        const int i = idx % k, c = idx / k;
        Y[i + c * ni] -= Lii[k + i * ni] * Y[k + c * ni];
      }
      __syncthreads();
    }
    }
    __syncthreads();
    keep_interior(a, e, Y, ni);
    const bool ok = iti_epilogue(a, e, Y, ni, S, f, perm, red_v, red_i);
    if (tid == 0) a.status[e] = (s_fail ? 1 : 0) | (ok ? 0 : 2);  // 1: singular L_ii
  }
}

// ---------------------------------------------------------------- v2
constexpr int PW = 16;  // panel width
#ifndef HPSB_TRAIL_BATCH
#define HPSB_TRAIL_BATCH 4
#endif
constexpr int kTrailBatch = HPSB_TRAIL_BATCH;  // trailing-update tiles per warp in flight

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__host__ __device__ inline int v2_ldp(int P) { return ((P - PW + 15) & ~15) + 4; }
constexpr int kLdq = PW + 4;
__host__ __device__ inline size_t v2_region(int P, int nbc, int nb) {
  const size_t panel = PW * PW + static_cast<size_t>(v2_ldp(P)) * PW + kLdq * nbc;
  const size_t epi = 2 * (static_cast<size_t>(nb) * nb + nb);
  return panel > epi ? panel : epi;
}

// v2: blocked right-looking Cholesky of the interior block, padded to P (a
// multiple of 16, identity on the padding), with the forward solve of the
// nb + 2 right-hand sides fused into each panel step; the trailing-matrix
// (SYRK) and right-hand-side (GEMM) updates run on the FP64 tensor cores
// (mma.sync m8n8k4, one 8 x 8 tile per warp step, panels staged in smem).
// The backward solve R^T X = Y is blocked the same way, right-looking from
// the last panel.  An indefinite L_ii (first failing pivot) marks the
// element for the pivoted-LU fallback (v1 kernel, status bit 4).
__global__ void __launch_bounds__(kThreads, 2) element_v2_kernel(ElemArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
  const int m = a.m, ni = a.ni, nb = a.nb, np = a.order + 1, N = a.order;
  const int P = a.npad, nbc = a.nbc, ldp = v2_ldp(P);
  double* D11 = reinterpret_cast<double*>(smem_raw);
  double* L21s = D11 + PW * PW;
  double* Bp = L21s + static_cast<size_t>(ldp) * PW;
  double2* S = reinterpret_cast<double2*>(smem_raw);
  double2* f = S + nb * nb;
  double* mass = reinterpret_cast<double*>(smem_raw) + v2_region(P, nbc, nb);
  int* perm = reinterpret_cast<int*>(mass + np);
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_fail;

  double* A = a.ws + blockIdx.x * a.ws_stride;  // P x P, ld P (lower triangle used)
  double* B = A + static_cast<size_t>(P) * P;    // P x nbc, ld P
  for (int i = tid; i < np; i += blockDim.x) mass[i] = a.mass[i];
  auto K = [&](int r, int c) { return __ldg(a.stiff + r + c * np); };
  const int count = a.elist ? a.nlist : a.ne;

  for (int ii = blockIdx.x; ii < count; ii += gridDim.x) {
    const int e = a.elist ? a.elist[ii] : ii;
    __syncthreads();
    if (tid == 0) s_fail = 0;
    const double* ce = a.coeff + static_cast<size_t>(e) * np * np;
    // assemble the lower triangle of L_ii (element.cpp:57-90), identity padding
    for (int idx = tid; idx < P * P; idx += blockDim.x) {
      const int r = idx % P, c = idx / P;
      if (c > r) continue;
      double v;
      if (r >= ni) {
        v = (r == c) ? 1.0 : 0.0;
      } else {
        const int i = r / m + 1, j = r % m + 1, k = c / m + 1, l = c % m + 1;
        v = 0.0;
        if (j == l) v += K(i, k) * mass[j];
        if (i == k) v += mass[i] * K(j, l);
        if (r == c) v -= __ldg(ce + i * np + j) * mass[i] * mass[j];
      }
      A[idx] = v;
    }
    // right-hand sides [L_iG | re b~ | im b~ | 0 ...]
    for (int idx = tid; idx < P * nbc; idx += blockDim.x) {
      const int q = idx % P, b = idx / P;
      double v = 0.0;
      if (q < ni && b < nb + 2) {
        const int i = q / m + 1, j = q % m + 1;
        if (b < nb) {
          const int side = b / m, t = b % m + 1;
          switch (side) {
            case 0: v = (j == t) ? K(i, 0) * mass[j] : 0.0; break;
            case 1: v = (j == t) ? K(i, N) * mass[j] : 0.0; break;
            case 2: v = (i == t) ? mass[i] * K(j, 0) : 0.0; break;
            default: v = (i == t) ? mass[i] * K(j, N) : 0.0; break;
          }
        } else if (a.source) {
          const double2 s = a.source[static_cast<size_t>(e) * ni + q];
          const double w = mass[i] * mass[j];
          v = (b == nb) ? s.x * w : s.y * w;
        }
      }
      B[idx] = v;
    }
    __syncthreads();

    // ---- factorisation + forward solve, panel by panel
    for (int k0 = 0; k0 < P; k0 += PW) {
      const int rem = P - k0 - PW;
      for (int idx = tid; idx < PW * PW; idx += blockDim.x) {
        const int r = idx % PW, c = idx / PW;
        D11[idx] = c <= r ? A[(k0 + r) + static_cast<size_t>(k0 + c) * P] : 0.0;
      }
      __syncthreads();
      if (warp == 0) {
        for (int j = 0; j < PW; ++j) {
          if (lane == 0) {
            const double d = D11[j + j * PW];
            if (!(d > 0.0)) s_fail = 1;
            D11[j + j * PW] = sqrt(fmax(d, 1e-300));
          }
          __syncwarp();
          const double inv = 1.0 / D11[j + j * PW];
          if (lane > j && lane < PW) D11[lane + j * PW] *= inv;
          __syncwarp();
          for (int p = lane; p < PW * PW; p += 32) {
            const int r = p % PW, c = p / PW;
            if (c > j && r >= c) D11[r + c * PW] -= D11[r + j * PW] * D11[c + j * PW];
          }
          __syncwarp();
        }
      }
      __syncthreads();
      if (s_fail) break;
      for (int idx = tid; idx < PW * PW; idx += blockDim.x) {
        const int r = idx % PW, c = idx / PW;
        if (c <= r) A[(k0 + r) + static_cast<size_t>(k0 + c) * P] = D11[idx];
      }
      // L21 = A21 L11^{-T} (one row per thread)
      for (int r = tid; r < rem; r += blockDim.x) {
        double x[PW];
        double* row = A + (k0 + PW + r) + static_cast<size_t>(k0) * P;
#pragma unroll
        for (int j = 0; j < PW; ++j) x[j] = row[static_cast<size_t>(j) * P];
#pragma unroll
        for (int j = 0; j < PW; ++j) {
          double s = x[j];
#pragma unroll
          for (int t = 0; t < j; ++t) s -= x[t] * D11[j + t * PW];
          x[j] = s / D11[j + j * PW];
          L21s[r + j * ldp] = x[j];
          row[static_cast<size_t>(j) * P] = x[j];
        }
      }
      // forward solve of the panel rows of B
      for (int c = tid; c < nbc; c += blockDim.x) {
        double y[PW];
        double* col = B + k0 + static_cast<size_t>(c) * P;
#pragma unroll
        for (int j = 0; j < PW; ++j) y[j] = col[j];
#pragma unroll
        for (int j = 0; j < PW; ++j) {
          double s = y[j];
#pragma unroll
          for (int t = 0; t < j; ++t) s -= D11[j + t * PW] * y[t];
          y[j] = s / D11[j + j * PW];
          Bp[j + c * kLdq] = y[j];
          col[j] = y[j];
        }
      }
      __syncthreads();
      // trailing SYRK (lower 8x8 tiles) and B update, DMMA
      const int nt = rem / 8, ntri = nt * (nt + 1) / 2, nbt = nbc / 8;
      const int total = ntri + nt * nbt;
      // Each warp takes kBatch tiles at a time: all C fragments are loaded
      // first (kBatch x 2 loads in flight), then the DMMAs, then the stores,
      // so the L2 latency of one tile overlaps the others'.
      constexpr int kBatch = kTrailBatch;
      constexpr int kWarps = kThreads / 32;
      for (int base = warp; base < total; base += kWarps * kBatch) {
        double* Cp[kBatch];
        const double* Ap[kBatch];
        const double* Bq[kBatch];
        int bstride[kBatch];
        double c0[kBatch], c1[kBatch];
#pragma unroll
        for (int q = 0; q < kBatch; ++q) {
          const int tile = base + q * kWarps;
          Cp[q] = nullptr;
          if (tile >= total) continue;
          if (tile < ntri) {
            int I = static_cast<int>((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
            while (I * (I + 1) / 2 > tile) --I;
            while ((I + 1) * (I + 2) / 2 <= tile) ++I;
            const int J = tile - I * (I + 1) / 2;
            Cp[q] = A + (k0 + PW + 8 * I + g) + static_cast<size_t>(k0 + PW + 8 * J + 2 * t4) * P;
            Ap[q] = L21s + 8 * I + g;
            Bq[q] = L21s + 8 * J + g;
            bstride[q] = ldp;
          } else {
            const int tt = tile - ntri, I = tt % nt, J = tt / nt;
            Cp[q] = B + (k0 + PW + 8 * I + g) + static_cast<size_t>(8 * J + 2 * t4) * P;
            Ap[q] = L21s + 8 * I + g;
            Bq[q] = Bp + (8 * J + g) * kLdq;
            bstride[q] = -1;  // Bp: k runs along the column (stride 1)
          }
          c0[q] = Cp[q][0];
          c1[q] = Cp[q][P];
        }
#pragma unroll
        for (int q = 0; q < kBatch; ++q) {
          if (!Cp[q]) continue;
#pragma unroll
          for (int kk = 0; kk < PW; kk += 4) {
            const double av = -Ap[q][(kk + t4) * ldp];
            const double bv = bstride[q] < 0 ? Bq[q][kk + t4] : Bq[q][(kk + t4) * ldp];
            dmma(c0[q], c1[q], av, bv);
          }
        }
#pragma unroll
        for (int q = 0; q < kBatch; ++q)
          if (Cp[q]) {
            Cp[q][0] = c0[q];
            Cp[q][P] = c1[q];
          }
      }
      __syncthreads();
    }
    if (s_fail) {
      if (tid == 0) a.status[e] = 4;  // indefinite: pivoted-LU fallback
      continue;
    }
    // ---- backward solve R^T X = Y, right-looking from the last panel
    for (int k0 = P - PW; k0 >= 0; k0 -= PW) {
      for (int idx = tid; idx < PW * PW; idx += blockDim.x) {
        const int r = idx % PW, c = idx / PW;
        D11[idx] = c <= r ? A[(k0 + r) + static_cast<size_t>(k0 + c) * P] : 0.0;
      }
      __syncthreads();
      for (int c = tid; c < nbc; c += blockDim.x) {
        double y[PW];
        double* col = B + k0 + static_cast<size_t>(c) * P;
#pragma unroll
        for (int j = 0; j < PW; ++j) y[j] = col[j];
#pragma unroll
        for (int j = PW - 1; j >= 0; --j) {
          double s = y[j];
#pragma unroll
          for (int t = j + 1; t < PW; ++t) s -= D11[t + j * PW] * y[t];
          y[j] = s / D11[j + j * PW];
        }
#pragma unroll
        for (int j = 0; j < PW; ++j) {
          col[j] = y[j];
          Bp[j + c * kLdq] = y[j];
        }
      }
      __syncthreads();
      const int nr = k0 / 8, nbt = nbc / 8;
      constexpr int kBatch = 4;
      constexpr int kWarps = kThreads / 32;
      for (int base = warp; base < nr * nbt; base += kWarps * kBatch) {
        double* Cp[kBatch];
        double c0[kBatch], c1[kBatch], av[kBatch][PW / 4];
#pragma unroll
        for (int q = 0; q < kBatch; ++q) {
          const int tile = base + q * kWarps;
          Cp[q] = nullptr;
          if (tile >= nr * nbt) continue;
          const int I = tile % nr, J = tile / nr;
          Cp[q] = B + (8 * I + g) + static_cast<size_t>(8 * J + 2 * t4) * P;
          c0[q] = Cp[q][0];
          c1[q] = Cp[q][P];
#pragma unroll
          for (int kk = 0; kk < PW / 4; ++kk)
            av[q][kk] = -A[(k0 + 4 * kk + t4) + static_cast<size_t>(8 * I + g) * P];
        }
#pragma unroll
        for (int q = 0; q < kBatch; ++q) {
          if (!Cp[q]) continue;
          const int J = (base + q * kWarps) / nr;
#pragma unroll
          for (int kk = 0; kk < PW / 4; ++kk)
            dmma(c0[q], c1[q], av[q][kk], Bp[(4 * kk + t4) + (8 * J + g) * kLdq]);
          Cp[q][0] = c0[q];
          Cp[q][P] = c1[q];
        }
      }
      __syncthreads();
    }
    keep_interior(a, e, B, P);
    const bool ok = iti_epilogue(a, e, B, P, S, f, perm, red_v, red_i);
    if (tid == 0) a.status[e] = ok ? 0 : 2;
  }
}

// ---------------------------------------------------------------- v4
// Left-looking blocked Cholesky (16-wide panels) with the interior block and
// right-hand sides in the per-CTA global workspace (L2).  Per panel k:
//   1. the panel's rows of L (16 x k0) are staged once in shared memory;
//   2. the panel column block is brought up to date with one GEMM
//      A[k0:, k0:k0+16] -= L[k0:, :k0] L[k0:k0+16, :k0]^T: every warp owns
//      8-row strips whose 8 x 16 accumulators stay in registers over the whole
//      K loop (the A operand streams from L2, each element read once per
//      panel; no read-modify-write of the trailing matrix as in v2);
//   3. likewise the panel rows of the right-hand sides,
//      B[k0:k0+16, :] -= L[k0:k0+16, :k0] Y[:k0, :];
//   4. the 16 x 16 diagonal block is factored (warp 0), the rows below solved
//      against it (TRSM) and the panel rows of B solved (forward).
// The backward solve is left-looking the same way:
//   X_k = L_kk^{-T} (Y_k - L[k0+16:, k]^T X[k0+16:]).
constexpr int kV4Ld = 8;  // smem padding of the staged panel rows
#ifndef HPSB_V4_UNROLL
#define HPSB_V4_UNROLL 8
#endif
constexpr int kV4Unroll = HPSB_V4_UNROLL;
__host__ __device__ inline size_t v4_region(int P, int nbc, int nb) {
  const size_t panel = static_cast<size_t>(PW) * (P + kV4Ld) + PW * PW + static_cast<size_t>(PW) * (nbc + 4);
  const size_t epi = 2 * (static_cast<size_t>(nb) * nb + nb);
  return panel > epi ? panel : epi;
}

__global__ void __launch_bounds__(kThreads, 2) element_v4_kernel(ElemArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
  constexpr int kWarps = kThreads / 32;
  const int m = a.m, ni = a.ni, nb = a.nb, np = a.order + 1, N = a.order;
  const int P = a.npad, nbc = a.nbc, ldk = P + kV4Ld;
  double* Ls = reinterpret_cast<double*>(smem_raw);        // [16][ldk]: L[k0 + n][k]
  double* D11 = Ls + static_cast<size_t>(PW) * ldk;         // 16 x 16
  double* Xp = D11 + PW * PW;                               // [16][nbc + 4]: panel rows of X
  const int ldx = nbc + 4;
  double2* S = reinterpret_cast<double2*>(smem_raw);        // epilogue overlay
  double2* f = S + nb * nb;
  double* mass = reinterpret_cast<double*>(smem_raw) + v4_region(P, nbc, nb);
  int* perm = reinterpret_cast<int*>(mass + np);
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_fail;

  double* A = a.ws + blockIdx.x * a.ws_stride;  // P x P, ld P (lower used)
  double* B = A + static_cast<size_t>(P) * P;    // P x nbc, ld P
  for (int i = tid; i < np; i += blockDim.x) mass[i] = a.mass[i];
  auto K = [&](int r, int c) { return __ldg(a.stiff + r + c * np); };
  const int count = a.elist ? a.nlist : a.ne;

  for (int ii = blockIdx.x; ii < count; ii += gridDim.x) {
    const int e = a.elist ? a.elist[ii] : ii;
    __syncthreads();
    if (tid == 0) s_fail = 0;
    const double* ce = a.coeff + static_cast<size_t>(e) * np * np;
    for (int idx = tid; idx < P * P; idx += blockDim.x) {
      const int r = idx % P, c = idx / P;
      if (c > r) continue;
      double v;
      if (r >= ni) {
        v = (r == c) ? 1.0 : 0.0;
      } else {
        const int i = r / m + 1, j = r % m + 1, k = c / m + 1, l = c % m + 1;
        v = 0.0;
        if (j == l) v += K(i, k) * mass[j];
        if (i == k) v += mass[i] * K(j, l);
        if (r == c) v -= __ldg(ce + i * np + j) * mass[i] * mass[j];
      }
      A[idx] = v;
    }
    for (int idx = tid; idx < P * nbc; idx += blockDim.x) {
      const int q = idx % P, b = idx / P;
      double v = 0.0;
      if (q < ni && b < nb + 2) {
        const int i = q / m + 1, j = q % m + 1;
        if (b < nb) {
          const int side = b / m, t = b % m + 1;
          switch (side) {
            case 0: v = (j == t) ? K(i, 0) * mass[j] : 0.0; break;
            case 1: v = (j == t) ? K(i, N) * mass[j] : 0.0; break;
            case 2: v = (i == t) ? mass[i] * K(j, 0) : 0.0; break;
            default: v = (i == t) ? mass[i] * K(j, N) : 0.0; break;
          }
        } else if (a.source) {
          const double2 sv = a.source[static_cast<size_t>(e) * ni + q];
          const double w = mass[i] * mass[j];
          v = (b == nb) ? sv.x * w : sv.y * w;
        }
      }
      B[idx] = v;
    }
    __syncthreads();

    // ---- factorisation + forward solve, left-looking
    for (int k0 = 0; k0 < P; k0 += PW) {
      // 1. panel rows of L (final) -> smem
      for (int idx = tid; idx < PW * k0; idx += blockDim.x) {
        const int n = idx % PW, k = idx / PW;
        Ls[n * ldk + k] = A[(k0 + n) + static_cast<size_t>(k) * P];
      }
      __syncthreads();
      const int nstrip = (P - k0) / 8, nbt = nbc / 8;
      // 2. + 3. GEMM updates: strips of the panel column block, then the
      //    panel rows of B (2 row tiles x nbt column tiles)
      for (int w = warp; w < nstrip + 2 * nbt; w += kWarps) {
        if (w < nstrip) {
          const int r0 = k0 + 8 * w;
          double* C0 = A + (r0 + g) + static_cast<size_t>(k0 + 2 * t4) * P;
          double* C1 = C0 + static_cast<size_t>(8) * P;
          double c00 = C0[0], c01 = C0[P], c10 = C1[0], c11 = C1[P];
          const double* Ar = A + (r0 + g) + static_cast<size_t>(t4) * P;
          int kk = 0;
          for (; kk + 4 * kV4Unroll <= k0; kk += 4 * kV4Unroll) {
            double av[kV4Unroll];  // kV4Unroll independent L2 loads in flight per lane
#pragma unroll
            for (int q = 0; q < kV4Unroll; ++q) av[q] = -Ar[static_cast<size_t>(kk + 4 * q) * P];
#pragma unroll
            for (int q = 0; q < kV4Unroll; ++q) {
              dmma(c00, c01, av[q], Ls[g * ldk + kk + 4 * q + t4]);
              dmma(c10, c11, av[q], Ls[(8 + g) * ldk + kk + 4 * q + t4]);
            }
          }
          for (; kk < k0; kk += 4) {
            const double av = -Ar[static_cast<size_t>(kk) * P];
            dmma(c00, c01, av, Ls[g * ldk + kk + t4]);
            dmma(c10, c11, av, Ls[(8 + g) * ldk + kk + t4]);
          }
          C0[0] = c00, C0[P] = c01, C1[0] = c10, C1[P] = c11;
        } else {
          const int tt = w - nstrip, I = tt % 2, J = tt / 2;
          double* Cp = B + (k0 + 8 * I + g) + static_cast<size_t>(8 * J + 2 * t4) * P;
          double c0 = Cp[0], c1 = Cp[P];
          const double* Yc = B + t4 + static_cast<size_t>(8 * J + g) * P;  // Y[k][8J + g]
          int kk = 0;
          for (; kk + 32 <= k0; kk += 32) {
            double ya[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) ya[q] = Yc[kk + 4 * q];
#pragma unroll
            for (int q = 0; q < 8; ++q) dmma(c0, c1, -Ls[(8 * I + g) * ldk + kk + 4 * q + t4], ya[q]);
          }
          for (; kk < k0; kk += 4)
            dmma(c0, c1, -Ls[(8 * I + g) * ldk + kk + t4], Yc[kk]);
          Cp[0] = c0, Cp[P] = c1;
        }
      }
      __syncthreads();
      // 4. diagonal block, TRSM below, forward solve of the panel rows of B
      for (int idx = tid; idx < PW * PW; idx += blockDim.x) {
        const int r = idx % PW, c = idx / PW;
        D11[idx] = c <= r ? A[(k0 + r) + static_cast<size_t>(k0 + c) * P] : 0.0;
      }
      __syncthreads();
      if (warp == 0) {
        for (int j = 0; j < PW; ++j) {
          if (lane == 0) {
            const double d = D11[j + j * PW];
            if (!(d > 0.0)) s_fail = 1;
            D11[j + j * PW] = sqrt(fmax(d, 1e-300));
          }
          __syncwarp();
          const double inv = 1.0 / D11[j + j * PW];
          if (lane > j && lane < PW) D11[lane + j * PW] *= inv;
          __syncwarp();
          for (int q = lane; q < PW * PW; q += 32) {
            const int r = q % PW, c = q / PW;
            if (c > j && r >= c) D11[r + c * PW] -= D11[r + j * PW] * D11[c + j * PW];
          }
          __syncwarp();
        }
      }
      __syncthreads();
      if (s_fail) break;
      const int rem = P - k0 - PW;
      for (int idx = tid; idx < PW * PW; idx += blockDim.x) {
        const int r = idx % PW, c = idx / PW;
        if (c <= r) A[(k0 + r) + static_cast<size_t>(k0 + c) * P] = D11[idx];
      }
      for (int r = tid; r < rem + nbc; r += blockDim.x) {
        double x[PW];
        if (r < rem) {
          double* row = A + (k0 + PW + r) + static_cast<size_t>(k0) * P;
#pragma unroll
          for (int j = 0; j < PW; ++j) x[j] = row[static_cast<size_t>(j) * P];
#pragma unroll
          for (int j = 0; j < PW; ++j) {
            double sacc = x[j];
#pragma unroll
            for (int t = 0; t < j; ++t) sacc -= x[t] * D11[j + t * PW];
            x[j] = sacc / D11[j + j * PW];
            row[static_cast<size_t>(j) * P] = x[j];
          }
        } else {
          double* col = B + k0 + static_cast<size_t>(r - rem) * P;
#pragma unroll
          for (int j = 0; j < PW; ++j) x[j] = col[j];
#pragma unroll
          for (int j = 0; j < PW; ++j) {
            double sacc = x[j];
#pragma unroll
            for (int t = 0; t < j; ++t) sacc -= D11[j + t * PW] * x[t];
            x[j] = sacc / D11[j + j * PW];
            col[j] = x[j];
          }
        }
      }
      __syncthreads();
    }
    if (s_fail) {
      if (tid == 0) a.status[e] = 4;  // indefinite: pivoted-LU fallback
      continue;
    }
    // ---- backward solve, left-looking: X_k = L_kk^{-T}(Y_k - L[k0+16:, k]^T X[k0+16:])
    for (int k0 = P - PW; k0 >= 0; k0 -= PW) {
      const int nbt = nbc / 8, kb = k0 + PW, klen = P - kb;
      for (int idx = tid; idx < PW * PW; idx += blockDim.x) {
        const int r = idx % PW, c = idx / PW;
        D11[idx] = c <= r ? A[(k0 + r) + static_cast<size_t>(k0 + c) * P] : 0.0;
      }
      for (int w = warp; w < 2 * nbt; w += kWarps) {
        const int I = w % 2, J = w / 2;
        double* Cp = B + (k0 + 8 * I + g) + static_cast<size_t>(8 * J + 2 * t4) * P;
        double c0 = Cp[0], c1 = Cp[P];
        // A-fragment (row 8I+g, k) = L[kb + k][k0 + 8I + g]; B-fragment (k, col 8J+g) = X[kb + k][8J + g]
        const double* Lc = A + kb + t4 + static_cast<size_t>(k0 + 8 * I + g) * P;
        const double* Xc = B + kb + t4 + static_cast<size_t>(8 * J + g) * P;
        int kk = 0;
        for (; kk + 32 <= klen; kk += 32) {
          double la[8], xa[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) la[q] = -Lc[kk + 4 * q], xa[q] = Xc[kk + 4 * q];
#pragma unroll
          for (int q = 0; q < 8; ++q) dmma(c0, c1, la[q], xa[q]);
        }
        for (; kk < klen; kk += 4) dmma(c0, c1, -Lc[kk], Xc[kk]);
        Cp[0] = c0, Cp[P] = c1;
      }
      __syncthreads();
      for (int c = tid; c < nbc; c += blockDim.x) {
        double y[PW];
        double* col = B + k0 + static_cast<size_t>(c) * P;
#pragma unroll
        for (int j = 0; j < PW; ++j) y[j] = col[j];
#pragma unroll
        for (int j = PW - 1; j >= 0; --j) {
          double sacc = y[j];
#pragma unroll
          for (int t = j + 1; t < PW; ++t) sacc -= D11[t + j * PW] * y[t];
          y[j] = sacc / D11[j + j * PW];
        }
#pragma unroll
        for (int j = 0; j < PW; ++j) col[j] = y[j];
      }
      __syncthreads();
    }
    (void)Xp, (void)ldx;
    keep_interior(a, e, B, P);
    const bool ok = iti_epilogue(a, e, B, P, S, f, perm, red_v, red_i);
    if (tid == 0) a.status[e] = ok ? 0 : 2;
  }
}

// ---------------------------------------------------------------- v3
// Shared-memory-resident variant for small interiors (P <= ~128, i.e. N <= 12):
// the whole interior block L_ii (column-major, ld P+4 so 8x8 DMMA fragments
// are bank-conflict free) and the right-hand sides [L_iG | b~] live in shared
// memory; one 512-thread CTA per SM loops over elements.  Blocked right-
// looking Cholesky with 16-wide panels (warp 0 factors the diagonal block,
// rows / columns of the panel solves on all threads), trailing SYRK and
// right-hand-side updates on DMMA tiles with every operand on-chip, blocked
// backward solve likewise.  No global-memory round trips inside the
// factorisation (the v2 kernel's trailing updates go through L2).
constexpr int kV3Threads = 512;
__host__ __device__ inline size_t v3_smem_doubles(int P, int nbc, int nb) {
  const size_t lda = P + 4;
  const size_t fact = lda * P + lda * nbc;              // A | B
  const size_t epi = 2 * (static_cast<size_t>(nb) * nb + nb) + lda * nbc;  // S, f over A; B kept
  return (fact > epi ? fact : epi);
}

__global__ void __launch_bounds__(kV3Threads, 1) element_v3_kernel(ElemArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
  constexpr int kWarps = kV3Threads / 32;
  const int m = a.m, ni = a.ni, nb = a.nb, np = a.order + 1, N = a.order;
  const int P = a.npad, nbc = a.nbc, lda = P + 4;
  double* A = reinterpret_cast<double*>(smem_raw);    // P x P (lower used), ld lda
  double* B = A + static_cast<size_t>(lda) * P;       // P x nbc, ld lda
  double2* S = reinterpret_cast<double2*>(smem_raw);  // epilogue overlay on A
  double2* f = S + nb * nb;
  __shared__ double mass[64];
  // the 1-D operators on chip: the large shared-memory carve-out leaves
  // little L1, and the assembly / epilogue index them in every inner loop
  __shared__ double stiff_s[64 * 64 / 2], diff_s[64 * 64 / 2];
  __shared__ int perm[128];
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_fail;
  for (int i = tid; i < np; i += kV3Threads) mass[i] = a.mass[i];
  for (int i = tid; i < np * np; i += kV3Threads) stiff_s[i] = a.stiff[i], diff_s[i] = a.diff[i];
  auto K = [&](int r, int c) { return stiff_s[r + c * np]; };
  const int count = a.elist ? a.nlist : a.ne;

  for (int ii = blockIdx.x; ii < count; ii += gridDim.x) {
    const int e = a.elist ? a.elist[ii] : ii;
    __syncthreads();
    if (tid == 0) s_fail = 0;
    const double* ce = a.coeff + static_cast<size_t>(e) * np * np;
    for (int idx = tid; idx < P * P; idx += kV3Threads) {
      const int r = idx % P, c = idx / P;
      if (c > r) continue;
      double v;
      if (r >= ni) {
        v = (r == c) ? 1.0 : 0.0;
      } else {
        const int i = r / m + 1, j = r % m + 1, k = c / m + 1, l = c % m + 1;
        v = 0.0;
        if (j == l) v += K(i, k) * mass[j];
        if (i == k) v += mass[i] * K(j, l);
        if (r == c) v -= __ldg(ce + i * np + j) * mass[i] * mass[j];
      }
      A[r + c * lda] = v;
    }
    for (int idx = tid; idx < P * nbc; idx += kV3Threads) {
      const int q = idx % P, b = idx / P;
      double v = 0.0;
      if (q < ni && b < nb + 2) {
        const int i = q / m + 1, j = q % m + 1;
        if (b < nb) {
          const int side = b / m, t = b % m + 1;
          switch (side) {
            case 0: v = (j == t) ? K(i, 0) * mass[j] : 0.0; break;
            case 1: v = (j == t) ? K(i, N) * mass[j] : 0.0; break;
            case 2: v = (i == t) ? mass[i] * K(j, 0) : 0.0; break;
            default: v = (i == t) ? mass[i] * K(j, N) : 0.0; break;
          }
        } else if (a.source) {
          const double2 sv = a.source[static_cast<size_t>(e) * ni + q];
          const double w = mass[i] * mass[j];
          v = (b == nb) ? sv.x * w : sv.y * w;
        }
      }
      B[q + b * lda] = v;
    }
    __syncthreads();

    // ---- factorisation + forward solve
    for (int k0 = 0; k0 < P; k0 += PW) {
      if (warp == 0) {  // Cholesky of the 16 x 16 diagonal block
        for (int j = 0; j < PW; ++j) {
          double* cj = A + (k0 + j) * lda + k0;
          if (lane == 0) {
            const double d = cj[j];
            if (!(d > 0.0)) s_fail = 1;
            cj[j] = sqrt(fmax(d, 1e-300));
          }
          __syncwarp();
          const double inv = 1.0 / cj[j];
          if (lane > j && lane < PW) cj[lane] *= inv;
          __syncwarp();
          for (int q = lane; q < PW * PW; q += 32) {
            const int r = q % PW, c = q / PW;
            if (c > j && r >= c) A[(k0 + r) + (k0 + c) * lda] -= cj[r] * cj[c];
          }
          __syncwarp();
        }
      }
      __syncthreads();
      if (s_fail) break;
      const int rem = P - k0 - PW;
      // L21 = A21 L11^{-T} (a row per thread) and the panel rows of B (a column per thread)
      for (int r = tid; r < rem + nbc; r += kV3Threads) {
        double x[PW];
        if (r < rem) {
          double* row = A + (k0 + PW + r) + k0 * lda;
#pragma unroll
          for (int j = 0; j < PW; ++j) x[j] = row[j * lda];
#pragma unroll
          for (int j = 0; j < PW; ++j) {
            double sacc = x[j];
#pragma unroll
            for (int t = 0; t < j; ++t) sacc -= x[t] * A[(k0 + j) + (k0 + t) * lda];
            x[j] = sacc / A[(k0 + j) + (k0 + j) * lda];
            row[j * lda] = x[j];
          }
        } else {
          double* col = B + k0 + (r - rem) * lda;
#pragma unroll
          for (int j = 0; j < PW; ++j) x[j] = col[j];
#pragma unroll
          for (int j = 0; j < PW; ++j) {
            double sacc = x[j];
#pragma unroll
            for (int t = 0; t < j; ++t) sacc -= A[(k0 + j) + (k0 + t) * lda] * x[t];
            x[j] = sacc / A[(k0 + j) + (k0 + j) * lda];
            col[j] = x[j];
          }
        }
      }
      __syncthreads();
      // trailing: A22 -= L21 L21^T (lower 8x8 tiles), B2 -= L21 B1 (DMMA, all in smem)
      const int nt = rem / 8, ntri = nt * (nt + 1) / 2, nbt = nbc / 8;
      const int total = ntri + nt * nbt;
      for (int tile = warp; tile < total; tile += kWarps) {
        double* Cp;
        int arow, brow;  // A-fragment row, B-fragment (col of result) row of L21 / column of B
        bool isB;
        if (tile < ntri) {
          int I = static_cast<int>((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
          while (I * (I + 1) / 2 > tile) --I;
          while ((I + 1) * (I + 2) / 2 <= tile) ++I;
          const int J = tile - I * (I + 1) / 2;
          Cp = A + (k0 + PW + 8 * I + g) + (k0 + PW + 8 * J + 2 * t4) * lda;
          arow = k0 + PW + 8 * I + g;
          brow = k0 + PW + 8 * J + g;
          isB = false;
        } else {
          const int tt = tile - ntri, I = tt % nt, J = tt / nt;
          Cp = B + (k0 + PW + 8 * I + g) + (8 * J + 2 * t4) * lda;
          arow = k0 + PW + 8 * I + g;
          brow = 8 * J + g;  // column of B
          isB = true;
        }
        double c0 = Cp[0], c1 = Cp[lda];
#pragma unroll
        for (int kk = 0; kk < PW; kk += 4) {
          const double av = -A[arow + (k0 + kk + t4) * lda];
          const double bv = isB ? B[(k0 + kk + t4) + brow * lda] : A[brow + (k0 + kk + t4) * lda];
          dmma(c0, c1, av, bv);
        }
        Cp[0] = c0;
        Cp[lda] = c1;
      }
      __syncthreads();
    }
    if (s_fail) {
      if (tid == 0) a.status[e] = 4;  // indefinite: pivoted-LU fallback
      continue;
    }
    // ---- backward solve R^T X = Y, from the last panel
    for (int k0 = P - PW; k0 >= 0; k0 -= PW) {
      for (int c = tid; c < nbc; c += kV3Threads) {
        double y[PW];
        double* col = B + k0 + c * lda;
#pragma unroll
        for (int j = 0; j < PW; ++j) y[j] = col[j];
#pragma unroll
        for (int j = PW - 1; j >= 0; --j) {
          double sacc = y[j];
#pragma unroll
          for (int t = j + 1; t < PW; ++t) sacc -= A[(k0 + t) + (k0 + j) * lda] * y[t];
          y[j] = sacc / A[(k0 + j) + (k0 + j) * lda];
        }
#pragma unroll
        for (int j = 0; j < PW; ++j) col[j] = y[j];
      }
      __syncthreads();
      const int nr = k0 / 8, nbt = nbc / 8;
      for (int tile = warp; tile < nr * nbt; tile += kWarps) {
        const int I = tile % nr, J = tile / nr;
        double* Cp = B + (8 * I + g) + (8 * J + 2 * t4) * lda;
        double c0 = Cp[0], c1 = Cp[lda];
#pragma unroll
        for (int kk = 0; kk < PW; kk += 4) {
          const double av = -A[(k0 + kk + t4) + (8 * I + g) * lda];
          const double bv = B[(k0 + kk + t4) + (8 * J + g) * lda];
          dmma(c0, c1, av, bv);
        }
        Cp[0] = c0;
        Cp[lda] = c1;
      }
      __syncthreads();
    }
    keep_interior(a, e, B, lda);
    __syncthreads();
    const bool ok = iti_epilogue(a, e, B, lda, S, f, perm, red_v, red_i, diff_s);
    if (tid == 0) a.status[e] = ok ? 0 : 2;
  }
}

}  // namespace

namespace {
// status bit 4 (indefinite interior block: redo with the pivoted LU) -> list
__global__ void collect_redo_kernel(const int* __restrict__ status, int ne, int* list, int* count) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x)
    if (status[e] & 4) list[atomicAdd(count, 1)] = e;
}
}  // namespace

std::unique_ptr<Elements> build_elements(Context* ctx, int n, int order, double eta,
                                         const double* coeff_dev, const double2* source_dev) {
  if (n < 2 || (n & (n - 1)) != 0)
    throw InvalidArgument("Mesh: elements per side must be a power of two >= 2");
  if (order < 2) throw InvalidArgument("Mesh: degree must be >= 2");
  if (!(eta > 0.0)) throw InvalidArgument("Mesh: kappa and eta must be positive");
  auto el = std::make_unique<Elements>();
  el->ctx = ctx;
  el->n = n, el->order = order, el->m = order - 1, el->nb = 4 * (order - 1);
  el->eta = eta, el->h = 1.0 / n;
  const int ne = n * n, np = order + 1, m = order - 1, ni = m * m, nb = 4 * m;

  // 1-D operators on the element edge (proj/src/spectral.cpp:89-98).
  const Gll g = gll_rule(order);
  const double h = el->h;
  std::vector<double> mass(np), diff(np * np), stiff(np * np, 0.0);
  for (int i = 0; i < np; ++i) mass[i] = (0.5 * h) * g.weights[i];
  for (int k = 0; k < np * np; ++k) diff[k] = (2.0 / h) * g.diff[k];
  for (int j = 0; j < np; ++j)
    for (int i = 0; i < np; ++i) {
      double s = 0.0;
      for (int q = 0; q < np; ++q) s += (diff[q + i * np] * mass[q]) * diff[q + j * np];
      stiff[i + j * np] = s;
    }
  DevBuf<double> d_mass, d_diff, d_stiff;
  d_mass.upload(mass, ctx->stream);
  d_diff.upload(diff, ctx->stream);
  d_stiff.upload(stiff, ctx->stream);

  el->T.alloc(static_cast<size_t>(ne) * nb * nb);
  el->H.alloc(static_cast<size_t>(ne) * nb);
  el->status.alloc(ne);
  el->Y.alloc(static_cast<size_t>(ne) * ni * (nb + 2));
  HPSB_CUDA(cudaMemsetAsync(el->status.p, 0, ne * sizeof(int), ctx->stream));
  // Sharded (one rank per GPU): build only this rank's quadtree subtree.
  el->part = make_partition(build_face_graph(n), ctx->world(), ctx->rank());
  DevBuf<int> d_own;
  const bool sharded = ctx->world() > 1;
  if (sharded) {
    HPSB_CUDA(cudaMemsetAsync(el->T.p, 0, el->T.bytes(), ctx->stream));
    HPSB_CUDA(cudaMemsetAsync(el->H.p, 0, el->H.bytes(), ctx->stream));
    d_own.upload(el->part.own_elems, ctx->stream);
  }
  const int nwork = sharded ? static_cast<int>(el->part.own_elems.size()) : ne;

  ElemArgs a{};
  a.ne = ne, a.order = order, a.m = m, a.ni = ni, a.nb = nb, a.eta = eta;
  a.mass = d_mass.p, a.diff = d_diff.p, a.stiff = d_stiff.p;
  a.coeff = coeff_dev, a.source = source_dev;
  a.T = el->T.p, a.H = el->H.p, a.status = el->status.p, a.Y = el->Y.p;
  a.npad = (ni + PW - 1) / PW * PW;
  a.nbc = (nb + 2 + 7) / 8 * 8;
  if (sharded) a.elist = d_own.p, a.nlist = nwork;

  // v3 (shared-memory resident) when the interior block fits, else v2
  DevBuf<double> ws;
  bool done = false;
  {
    const size_t smem3 = sizeof(double) * v3_smem_doubles(a.npad, a.nbc, nb);
    // Opt-in (HPSB_ELEMENT_V3=1): measured slower than v2 at cfg4 (132 vs 113 ms):
    // with one 512-thread CTA per SM the serial panel / pivot steps leave 15
    // warps waiting (ncu: 20% of stall samples at the panel barrier).
    if (smem3 <= 200u * 1024 && np * np <= 2048 && nb <= 128 && std::getenv("HPSB_ELEMENT_V3")) {
      allow_smem<element_v3_kernel>(smem3);
      const int slots3 = std::min(nwork, ctx->num_sms);
      HPSB_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
      {
        const double fe = ni * double(ni) * ni / 3.0 + 2.0 * ni * double(ni) * nb + 8.0 * nb * double(nb) * nb;
        KernelScope ks(ctx, "element_iti", 8.0 * nwork * (np * np + 2 * ni + 2 * nb * nb + 2 * nb),
                       fe * nwork);
        element_v3_kernel<<<slots3, kV3Threads, smem3, ctx->stream>>>(a);
        HPSB_LAUNCHED(ctx);
      }
      done = true;
    }
  }
  if (!done && !std::getenv("HPSB_ELEMENT_V2")) {
    // v5 (batched blocked Cholesky over element chunks, element_v5.cu)
    HPSB_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
    done = element_v5_build(ctx, a, nwork);
  }
  if (!done && !std::getenv("HPSB_ELEMENT_V2")) {
    // v4 (left-looking, DMMA GEMM panels)
    const size_t smem4 = sizeof(double) * (v4_region(a.npad, a.nbc, nb) + np) + sizeof(int) * nb + 16;
    allow_smem<element_v4_kernel>(smem4);
    int per_sm = 0;
    HPSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, element_v4_kernel, kThreads, smem4));
    const int slots4 = std::min(nwork, std::max(1, std::min(per_sm, 3)) * ctx->num_sms);
    const size_t stride4 = static_cast<size_t>(a.npad) * (a.npad + a.nbc);
    ws.alloc(stride4 * slots4);
    a.ws = ws.p, a.ws_stride = stride4;
    HPSB_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
    {
      const double fe = ni * double(ni) * ni / 3.0 + 2.0 * ni * double(ni) * nb + 8.0 * nb * double(nb) * nb;
      KernelScope ks(ctx, "element_iti", 8.0 * nwork * (np * np + 2 * ni + 2 * nb * nb + 2 * nb),
                     fe * nwork);
      element_v4_kernel<<<slots4, kThreads, smem4, ctx->stream>>>(a);
      HPSB_LAUNCHED(ctx);
    }
    done = true;
  }
  if (!done) {
  // v2 (blocked, DMMA) for every element
  const size_t smem2 = sizeof(double) * (v2_region(a.npad, a.nbc, nb) + np) + sizeof(int) * nb + 16;
  allow_smem<element_v2_kernel>(smem2);
  int per_sm = 0;
  HPSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, element_v2_kernel, kThreads, smem2));
  const int slots2 = std::min(nwork, std::max(1, std::min(per_sm, 3)) * ctx->num_sms);
  const size_t stride2 = static_cast<size_t>(a.npad) * (a.npad + a.nbc);
  ws.alloc(stride2 * slots2);
  a.ws = ws.p, a.ws_stride = stride2;
  HPSB_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  {
    // pinned algorithmic flops: ni^3/3 + 2 ni^2 nb + 8 nb^3 per element
    const double fe = ni * double(ni) * ni / 3.0 + 2.0 * ni * double(ni) * nb + 8.0 * nb * double(nb) * nb;
    KernelScope ks(ctx, "element_iti", 8.0 * nwork * (np * np + 2 * ni + 2 * nb * nb + 2 * nb),
                   fe * nwork);
    element_v2_kernel<<<slots2, kThreads, smem2, ctx->stream>>>(a);
    HPSB_LAUNCHED(ctx);
  }
  }
  // Pivoted-LU fallback (v1) for elements whose interior block is
  // indefinite (status bit 4), without a host round trip: the flagged
  // elements are listed on the device and the v1 launch reads the count.
  {
    DevBuf<int> d_redo(ne + 1);
    HPSB_CUDA(cudaMemsetAsync(d_redo.p + ne, 0, sizeof(int), ctx->stream));
    collect_redo_kernel<<<std::max(1, std::min((ne + 255) / 256, 4 * ctx->num_sms)), 256, 0,
                          ctx->stream>>>(el->status.p, ne, d_redo.p, d_redo.p + ne);
    HPSB_LAUNCHED(ctx);
    const int slots = std::min(ne, ctx->num_sms);
    const size_t stride = static_cast<size_t>(ni) * ni + static_cast<size_t>(ni) * (nb + 2);
    ws.alloc(stride * slots);
    a.ws = ws.p, a.ws_stride = stride;
    a.elist = d_redo.p, a.nlist = ne, a.nlist_dev = d_redo.p + ne;
    const size_t smem = sizeof(double2) * (nb * nb + nb) + sizeof(double) * (ni + np) +
                        sizeof(int) * nb + 16;
    allow_smem<element_kernel>(smem);
    KernelScope ks(ctx, "element_iti_lu", 0.0, 0.0);
    element_kernel<<<slots, kThreads, smem, ctx->stream>>>(a);
    HPSB_LAUNCHED(ctx);
    // h_status[ne] = number of elements the fallback redid
    el->h_status = pinned_ints_acquire(ne + 1, &el->h_status_cap);
    HPSB_CUDA(cudaMemcpyAsync(el->h_status, el->status.p, ne * sizeof(int),
                              cudaMemcpyDeviceToHost, ctx->stream));
    HPSB_CUDA(cudaMemcpyAsync(el->h_status + ne, d_redo.p + ne, sizeof(int),
                              cudaMemcpyDeviceToHost, ctx->stream));
  }
  HPSB_CUDA(cudaEventCreateWithFlags(&el->done, cudaEventDisableTiming));
  HPSB_CUDA(cudaEventRecord(el->done, ctx->stream));
  el->pending = true;
  if (std::getenv("HPSB_ELEMENTS_SYNC")) elements_wait(el.get());
  return el;
}

// Pinned status buffers are recycled, never freed: cudaFreeHost (and often
// cudaMallocHost) synchronises the whole device, which would stall the next
// setup's overlapped pipeline when the previous Elements is released.
namespace {
std::mutex g_pinned_mu;
std::vector<std::pair<int*, size_t>> g_pinned_free;
}  // namespace

int* pinned_ints_acquire(size_t n, size_t* cap) {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    for (size_t i = 0; i < g_pinned_free.size(); ++i)
      if (g_pinned_free[i].second >= n) {
        auto pr = g_pinned_free[i];
        g_pinned_free.erase(g_pinned_free.begin() + i);
        *cap = pr.second;
        return pr.first;
      }
  }
  int* p = nullptr;
  HPSB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p), n * sizeof(int)));
  *cap = n;
  return p;
}

Elements::~Elements() {
  if (done) cudaEventDestroy(done);
  if (h_status) {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    g_pinned_free.emplace_back(h_status, h_status_cap);
  }
}

void elements_wait(Elements* el) {
  if (!el || !el->pending) return;
  HPSB_CUDA(cudaEventSynchronize(el->done));
  el->pending = false;
  const int ne = el->n * el->n;
  el->fallbacks = el->h_status[ne];
  for (int e = 0; e < ne; ++e)
    if (el->h_status[e]) {
      // mesh.cpp:82-84 annotates element failures with the element id.
      throw std::runtime_error("element " + std::to_string(e) + ": " +
                               ((el->h_status[e] & 1) ? "singular interior block"
                                                      : "singular local operator"));
    }
}

}  // namespace hpsb
