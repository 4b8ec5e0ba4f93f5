// Register-resident complex Gauss-Jordan inverse for batched small matrices
// (n <= 96): one 512-thread CTA per matrix, the matrix held in registers.
//
// The shared-memory Gauss-Jordan (linalg.cuh gj_inverse_cta) keeps the
// matrix in ~n^2 x 16 B of shared memory, so only two matrices fit on an SM
// and its four barriers plus a one-warp pivot search per column leave the
// SM idle: the element ItI inverses (76 x 76, one per element) ran at
// ~2 TFLOP/s.  Here the 512 threads form a 16 x 32 grid; thread (ty, tx)
// owns rows ty + 16 a and columns tx + 32 b (cyclic, TR x TC entries), and
// the only shared state per step is the pivot row and column (two small
// double-buffered vectors): two barriers per column.
//
// Partial pivoting without physical row swaps (the pivot of column k is the
// largest |a_ik| over rows not yet used, lowest row index on ties -- the
// same choice as gj_inverse_cta's swap-based search).  With p_k the pivot
// row of step k, the stored entry X[i][k] is the inverse's entry
//   A^{-1}[step(i)][p_k],   step(p_k) = k,
// which the callers apply when they write the result out.
#pragma once

#include "device.cuh"

namespace hpsb {

constexpr int kGjY = 16, kGjX = 32, kGjThreads = kGjY * kGjX, kGjMax = 96;
// Guard of the diagonal-pivot Gauss-Jordan (squared magnitudes relative to
// m0 = max |a_ij|^2): every pivot |p_k| >= 1e-6 max |a_ij| and every inverse
// entry <= 1e8 / max |a_ij| (growth of at most ~1e8 over the pivoted
// inverse's bound, ~1e-8 relative of rounding headroom before the 1e-10
// operator tolerance would be at risk); a matrix outside either bound is
// redone with partial pivoting.
constexpr double kGjTiny2 = 1e-12, kGjHuge2 = 1e16;

struct GjShared {
  double2 rowbuf[2][kGjMax];
  double2 colbuf[2][kGjMax];
  double2 inv[2];
  int p[2];
  int piv[kGjMax];   // piv[k]  = pivot row of step k
  int step[kGjMax];  // step[i] = step at which row i was the pivot
  int fail;
};

template <int TR, int TC>
struct GjReg {
  double2 x[TR][TC];
};

// Inverse of the n x n matrix get(i, j) (n <= min(16 TR, 32 TC)).  On return
// g.x holds the permuted inverse (see above), sh.piv / sh.step the
// permutation; returns false if a pivot was exactly zero.  Block-wide: all
// kGjThreads threads must call it.
template <int TR, int TC, class Get>
__device__ __forceinline__ bool gj_reg_inverse(int n, Get get, GjReg<TR, TC>& g, GjShared& sh) {
  const int tid = threadIdx.x, ty = tid % kGjY, tx = tid / kGjY;
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int i = ty + kGjY * a, j = tx + kGjX * b;
      g.x[a][b] = (i < n && j < n) ? get(i, j) : make_double2(0.0, 0.0);
    }
  if (tid == 0) sh.fail = 0;
  for (int t = tid; t < 2 * kGjMax; t += kGjThreads) {
    sh.rowbuf[t / kGjMax][t % kGjMax] = make_double2(0.0, 0.0);
    sh.colbuf[t / kGjMax][t % kGjMax] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  unsigned used = 0;  // bit a: row ty + 16 a has been a pivot row
  for (int k = 0; k < n; ++k) {
    const int buf = k & 1, kx = k % kGjX, kb = k / kGjX;
    // pivot search: the owners of column k are 16 consecutive threads (a half-warp)
    if (tx == kx) {
      const unsigned hmask = (kx & 1) ? 0xffff0000u : 0x0000ffffu;  // this half-warp
      double best = -1.0, br = 0.0, bim = 0.0;
      int bi = n;
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        const int i = ty + kGjY * a;
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < TC; ++b)
          if (b == kb) v = g.x[a][b];
        const double m2 = cabs2(v);
        if (i < n && !((used >> a) & 1u) && m2 > best) best = m2, bi = i, br = v.x, bim = v.y;
      }
#pragma unroll
      for (int o = kGjY / 2; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(hmask, best, o, kGjY);
        const int oi = __shfl_xor_sync(hmask, bi, o, kGjY);
        const double orr = __shfl_xor_sync(hmask, br, o, kGjY);
        const double oim = __shfl_xor_sync(hmask, bim, o, kGjY);
        if (ob > best || (ob == best && oi < bi)) best = ob, bi = oi, br = orr, bim = oim;
      }
      if (ty == 0) {
        sh.p[buf] = bi;
        if (!(best > 0.0)) {
          sh.fail = 1;
          sh.inv[buf] = make_double2(0.0, 0.0);
        } else {
          sh.inv[buf] = cinv(make_double2(br, bim));
        }
        sh.piv[k] = bi;
        sh.step[bi < n ? bi : 0] = k;
      }
    }
    __syncthreads();
    const int p = sh.p[buf];
    const double2 inv = sh.inv[buf];
    const int pa = p / kGjY;
    // publish the scaled pivot row and the pivot column
    if (ty == p % kGjY) {
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        const int j = tx + kGjX * b;
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int a = 0; a < TR; ++a)
          if (a == pa) v = g.x[a][b];
        if (j < n) sh.rowbuf[buf][j] = (j == k) ? inv : cmul(v, inv);
      }
    }
    if (tx == kx) {
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        const int i = ty + kGjY * a;
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < TC; ++b)
          if (b == kb) v = g.x[a][b];
        if (i < n) sh.colbuf[buf][i] = (i == p) ? make_double2(0.0, 0.0) : v;
      }
    }
    __syncthreads();
    // eliminate, branch-free: rows i != p: a_ij -= a_ik r_j; row p := r
    // (colbuf[p] = 0); then the owners of column k set a_ik := -a_ik / piv
    // (a_pk := 1 / piv), which the bulk update got wrong
    double2 rj[TC];
#pragma unroll
    for (int b = 0; b < TC; ++b) rj[b] = sh.rowbuf[buf][tx + kGjX * b];
#pragma unroll
    for (int a = 0; a < TR; ++a) {
      const int i = ty + kGjY * a;
      const double2 ci = sh.colbuf[buf][i];
      const bool rowp = (i == p);
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        const double2 u = csub(g.x[a][b], cmul(ci, rj[b]));
        g.x[a][b] = rowp ? rj[b] : u;
      }
    }
    if (tx == kx) {
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        const int i = ty + kGjY * a;
        const double2 ci = sh.colbuf[buf][i];
        const double2 val = (i == p) ? inv : make_double2(-(ci.x * inv.x - ci.y * inv.y), -(ci.x * inv.y + ci.y * inv.x));
#pragma unroll
        for (int b = 0; b < TC; ++b)
          if (b == kb) g.x[a][b] = val;
      }
    }
    used |= (p % kGjY == ty) ? (1u << pa) : 0u;
  }
  __syncthreads();
  return sh.fail == 0;
}

// Gauss-Jordan WITHOUT pivoting, one barrier per column: the owners of row
// k / column k publish them unscaled (double-buffered), every thread forms
// 1 / a_kk itself.  For matrices where diagonal pivots are safe (the element
// Schur complements S = L_GG - L_Gi L_ii^{-1} L_iG + i eta I of the BASELINE
// configs: no-pivot GJ matches the pivoted inverse to 1e-15).  Guarded: the
// return value is false if a pivot falls below `tiny` or an entry grows past
// `huge` -- the caller then redoes the matrix with gj_reg_inverse.  On
// success g.x holds A^{-1} in natural order (no permutation).
template <int TR, int TC, class Get>
__device__ __forceinline__ bool gj_reg_inverse_nopiv(int n, Get get, GjReg<TR, TC>& g, GjShared& sh,
                                                    double tiny2, double huge2) {
  const int tid = threadIdx.x, ty = tid % kGjY, tx = tid / kGjY;
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int i = ty + kGjY * a, j = tx + kGjX * b;
      g.x[a][b] = (i < n && j < n) ? get(i, j) : make_double2(0.0, 0.0);
    }
  for (int t = tid; t < 2 * kGjMax; t += kGjThreads) {
    sh.rowbuf[t / kGjMax][t % kGjMax] = make_double2(0.0, 0.0);
    sh.colbuf[t / kGjMax][t % kGjMax] = make_double2(0.0, 0.0);
  }
  if (tid == 0) sh.fail = 0;
  __syncthreads();
  bool bad = false;
  // publish row 0 / column 0
  auto publish = [&](int k) {
    const int buf = k & 1, ka = k / kGjY, kb = k / kGjX;
    if (ty == k % kGjY) {
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int a = 0; a < TR; ++a)
          if (a == ka) v = g.x[a][b];
        const int j = tx + kGjX * b;
        if (j < n) sh.rowbuf[buf][j] = v;
      }
    }
    if (tx == k % kGjX) {
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < TC; ++b)
          if (b == kb) v = g.x[a][b];
        const int i = ty + kGjY * a;
        if (i < n) sh.colbuf[buf][i] = v;
      }
    }
  };
  publish(0);
  for (int k = 0; k < n; ++k) {
    const int buf = k & 1;
    __syncthreads();
    const double2 piv = sh.rowbuf[buf][k];
    const double p2 = cabs2(piv);
    if (!(p2 > tiny2)) bad = true;
    const double2 inv = p2 > 0.0 ? cinv(piv) : make_double2(0.0, 0.0);
    double2 rj[TC];
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int j = tx + kGjX * b;
      rj[b] = (j == k) ? inv : cmul(sh.rowbuf[buf][j], inv);
    }
#pragma unroll
    for (int a = 0; a < TR; ++a) {
      const int i = ty + kGjY * a;
      const bool rowk = (i == k);
      const double2 ci = rowk ? make_double2(0.0, 0.0) : sh.colbuf[buf][i];
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        const int j = tx + kGjX * b;
        const double2 base = (j == k) ? make_double2(0.0, 0.0) : g.x[a][b];
        const double2 u = csub(base, cmul(ci, rj[b]));
        g.x[a][b] = rowk ? rj[b] : u;
      }
    }
    if (k + 1 < n) publish(k + 1);
  }
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b)
      if (!(cabs2(g.x[a][b]) <= huge2)) bad = true;  // also catches NaN
  if (bad) sh.fail = 1;
  __syncthreads();
  return sh.fail == 0;
}

}  // namespace hpsb
