// Device side of the GEMV work items (shared by the plan kernel and the fused
// coarse-solve kernel).
#pragma once

#include "device.cuh"
#include "internal.hpp"

namespace hpsb {

constexpr int kGemvThreads = 256;

// Rows per CTA when an item is split across a cluster of cs CTAs: 8 / 16 /
// multiple-of-32 blocks (the row-block shapes gemv_item_rows maps well).
__host__ __device__ __forceinline__ int cluster_chunk(int rows, int cs) {
  const int c = (rows + cs - 1) / cs;
  return c <= 8 ? 8 : c <= 16 ? 16 : (c + 31) & ~31;
}

__device__ __forceinline__ double2 ld_vec(const double2* base, const int* idx, int j) {
  if (idx) {
    const int k = __ldg(idx + j);
    return k >= 0 ? __ldcg(base + k) : make_double2(0.0, 0.0);
  }
  return __ldcg(base + j);
}

// Rows [rb, re) of item I:  y[yi] = beta y[yi] + gamma z[zi] + alpha A x[xi].
// x / z / y may be overridden (coarse solve: the Krylov vector of the step).
// xs: shared staging for x (>= I.cols), red: kGemvThreads shared double2.
// Latency matters as much as bandwidth here (a level is a chain of dependent
// items), so everything that does not depend on x -- the first four A
// columns of each thread, the output index and the z / y operands of the
// first row block -- is loaded before the barrier that publishes x.
// kSmemA: rows [rb, re) of A were staged in shared memory (As, ld lds) by the
// caller (cp.async issued before the kernel's PDL wait); the caller waits for
// its copies and synchronises the block before the first item.
template <bool kSmemA = false>
__device__ __forceinline__ void gemv_item_rows(const VItem& I, int rb, int re, const double2* x,
                                               const double2* z, double2* y, double2* xs,
                                               double2* red, const double2* As = nullptr,
                                               int lds = 0) {
  auto lda_ld = [](const double2* p) { return kSmemA ? *p : ldg2(p); };
  const int tid = threadIdx.x;
  if (I.A)
    for (int j = tid; j < I.cols; j += kGemvThreads) xs[j] = ld_vec(x, I.xi, j);
  bool first = true;
  for (int r0 = rb; r0 < re; r0 += kGemvThreads) {
    const int rows = min(re - r0, kGemvThreads);
    // 8 / 16-row blocks keep every lane busy (a warp then reads 4 / 2 column
    // segments of 128 / 256 B per load) for short row blocks.
    const int rpad = rows <= 8 ? 8 : rows <= 16 ? 16 : (rows + 31) & ~31;
    const int groups = kGemvThreads / rpad;
    const int r = tid % rpad, g = tid / rpad;
    const bool active = I.A && g < groups && r < rows;
    const double2* Ar = I.A ? (kSmemA ? As + (r0 - rb) + r : I.A + r0 + r) : nullptr;
    const size_t lda = kSmemA ? static_cast<size_t>(lds) : static_cast<size_t>(I.lda);
    double2 a_pre[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = g + q * groups;
      a_pre[q] = (active && j < I.cols) ? lda_ld(Ar + j * lda) : make_double2(0.0, 0.0);
    }
    int yk = -1;
    double2 zv = make_double2(0.0, 0.0), yv = make_double2(0.0, 0.0);
    if (tid < rows) {
      const int row = r0 + tid;
      yk = I.yi ? __ldg(I.yi + row) : row;
      if (yk >= 0) {
        if (I.gamma != 0.0) zv = ld_vec(z, I.zi, row);
        if (I.beta != 0.0) yv = __ldcg(y + yk);
      }
    }
    if (first) __syncthreads();  // xs published
    first = false;
    double2 acc = make_double2(0.0, 0.0);
    if (active) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = g + q * groups;
        if (j < I.cols) acc = cfma(a_pre[q], xs[j], acc);
      }
      int j = g + 4 * groups;
      // 8 independent 16-byte loads in flight per thread (Little's law:
      // ~35 KB in flight per SM are needed to cover HBM latency).
      double2 acc2 = make_double2(0.0, 0.0);
      for (; j + 7 * groups < I.cols; j += 8 * groups) {
        double2 a[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = lda_ld(Ar + (j + q * groups) * lda);
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          acc = cfma(a[q], xs[j + q * groups], acc);
          acc2 = cfma(a[q + 1], xs[j + (q + 1) * groups], acc2);
        }
      }
      acc = cadd(acc, acc2);
      for (; j + 3 * groups < I.cols; j += 4 * groups) {
        const double2 a0 = lda_ld(Ar + j * lda);
        const double2 a1 = lda_ld(Ar + (j + groups) * lda);
        const double2 a2 = lda_ld(Ar + (j + 2 * groups) * lda);
        const double2 a3 = lda_ld(Ar + (j + 3 * groups) * lda);
        acc = cfma(a0, xs[j], acc);
        acc = cfma(a1, xs[j + groups], acc);
        acc = cfma(a2, xs[j + 2 * groups], acc);
        acc = cfma(a3, xs[j + 3 * groups], acc);
      }
      for (; j < I.cols; j += groups) acc = cfma(lda_ld(Ar + j * lda), xs[j], acc);
    }
    red[tid] = acc;
    __syncthreads();
    if (tid < rows && yk >= 0) {
      double2 s = red[tid];
      for (int gg = 1; gg < groups; ++gg) s = cadd(s, red[tid + gg * rpad]);
      double2 v = cscale(s, I.alpha);
      if (I.gamma != 0.0) v = cadd(v, cscale(zv, I.gamma));
      if (I.beta != 0.0) v = cadd(v, cscale(yv, I.beta));
      __stcg(y + yk, v);
    }
    __syncthreads();
  }
  if (first) __syncthreads();
}

}  // namespace hpsb
