// K6: restarted flexible GMRES on the skeleton system.
//
// Follows gmres_driver (proj/src/krylov.cpp:45-178) in flexible mode: the
// same cycle / restart / breakdown / true-residual logic, complex Givens
// rotations and convergence test on |g_{j+1}| / ||b||.  The Arnoldi
// orthogonalisation is classical Gram-Schmidt applied twice (CGS2) instead of
// the reference's modified Gram-Schmidt + reorthogonalisation pass: the same
// two passes over the basis, but each pass is one batched dot kernel (V^H w)
// and one batched axpy, so it streams the basis twice per pass instead of
// 2(j+1) dependent dot/axpy launches.  The (restart+1) x restart Hessenberg
// matrix and the Givens rotations live on the host (a few KB); the vectors
// stay in HBM.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <complex>

#include "device.cuh"
#include "tma.cuh"
#include "internal.hpp"
#include "zgemv_batch.hpp"

namespace hpsb {

namespace {
constexpr int kRowsPerThread = 4;
constexpr int kThreads = 256;
constexpr int kRowsPerBlock = kThreads * kRowsPerThread;

// partial[b * ncols + i] = sum_{rows of block b} conj(V[k, i]) w[k]
__global__ void __launch_bounds__(kThreads) dots_kernel(const double2* __restrict__ V, int64_t ld,
                                                       int ncols, const double2* __restrict__ w,
                                                       int64_t n, double2* partial) {
  __shared__ double2 sh[kThreads / 32][104];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock;
  double2 wv[kRowsPerThread];
#pragma unroll
  for (int r = 0; r < kRowsPerThread; ++r) {
    const int64_t k = base + threadIdx.x + r * kThreads;
    wv[r] = k < n ? w[k] : make_double2(0.0, 0.0);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = 0; i < ncols; ++i) {
    const double2* Vi = V + i * ld;
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < kRowsPerThread; ++r) {
      const int64_t k = base + threadIdx.x + r * kThreads;
      if (k < n) acc = cfma_conj(ldg2(Vi + k), wv[r], acc);
    }
    acc.x = warp_sum(acc.x);
    acc.y = warp_sum(acc.y);
    if (lane == 0) sh[warp][i] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ncols; i += kThreads) {
    double2 s = make_double2(0.0, 0.0);
    for (int q = 0; q < kThreads / 32; ++q) s = cadd(s, sh[q][i]);
    partial[static_cast<int64_t>(blockIdx.x) * ncols + i] = s;
  }
}

// out[0..ncols) = V^H w in one launch: block b reduces rows
// [b*chunk, (b+1)*chunk) into partial[b*ncols + i]; the last block to finish
// (atomic ticket) sums the partials in fixed block order (deterministic).
__global__ void __launch_bounds__(kThreads) dots_fused_kernel(
    const double2* __restrict__ V, int64_t ld, int ncols, const double2* __restrict__ w,
    int64_t n, int64_t chunk, double2* partial, double2* out, unsigned* ticket) {
  __shared__ double2 sh[kThreads / 32][104];
  __shared__ bool last;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = 0; i < ncols; ++i) {
    const double2* Vi = V + i * ld;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t k = r0 + threadIdx.x; k < r1; k += kThreads)
      acc = cfma_conj(ldg2(Vi + k), __ldcg(w + k), acc);
    acc.x = warp_sum(acc.x);
    acc.y = warp_sum(acc.y);
    if (lane == 0) sh[warp][i] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ncols; i += kThreads) {
    double2 s = make_double2(0.0, 0.0);
    for (int q = 0; q < kThreads / 32; ++q) s = cadd(s, sh[q][i]);
    __stcg(partial + static_cast<int64_t>(blockIdx.x) * ncols + i, s);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = warp; i < ncols; i += kThreads / 32) {  // one warp per column (fixed order)
      double2 s = make_double2(0.0, 0.0);
      for (unsigned b = lane; b < gridDim.x; b += 32) s = cadd(s, __ldcg(partial + b * ncols + i));
      s.x = warp_sum(s.x);
      s.y = warp_sum(s.y);
      if (lane == 0) out[i] = s;
    }
  }
  if (threadIdx.x == 0) *ticket = 0;  // ready for the next launch (stream-ordered)
}

// One pass of CGS2 over the rows of a block (kOrthThreads x R rows per block,
// w's rows kept in registers):
//   kUpdate: w -= V h_upd (the previous pass's projection), written back;
//   then partial[b, i] = sum_rows conj(V[k, vdot + i]) w[k] for i < ncols,
//   or, with ncols == 0, partial[b, 0] = sum_rows |w[k]|^2.
// A modified Gram-Schmidt step is the same pass with one update column and
// one dot column (vdot = 1): w -= h_{i-1} V_{i-1}, then h_i = V_i^H w.
// With `fused`, the last block to finish (atomic ticket) sums the partials in
// fixed block order into out (deterministic); else reduce_kernel does.
constexpr int kOrthThreads = 128;
constexpr int kOrthMaxR = 8;
// Multi-RHS: blockIdx.y selects the right-hand side; its basis, vector,
// coefficients, partials and ticket sit at the given strides.
struct OrthStride {
  int64_t v = 0, w = 0, p = 0;
  int h = 0;
};
template <bool kUpdate>
__global__ void __launch_bounds__(kOrthThreads) orth_kernel(
    const double2* __restrict__ V, int64_t ld, int ncols, const double2* __restrict__ h_upd,
    int nupd, double2* w, int64_t n, int R, double2* partial, double2* out, unsigned* ticket,
    int fused, OrthStride bs, const int* jdev, int vdot, const int* __restrict__ rows) {
  __shared__ double2 sh[kOrthThreads / 32][104];
  __shared__ double2 hs[104];
  __shared__ bool last;
  pdl_trigger();
  pdl_wait();
  if (jdev) {  // device-driven cycle: nonzero counts mean "j + 1" (j from the device state)
    const int j1 = *jdev + 1;
    ncols = ncols ? j1 : 0;
    nupd = nupd ? j1 : 0;
  }
  {
    const int b = blockIdx.y;
    V += b * bs.v, w += b * bs.w, partial += b * bs.p, ticket += b;
    if (h_upd) h_upd += b * bs.h;
    out += b * bs.h;
  }
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kOrthThreads * R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (kUpdate) {
    for (int i = threadIdx.x; i < nupd; i += kOrthThreads) hs[i] = h_upd[i];
    __syncthreads();
  }
  // rows (sharded): compact row k is vector row rows[k], or -(rows[k] + 1)
  // for a row that is updated but left out of the dot products
  double2 wv[kOrthMaxR];
  int64_t kx[kOrthMaxR];
  bool cnt[kOrthMaxR];
#pragma unroll
  for (int r = 0; r < kOrthMaxR; ++r) {
    const int64_t kc = base + threadIdx.x + r * kOrthThreads;
    kx[r] = -1, cnt[r] = false;
    if (r < R && kc < n) {
      const int64_t rr = rows ? rows[kc] : kc;
      kx[r] = rr >= 0 ? rr : -rr - 1;
      cnt[r] = rr >= 0;
    }
    const int64_t k = kx[r];
    wv[r] = k >= 0 ? __ldcg(w + k) : make_double2(0.0, 0.0);
    if (kUpdate && k >= 0) {
      double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
      int i = 0;
      for (; i + 8 <= nupd; i += 8) {  // 8 independent loads in flight
        double2 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = ldg2(V + (i + q) * ld + k);
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          acc = cfma(hs[i + q], v[q], acc);
          acc2 = cfma(hs[i + q + 1], v[q + 1], acc2);
        }
      }
      for (; i < nupd; ++i) acc = cfma(hs[i], ldg2(V + i * ld + k), acc);
      wv[r] = csub(wv[r], cadd(acc, acc2));
      __stcg(w + k, wv[r]);
    }
  }
  const int nout = ncols > 0 ? ncols : 1;
  if (ncols == 0) {
    double a = 0.0;
#pragma unroll
    for (int r = 0; r < kOrthMaxR; ++r)
      if (cnt[r]) a += cabs2(wv[r]);
    a = warp_sum(a);
    if (lane == 0) sh[warp][0] = make_double2(a, 0.0);
  } else {
    // 8 columns at a time: all their loads are issued before any reduction.
    for (int i0 = 0; i0 < ncols; i0 += 8) {
      double2 acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = make_double2(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < kOrthMaxR; ++r) {
        const int64_t k = kx[r];
        if (cnt[r]) {
          double2 v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            v[q] = i0 + q < ncols ? ldg2(V + (vdot + i0 + q) * ld + k) : make_double2(0.0, 0.0);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = cfma_conj(v[q], wv[r], acc[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        acc[q].x = warp_sum(acc[q].x);
        acc[q].y = warp_sum(acc[q].y);
        if (lane == 0 && i0 + q < ncols) sh[warp][i0 + q] = acc[q];
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nout; i += kOrthThreads) {
    double2 s = make_double2(0.0, 0.0);
    for (int q = 0; q < kOrthThreads / 32; ++q) s = cadd(s, sh[q][i]);
    __stcg(partial + static_cast<int64_t>(blockIdx.x) * nout + i, s);
  }
  if (!fused) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // one warp per column: lanes stride over the blocks (loads in flight in
  // parallel), then a butterfly -- a fixed order, so still deterministic
  for (int i = warp; i < nout; i += kOrthThreads / 32) {
    double2 s = make_double2(0.0, 0.0);
    for (unsigned b = lane; b < gridDim.x; b += 32) s = cadd(s, __ldcg(partial + b * nout + i));
    s.x = warp_sum(s.x);
    s.y = warp_sum(s.y);
    if (lane == 0) out[i] = s;
  }
  if (threadIdx.x == 0) *ticket = 0;  // ready for the next launch (stream-ordered)
}

// One CGS2 pass as orth_kernel (single right-hand side, full-length rows),
// with V streamed by TMA bulk copies: a CTA owns kOsRows rows; a producer
// warp copies each needed column's row segment (8 KB) into a ring of
// shared-memory slots.  The update runs row-parallel (2 rows per thread, w in
// registers); the dot products column-parallel (a warp per column, lanes
// over the rows of w' kept in shared memory), so each column costs one warp
// reduction instead of one per warp.  The dots re-stream the columns, which
// the update just pulled through L2.  out: per-block partials (reduce_kernel).
// (orth_kernel at cfg3: 148 registers, 19% occupancy, 32-40% of DRAM
// bandwidth, long-scoreboard bound.)
constexpr int kOsRows = 512, kOsWarps = 8, kOsSlots = 8;
constexpr size_t kOsSmem = sizeof(double2) * (static_cast<size_t>(kOsSlots) * kOsRows + kOsRows) +
                           2 * kOsSlots * sizeof(unsigned long long);
template <bool kUpdate>
__global__ void __launch_bounds__(32 * (kOsWarps + 1)) orth_stream_kernel(
    const double2* __restrict__ V, int64_t ld, int ncols, const double2* __restrict__ h_upd, int nupd, double2* w,
    int64_t n, double2* partial, int vdot, OrthStride bs) {
  constexpr int NT = 32 * kOsWarps;
  {  // multi-RHS: blockIdx.y selects the right-hand side
    const int b = blockIdx.y;
    V += b * bs.v, w += b * bs.w, partial += b * bs.p;
    if (h_upd) h_upd += b * bs.h;
  }
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* ring = reinterpret_cast<double2*>(smem_raw);
  double2* wsm = ring + static_cast<size_t>(kOsSlots) * kOsRows;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(wsm + kOsRows);
  unsigned long long* empty = full + kOsSlots;
  __shared__ double2 hs[104];
  __shared__ double nsum[kOsWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kOsRows;
  const int rows = static_cast<int>(n - r0 < kOsRows ? n - r0 : kOsRows);
  const int nu = kUpdate ? nupd : 0;
  if (tid == 0) {
    for (int q = 0; q < kOsSlots; ++q) tma_mbar_init(full + q, 1), tma_mbar_init(empty + q, kOsWarps);
    tma_mbar_init_fence();
  }
  __syncthreads();
  pdl_trigger();
  if (warp == kOsWarps) {  // producer: update columns, then dot columns (V is static here)
    if (lane == 0) {
      const unsigned bytes = static_cast<unsigned>(sizeof(double2) * rows);
      for (int q = 0; q < nu + ncols; ++q) {
        const int slot = q % kOsSlots;
        if (q >= kOsSlots) tma_wait(empty + slot, (q / kOsSlots - 1) & 1u);
        const int col = q < nu ? q : vdot + (q - nu);
        tma_expect_tx(full + slot, bytes);
        tma_load(ring + static_cast<size_t>(slot) * kOsRows, V + static_cast<int64_t>(col) * ld + r0, bytes, full + slot);
      }
    }
    return;
  }
  pdl_wait();
  if (kUpdate)
    for (int i = tid; i < nu; i += NT) hs[i] = h_upd[i];
  double2 wr[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int rr = tid + e * NT;
    wr[e] = rr < rows ? __ldcg(w + r0 + rr) : make_double2(0.0, 0.0);
  }
  named_bar(1, NT);  // hs
  int q = 0;
  if (kUpdate) {
    for (; q < nu; ++q) {
      const int slot = q % kOsSlots;
      tma_wait(full + slot, (q / kOsSlots) & 1u);
      const double2* col = ring + static_cast<size_t>(slot) * kOsRows;
      const double2 h = hs[q];
#pragma unroll
      for (int e = 0; e < 2; ++e) wr[e] = csub(wr[e], cmul(h, col[tid + e * NT]));
      tma_release(empty + slot, lane);
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {  // (rows past the vector: stale slot entries, drop them)
      const int rr = tid + e * NT;
      if (rr < rows) __stcg(w + r0 + rr, wr[e]);
      else wr[e] = make_double2(0.0, 0.0);
    }
  }
  if (ncols == 0) {  // ||w||^2 partial
    double a = cabs2(wr[0]) + cabs2(wr[1]);
    a = warp_sum(a);
    if (lane == 0) nsum[warp] = a;
    named_bar(1, NT);
    if (tid == 0) {
      double t = 0.0;
      for (int k = 0; k < kOsWarps; ++k) t += nsum[k];
      partial[blockIdx.x] = make_double2(t, 0.0);
    }
    return;
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) wsm[tid + e * NT] = wr[e];  // rows >= rows hold zeros
  named_bar(1, NT);
  for (int i = 0; i < ncols; ++i, ++q) {
    const int slot = q % kOsSlots;
    tma_wait(full + slot, (q / kOsSlots) & 1u);
    if ((i % kOsWarps) == warp) {
      const double2* col = ring + static_cast<size_t>(slot) * kOsRows;
      double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
      for (int rr = lane; rr < rows; rr += 64) {
        acc = cfma_conj(col[rr], wsm[rr], acc);
        if (rr + 32 < rows) acc2 = cfma_conj(col[rr + 32], wsm[rr + 32], acc2);
      }
      acc = cadd(acc, acc2);
      acc.x = warp_sum(acc.x);
      acc.y = warp_sum(acc.y);
      if (lane == 0) partial[static_cast<int64_t>(blockIdx.x) * ncols + i] = acc;
    }
    tma_release(empty + slot, lane);
  }
}

// dst[b] = s[b] * src[b] for the R vectors of a block (strides ls / ld)
__global__ void scale_batch_kernel(const double2* __restrict__ src, int64_t ls,
                                   const double* __restrict__ s, double2* dst, int64_t ld, int64_t n) {
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.y;
  const double f = s[b];
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double2 v = src[b * ls + k];
    dst[b * ld + k] = make_double2(v.x * f, v.y * f);
  }
}

// w[b] += sum_i h[b][i] V[i][b] (V: column i of RHS b at V + i * ldc + b * n)
__global__ void __launch_bounds__(kThreads) axpy_batch_kernel(const double2* __restrict__ V,
                                                             int64_t ldc, int ncols,
                                                             const double2* __restrict__ h, int hs,
                                                             double2* w, int64_t n) {
  __shared__ double2 hv[104];
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.y;
  for (int i = threadIdx.x; i < ncols; i += blockDim.x) hv[i] = h[b * hs + i];
  __syncthreads();
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < ncols; ++i) acc = cfma(hv[i], ldg2(V + i * ldc + b * n + k), acc);
    w[b * n + k] = cadd(w[b * n + k], acc);
  }
}

// out[i] = sum_b partial[b * ncols + i]  (fixed order: deterministic)
__global__ void reduce_kernel(const double2* __restrict__ partial, int nblocks, int ncols,
                              double2* out, const int* jdev = nullptr) {
  pdl_trigger();
  pdl_wait();
  __shared__ double2 sh[256];
  if (jdev) ncols = ncols ? *jdev + 1 : 1;  // device-driven cycle (see orth_kernel)
  const int i = blockIdx.x;
  if (i >= ncols) return;
  double2 s = make_double2(0.0, 0.0);
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x)
    s = cadd(s, partial[static_cast<int64_t>(b) * ncols + i]);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = cadd(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[i] = sh[0];
}

// out[b * hstride + i] = sum_blk partial[b * pstride + blk * ncols + i]
// (multi-RHS partials of orth_stream_kernel; fixed order: deterministic)
__global__ void reduce_batch_kernel(const double2* __restrict__ partial, int64_t pstride, int nblocks, int ncols,
                                    double2* out, int hstride) {
  pdl_trigger();
  pdl_wait();
  __shared__ double2 sh[256];
  const int i = blockIdx.x, b = blockIdx.y;
  partial += b * pstride;
  double2 s = make_double2(0.0, 0.0);
  for (int k = threadIdx.x; k < nblocks; k += blockDim.x) s = cadd(s, partial[static_cast<int64_t>(k) * ncols + i]);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = cadd(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[b * hstride + i] = sh[0];
}

// w[k] += sign * sum_i h[i] V[k, i]
__global__ void __launch_bounds__(kThreads) axpy_kernel(const double2* __restrict__ V, int64_t ld,
                                                       int ncols, const double2* __restrict__ h,
                                                       double sign, double2* w, int64_t n) {
  pdl_trigger();
  pdl_wait();
  __shared__ double2 hs[104];
  for (int i = threadIdx.x; i < ncols; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < ncols; ++i) acc = cfma(hs[i], ldg2(V + i * ld + k), acc);
    w[k] = make_double2(w[k].x + sign * acc.x, w[k].y + sign * acc.y);
  }
}

__global__ void scale_kernel(const double2* __restrict__ src, double s, double2* dst, int64_t n) {
  pdl_trigger();
  pdl_wait();
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[k] = make_double2(src[k].x * s, src[k].y * s);
}

// r = b - y
__global__ void sub_kernel(const double2* __restrict__ b, const double2* __restrict__ y, double2* r,
                           int64_t n) {
  pdl_trigger();
  pdl_wait();
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    r[k] = csub(b[k], y[k]);
}

// ---------------------------------------------------------------- device-driven Arnoldi cycle
// One restart cycle of fgmres as a CUDA graph: a WHILE conditional node whose
// body is one Arnoldi step (preconditioner on a fixed input buffer, Z_j copy,
// interface matvec, the three CGS2 passes with the column count read from the
// device state, the Givens update, V_{j+1}).  The Givens update runs on the
// device and ends the loop exactly where the host loop would (krylov.cpp:
// 92-123: converged estimate, breakdown, restart length, max_iters), so a
// cycle needs no host round trip per iteration.
struct CycleState {
  int j, total, stop, pad;  // stop: 0 running, 1 converged estimate, 2 breakdown, 3 cycle end
  double bnorm, tol, inv_h, pad2;
};

__device__ void dev_make_givens(double2 a, double2 b, double& c, double2& s) {  // krylov.cpp:17-31
  c = 1.0;
  s = make_double2(0.0, 0.0);
  const double na = hypot(a.x, a.y), nb = hypot(b.x, b.y);
  if (nb == 0.0) return;
  const double r = hypot(na, nb);
  if (na == 0.0) {
    c = 0.0;
    s = make_double2(b.x / nb, -b.y / nb);
  } else {
    c = na / r;
    const double2 t = cmul(make_double2(a.x / na, a.y / na), make_double2(b.x, -b.y));
    s = make_double2(t.x / r, t.y / r);
  }
}
__device__ void dev_apply_givens(double c, double2 s, double2& a, double2& b) {  // krylov.cpp:33-37
  const double2 t = cadd(cscale(a, c), cmul(s, b));
  b = cadd(cmul(make_double2(-s.x, s.y), a), cscale(b, c));
  a = t;
}

__global__ void arn_init_kernel(CycleState* st, double2* gv, int restart, int total, double beta,
                                double bnorm, double tol) {
  pdl_trigger();
  pdl_wait();
  for (int i = threadIdx.x; i <= restart; i += blockDim.x) gv[i] = make_double2(i == 0 ? beta : 0.0, 0.0);
  if (threadIdx.x == 0) {
    st->j = 0, st->total = total, st->stop = 0;
    st->bnorm = bnorm, st->tol = tol, st->inv_h = 0.0;
  }
}

// dst_base[j] = src (j from the device state)
__global__ void arn_copy_col_kernel(const double2* __restrict__ src, double2* dst_base, int64_t n,
                                    const CycleState* st) {
  pdl_trigger();
  pdl_wait();
  double2* dst = dst_base + static_cast<int64_t>(st->j) * n;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[k] = src[k];
}

// Rows per thread cap of the multi-RHS CGS2 passes (cfg4: 8 and 2 measured
// equal, 5.2-5.3 TB/s).
constexpr int orth_rr_cap() { return kOrthMaxR; }

// Hessenberg column j from the CGS2 coefficients (h = h1 + h2, h_{j+1,j} =
// ||w||), previous rotations, the new rotation, the residual estimate and the
// loop decision -- the host loop body of fgmres (krylov.cpp:102-123).
__global__ void arn_givens_kernel(CycleState* st, const double2* __restrict__ hd, int R1, double2* H,
                                  double* rc, double2* rs, double2* gv, double* hist, int restart,
                                  int max_iters, cudaGraphConditionalHandle cond) {
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x != 0) return;
  const int j = st->j;
  double2* Hj = H + static_cast<size_t>(j) * R1;
  for (int i = 0; i <= j; ++i) Hj[i] = cadd(hd[i], hd[R1 + i]);
  const double hnext = sqrt(fmax(hd[2 * R1].x, 0.0));
  Hj[j + 1] = make_double2(hnext, 0.0);
  for (int i = 0; i < j; ++i) dev_apply_givens(rc[i], rs[i], Hj[i], Hj[i + 1]);
  double c;
  double2 sg;
  dev_make_givens(Hj[j], Hj[j + 1], c, sg);
  rc[j] = c, rs[j] = sg;
  dev_apply_givens(c, sg, Hj[j], Hj[j + 1]);
  dev_apply_givens(c, sg, gv[j], gv[j + 1]);
  const double rel = hypot(gv[j + 1].x, gv[j + 1].y) / st->bnorm;
  if (hist) hist[st->total] = rel;
  int stop = 0;
  if (hnext <= 1e-14 * st->bnorm) {
    stop = 2;
  } else {
    st->inv_h = 1.0 / hnext;
    if (rel <= st->tol) stop = 1;
  }
  const int jn = j + 1, tn = st->total + 1;
  if (!stop && (jn >= restart || tn >= max_iters)) stop = 3;
  st->j = jn, st->total = tn, st->stop = stop;
  cudaGraphSetConditional(cond, stop ? 0u : 1u);
}

// V_{j+1} = w / h_{j+1,j}, also into the preconditioner's fixed input buffer
__global__ void arn_scale_kernel(const double2* __restrict__ w, double2* Vbase, double2* vin, int64_t n,
                                 const CycleState* st) {
  pdl_trigger();
  pdl_wait();
  if (st->stop == 2) return;  // breakdown: no next basis vector (krylov.cpp:111-114)
  const double f = st->inv_h;
  double2* dst = Vbase + static_cast<int64_t>(st->j) * n;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double2 v = w[k];
    const double2 o = make_double2(v.x * f, v.y * f);
    dst[k] = o;
    vin[k] = o;
  }
}

using cd = std::complex<double>;

struct Givens {
  double c = 1.0;
  cd s{0.0, 0.0};
};
Givens make_givens(cd a, cd b) {  // krylov.cpp:17-31
  Givens g;
  const double na = std::abs(a), nb = std::abs(b);
  if (nb == 0.0) return g;
  const double r = std::hypot(na, nb);
  if (na == 0.0) {
    g.c = 0.0;
    g.s = std::conj(b) / nb;
  } else {
    g.c = na / r;
    g.s = (a / na) * std::conj(b) / r;
  }
  return g;
}
void apply_givens(const Givens& g, cd& a, cd& b) {  // krylov.cpp:33-37
  const cd t = g.c * a + g.s * b;
  b = -std::conj(g.s) * a + g.c * b;
  a = t;
}

// The orthogonalisation kernels keep their coefficients in shared memory
// (<= 104 columns per launch).  orth_any issues one logical pass over any
// number of columns as launches of at most kOrthChunk columns:
//   w -= V[0..nupd) h_upd, then out = V[vdot..vdot+ncols)^H w (ncols > 0) or
//   out[0] = ||w||^2 (ncols == 0).
// launch(Vbase, ncols, h_upd, nupd, out, vdot) is one kernel launch of that
// form; `scratch` receives the discarded norms of intermediate update chunks.
constexpr int kOrthChunk = 96;
template <class L>
void orth_any(L&& launch, const double2* V, int64_t ld, int ncols, const double2* h_upd, int nupd,
              double2* out, int vdot, double2* scratch) {
  if (ncols <= kOrthChunk && nupd <= kOrthChunk) {
    launch(V, ncols, h_upd, nupd, out, vdot);
    return;
  }
  for (int u0 = 0; u0 < nupd; u0 += kOrthChunk) {
    const int cu = std::min(kOrthChunk, nupd - u0);
    const bool last = u0 + cu >= nupd;
    launch(V + u0 * ld, 0, h_upd + u0, cu, (last && ncols == 0) ? out : scratch, 0);
  }
  if (ncols == 0 && nupd > 0) return;
  for (int d0 = 0; d0 < ncols; d0 += kOrthChunk)
    launch(V, std::min(kOrthChunk, ncols - d0), nullptr, 0, out + d0, vdot + d0);
}

struct Work {
  Context* ctx;
  int64_t n;
  int blocks;
  int64_t chunk;
  DevBuf<double2> partial, hdev;
  DevBuf<unsigned> ticket;
  // Sharded: the dot products run over this rank's rows (rows / on, see
  // Skeleton::dist_rows) and are summed over the ranks (one allreduce of the
  // few coefficients per pass); elementwise updates stay full length.
  const int* rows = nullptr;
  int64_t on = 0;
  bool sharded() const { return ctx->world() > 1; }
  explicit Work(Context* c, int64_t dim, int maxcols) : ctx(c), n(dim), on(dim) {
    blocks = static_cast<int>((dim + kRowsPerBlock - 1) / kRowsPerBlock);
    chunk = kRowsPerBlock;
    partial.alloc(static_cast<size_t>((dim + kOrthThreads - 1) / kOrthThreads + blocks) * maxcols);
    hdev.alloc(3 * static_cast<size_t>(maxcols) + 4);  // h1 | h2 | norm ... | scratch (last)
    ticket.alloc(1);
    HPSB_CUDA(cudaMemsetAsync(ticket.p, 0, sizeof(unsigned), c->stream));
  }
  int grid() const { return static_cast<int>(std::min<int64_t>((n + 255) / 256, 8 * ctx->num_sms)); }
  // rows per thread: enough blocks for ~2 per SM, at most kOrthMaxR
  // At most 2 rows per thread: the update-and-project pass reads each V row
  // twice, and with short row blocks the second read still hits L2 (cfg3:
  // R = 8 / 4 / 2 / 1 -> 27.9 / 25.6 / 23.1 / 28.7 ms of orthogonalisation).
  void orth_grid(int& R, int& nb) const {
    R = 1;
    while (R < 2 && (on + kOrthThreads * 2 * R - 1) / (kOrthThreads * 2 * R) >= 2 * ctx->num_sms)
      R *= 2;
    nb = static_cast<int>((on + kOrthThreads * R - 1) / (kOrthThreads * R));
  }
  void reserve(int maxcols) {  // partial sums for maxcols columns (before a graph capture)
    int R, nb;
    orth_grid(R, nb);
    if (static_cast<size_t>(nb) * maxcols > partial.n) partial.alloc(static_cast<size_t>(nb) * maxcols);
  }
  // One CGS2 pass (orth_kernel): optionally w -= V h_upd, then out = V^H w
  // (ncols > 0) or out[0] = ||w||^2 (ncols == 0).
  // any column count (orth_any); jdev (device-driven cycle) needs <= kOrthChunk
  void orth(const double2* V, int ncols, const double2* h_upd, int nupd, double2* w, double2* out,
            const int* jdev = nullptr, int maxcols = 0, int vdot = 0) {
    if (jdev) return orth1(V, ncols, h_upd, nupd, w, out, jdev, maxcols, vdot);
    orth_any([&](const double2* Vb, int nc, const double2* hu, int nu, double2* o, int vd) {
               orth1(Vb, nc, hu, nu, w, o, nullptr, 0, vd);
             },
             V, n, ncols, h_upd, nupd, out, vdot, hdev.p + hdev.n - 1);
  }
  void orth1(const double2* V, int ncols, const double2* h_upd, int nupd, double2* w, double2* out,
             const int* jdev, int maxcols, int vdot) {
    int R, nb;
    orth_grid(R, nb);
    // (device-driven: ncols / nupd are flags, the counts come from *jdev; the
    // launch is sized for maxcols columns)
    const int nout = jdev ? maxcols : (ncols > 0 ? ncols : 1);
    const bool fused = nb <= 4 * ctx->num_sms;
    if (static_cast<size_t>(nb) * nout > partial.n) partial.alloc(static_cast<size_t>(nb) * nout);
    KernelScope ks(ctx, "gmres_orth", 16.0 * n * (nout + nupd + (h_upd ? 2 : 1)),
                   8.0 * n * (ncols + nupd));
    if (!jdev && !rows && !sharded() && n >= 64LL * kOsRows) {
      const int nbs = static_cast<int>((n + kOsRows - 1) / kOsRows);
      if (static_cast<size_t>(nbs) * nout > partial.n) partial.alloc(static_cast<size_t>(nbs) * nout);
      allow_smem<orth_stream_kernel<true>>(kOsSmem);
      allow_smem<orth_stream_kernel<false>>(kOsSmem);
      if (h_upd)
        launch_k(ctx, orth_stream_kernel<true>, dim3(nbs), dim3(32 * (kOsWarps + 1)), kOsSmem, 1, V, n, ncols,
                 h_upd, nupd, w, n, partial.p, vdot, OrthStride{});
      else
        launch_k(ctx, orth_stream_kernel<false>, dim3(nbs), dim3(32 * (kOsWarps + 1)), kOsSmem, 1, V, n, ncols,
                 h_upd, nupd, w, n, partial.p, vdot, OrthStride{});
      launch_k(ctx, reduce_kernel, dim3(nout), dim3(256), 0, 1, static_cast<const double2*>(partial.p), nbs, nout,
               out, static_cast<const int*>(nullptr));
      return;
    }
    if (h_upd)
      launch_k(ctx, orth_kernel<true>, dim3(nb), dim3(kOrthThreads), 0, 1, V, n, ncols, h_upd, nupd,
               w, on, R, partial.p, out, ticket.p, fused ? 1 : 0, OrthStride{}, jdev, vdot, rows);
    else
      launch_k(ctx, orth_kernel<false>, dim3(nb), dim3(kOrthThreads), 0, 1, V, n, ncols, h_upd, nupd,
               w, on, R, partial.p, out, ticket.p, fused ? 1 : 0, OrthStride{}, jdev, vdot, rows);
    if (!fused)
      launch_k(ctx, reduce_kernel, dim3(nout), dim3(256), 0, 1,
               static_cast<const double2*>(partial.p), nb, jdev ? ncols : nout, out, jdev);
    if (sharded()) ctx->comm->allreduce_sum(out, nout, ctx);  // GMRES inner products (NCCL)
  }
  // out[0..ncols) = V^H w.  Short vectors: one launch (last-block reduction);
  // long vectors: many row blocks + a column-parallel reduce launch.
  void dots(const double2* V, int ncols, const double2* w, double2* out) {
    KernelScope ks(ctx, "gmres_dots", 16.0 * n * (ncols + 1), 8.0 * n * ncols);
    if (blocks <= 64) {
      dots_fused_kernel<<<blocks, kThreads, 0, ctx->stream>>>(V, n, ncols, w, n, chunk, partial.p,
                                                              out, ticket.p);
      HPSB_LAUNCHED(ctx);
    } else {
      dots_kernel<<<blocks, kThreads, 0, ctx->stream>>>(V, n, ncols, w, n, partial.p);
      HPSB_LAUNCHED(ctx);
      reduce_kernel<<<ncols, 256, 0, ctx->stream>>>(partial.p, blocks, ncols, out, nullptr);
      HPSB_LAUNCHED(ctx);
    }
  }
  void axpy(const double2* V, int ncols, const double2* h, double sign, double2* w) {
    KernelScope ks(ctx, "gmres_axpy", 16.0 * n * (ncols + 2), 8.0 * n * ncols);
    for (int c0 = 0; c0 < ncols; c0 += kOrthChunk)
      launch_k(ctx, axpy_kernel, dim3(grid()), dim3(kThreads), 0, 1, V + c0 * n, n,
               std::min(kOrthChunk, ncols - c0), h + c0, sign, w, n);
  }
  double norm(const double2* w) {
    if (sharded())
      orth1(w, 0, nullptr, 0, const_cast<double2*>(w), hdev.p, nullptr, 0, 0);
    else
      dots(w, 1, w, hdev.p);
    double2 v;
    HPSB_CUDA(cudaMemcpyAsync(&v, hdev.p, sizeof(v), cudaMemcpyDeviceToHost, ctx->stream));
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    return std::sqrt(std::max(v.x, 0.0));
  }
  void scale(const double2* src, double s, double2* dst) {
    KernelScope ks(ctx, "gmres_scale", 32.0 * n, 0.0);
    launch_k(ctx, scale_kernel, dim3(grid()), dim3(256), 0, 1, src, s, dst, n);
  }
  void sub(const double2* b, const double2* y, double2* r) {
    KernelScope ks(ctx, "gmres_sub", 48.0 * n, 0.0);
    launch_k(ctx, sub_kernel, dim3(grid()), dim3(256), 0, 1, b, y, r, n);
  }
};
}  // namespace

// The device-driven restart cycle (see arn_givens_kernel): buffers, the
// captured graph and the host copies of its outcome.
struct CycleGraph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  DevBuf<double2> vin, zout, Hd, rsd, gvd;
  DevBuf<double> rcd, histd;
  DevBuf<CycleState> st;
  CycleState hs{};
  std::vector<double2> Hh, gh;
  std::vector<double> hist_h;
  int R1 = 0;
  ~CycleGraph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
  void build(Context* ctx, Skeleton* sk, Precond* pc, Work& wk, double2* V, double2* Z, double2* w,
             int64_t n, int restart, int max_iters, bool record) {
    R1 = restart + 1;
    vin.alloc(n), zout.alloc(pc ? n : 0), Hd.alloc(static_cast<size_t>(R1) * restart);
    rsd.alloc(restart), gvd.alloc(R1), rcd.alloc(restart), st.alloc(1);
    histd.alloc(record ? max_iters : 0);
    Hh.resize(static_cast<size_t>(R1) * restart), gh.resize(R1), hist_h.resize(record ? max_iters : 0);
    wk.reserve(R1);
    HPSB_CUDA(cudaMemsetAsync(Hd.p, 0, Hd.bytes(), ctx->stream));
    HPSB_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle cond;
    HPSB_CUDA(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    HPSB_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    HPSB_CUDA(cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0,
                                            cudaStreamCaptureModeThreadLocal));
    bool ok = true;
    try {
      const int* jdev = reinterpret_cast<const int*>(st.p);
      const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 8 * ctx->num_sms));
      if (pc) {
        precond_apply(pc, vin.p, zout.p);
        launch_k(ctx, arn_copy_col_kernel, dim3(blocks), dim3(256), 0, 1,
                 static_cast<const double2*>(zout.p), Z, n, static_cast<const CycleState*>(st.p));
        skeleton_apply(sk, zout.p, w);
      } else {
        skeleton_apply(sk, vin.p, w);
      }
      double2* h1 = wk.hdev.p;
      double2* h2 = wk.hdev.p + R1;
      double2* nn = wk.hdev.p + 2 * R1;
      wk.orth(V, 1, nullptr, 0, w, h1, jdev, R1);  // h1 = V^H w
      wk.orth(V, 1, h1, 1, w, h2, jdev, R1);       // w -= V h1; h2 = V^H w
      wk.orth(V, 0, h2, 1, w, nn, jdev, R1);       // w -= V h2; nn = ||w||^2
      launch_k(ctx, arn_givens_kernel, dim3(1), dim3(32), 0, 1, st.p,
               static_cast<const double2*>(wk.hdev.p), R1, Hd.p, rcd.p, rsd.p, gvd.p,
               record ? histd.p : static_cast<double*>(nullptr), restart, max_iters, cond);
      launch_k(ctx, arn_scale_kernel, dim3(blocks), dim3(256), 0, 1, static_cast<const double2*>(w), V,
               vin.p, n, static_cast<const CycleState*>(st.p));
    } catch (...) {
      ok = false;
    }
    cudaGraph_t captured = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &captured);
    const cudaError_t ei = (ok && ec == cudaSuccess) ? cudaGraphInstantiate(&exec, graph, 0) : cudaErrorUnknown;
    if (std::getenv("HPSB_TRACE"))
      std::fprintf(stderr, "[hpsb cycle graph] capture %s (%s), instantiate %s\n", ok ? "ok" : "threw",
                   cudaGetErrorString(ec), cudaGetErrorString(ei));
    if (ei != cudaSuccess) {
      cudaGetLastError();  // clear; fall back to the host-driven loop
      if (exec) cudaGraphExecDestroy(exec);
      exec = nullptr;
    }
  }
  void run(Context* ctx, const double2* V0, int64_t n, int restart, int total, double beta, double bnorm,
           double tol) {
    zcopy(ctx, vin.p, V0, n);
    launch_k(ctx, arn_init_kernel, dim3(1), dim3(128), 0, 1, st.p, gvd.p, restart, total, beta, bnorm, tol);
    HPSB_CUDA(cudaGraphLaunch(exec, ctx->stream));
    HPSB_CUDA(cudaMemcpyAsync(&hs, st.p, sizeof(hs), cudaMemcpyDeviceToHost, ctx->stream));
    HPSB_CUDA(cudaMemcpyAsync(Hh.data(), Hd.p, Hd.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
    HPSB_CUDA(cudaMemcpyAsync(gh.data(), gvd.p, gvd.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
    if (histd.n)
      HPSB_CUDA(cudaMemcpyAsync(hist_h.data(), histd.p, histd.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
};

// right = true: gmres with a fixed right preconditioner (krylov.cpp:180-186):
// w = M P(V_j), and at the end of a cycle x += P(V y); else flexible GMRES
// (fgmres, krylov.cpp:188-192) storing Z_j = P(V_j) and x += Z y.
hpsb_status fgmres(Skeleton* sk, Precond* pc, const double2* rhs, double2* x,
                   const hpsb_krylov_config& cfg, hpsb_solve_report* rep, bool right) {
  if (cfg.restart < 1) throw InvalidArgument("gmres: restart must be >= 1");
  if (!(cfg.tol > 0.0 && cfg.tol < 1.0)) throw InvalidArgument("gmres: tol must lie in (0, 1)");
  if (cfg.max_iters < 1) throw InvalidArgument("gmres: max_iters must be >= 1");
  Context* ctx = sk->ctx;
  const int64_t n = sk->dim;
  const int restart = cfg.restart;
  *rep = hpsb_solve_report{};
  Work wk(ctx, n, restart + 2);
  const bool dist = ctx->world() > 1;  // sharded: distributed vectors (Skeleton::dist_rows)
  if (dist) wk.rows = sk->dist_rows.p, wk.on = sk->n_dist_rows;
  ctx->history.clear();
  DevBuf<double2> V(static_cast<size_t>(n) * (restart + 1));
  if (!pc) right = false;
  DevBuf<double2> Z(pc && !right ? static_cast<size_t>(n) * restart : 0);
  DevBuf<double2> w(n), tmp(n), pz(right ? n : 0), pu(right ? n : 0);
  if (pc) {
    rep->precond_memory = precond_memory(pc);
    rep->wall_build = precond_build_seconds(pc);
  }
  HPSB_CUDA(cudaEventRecord(ctx->ev[2], ctx->stream));
  HPSB_CUDA(cudaMemsetAsync(x, 0, sizeof(double2) * n, ctx->stream));
  const double bnorm = wk.norm(rhs);
  auto finish_time = [&] {
    HPSB_CUDA(cudaEventRecord(ctx->ev[3], ctx->stream));
    HPSB_CUDA(cudaEventSynchronize(ctx->ev[3]));
    float ms = 0;
    HPSB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]));
    rep->seconds = ms * 1e-3;
    rep->wall_solve = rep->seconds;
  };
  if (bnorm == 0.0) {
    rep->converged = 1;
    finish_time();
    return HPSB_OK;
  }
  auto true_residual = [&]() {
    skeleton_apply(sk, x, tmp.p, dist);
    wk.sub(rhs, tmp.p, tmp.p);
    return wk.norm(tmp.p) / bnorm;
  };
  std::vector<cd> H(static_cast<size_t>(restart + 1) * restart), gv(restart + 1);
  std::vector<Givens> rot(restart);
  std::vector<double2> hh(2 * (restart + 1) + 1);
  auto Hm = [&](int i, int j) -> cd& { return H[i + static_cast<size_t>(j) * (restart + 1)]; };
  int total = 0;
  bool converged = false;
  CycleGraph cg;
  // Opt-in (HPSB_CYCLE_GRAPH=1): measured equal to the host-driven loop at
  // cfg1 / cfg2 (191 vs 193 us per iteration at cfg1: the device, not the
  // per-iteration host round trip, is the bound) and the first graph in a
  // process costs ~60 ms of one-time setup.
  // reorthogonalize (KrylovConfig, krylov.hpp:19): two classical passes
  // (CGS2); off: the reference's single modified Gram-Schmidt pass.
  const bool reorth = cfg.reorthogonalize != 0;
  if (!ctx->profile && ctx->world() == 1 && (!pc || precond_graph_safe(pc)) && reorth && !right &&
      restart + 1 <= kOrthChunk && std::getenv("HPSB_CYCLE_GRAPH"))
    cg.build(ctx, sk, pc, wk, V.p, Z.p, w.p, n, restart, cfg.max_iters, cfg.record_history != 0);
  while (total < cfg.max_iters && !converged) {
    double beta;
    if (total == 0) {
      zcopy(ctx, tmp.p, rhs, n);
      beta = bnorm;
    } else {
      beta = true_residual() * bnorm;  // r0 = rhs - M x (krylov.cpp:72-73)
    }
    if (beta / bnorm <= cfg.tol) {
      converged = true;
      break;
    }
    wk.scale(tmp.p, 1.0 / beta, V.p);
    std::fill(gv.begin(), gv.end(), cd(0.0, 0.0));
    gv[0] = beta;
    int j = 0;
    bool breakdown = false;
    if (cg.exec) {
      // the whole cycle on the device (CycleGraph); read back its outcome
      const int t0 = total;
      cg.run(ctx, V.p, n, restart, total, beta, bnorm, cfg.tol);
      j = cg.hs.j, total = cg.hs.total, breakdown = cg.hs.stop == 2;
      for (int c = 0; c < j; ++c)
        for (int i = 0; i <= c + 1; ++i) {
          const double2 v = cg.Hh[i + static_cast<size_t>(c) * (restart + 1)];
          Hm(i, c) = cd(v.x, v.y);
        }
      for (int i = 0; i <= j; ++i) gv[i] = cd(cg.gh[i].x, cg.gh[i].y);
      if (cfg.record_history)
        for (int t = t0; t < total; ++t) ctx->history.push_back(cg.hist_h[t]);
    }
    for (; !cg.exec && j < restart && total < cfg.max_iters; ++j, ++total) {
      double2* Vj = V.p + static_cast<size_t>(j) * n;
      if (right) {
        precond_apply(pc, Vj, pz.p, dist);
        skeleton_apply(sk, pz.p, w.p, dist);
      } else if (pc) {
        double2* Zj = Z.p + static_cast<size_t>(j) * n;
        precond_apply(pc, Vj, Zj, dist);
        skeleton_apply(sk, Zj, w.p, dist);
      } else {
        skeleton_apply(sk, Vj, w.p, dist);
      }
      double2* h1 = wk.hdev.p;
      double2* h2 = wk.hdev.p + (j + 1);
      double2* nn = wk.hdev.p + 2 * (j + 1);
      if (reorth) {
        // CGS2: two passes of h = V^H w, w -= V h
        wk.orth(V.p, j + 1, nullptr, 0, w.p, h1);  // h1 = V^H w
        wk.orth(V.p, j + 1, h1, j + 1, w.p, h2);   // w -= V h1; h2 = V^H w
        wk.orth(V.p, 0, h2, j + 1, w.p, nn);       // w -= V h2; nn = ||w||^2
      } else {
        // single-pass modified Gram-Schmidt (krylov.cpp:98-102): h_i = V_i^H w,
        // w -= h_i V_i for i = 0..j in order, each step one pass over w
        HPSB_CUDA(cudaMemsetAsync(h2, 0, sizeof(double2) * (j + 1), ctx->stream));
        wk.orth(V.p, 1, nullptr, 0, w.p, h1);
        for (int i = 1; i <= j; ++i)
          wk.orth(V.p + static_cast<size_t>(i - 1) * n, 1, h1 + i - 1, 1, w.p, h1 + i, nullptr, 0, 1);
        wk.orth(V.p + static_cast<size_t>(j) * n, 0, h1 + j, 1, w.p, nn);
      }
      HPSB_CUDA(cudaMemcpyAsync(hh.data(), wk.hdev.p, sizeof(double2) * (2 * (j + 1) + 1),
                                cudaMemcpyDeviceToHost, ctx->stream));
      HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
      for (int i = 0; i <= j; ++i)
        Hm(i, j) = cd(hh[i].x + hh[j + 1 + i].x, hh[i].y + hh[j + 1 + i].y);
      const double hnext = std::sqrt(std::max(hh[2 * (j + 1)].x, 0.0));
      Hm(j + 1, j) = hnext;
      for (int i = 0; i < j; ++i) apply_givens(rot[i], Hm(i, j), Hm(i + 1, j));
      rot[j] = make_givens(Hm(j, j), Hm(j + 1, j));
      apply_givens(rot[j], Hm(j, j), Hm(j + 1, j));
      apply_givens(rot[j], gv[j], gv[j + 1]);
      const double rel = std::abs(gv[j + 1]) / bnorm;
      if (cfg.record_history) ctx->history.push_back(rel);
      if (hnext <= 1e-14 * bnorm) {
        breakdown = true;
        ++j;
        ++total;
        break;
      }
      wk.scale(w.p, 1.0 / hnext, V.p + static_cast<size_t>(j + 1) * n);
      if (rel <= cfg.tol) {
        ++j;
        ++total;
        break;
      }
    }
    if (j > 0) {
      std::vector<cd> y(j);
      for (int i = j - 1; i >= 0; --i) {
        cd s = gv[i];
        for (int k = i + 1; k < j; ++k) s -= Hm(i, k) * y[k];
        y[i] = s / Hm(i, i);
      }
      std::vector<double2> yd(j + 1);
      for (int i = 0; i < j; ++i) yd[i] = make_double2(y[i].real(), y[i].imag());
      yd[j] = make_double2(1.0, 0.0);
      HPSB_CUDA(cudaMemcpyAsync(wk.hdev.p, yd.data(), sizeof(double2) * (j + 1),
                                cudaMemcpyHostToDevice, ctx->stream));
      if (right) {  // x += P(V y)
        zfill(ctx, pu.p, n, make_double2(0.0, 0.0));
        wk.axpy(V.p, j, wk.hdev.p, 1.0, pu.p);
        precond_apply(pc, pu.p, pz.p, dist);
        wk.axpy(pz.p, 1, wk.hdev.p + j, 1.0, x);
      } else {
        wk.axpy(pc ? Z.p : V.p, j, wk.hdev.p, 1.0, x);
      }
      HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    if (cfg.record_history && j > 0) {
      // basis orthogonality over the cycle's first j basis vectors
      // (krylov.cpp:149-160): max | |<V_a, V_b>| - delta_ab |, b <= a
      std::vector<double2> g(j);
      for (int a = 0; a < j; ++a) {
        double2* Va = V.p + static_cast<size_t>(a) * n;
        wk.orth(V.p, a + 1, nullptr, 0, Va, wk.hdev.p);
        HPSB_CUDA(cudaMemcpyAsync(g.data(), wk.hdev.p, sizeof(double2) * (a + 1),
                                  cudaMemcpyDeviceToHost, ctx->stream));
        HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int b = 0; b <= a; ++b)
          rep->basis_orthogonality =
              std::max(rep->basis_orthogonality,
                       std::abs(std::hypot(g[b].x, g[b].y) - (a == b ? 1.0 : 0.0)));
      }
    }
    const double true_rel = true_residual();
    rep->final_residual = true_rel;
    if (true_rel <= cfg.tol) converged = true;
    if (breakdown && !converged) {
      finish_time();
      rep->iterations = total;
      throw std::runtime_error("gmres: numerical breakdown before convergence");
    }
  }
  rep->iterations = total;
  rep->final_residual = true_residual();
  rep->converged = rep->final_residual <= cfg.tol;
  if (dist) gather_distributed(sk, x);  // the ABI's x is the full vector on every rank
  finish_time();
  return rep->converged ? HPSB_OK : HPSB_NO_CONVERGENCE;
}


// ------------------------------------------------------------- multi-RHS
// R independent restarted FGMRES solves (gmres_driver per right-hand side,
// krylov.cpp:45-178) advanced in lockstep: each iteration applies the
// preconditioner and the interface operator to the R current basis vectors
// at once (multi-RHS DMMA GEMMs, zgemv_batch.cu) -- the operators stream
// once per iteration instead of R times.  The Arnoldi recurrences, Givens
// rotations, restarts and convergence tests stay per right-hand side and
// follow the single-RHS driver above exactly; a right-hand side that has
// converged (or finished its cycle) is frozen with zero basis vectors.
// Layout: basis column j of RHS b at V + (j * R + b) * n.
namespace {
hpsb_status fgmres_group(Skeleton* sk, Precond* pc, const double2* rhs, double2* x, int R,
                         const hpsb_krylov_config& cfg, hpsb_solve_report* reps);
}

// Device memory the stream-ordered pool can still hand out: free memory plus
// what the pool holds but does not use.
static size_t available_device_bytes(int device) {
  size_t fr = 0, tot = 0;
  HPSB_CUDA(cudaMemGetInfo(&fr, &tot));
  cudaMemPool_t pool;
  HPSB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t reserved = 0, used = 0;
  HPSB_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
  HPSB_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  return fr + static_cast<size_t>(reserved > used ? reserved - used : 0);
}

// Right-hand sides are solved in groups sized to the device memory: a group
// of G needs (2 restart + 4) G dim complex vectors (basis V, preconditioned
// basis Z, work vectors).
hpsb_status fgmres_batch(Skeleton* sk, Precond* pc, const double2* rhs, double2* x, int R,
                         const hpsb_krylov_config& cfg, hpsb_solve_report* reps) {
  if (R < 1 || R > kBatchMaxRhs) throw InvalidArgument("gmres: 1 <= nrhs <= 32");
  const int64_t n = sk->dim;
  const double per_rhs = 16.0 * n * (2.0 * std::max(cfg.restart, 1) + 4.0);
  const double avail = 0.85 * static_cast<double>(available_device_bytes(sk->ctx->device));
  int G = std::max(1, std::min(R, static_cast<int>(avail / per_rhs)));
  const int ngroups = (R + G - 1) / G;
  G = (R + ngroups - 1) / ngroups;  // balanced groups
  hpsb_status rc = HPSB_OK;
  double seconds = 0;
  for (int b0 = 0; b0 < R; b0 += G) {
    const int g = std::min(G, R - b0);
    const hpsb_status s = fgmres_group(sk, pc, rhs + static_cast<size_t>(b0) * n,
                                       x + static_cast<size_t>(b0) * n, g, cfg, reps + b0);
    seconds += reps[b0].seconds;
    if (s != HPSB_OK) rc = s;
  }
  for (int b = 0; b < R; ++b) reps[b].seconds = seconds;
  return rc;
}

namespace {
hpsb_status fgmres_group(Skeleton* sk, Precond* pc, const double2* rhs, double2* x, int R,
                         const hpsb_krylov_config& cfg, hpsb_solve_report* reps) {
  if (cfg.restart < 1) throw InvalidArgument("gmres: restart must be >= 1");
  if (!(cfg.tol > 0.0 && cfg.tol < 1.0)) throw InvalidArgument("gmres: tol must lie in (0, 1)");
  if (cfg.max_iters < 1) throw InvalidArgument("gmres: max_iters must be >= 1");
  if (R < 1 || R > kBatchMaxRhs) throw InvalidArgument("gmres: 1 <= nrhs <= 32");
  Context* ctx = sk->ctx;
  // Sharded: distributed vectors as the single-RHS driver (Skeleton::dist_rows;
  // the R columns' coefficients are summed over the ranks in one allreduce).
  const bool dist = ctx->world() > 1;
  const int* rows = dist ? sk->dist_rows.p : nullptr;
  const int64_t n = sk->dim, on = dist ? sk->n_dist_rows : sk->dim;
  DevBuf<double2> xch;
  const int restart = cfg.restart;
  const int hs = 2 * (restart + 2) + 1;  // per-RHS slots: h1 | h2 | nn (and y)
  const bool reorth = cfg.reorthogonalize != 0;  // CGS2, else single-pass MGS
  for (int b = 0; b < R; ++b) reps[b] = hpsb_solve_report{};
  DevBuf<double2> V(static_cast<size_t>(restart + 1) * R * n);
  DevBuf<double2> Z(pc ? static_cast<size_t>(restart) * R * n : 0);
  DevBuf<double2> w(static_cast<size_t>(R) * n), tmp(static_cast<size_t>(R) * n);
  DevBuf<double2> hdev(static_cast<size_t>(R) * hs);
  DevBuf<double> sdev(R);
  DevBuf<unsigned> tickets(R);
  HPSB_CUDA(cudaMemsetAsync(tickets.p, 0, sizeof(unsigned) * R, ctx->stream));
  int RR = 1;  // rows per thread of the orth kernel
  while (RR < orth_rr_cap() && (on + kOrthThreads * 2 * RR - 1) / (kOrthThreads * 2 * RR) >= 2 * ctx->num_sms)
    RR *= 2;
  const int nb = static_cast<int>((on + kOrthThreads * RR - 1) / (kOrthThreads * RR));
  const int64_t pstride = static_cast<int64_t>(nb) * (restart + 2);
  DevBuf<double2> partial(static_cast<size_t>(R) * pstride);
  // one CGS2 pass for all R: optional w -= V h_upd, then V^H w / ||w||^2
  auto orth1 = [&](int ncols, const double2* h_upd, int nupd, double2* wv, double2* out,
                   const double2* Vb, int vdot) {
    OrthStride st;
    st.v = n, st.w = n, st.p = pstride, st.h = hs;
    const int nout = ncols > 0 ? ncols : 1;
    KernelScope ks(ctx, "gmres_orth", 16.0 * n * R * (nout + nupd + (h_upd ? 2 : 1)),
                   8.0 * n * R * (ncols + nupd));
    const int nbs = static_cast<int>((n + kOsRows - 1) / kOsRows);
    if (!dist && n >= 64LL * kOsRows && static_cast<int64_t>(nbs) * nout <= pstride) {
      // TMA-streamed pass (as the single-RHS driver), a batched reduction
      allow_smem<orth_stream_kernel<true>>(kOsSmem);
      allow_smem<orth_stream_kernel<false>>(kOsSmem);
      st.p = pstride;
      if (h_upd)
        launch_k(ctx, orth_stream_kernel<true>, dim3(nbs, R), dim3(32 * (kOsWarps + 1)), kOsSmem, 1, Vb,
                 static_cast<int64_t>(R) * n, ncols, h_upd, nupd, wv, n, partial.p, vdot, st);
      else
        launch_k(ctx, orth_stream_kernel<false>, dim3(nbs, R), dim3(32 * (kOsWarps + 1)), kOsSmem, 1, Vb,
                 static_cast<int64_t>(R) * n, ncols, h_upd, nupd, wv, n, partial.p, vdot, st);
      launch_k(ctx, reduce_batch_kernel, dim3(nout, R), dim3(256), 0, 1, static_cast<const double2*>(partial.p),
               pstride, nbs, nout, out, hs);
      return;
    }
    if (h_upd)
      launch_k(ctx, orth_kernel<true>, dim3(nb, R), dim3(kOrthThreads), 0, 1,
               Vb, static_cast<int64_t>(R) * n, ncols, h_upd, nupd, wv, on,
               RR, partial.p, out, tickets.p, 1, st, static_cast<const int*>(nullptr), vdot, rows);
    else
      launch_k(ctx, orth_kernel<false>, dim3(nb, R), dim3(kOrthThreads), 0, 1,
               Vb, static_cast<int64_t>(R) * n, ncols, h_upd, nupd, wv, on,
               RR, partial.p, out, tickets.p, 1, st, static_cast<const int*>(nullptr), vdot, rows);
    if (dist) exchange_deltas(ctx, xch, {{out, nullptr, nout, R, hs, 0}});  // NCCL allreduce
  };
  auto orth = [&](int ncols, const double2* h_upd, int nupd, double2* wv, double2* out,
                  const double2* Vb, int vdot) {
    orth_any([&](const double2* V0, int nc, const double2* hu, int nu, double2* o, int vd) {
               orth1(nc, hu, nu, wv, o, V0, vd);
             },
             Vb, static_cast<int64_t>(R) * n, ncols, h_upd, nupd, out, vdot, hdev.p + hs - 1);
  };
  const int vblocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 2 * ctx->num_sms));
  auto scale = [&](const double2* src, int64_t ls, const std::vector<double>& f, double2* dst, int64_t ld) {
    HPSB_CUDA(cudaMemcpyAsync(sdev.p, f.data(), sizeof(double) * R, cudaMemcpyHostToDevice, ctx->stream));
    KernelScope ks(ctx, "gmres_scale", 32.0 * n * R, 0.0);
    launch_k(ctx, scale_batch_kernel, dim3(vblocks, R), dim3(256), 0, 1, src, ls,
             static_cast<const double*>(sdev.p), dst, ld, n);
  };
  std::vector<double2> hh(static_cast<size_t>(R) * hs);
  auto norms = [&](double2* vecs, std::vector<double>& out) {  // ||vecs[b]|| for all b
    orth(0, nullptr, 0, vecs, hdev.p, V.p, 0);
    HPSB_CUDA(cudaMemcpyAsync(hh.data(), hdev.p, sizeof(double2) * R * hs, cudaMemcpyDeviceToHost,
                              ctx->stream));
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    out.resize(R);
    for (int b = 0; b < R; ++b) out[b] = std::sqrt(std::max(hh[static_cast<size_t>(b) * hs].x, 0.0));
  };
  HPSB_CUDA(cudaEventRecord(ctx->ev[2], ctx->stream));
  HPSB_CUDA(cudaMemsetAsync(x, 0, sizeof(double2) * R * n, ctx->stream));
  std::vector<double> bnorm, beta(R, 0.0), rel(R, 0.0), fac(R, 0.0);
  HPSB_CUDA(cudaMemcpyAsync(tmp.p, rhs, sizeof(double2) * R * n, cudaMemcpyDeviceToDevice, ctx->stream));
  norms(tmp.p, bnorm);
  auto true_residual = [&](std::vector<double>& out) {  // ||rhs - M x|| / ||rhs||
    skeleton_apply_batch(sk, x, tmp.p, R, dist);
    {
      KernelScope ks(ctx, "gmres_sub", 48.0 * n * R, 0.0);
      launch_k(ctx, sub_kernel, dim3(vblocks), dim3(256), 0, 1, rhs, static_cast<const double2*>(tmp.p),
               tmp.p, static_cast<int64_t>(R) * n);
    }
    norms(tmp.p, out);
    for (int b = 0; b < R; ++b) out[b] = bnorm[b] > 0.0 ? out[b] / bnorm[b] : 0.0;
  };
  std::vector<char> active(R), breakdown(R, 0), in_cycle(R);
  std::vector<int> total(R, 0), jlen(R, 0);
  for (int b = 0; b < R; ++b) {
    active[b] = bnorm[b] > 0.0;
    if (!active[b]) reps[b].converged = 1;
  }
  const int ldh = restart + 1;
  std::vector<std::vector<cd>> H(R, std::vector<cd>(static_cast<size_t>(ldh) * restart)),
      gv(R, std::vector<cd>(restart + 1));
  std::vector<std::vector<Givens>> rot(R, std::vector<Givens>(restart));
  bool first = true;
  auto any = [&](const std::vector<char>& f) {
    for (char c : f)
      if (c) return true;
    return false;
  };
  while (any(active)) {
    std::vector<double> res;
    if (first) {
      beta = bnorm;  // tmp = rhs
    } else {
      true_residual(res);
      for (int b = 0; b < R; ++b) beta[b] = res[b] * bnorm[b];
    }
    first = false;
    for (int b = 0; b < R; ++b)
      if (active[b] && (beta[b] / bnorm[b] <= cfg.tol || total[b] >= cfg.max_iters)) active[b] = 0;
    if (!any(active)) break;
    for (int b = 0; b < R; ++b) {
      fac[b] = active[b] ? 1.0 / beta[b] : 0.0;
      in_cycle[b] = active[b];
      jlen[b] = 0;
      std::fill(gv[b].begin(), gv[b].end(), cd(0.0, 0.0));
      gv[b][0] = beta[b];
    }
    scale(tmp.p, n, fac, V.p, n);
    for (int j = 0; j < restart && any(in_cycle); ++j) {
      double2* Vj = V.p + static_cast<size_t>(j) * R * n;
      double2* src = Vj;
      if (pc) {
        src = Z.p + static_cast<size_t>(j) * R * n;
        precond_apply_batch(pc, Vj, src, R, dist);
      }
      skeleton_apply_batch(sk, src, w.p, R, dist);
      if (reorth) {
        orth(j + 1, nullptr, 0, w.p, hdev.p, V.p, 0);                       // h1 = V^H w
        orth(j + 1, hdev.p, j + 1, w.p, hdev.p + (j + 1), V.p, 0);          // w -= V h1; h2 = V^H w
        orth(0, hdev.p + (j + 1), j + 1, w.p, hdev.p + 2 * (j + 1), V.p, 0);  // w -= V h2; ||w||^2
      } else {  // single-pass MGS, as the single-RHS driver
        HPSB_CUDA(cudaMemsetAsync(hdev.p, 0, hdev.bytes(), ctx->stream));
        orth(1, nullptr, 0, w.p, hdev.p, V.p, 0);
        for (int i = 1; i <= j; ++i)
          orth(1, hdev.p + i - 1, 1, w.p, hdev.p + i, V.p + static_cast<size_t>(i - 1) * R * n, 1);
        orth(0, hdev.p + j, 1, w.p, hdev.p + 2 * (j + 1), V.p + static_cast<size_t>(j) * R * n, 0);
      }
      HPSB_CUDA(cudaMemcpyAsync(hh.data(), hdev.p, sizeof(double2) * R * hs, cudaMemcpyDeviceToHost,
                                ctx->stream));
      HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
      for (int b = 0; b < R; ++b) {
        fac[b] = 0.0;
        if (!in_cycle[b]) continue;
        const double2* hb = hh.data() + static_cast<size_t>(b) * hs;
        auto Hm = [&](int i, int c) -> cd& { return H[b][i + static_cast<size_t>(c) * ldh]; };
        for (int i = 0; i <= j; ++i) Hm(i, j) = cd(hb[i].x + hb[j + 1 + i].x, hb[i].y + hb[j + 1 + i].y);
        const double hnext = std::sqrt(std::max(hb[2 * (j + 1)].x, 0.0));
        Hm(j + 1, j) = hnext;
        for (int i = 0; i < j; ++i) apply_givens(rot[b][i], Hm(i, j), Hm(i + 1, j));
        rot[b][j] = make_givens(Hm(j, j), Hm(j + 1, j));
        apply_givens(rot[b][j], Hm(j, j), Hm(j + 1, j));
        apply_givens(rot[b][j], gv[b][j], gv[b][j + 1]);
        rel[b] = std::abs(gv[b][j + 1]) / bnorm[b];
        ++total[b];
        jlen[b] = j + 1;
        if (hnext <= 1e-14 * bnorm[b]) {
          breakdown[b] = 1;
          in_cycle[b] = 0;
          continue;
        }
        fac[b] = 1.0 / hnext;
        if (rel[b] <= cfg.tol || total[b] >= cfg.max_iters) in_cycle[b] = 0;
      }
      if (j + 1 < restart + 1) scale(w.p, n, fac, V.p + static_cast<size_t>(j + 1) * R * n, n);
    }
    // x[b] += Z[b] y[b] (V[b] y[b] without preconditioner), y from H[b] y = g[b]
    int jmax = 0;
    std::vector<double2> yd(static_cast<size_t>(R) * hs, make_double2(0.0, 0.0));
    for (int b = 0; b < R; ++b) {
      const int j = active[b] ? jlen[b] : 0;
      jmax = std::max(jmax, j);
      std::vector<cd> y(j);
      for (int i = j - 1; i >= 0; --i) {
        cd sacc = gv[b][i];
        for (int k = i + 1; k < j; ++k) sacc -= H[b][i + static_cast<size_t>(k) * ldh] * y[k];
        y[i] = sacc / H[b][i + static_cast<size_t>(i) * ldh];
      }
      for (int i = 0; i < j; ++i) yd[static_cast<size_t>(b) * hs + i] = make_double2(y[i].real(), y[i].imag());
    }
    if (jmax > 0) {
      HPSB_CUDA(cudaMemcpyAsync(hdev.p, yd.data(), sizeof(double2) * R * hs, cudaMemcpyHostToDevice,
                                ctx->stream));
      KernelScope ks(ctx, "gmres_axpy", 16.0 * n * R * (jmax + 2), 8.0 * n * R * jmax);
      for (int c0 = 0; c0 < jmax; c0 += kOrthChunk)
        launch_k(ctx, axpy_batch_kernel, dim3(vblocks, R), dim3(kThreads), 0, 1,
                 static_cast<const double2*>(pc ? Z.p : V.p) + static_cast<size_t>(c0) * R * n,
                 static_cast<int64_t>(R) * n, std::min(kOrthChunk, jmax - c0),
                 static_cast<const double2*>(hdev.p) + c0, hs, x, n);
    }
    true_residual(res);
    for (int b = 0; b < R; ++b) {
      if (!active[b]) continue;
      reps[b].final_residual = res[b];
      if (res[b] <= cfg.tol) active[b] = 0;
      if (breakdown[b] && active[b]) {
        HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
        throw std::runtime_error("gmres: numerical breakdown before convergence (rhs " +
                                 std::to_string(b) + ")");
      }
    }
  }
  std::vector<double> fin;
  true_residual(fin);
  if (dist) gather_distributed(sk, x, R);  // full solutions on every rank
  HPSB_CUDA(cudaEventRecord(ctx->ev[3], ctx->stream));
  HPSB_CUDA(cudaEventSynchronize(ctx->ev[3]));
  float ms = 0;
  HPSB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]));
  bool all = true;
  for (int b = 0; b < R; ++b) {
    reps[b].iterations = total[b];
    reps[b].final_residual = fin[b];
    reps[b].converged = fin[b] <= cfg.tol;
    reps[b].seconds = ms * 1e-3;
    all = all && reps[b].converged;
  }
  return all ? HPSB_OK : HPSB_NO_CONVERGENCE;
}
}  // namespace

}  // namespace hpsb
