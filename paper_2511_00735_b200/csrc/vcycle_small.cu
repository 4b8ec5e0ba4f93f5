// Fused V-cycle step for small merges: one CTA per merge, operators in smem.
//
// For the low levels of the hierarchy a merge's operators are a few tens of
// KB, and the generic work-list execution is bound by the latency of its
// dependent GEMV chain (each item waits for the previous item's output in
// L2).  Here a CTA first issues ONE burst of cp.async copies for everything
// the step needs -- the [T_ps; T_ss] (down) or [T_sp, T_ss] (up) column /
// row blocks of both children (contiguous / 2-D slices of the stored
// [p | s]-permuted maps) and W -- together with the vector gathers, then runs
// the whole chain of multigrid.cpp:47-98 out of shared memory:
//   down: t = r1 - T2_ss r2, x1 = W t, x2 = r2 - T1_ss x1,
//         out[s] = (x1, x2), r[out_k,p] -= T_k,ps x_k
//   up:   b1 = T2_sp u2, b2 = T1_sp u1, t = b1 - T2_ss b2, y1 = W t,
//         out[s2] += T1_ss y1 - b2, out[s1] -= y1
#include <algorithm>

#include "device.cuh"
#include "hierarchy.hpp"
#include "vcycle_device.cuh"
#include "vcycle_small.hpp"

namespace hpsb {

namespace {
constexpr int kThreads = 256;

// One merge's step, whole CTA (shared by the per-level and the subtree kernels).
__device__ __forceinline__ void small_step(const SmallMerge& M, int down, double2* r, double2* out,
                                           unsigned char* smem_raw, double2* red) {
  const int tid = threadIdx.x, s = M.s, p1 = M.p1, p2 = M.p2, P1 = M.P1, P2 = M.P2;
  double2* A1 = reinterpret_cast<double2*>(smem_raw);
  double2* A2 = A1 + static_cast<size_t>(P1) * s;
  double2* Ws = A2 + static_cast<size_t>(P2) * s;
  double2* v1 = Ws + static_cast<size_t>(s) * s;
  double2* v2 = v1 + s;
  double2* t = v2 + s;
  double2* w1 = t + s;
  double2* u1 = w1 + s;
  double2* u2 = u1 + p1;
  pdl_trigger();

  // ---- one burst of asynchronous copies: operators (+ W); they never depend
  // on the vectors, so they are issued before the PDL wait
  // (overlapping the previous kernel's tail).
  if (down) {
    const double2* g1 = M.T1 + static_cast<size_t>(p1) * P1;  // [T1_ps; T1_ss], P1 x s
    const double2* g2 = M.T2 + static_cast<size_t>(p2) * P2;
    for (int k = tid; k < P1 * s; k += kThreads) cp_async16(A1 + k, g1 + k);
    for (int k = tid; k < P2 * s; k += kThreads) cp_async16(A2 + k, g2 + k);
  } else {
    for (int k = tid; k < s * P1; k += kThreads)  // [T1_sp, T1_ss], s x P1 (ld s)
      cp_async16(A1 + k, M.T1 + p1 + (k % s) + static_cast<size_t>(k / s) * P1);
    for (int k = tid; k < s * P2; k += kThreads)
      cp_async16(A2 + k, M.T2 + p2 + (k % s) + static_cast<size_t>(k / s) * P2);
  }
  for (int k = tid; k < s * s; k += kThreads) cp_async16(Ws + k, M.W + k);
  asm volatile("cp.async.commit_group;\n" ::);
  pdl_wait();
  // vector gathers overlap the copies
  if (down) {
    for (int k = tid; k < s; k += kThreads) {
      v1[k] = __ldcg(r + M.in1s[k]);
      v2[k] = __ldcg(r + M.in2s[k]);
    }
  } else {
    for (int k = tid; k < p1; k += kThreads) u1[k] = __ldcg(out + M.in1p[k]);
    for (int k = tid; k < p2; k += kThreads) u2[k] = __ldcg(out + M.in2p[k]);
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();

  if (down) {
    const double2 *T1ps = A1, *T1ss = A1 + p1, *T2ps = A2, *T2ss = A2 + p2;
    double2 y = smem_gemv<kThreads>(T2ss, P2, s, s, v2, red);  // t = v1 - T2_ss v2
    if (tid < s) t[tid] = csub(v1[tid], y);
    __syncthreads();
    y = smem_gemv<kThreads>(Ws, s, s, s, t, red);  // x1 = W t
    if (tid < s) {
      w1[tid] = y;
      __stcg(out + M.in1s[tid], y);
    }
    __syncthreads();
    y = smem_gemv<kThreads>(T1ss, P1, s, s, w1, red);  // x2 = v2 - T1_ss x1
    if (tid < s) {
      const double2 x2 = csub(v2[tid], y);
      t[tid] = x2;
      __stcg(out + M.in2s[tid], x2);
    }
    __syncthreads();
    for (int r0 = 0; r0 < p1; r0 += kThreads) {  // r[out1_p] -= T1_ps x1
      y = smem_gemv<kThreads>(T1ps + r0, P1, min(p1 - r0, kThreads), s, w1, red);
      if (tid < p1 - r0) {
        const int o = M.out1p[r0 + tid];
        __stcg(r + o, csub(__ldcg(r + o), y));
      }
    }
    for (int r0 = 0; r0 < p2; r0 += kThreads) {  // r[out2_p] -= T2_ps x2
      y = smem_gemv<kThreads>(T2ps + r0, P2, min(p2 - r0, kThreads), s, t, red);
      if (tid < p2 - r0) {
        const int o = M.out2p[r0 + tid];
        __stcg(r + o, csub(__ldcg(r + o), y));
      }
    }
  } else {
    const double2 *T1sp = A1, *T1ss = A1 + static_cast<size_t>(p1) * s, *T2sp = A2,
                  *T2ss = A2 + static_cast<size_t>(p2) * s;
    double2 b1 = smem_gemv<kThreads>(T2sp, s, s, p2, u2, red);  // b1 = T2_sp u2
    double2 b2 = smem_gemv<kThreads>(T1sp, s, s, p1, u1, red);  // b2 = T1_sp u1
    if (tid < s) v1[tid] = b1, v2[tid] = b2;
    __syncthreads();
    double2 y = smem_gemv<kThreads>(T2ss, s, s, s, v2, red);  // t = b1 - T2_ss b2
    if (tid < s) t[tid] = csub(v1[tid], y);
    __syncthreads();
    y = smem_gemv<kThreads>(Ws, s, s, s, t, red);  // y1 = W t
    if (tid < s) w1[tid] = y;
    __syncthreads();
    const double2 z = smem_gemv<kThreads>(T1ss, s, s, s, w1, red);  // T1_ss y1
    if (tid < s) {
      const int o2 = M.in2s[tid], o1 = M.in1s[tid];
      __stcg(out + o2, cadd(__ldcg(out + o2), csub(z, v2[tid])));
      __stcg(out + o1, csub(__ldcg(out + o1), w1[tid]));
    }
  }
}
__global__ void __launch_bounds__(kThreads) merge_small_kernel(const SmallMerge* __restrict__ ms,
                                                               int down, double2* r,
                                                               double2* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double2 red[kThreads];
  const SmallMerge M = ms[blockIdx.x];
  small_step(M, down, r, out, smem_raw, red);
}


// Multi-RHS variant: the same fused chain for R right-hand sides (vectors
// with RHS stride ld); every GEMV becomes a small GEMM on shared memory,
// Y (rows x R) = A (rows x K, ld lda) X (K x R, ld ldx), on the FP64 tensor
// cores: a warp owns 8-row x 16-column output tiles (two 8 x 8 fragments,
// complex = four real DMMAs each), k in steps of 4 straight from shared
// memory; rows, K and R are masked to the problem (merge sizes are multiples
// of N - 1).  The scalar version (one output per thread pass, two 16-byte
// shared-memory loads per complex FMA) stays for separators below 16 nodes,
// where the 8 x 16 tiles are mostly padding (cfg4 level 1, s = 11: 1.79 ms
// scalar, 2.24 ms DMMA; levels 2-3, s = 22: 5.06 -> 4.43 ms).  These levels
// remain bound by the per-merge latency chain at one or two CTAs per SM, not
// by the arithmetic.
__device__ __forceinline__ void sdmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
template <class F>
__device__ __forceinline__ void smem_gemm_scalar(const double2* A, int lda, int rows, int K,
                                                 const double2* X, int ldx, int R, F&& emit) {
  for (int idx = threadIdx.x; idx < rows * R; idx += kThreads) {
    const int r = idx % rows, b = idx / rows;
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < K; ++k) acc = cfma(A[r + k * lda], X[k + b * ldx], acc);
    emit(r, b, acc);
  }
}
template <class F>
__device__ __forceinline__ void smem_gemm_dmma(const double2* A, int lda, int rows, int K,
                                               const double2* X, int ldx, int R, F&& emit) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  const int nrt = (rows + 7) >> 3, nct = (R + 15) >> 4;
  const double2 zero = make_double2(0.0, 0.0);
  for (int unit = warp; unit < nrt * nct; unit += kThreads / 32) {
    const int rt = unit % nrt, ct = unit / nrt;
    const int row = 8 * rt + g, col0 = 16 * ct + g;
    double cr[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, ci[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int k0 = 0; k0 < K; k0 += 4) {
      const int k = k0 + t4;
      const bool kin = k < K;
      const double2 a = (kin && row < rows) ? A[row + k * lda] : zero;
      double2 b[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = (kin && col0 + 8 * j < R) ? X[k + (col0 + 8 * j) * ldx] : zero;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        sdmma(cr[j][0], cr[j][1], a.x, b[j].x);
        sdmma(ci[j][0], ci[j][1], a.x, b[j].y);
        sdmma(cr[j][0], cr[j][1], -a.y, b[j].y);
        sdmma(ci[j][0], ci[j][1], a.y, b[j].x);
      }
    }
    // fragment (g, t4) holds C[8 rt + g][16 ct + 8 j + 2 t4 + h]
    if (row < rows) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 16 * ct + 8 * j + 2 * t4 + h;
          if (col < R) emit(row, col, make_double2(cr[j][h], ci[j][h]));
        }
    }
  }
}

template <bool DMMA, class F>
__device__ __forceinline__ void smem_gemm_r(const double2* A, int lda, int rows, int K,
                                            const double2* X, int ldx, int R, F&& emit) {
  if (DMMA) smem_gemm_dmma(A, lda, rows, K, X, ldx, R, emit);
  else smem_gemm_scalar(A, lda, rows, K, X, ldx, R, emit);
}

template <bool DMMA>
__global__ void __launch_bounds__(kThreads) merge_small_batch_kernel(
    const SmallMerge* __restrict__ ms, int down, double2* r, double2* out, int R, int64_t ld) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SmallMerge M = ms[blockIdx.x];
  const int tid = threadIdx.x, s = M.s, p1 = M.p1, p2 = M.p2, P1 = M.P1, P2 = M.P2;
  double2* A1 = reinterpret_cast<double2*>(smem_raw);
  double2* A2 = A1 + static_cast<size_t>(P1) * s;
  double2* Ws = A2 + static_cast<size_t>(P2) * s;
  // Vectors (s x R each): down v1 v2 t w1; up v1 v2 and ONE perimeter buffer
  // ub (max(p1, p2, 2 s) x R) that holds u2, then u1, then t and w1 (u1 is
  // dead once b2 is formed).  Sized per direction, so the level fits two CTAs
  // per SM where the single layout fitted one (cfg4 level 3: 126 -> 92 / 98 KB).
  double2* v1 = Ws + static_cast<size_t>(s) * s;
  double2* v2 = v1 + static_cast<size_t>(s) * R;
  double2* ub = v2 + static_cast<size_t>(s) * R;
  double2* t = ub;
  double2* w1 = t + static_cast<size_t>(s) * R;
  pdl_trigger();
  if (down) {
    const double2* g1 = M.T1 + static_cast<size_t>(p1) * P1;
    const double2* g2 = M.T2 + static_cast<size_t>(p2) * P2;
    for (int k = tid; k < P1 * s; k += kThreads) cp_async16(A1 + k, g1 + k);
    for (int k = tid; k < P2 * s; k += kThreads) cp_async16(A2 + k, g2 + k);
  } else {
    for (int k = tid; k < s * P1; k += kThreads)
      cp_async16(A1 + k, M.T1 + p1 + (k % s) + static_cast<size_t>(k / s) * P1);
    for (int k = tid; k < s * P2; k += kThreads)
      cp_async16(A2 + k, M.T2 + p2 + (k % s) + static_cast<size_t>(k / s) * P2);
  }
  for (int k = tid; k < s * s; k += kThreads) cp_async16(Ws + k, M.W + k);
  cp_async_commit();
  pdl_wait();
  if (down) {
    for (int k = tid; k < s * R; k += kThreads) {
      const int i = k % s, b = k / s;
      v1[k] = __ldcg(r + b * ld + M.in1s[i]);
      v2[k] = __ldcg(r + b * ld + M.in2s[i]);
    }
  } else {
    for (int k = tid; k < p2 * R; k += kThreads)
      ub[k] = __ldcg(out + (k / p2) * ld + M.in2p[k % p2]);
  }
  cp_async_wait_all();
  __syncthreads();
  if (down) {
    const double2 *T1ps = A1, *T1ss = A1 + p1, *T2ps = A2, *T2ss = A2 + p2;
    // t = v1 - T2_ss v2
    smem_gemm_r<DMMA>(T2ss, P2, s, s, v2, s, R, [&](int i, int b, double2 y) {
      t[i + b * s] = csub(v1[i + b * s], y);
    });
    __syncthreads();
    // x1 = W t
    smem_gemm_r<DMMA>(Ws, s, s, s, t, s, R, [&](int i, int b, double2 y) {
      w1[i + b * s] = y;
      __stcg(out + b * ld + M.in1s[i], y);
    });
    __syncthreads();
    // x2 = v2 - T1_ss x1  (into t)
    smem_gemm_r<DMMA>(T1ss, P1, s, s, w1, s, R, [&](int i, int b, double2 y) {
      const double2 x2 = csub(v2[i + b * s], y);
      t[i + b * s] = x2;
      __stcg(out + b * ld + M.in2s[i], x2);
    });
    // r[out1_p] -= T1_ps x1 (independent of the x2 rows above)
    smem_gemm_r<DMMA>(T1ps, P1, p1, s, w1, s, R, [&](int i, int b, double2 y) {
      double2* q = r + b * ld + M.out1p[i];
      __stcg(q, csub(__ldcg(q), y));
    });
    __syncthreads();
    smem_gemm_r<DMMA>(T2ps, P2, p2, s, t, s, R, [&](int i, int b, double2 y) {
      double2* q = r + b * ld + M.out2p[i];
      __stcg(q, csub(__ldcg(q), y));
    });
  } else {
    const double2 *T1sp = A1, *T1ss = A1 + static_cast<size_t>(p1) * s, *T2sp = A2,
                  *T2ss = A2 + static_cast<size_t>(p2) * s;
    // b1 = T2_sp u2 (v1), then b2 = T1_sp u1 (v2), through the one buffer
    smem_gemm_r<DMMA>(T2sp, s, s, p2, ub, p2, R, [&](int i, int b, double2 y) { v1[i + b * s] = y; });
    __syncthreads();
    for (int k = tid; k < p1 * R; k += kThreads)
      ub[k] = __ldcg(out + (k / p1) * ld + M.in1p[k % p1]);
    __syncthreads();
    smem_gemm_r<DMMA>(T1sp, s, s, p1, ub, p1, R, [&](int i, int b, double2 y) { v2[i + b * s] = y; });
    __syncthreads();
    // t = b1 - T2_ss b2
    smem_gemm_r<DMMA>(T2ss, s, s, s, v2, s, R, [&](int i, int b, double2 y) {
      t[i + b * s] = csub(v1[i + b * s], y);
    });
    __syncthreads();
    // y1 = W t
    smem_gemm_r<DMMA>(Ws, s, s, s, t, s, R, [&](int i, int b, double2 y) { w1[i + b * s] = y; });
    __syncthreads();
    // out[s2] += T1_ss y1 - b2,  out[s1] -= y1
    smem_gemm_r<DMMA>(T1ss, s, s, s, w1, s, R, [&](int i, int b, double2 y) {
      double2* q2 = out + b * ld + M.in2s[i];
      __stcg(q2, cadd(__ldcg(q2), csub(y, v2[i + b * s])));
      double2* q1 = out + b * ld + M.in1s[i];
      __stcg(q1, csub(__ldcg(q1), w1[i + b * s]));
    });
  }
}
}  // namespace

// vector entries per right-hand side of one direction (see the kernel's layout)
size_t small_merge_batch_vec(int s, int p1, int p2, bool down) {
  return down ? 4 * static_cast<size_t>(s)
              : 2 * static_cast<size_t>(s) + std::max<size_t>(std::max(p1, p2), 2 * static_cast<size_t>(s));
}
size_t small_merge_batch_smem(int s, int p1, int p2, int R) {  // the larger direction
  const size_t P1 = p1 + s, P2 = p2 + s;
  return sizeof(double2) * ((P1 + P2 + s) * s +
                            static_cast<size_t>(R) * std::max(small_merge_batch_vec(s, p1, p2, true),
                                                              small_merge_batch_vec(s, p1, p2, false)));
}

void SmallLevel::run_batch(Context* ctx, bool down, double2* r, double2* out, int R, int64_t ld) const {
  if (!count) return;
  const size_t smem = batch_ops + sizeof(double2) * R * (down ? batch_vec_down : batch_vec_up);
  allow_smem<merge_small_batch_kernel<false>>(smem);
  allow_smem<merge_small_batch_kernel<true>>(smem);
  KernelScope ks(ctx, label.empty() ? (down ? "vcycle_down_batch" : "vcycle_up_batch") : label.c_str(),
                 down ? bytes_down : bytes_up, 0.0);
  if (max_s >= 16)
    launch_k(ctx, merge_small_batch_kernel<true>, dim3(count), dim3(kThreads), smem, 1,
             static_cast<const SmallMerge*>(d.p), down ? 1 : 0, r, out, R, ld);
  else
    launch_k(ctx, merge_small_batch_kernel<false>, dim3(count), dim3(kThreads), smem, 1,
             static_cast<const SmallMerge*>(d.p), down ? 1 : 0, r, out, R, ld);
}


size_t small_merge_smem(int s, int p1, int p2) {
  const size_t P1 = p1 + s, P2 = p2 + s;
  return sizeof(double2) * ((P1 + P2 + s) * s + 4 * static_cast<size_t>(s) + p1 + p2);
}

void SmallLevel::run(Context* ctx, bool down, double2* r, double2* out) const {
  if (!count) return;
  allow_smem<merge_small_kernel>(smem);
  KernelScope ks(ctx, label.empty() ? (down ? "vcycle_down" : "vcycle_up") : label.c_str(),
                 down ? bytes_down : bytes_up, 0.0);
  launch_k(ctx, merge_small_kernel, dim3(count), dim3(kThreads), smem, 1,
           static_cast<const SmallMerge*>(d.p), down ? 1 : 0, r, out);
}

}  // namespace hpsb
