// V-cycle level step for levels of many small / medium merges: one CTA per
// merge at a time (persistent over the level's merges), operators streamed
// through a CTA ring of shared-memory slots filled by TMA bulk copies
// (cp.async.bulk + mbarrier transaction counts) from a producer warp.
//
// The chain of multigrid.cpp:47-98 on one merge is four dependent GEMVs, so
// a CTA that loads a stage's operator, waits, reduces and synchronises
// before it can touch the next stage keeps little of the HBM stream in
// flight (cfg3 levels 1-5 ran at 2.3-4.0 TB/s).  The operators are static,
// so here the copies run ahead of the arithmetic: the producer warp walks
// the column pieces of every operator of every merge the CTA owns, in the
// order the chain consumes them, and refills a slot as soon as the consumer
// warps release it; the chain's data dependencies only gate the arithmetic.
// Consumer warps split a piece into row groups of 32 (one row per lane) x
// column groups; the column-group partial sums are reduced through shared
// memory at the end of each operator (two named barriers per operator).
//
// Operators in consumption order (contiguous columns of one operator per
// slot; strided sub-blocks are copied column by column):
//   down: T2_ss (x = r2)  -> t = r1 - T2_ss r2
//         W     (x = t)   -> x1 = W t                    -> out[in1s]
//         [T1_ps; T1_ss] (x = x1, one pass over the stored P1 x s column
//                block)   -> r[out1p] -= T1_ps x1,  x2 = r2 - T1_ss x1 -> out[in2s]
//         T2_ps (x = x2)  -> r[out2p] -= T2_ps x2
//   up:   T1_sp (x = u1)  -> b2 = T1_sp u1 (kept negated right behind u2)
//         [T2_sp, T2_ss] (x = [u2; -b2], one pass over the s x P2 row block)
//                         -> t = b1 - T2_ss b2
//         W     (x = t)   -> y1 = W t                    -> out[in1s] -= y1
//         T1_ss (x = y1)  -> out[in2s] += T1_ss y1 - b2
// Every operator byte is read once per step (3 s^2 + s (p1 + p2) entries).
#include <algorithm>
#include <type_traits>

#include "device.cuh"
#include "hierarchy.hpp"
#include "vcycle_device.cuh"
#include "vcycle_small.hpp"

namespace hpsb {

namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// One operator of a merge's step: src rows x cols (column-major, ld); x_off:
// offset of its input vector in the merge's vector scratch.
struct Op {
  const double2* src;
  int rows, cols, ld, x_off;
};

__device__ __forceinline__ Op merge_op(const SmallMerge& M, int down, int k) {
  const int s = M.s, p1 = M.p1, p2 = M.p2, P1 = M.P1, P2 = M.P2;
  if (down) {  // scratch r1 | r2 | t | x1 | x2
    switch (k) {
      case 0: return {M.T2 + p2 + static_cast<size_t>(p2) * P2, s, s, P2, s};          // T2_ss
      case 1: return {M.W, s, s, s, 2 * s};                                              // W
      case 2: return {M.T1 + static_cast<size_t>(p1) * P1, P1, s, P1, 3 * s};            // [T1_ps; T1_ss]
      default: return {M.T2 + static_cast<size_t>(p2) * P2, p2, p2 ? s : 0, P2, 4 * s};  // T2_ps
    }
  }
  switch (k) {  // scratch u1 | u2 | -b2 | t | y1
    case 0: return {M.T1 + p1, s, p1, P1, 0};                                            // T1_sp
    case 1: return {M.T2 + p2, s, P2, P2, p1};                                           // [T2_sp, T2_ss]
    case 2: return {M.W, s, s, s, p1 + p2 + s};                                          // W
    default: return {M.T1 + p1 + static_cast<size_t>(p1) * P1, s, s, P1, p1 + p2 + 2 * s};  // T1_ss
  }
}

__device__ __forceinline__ void bar_consumers(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

constexpr int kStreamMaxSlots = 8;

// CW consumer warps + 1 producer warp.  Ring: ns slots of slot_entries
// (+ 32 padding entries read by lanes past an operator's last row).
template <int CW>
__global__ void __launch_bounds__(32 * (CW + 1)) merge_stream_kernel(const SmallMerge* __restrict__ ms, int count,
                                                                     int down, double2* r, double2* out, int ns,
                                                                     int slot_entries, int vec_entries, int pre_out) {
  constexpr int U = 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot_stride = slot_entries + 32;
  double2* ring = reinterpret_cast<double2*>(smem_raw);
  double2* red = ring + static_cast<size_t>(ns) * slot_stride;  // [CW * 32]
  double2* vbuf = red + 32 * CW;  // two vector scratch areas (this merge / the next)
  unsigned long long* full = reinterpret_cast<unsigned long long*>(vbuf + 2 * vec_entries);
  unsigned long long* empty = full + kStreamMaxSlots;
  // No early launch_dependents: the dependents are scheduled when this grid
  // exits (an early trigger let them occupy the SMs while this persistent
  // grid still streams: cfg3 V-cycle 3.87 -> 4.44 ms).
  if (tid == 0) {
    for (int q = 0; q < ns; ++q) mbar_init(full + q, 1), mbar_init(empty + q, CW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CW) {
    // ---- producer warp: every piece of every merge of this CTA, in order
    // (operators are static: no PDL wait needed)
    unsigned q = 0;
    for (int m = blockIdx.x; m < count; m += gridDim.x) {
      const SmallMerge M = ms[m];
      for (int k = 0; k < 4; ++k) {
        const Op op = merge_op(M, down, k);
        const int ncp = op.rows ? max(1, slot_entries / op.rows) : 1;
        for (int c0 = 0; c0 < op.cols; c0 += ncp, ++q) {
          const int nc = min(ncp, op.cols - c0), slot = static_cast<int>(q % ns);
          if (q >= static_cast<unsigned>(ns)) mbar_wait(empty + slot, (q / ns - 1) & 1u);
          const unsigned bytes = static_cast<unsigned>(sizeof(double2) * op.rows * nc);
          if (lane == 0) mbar_expect_tx(full + slot, bytes);
          __syncwarp();
          double2* dst = ring + static_cast<size_t>(slot) * slot_stride;
          const double2* src = op.src + static_cast<size_t>(c0) * op.ld;
          if (op.ld == op.rows) {
            if (lane == 0) bulk_g2s(dst, src, bytes, full + slot);
          } else {
            const unsigned cb = static_cast<unsigned>(sizeof(double2) * op.rows);
            for (int j = lane; j < nc; j += 32)
              bulk_g2s(dst + static_cast<size_t>(j) * op.rows, src + static_cast<size_t>(j) * op.ld, cb, full + slot);
          }
        }
      }
    }
    return;
  }

  // ---- consumer warps
  // A merge's input vector (down r1 | r2, up u1 | u2) is gathered during the
  // previous merge: its indices are loaded at that merge's start and the
  // gathers issued as cp.async after its first operator, so neither L2
  // round trip sits on the chain.  (Same-level merges touch disjoint rows.)
  constexpr int NT = 32 * CW;
  pdl_wait();
  const double2* src = down ? r : out;
  // A merge's gathered rows, in scratch order: its inputs (down r1 | r2 at 0,
  // up u1 | u2 at 0) and the bases of its read-modify-write outputs (down
  // r[out1p] | r[out2p] at 5s, up out[in1s] | out[in2s] at p1 + p2 + 3s).
  auto gather_row = [&](const SmallMerge& X, int i, int& dst) -> int {
    const int s2 = X.s, q1 = X.p1, q2 = X.p2;
    if (down) {
      if (i < s2) return dst = i, X.in1s[i];
      if (i < 2 * s2) return dst = i, X.in2s[i - s2];
      if (i < 2 * s2 + q1) return dst = 5 * s2 + (i - 2 * s2), X.out1p[i - 2 * s2];
      return dst = 5 * s2 + q1 + (i - 2 * s2 - q1), X.out2p[i - 2 * s2 - q1];
    }
    if (i < q1) return dst = i, X.in1p[i];
    if (i < q1 + q2) return dst = i, X.in2p[i - q1];
    if (i < q1 + q2 + s2) return dst = q1 + q2 + 3 * s2 + (i - q1 - q2), X.in1s[i - q1 - q2];
    return dst = q1 + q2 + 4 * s2 + (i - q1 - q2 - s2), X.in2s[i - q1 - q2 - s2];
  };
  // (pre_out: the output bases too -- levels of small merges, where the extra
  // scratch does not shrink the ring; cfg3 levels 1-2 -8% / -4%, levels 4-6 +5%)
  auto n_gather = [&](const SmallMerge& X) { return pre_out ? 2 * X.s + X.p1 + X.p2 : (down ? 2 * X.s : X.p1 + X.p2); };
  auto zero_b2 = [&](const SmallMerge& X, double2* vv) {  // up without T1_sp: b2 = 0
    if (!down && X.p1 == 0)
      for (int i = tid; i < X.s; i += NT) vv[X.p1 + X.p2 + i] = make_double2(0.0, 0.0);
  };
  if (blockIdx.x < count) {  // the first merge's rows
    const SmallMerge& X = ms[blockIdx.x];
    const int ng = n_gather(X);
    for (int i = tid; i < ng; i += NT) {
      int dst;
      const int row = gather_row(X, i, dst);
      cp_async16(vbuf + dst, src + row);
    }
    cp_async_commit();
    zero_b2(X, vbuf);
  }
  unsigned q = 0;
  int it = 0;
  for (int m = blockIdx.x; m < count; m += gridDim.x, ++it) {
    const SmallMerge& M = ms[m];
    const int s = M.s, p1 = M.p1, p2 = M.p2;
    double2* v = vbuf + (it & 1) * vec_entries;
    double2* vn = vbuf + ((it + 1) & 1) * vec_entries;
    cp_async_wait_all();
    bar_consumers(NT);
    // next merge: row indices now (their loads overlap operator 0), gathers after it
    const int mn = m + gridDim.x;
    int pidx[2] = {-1, -1}, pdst[2] = {0, 0};
    if (mn < count) {
      const SmallMerge& X = ms[mn];
      const int ng = n_gather(X);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = tid + e * NT;
        if (i < ng) pidx[e] = gather_row(X, i, pdst[e]);
      }
      for (int i = tid + 2 * NT; i < ng; i += NT) {  // (beyond two per thread: issued now)
        int dst;
        const int row = gather_row(X, i, dst);
        cp_async16(vn + dst, src + row);
      }
    }
    for (int k = 0; k < 4; ++k) {
      const Op op = merge_op(M, down, k);
      if (op.cols == 0) continue;
      const int rows = op.rows, ncp = max(1, slot_entries / rows);
      const int RG = (rows + 31) >> 5, CG = CW / RG;
      const int rg = warp % RG, cg = warp / RG;
      const bool active = cg < CG;
      const double2* x = v + op.x_off;
      double2 acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = make_double2(0.0, 0.0);
      for (int c0 = 0; c0 < op.cols; c0 += ncp, ++q) {
        const int nc = min(ncp, op.cols - c0), slot = static_cast<int>(q % ns);
        mbar_wait(full + slot, (q / ns) & 1u);
        if (active) {
          const double2* A = ring + static_cast<size_t>(slot) * slot_stride + rg * 32 + lane;
          const double2* xp = x + c0;
          int c = cg;
          for (; c + (U - 1) * CG < nc; c += U * CG) {
#pragma unroll
            for (int u = 0; u < U; ++u) acc[u] = cfma(A[(c + u * CG) * rows], xp[c + u * CG], acc[u]);
          }
          for (; c < nc; c += CG) acc[0] = cfma(A[c * rows], xp[c], acc[0]);
        }
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads before the next TMA write
        if (lane == 0) mbar_arrive(empty + slot);
      }
      if (active) {
        double2 y = acc[0];
#pragma unroll
        for (int u = 1; u < U; ++u) y = cadd(y, acc[u]);
        red[cg * (RG * 32) + rg * 32 + lane] = y;
      }
      bar_consumers(NT);
      // reduce the column groups, then the chain's epilogue for stage k
      for (int i = tid; i < rows; i += NT) {
        double2 y = red[i];
        for (int g = 1; g < CG; ++g) y = cadd(y, red[g * (RG * 32) + i]);
        if (down) {
          double2 *r1 = v, *r2 = v + s, *t = v + 2 * s, *x1 = v + 3 * s, *x2 = v + 4 * s;
          if (k == 0) {
            t[i] = csub(r1[i], y);
          } else if (k == 1) {
            x1[i] = y;
            __stcg(out + M.in1s[i], y);
          } else if (k == 2) {
            if (i < p1) {
              double2* qp = r + M.out1p[i];
              __stcg(qp, csub(pre_out ? v[5 * s + i] : __ldcg(qp), y));
            } else {
              const double2 xv = csub(r2[i - p1], y);
              x2[i - p1] = xv;
              __stcg(out + M.in2s[i - p1], xv);
            }
          } else {
            double2* qp = r + M.out2p[i];
            __stcg(qp, csub(pre_out ? v[5 * s + p1 + i] : __ldcg(qp), y));
          }
        } else {
          double2 *nb2 = v + p1 + p2, *t = nb2 + s, *y1 = t + s;
          if (k == 0) {
            nb2[i] = make_double2(-y.x, -y.y);
          } else if (k == 1) {
            t[i] = y;
          } else if (k == 2) {
            y1[i] = y;
            double2* qp = out + M.in1s[i];
            __stcg(qp, csub(pre_out ? y1[s + i] : __ldcg(qp), y));  // base out[in1s] at p1 + p2 + 3s
          } else {
            double2* qp = out + M.in2s[i];
            __stcg(qp, cadd(pre_out ? y1[2 * s + i] : __ldcg(qp), cadd(y, nb2[i])));  // base at p1 + p2 + 4s
          }
        }
      }
      if (k == 0 || (k == 1 && pidx[0] != -2)) {  // after the first operator that ran
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (pidx[e] >= 0) cp_async16(vn + pdst[e], src + pidx[e]);
        cp_async_commit();
        if (mn < count) zero_b2(ms[mn], vn);
        pidx[0] = pidx[1] = -2;
      }
      bar_consumers(NT);
    }
    if (pidx[0] != -2) {  // (no operator ran)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (pidx[e] >= 0) cp_async16(vn + pdst[e], src + pidx[e]);
      cp_async_commit();
      if (mn < count) zero_b2(ms[mn], vn);
    }
  }
}

// Independent GEMVs y[yi] = x[yi] + A x[xi] (A contiguous rows x cols; an
// index < 0 reads zero / skips the row) -- the interface matvec over the
// element maps (block_matrix.cpp:23-31).  Persistent CTAs over the items, the
// producer warp streams each A through the TMA ring (contiguous bulk copies),
// the next item's gathered x is prefetched with cp.async while this item runs.
__device__ __forceinline__ void cp_async16z(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(valid ? 16 : 0));
}

template <int CW>
__global__ void __launch_bounds__(32 * (CW + 1)) gemv_stream_kernel(const GemvItem* __restrict__ items, int count,
                                                                    const double2* x, double2* y, int ns,
                                                                    int slot_entries, int xs_entries) {
  constexpr int U = 2, NT = 32 * CW;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot_stride = slot_entries + 32;
  double2* ring = reinterpret_cast<double2*>(smem_raw);
  double2* red = ring + static_cast<size_t>(ns) * slot_stride;  // [CW * 32]
  double2* xbuf = red + 32 * CW;                                 // [2][xs_entries]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(xbuf + 2 * xs_entries);
  unsigned long long* empty = full + kStreamMaxSlots;
  if (tid == 0) {
    for (int q = 0; q < ns; ++q) mbar_init(full + q, 1), mbar_init(empty + q, CW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == CW) {  // producer: the operators are static (no PDL wait)
    unsigned q = 0;
    for (int t = blockIdx.x; t < count; t += gridDim.x) {
      const GemvItem T = items[t];
      const int ncp = max(1, slot_entries / T.rows);
      for (int c0 = 0; c0 < T.cols; c0 += ncp, ++q) {
        const int nc = min(ncp, T.cols - c0), slot = static_cast<int>(q % ns);
        if (q >= static_cast<unsigned>(ns)) mbar_wait(empty + slot, (q / ns - 1) & 1u);
        const unsigned bytes = static_cast<unsigned>(sizeof(double2) * T.rows * nc);
        if (lane == 0) {
          mbar_expect_tx(full + slot, bytes);
          bulk_g2s(ring + static_cast<size_t>(slot) * slot_stride, T.A + static_cast<size_t>(c0) * T.rows, bytes,
                   full + slot);
        }
        __syncwarp();
      }
    }
    return;
  }
  pdl_wait();
  auto prefetch = [&](int t, double2* xb) {
    const GemvItem T = items[t];
    for (int c = tid; c < T.cols; c += NT) {
      const int i = T.xi[c];
      cp_async16z(xb + c, x + (i >= 0 ? i : 0), i >= 0);
    }
    cp_async_commit();
  };
  if (blockIdx.x < count) prefetch(blockIdx.x, xbuf);
  unsigned q = 0;
  int it = 0;
  for (int t = blockIdx.x; t < count; t += gridDim.x, ++it) {
    const GemvItem T = items[t];
    const double2* xs = xbuf + (it & 1) * xs_entries;
    cp_async_wait_all();
    bar_consumers(NT);
    if (t + static_cast<int>(gridDim.x) < count) prefetch(t + gridDim.x, xbuf + ((it + 1) & 1) * xs_entries);
    const int rows = T.rows, ncp = max(1, slot_entries / rows);
    const int RG = (rows + 31) >> 5, CG = CW / RG;
    const int rg = warp % RG, cg = warp / RG;
    const bool active = cg < CG;
    double2 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = make_double2(0.0, 0.0);
    for (int c0 = 0; c0 < T.cols; c0 += ncp, ++q) {
      const int nc = min(ncp, T.cols - c0), slot = static_cast<int>(q % ns);
      mbar_wait(full + slot, (q / ns) & 1u);
      if (active) {
        const double2* A = ring + static_cast<size_t>(slot) * slot_stride + rg * 32 + lane;
        const double2* xp = xs + c0;
        int c = cg;
        for (; c + (U - 1) * CG < nc; c += U * CG) {
#pragma unroll
          for (int u = 0; u < U; ++u) acc[u] = cfma(A[(c + u * CG) * rows], xp[c + u * CG], acc[u]);
        }
        for (; c < nc; c += CG) acc[0] = cfma(A[c * rows], xp[c], acc[0]);
      }
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads before the next TMA write
      if (lane == 0) mbar_arrive(empty + slot);
    }
    if (active) red[cg * (RG * 32) + rg * 32 + lane] = cadd(acc[0], acc[1]);
    bar_consumers(NT);
    for (int i = tid; i < rows; i += NT) {
      const int o = T.yi[i];
      if (o < 0) continue;
      double2 v = red[i];
      for (int g = 1; g < CG; ++g) v = cadd(v, red[g * (RG * 32) + i]);
      __stcg(y + o, cadd(__ldcg(x + o), v));
    }
  }
}

}  // namespace

StreamLevel::Shape stream_level_shape(int rows_max, int vec_in, int vec_all, int merges, int sms) {
  StreamLevel::Shape sh;
  if (rows_max > 512 || merges < sms) return sh;
  // one row group of 32 per consumer warp (and column groups on top): 4
  // consumer warps (rows <= 128) x 5 CTAs per SM, 8 x 4, or 16 x 2 -- several
  // merges in flight per SM hide each merge's per-operator barriers
  const int cw = rows_max <= 128 ? 4 : rows_max <= 256 ? 8 : 16;
  const int ctas_per_sm = cw == 4 ? 5 : cw == 8 ? 4 : 2;  // (measured: 4/3/2 -> 186.3 ms, 5/4/2 -> 184.9, 6/5/3 -> 194.4)
  sh.pre_out = cw == 4;
  const int vec = ((sh.pre_out ? vec_all : vec_in) + 7) & ~7;
  const size_t budget = (220u << 10) / ctas_per_sm;
  const size_t fixed = sizeof(double2) * (32 * static_cast<size_t>(cw) + 2 * static_cast<size_t>(vec)) +
                       2 * sizeof(unsigned long long) * kStreamMaxSlots;
  if (fixed >= budget) return sh;
  // ns slots of whole columns: 4 slots, each as large as the budget allows
  const int ns = 2;  // (cfg3 A/B: 4 / 3 / 2 slots -> solve 186.3 / 185.4 / 183.4 ms at 5 / 4 / 2 CTAs per SM)
  const int slot = static_cast<int>((budget - fixed) / (sizeof(double2) * ns)) - 32;
  if (slot < rows_max) return sh;
  sh.ok = true, sh.warps = cw, sh.ns = ns, sh.slot_entries = slot, sh.vec_entries = vec;
  sh.rpl = ctas_per_sm;
  sh.smem = fixed + sizeof(double2) * ns * (static_cast<size_t>(slot) + 32);
  return sh;
}

void StreamLevel::run(Context* ctx, bool down, double2* r, double2* out) const {
  if (!count) return;
  KernelScope ks(ctx, label.empty() ? (down ? "vcycle_down" : "vcycle_up") : label.c_str(),
                 down ? bytes_down : bytes_up, 0.0);
  const int ctas = std::max(1, std::min(ctx->num_sms * shape.rpl, count));
  auto go = [&](auto kern) {
    allow_smem<decltype(kern)::value>(shape.smem);
    launch_k(ctx, decltype(kern)::value, dim3(ctas), dim3(32 * (shape.warps + 1)), shape.smem, 1,
             static_cast<const SmallMerge*>(d.p), count, down ? 1 : 0, r, out, shape.ns, shape.slot_entries,
             shape.vec_entries, shape.pre_out ? 1 : 0);
  };
  if (shape.warps == 4) go(std::integral_constant<decltype(&merge_stream_kernel<4>), &merge_stream_kernel<4>>{});
  else if (shape.warps == 8) go(std::integral_constant<decltype(&merge_stream_kernel<8>), &merge_stream_kernel<8>>{});
  else go(std::integral_constant<decltype(&merge_stream_kernel<16>), &merge_stream_kernel<16>>{});
}

}  // namespace hpsb

namespace hpsb {

GemvStream::Shape gemv_stream_shape(int rows_max, int cols_max) {
  GemvStream::Shape sh;
  if (rows_max > 256 || rows_max < 1) return sh;
  sh.warps = 8;
  sh.ctas_per_sm = 4;  // (2 / 3 / 4 / 6 per SM: interface matvec 17.5 / 16.3 / 15.3 / 19.1 ms per cfg3 solve)
  const size_t budget = (220u << 10) / sh.ctas_per_sm;
  const int xs = (cols_max + 7) & ~7;
  const size_t fixed = sizeof(double2) * (32 * static_cast<size_t>(sh.warps) + 2 * static_cast<size_t>(xs)) +
                       2 * sizeof(unsigned long long) * kStreamMaxSlots;
  if (fixed >= budget) return sh;
  sh.ns = 4;
  sh.slot_entries = static_cast<int>((budget - fixed) / (sizeof(double2) * sh.ns)) - 32;
  if (sh.slot_entries < rows_max) return sh;
  sh.xs_entries = xs;
  sh.smem = fixed + sizeof(double2) * sh.ns * (static_cast<size_t>(sh.slot_entries) + 32);
  sh.ok = true;
  return sh;
}

void GemvStream::run(Context* ctx, const double2* x, double2* y) const {
  if (!count) return;
  KernelScope ks(ctx, label.c_str(), bytes, 0.0);
  const int ctas = std::max(1, std::min(ctx->num_sms * shape.ctas_per_sm, count));
  allow_smem<gemv_stream_kernel<8>>(shape.smem);
  launch_k(ctx, gemv_stream_kernel<8>, dim3(ctas), dim3(32 * (shape.warps + 1)), shape.smem, 1,
           static_cast<const GemvItem*>(d.p), count, x, y, shape.ns, shape.slot_entries, shape.xs_entries);
}

}  // namespace hpsb
