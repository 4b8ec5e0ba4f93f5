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
                                                                     int slot_entries, int vec_entries) {
  constexpr int U = 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot_stride = slot_entries + 32;
  double2* ring = reinterpret_cast<double2*>(smem_raw);
  double2* red = ring + static_cast<size_t>(ns) * slot_stride;  // [CW * 32]
  double2* v = red + 32 * CW;                                    // vector scratch
  unsigned long long* full = reinterpret_cast<unsigned long long*>(v + vec_entries);
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
  constexpr int NT = 32 * CW;
  pdl_wait();
  unsigned q = 0;
  for (int m = blockIdx.x; m < count; m += gridDim.x) {
    const SmallMerge& M = ms[m];
    const int s = M.s, p1 = M.p1, p2 = M.p2;
    if (down) {
      const int *i1 = M.in1s, *i2 = M.in2s;
      for (int i = tid; i < s; i += NT) {
        v[i] = __ldcg(r + i1[i]);
        v[s + i] = __ldcg(r + i2[i]);
      }
    } else {
      const int *i1 = M.in1p, *i2 = M.in2p;
      for (int i = tid; i < p1; i += NT) v[i] = __ldcg(out + i1[i]);
      for (int i = tid; i < p2; i += NT) v[p1 + i] = __ldcg(out + i2[i]);
      if (p1 == 0)  // no T1_sp: b2 = 0
        for (int i = tid; i < s; i += NT) v[p1 + p2 + i] = make_double2(0.0, 0.0);
    }
    bar_consumers(NT);
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
              const int o = M.out1p[i];
              __stcg(r + o, csub(__ldcg(r + o), y));
            } else {
              const double2 xv = csub(r2[i - p1], y);
              x2[i - p1] = xv;
              __stcg(out + M.in2s[i - p1], xv);
            }
          } else {
            const int o = M.out2p[i];
            __stcg(r + o, csub(__ldcg(r + o), y));
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
            __stcg(qp, csub(__ldcg(qp), y));
          } else {
            double2* qp = out + M.in2s[i];
            __stcg(qp, cadd(__ldcg(qp), cadd(y, nb2[i])));
          }
        }
      }
      bar_consumers(NT);
    }
  }
}

}  // namespace

StreamLevel::Shape stream_level_shape(int rows_max, int s_max, int vec_max, int merges, int sms) {
  StreamLevel::Shape sh;
  (void)s_max;
  if (rows_max > 512 || merges < sms) return sh;
  // one row group of 32 per consumer warp (and column groups on top): 4
  // consumer warps (rows <= 128) x 4 CTAs per SM, 8 x 3, or 16 x 2 -- several
  // merges in flight per SM hide each merge's per-operator barriers
  const int cw = rows_max <= 128 ? 4 : rows_max <= 256 ? 8 : 16;
  const int ctas_per_sm = cw == 4 ? 4 : cw == 8 ? 3 : 2;
  const int vec = (vec_max + 7) & ~7;
  const size_t budget = (220u << 10) / ctas_per_sm;
  const size_t fixed = sizeof(double2) * (32 * static_cast<size_t>(cw) + vec) +
                       2 * sizeof(unsigned long long) * kStreamMaxSlots;
  if (fixed >= budget) return sh;
  // ns slots of whole columns: 4 slots, each as large as the budget allows
  const int ns = 4;
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
             shape.vec_entries);
  };
  if (shape.warps == 4) go(std::integral_constant<decltype(&merge_stream_kernel<4>), &merge_stream_kernel<4>>{});
  else if (shape.warps == 8) go(std::integral_constant<decltype(&merge_stream_kernel<8>), &merge_stream_kernel<8>>{});
  else go(std::integral_constant<decltype(&merge_stream_kernel<16>), &merge_stream_kernel<16>>{});
}

}  // namespace hpsb
