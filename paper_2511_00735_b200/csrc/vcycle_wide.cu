// V-cycle level step for levels of few, large merges (the top of the
// quadtree): ONE persistent launch per level step over every SM, the four
// dependent GEMV stages of multigrid.cpp:47-98 separated by grid-wide
// barriers instead of kernel boundaries.
//
// Each stage's rows (all merges of the level, times a few column blocks
// when there are fewer than ~32 rows per CTA) are split into equal
// contiguous ranges, one per CTA (a range crossing a merge or column-block
// boundary becomes two tiles).  A producer warp per CTA streams
// its tiles' column segments through a TMA bulk-copy ring (cp.async.bulk +
// mbarrier transaction counts); it never waits for the grid barriers (the
// operators are static), so the next stage's tiles are already in flight
// while the consumers synchronise.  Consumer warps split a tile into row
// groups of 32 x column groups, reduce through shared memory and write the
// tile's partial product to a per-stage partial buffer [column block][row].
// The next stage's input vector is formed from those partials (summed in
// column-block order, deterministic) by whichever tile needs it; the
// stage's global writes (out / r updates) are distributed over the CTAs in
// the following stage.  Four grid barriers per level step.
//
//   down  S0 y0 = T2_ss r2                       (t  = r1 - y0)
//         S1 y1 = W t                             (x1 = y1 -> out[in1s])
//         S2 y2 = [T1_ps; T1_ss] x1               (r[out1p] -= y2[:p1], x2 = r2 - y2[p1:] -> out[in2s])
//         S3 y3 = T2_ps x2                        (r[out2p] -= y3)
//   up    S0 y0 = T1_sp u1                        (b2 = y0)
//         S1 y1 = [T2_sp, T2_ss] [u2; -b2]        (t = y1)
//         S2 y2 = W t                             (y1 -> out[in1s] -= y1)
//         S3 y3 = T1_ss y1                        (out[in2s] += y3 - b2)
#include <algorithm>
#include <type_traits>

#include "device.cuh"
#include "hierarchy.hpp"
#include "vcycle_small.hpp"

namespace hpsb {

namespace {

__device__ __forceinline__ unsigned wsmem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void wmbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(wsmem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void wmbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(wsmem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void wmbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(wsmem_u32(bar)) : "memory");
}
__device__ __forceinline__ void wmbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(wsmem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void wbulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          wsmem_u32(dst)),
      "l"(src), "r"(bytes), "r"(wsmem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void wbar_consumers(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

constexpr int kWideSlots = 4;

__device__ void make_givens_w(double2 a, double2 b, double& c, double2& s) {  // krylov.cpp:17-31
  c = 1.0;
  s = make_double2(0.0, 0.0);
  const double na = hypot(a.x, a.y), nb = hypot(b.x, b.y);
  if (nb == 0.0) return;
  const double r = hypot(na, nb);
  const double2 cb = make_double2(b.x, -b.y);
  if (na == 0.0) {
    c = 0.0;
    s = make_double2(cb.x / nb, cb.y / nb);
  } else {
    c = na / r;
    const double2 an = make_double2(a.x / na, a.y / na);
    s = cmul(an, make_double2(cb.x / r, cb.y / r));
  }
}
__device__ void apply_givens_w(double c, double2 s, double2& a, double2& b) {  // krylov.cpp:33-37
  const double2 t = cadd(cscale(a, c), cmul(s, b));
  b = cadd(cmul(make_double2(-s.x, s.y), a), cscale(b, c));
  a = t;
}

// CTA b's tiles of stage k: [cta_tiles[k][b], cta_tiles[k][b + 1])
__device__ __forceinline__ void stage_range(const WideArgs& a, int k, int b, int G, int& t0, int& t1) {
  const int* o = a.cta_tiles + k * (G + 1);
  t0 = o[b], t1 = o[b + 1];
}

// sum over the column blocks of stage k's partial product, row i of merge m
// (eight loads in flight, summed in column-block order)
__device__ __forceinline__ double2 part_sum(const WideArgs& a, const WideMerge& M, int k, int i) {
  const double2* p = a.part + M.part[k] + i;
  const int n = M.ncb[k];
  const size_t ld = static_cast<size_t>(M.R[k]);
  double2 y = make_double2(0.0, 0.0);
  for (int cb0 = 0; cb0 < n; cb0 += 8) {
    double2 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = cb0 + j < n ? __ldcg(p + (cb0 + j) * ld) : make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < 8; ++j) y = cadd(y, v[j]);
  }
  return y;
}

// column c of stage k's input vector for merge m
__device__ __forceinline__ double2 stage_x(const WideArgs& a, const WideMerge& M, int k, int c) {
  if (a.down) {
    switch (k) {
      case 0: return __ldcg(a.r + M.in2s[c]);                                // r2
      case 1: return csub(__ldcg(a.r + M.in1s[c]), part_sum(a, M, 0, c));   // t = r1 - T2_ss r2
      case 2: return part_sum(a, M, 1, c);                                   // x1
      default: return csub(__ldcg(a.r + M.in2s[c]), part_sum(a, M, 2, M.p1 + c));  // x2
    }
  }
  switch (k) {
    case 0: return __ldcg(a.out + M.in1p[c]);  // u1
    case 1: {
      if (c < M.p2) return __ldcg(a.out + M.in2p[c]);  // u2
      const double2 b2 = part_sum(a, M, 0, c - M.p2);
      return make_double2(-b2.x, -b2.y);  // -b2
    }
    default: return part_sum(a, M, k - 1, c);  // t (k = 2), y1 (k = 3)
  }
}

// the global writes of stage k's output, row i of merge m
__device__ __forceinline__ void stage_write(const WideArgs& a, const WideMerge& M, int k, int i) {
  if (a.down) {
    if (k == 1) {
      __stcg(a.out + M.in1s[i], part_sum(a, M, 1, i));
    } else if (k == 2) {
      const double2 y = part_sum(a, M, 2, i);
      if (i < M.p1) {
        double2* q = a.r + M.out1p[i];
        __stcg(q, csub(__ldcg(q), y));
      } else {
        const int j = i - M.p1;
        __stcg(a.out + M.in2s[j], csub(__ldcg(a.r + M.in2s[j]), y));
      }
    } else if (k == 3) {
      double2* q = a.r + M.out2p[i];
      __stcg(q, csub(__ldcg(q), part_sum(a, M, 3, i)));
    }
  } else {
    if (k == 2) {
      double2* q = a.out + M.in1s[i];
      __stcg(q, csub(__ldcg(q), part_sum(a, M, 2, i)));
    } else if (k == 3) {
      double2* q = a.out + M.in2s[i];
      __stcg(q, cadd(__ldcg(q), csub(part_sum(a, M, 3, i), part_sum(a, M, 0, i))));
    }
  }
}

// distribute stage k's output rows (all merges) over the CTAs
__device__ __forceinline__ void stage_writes(const WideArgs& a, int k, int b, int G, int tid, int nt) {
  const bool any = a.down ? k >= 1 : k >= 2;
  if (!any) return;
  const int* pre = a.row_prefix + k * (a.nm + 1);
  const int n = pre[a.nm];
  const int i0 = static_cast<int>((static_cast<long long>(n) * b) / G);
  const int i1 = static_cast<int>((static_cast<long long>(n) * (b + 1)) / G);
  int m = 0;
  for (int f = i0 + tid; f < i1; f += nt) {
    while (pre[m + 1] <= f) ++m;  // rows ascend with f within a thread
    stage_write(a, a.merges[m], k, f - pre[m]);
  }
}

// grid-wide barrier of the consumer threads (generation counter; every
// CTA of the grid is resident: the grid is sized to the occupancy)
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned G, int nt) {
  wbar_consumers(nt);
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    const unsigned g = *vgen;
    __threadfence();
    if (atomicAdd(bar, 1u) == G - 1) {
      *reinterpret_cast<volatile unsigned*>(bar) = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == g) __nanosleep(64);
    }
    __threadfence();
  }
  wbar_consumers(nt);
}

template <int CW>
__global__ void __launch_bounds__(32 * (CW + 1)) merge_wide_kernel(const __grid_constant__ WideArgs a) {
  constexpr int U = 2, NT = 32 * CW;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, b = blockIdx.x;
  const int ns = kWideSlots, slot_stride = a.slot_entries + 32;
  double2* ring = reinterpret_cast<double2*>(smem_raw);
  double2* red = ring + static_cast<size_t>(ns) * slot_stride;  // [CW * 32]
  double2* xs = red + 32 * CW;                                   // [tc_max]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(xs + a.tc_max);
  unsigned long long* empty = full + kWideSlots;
  if (tid == 0) {
    for (int q = 0; q < ns; ++q) wmbar_init(full + q, 1), wmbar_init(empty + q, CW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CW) {
    // ---- producer: the column segments of this CTA's tiles, stage by stage
    unsigned q = 0;
    for (int k = 0; k < 4; ++k) {
      int t0, t1;
      stage_range(a, k, b, G, t0, t1);
      for (int t = t0; t < t1; ++t) {
        const WideTile T = a.tiles[t];
        const int ncp = max(1, a.slot_entries / T.rows);
        for (int c0 = 0; c0 < T.cols; c0 += ncp, ++q) {
          const int nc = min(ncp, T.cols - c0), slot = static_cast<int>(q % ns);
          if (q >= static_cast<unsigned>(ns)) wmbar_wait(empty + slot, (q / ns - 1) & 1u);
          const unsigned cb = static_cast<unsigned>(sizeof(double2) * T.rows);
          if (lane == 0) wmbar_expect_tx(full + slot, cb * nc);
          __syncwarp();
          double2* dst = ring + static_cast<size_t>(slot) * slot_stride;
          const double2* src = T.A + static_cast<size_t>(c0) * T.ld;
          for (int j = lane; j < nc; j += 32)
            wbulk_g2s(dst + static_cast<size_t>(j) * T.rows, src + static_cast<size_t>(j) * T.ld, cb, full + slot);
        }
      }
    }
    return;
  }

  // ---- consumers
  pdl_wait();
  unsigned q = 0;
  for (int k = 0; k < 4; ++k) {
    if (k > 0) {
      grid_sync(a.bar, G, NT);
      stage_writes(a, k - 1, b, G, tid, NT);  // stage k-1's global writes
    }
    int t0, t1;
    stage_range(a, k, b, G, t0, t1);
    for (int t = t0; t < t1; ++t) {
      const WideTile T = a.tiles[t];
      const WideMerge& M = a.merges[T.m];
      for (int c = tid; c < T.cols; c += NT) xs[c] = stage_x(a, M, k, T.c0 + c);
      wbar_consumers(NT);
      const int rows = T.rows, ncp = max(1, a.slot_entries / rows);
      const int RG = (rows + 31) >> 5, CG = CW / RG;
      const int rg = warp % RG, cg = warp / RG;
      const bool active = cg < CG;
      double2 acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = make_double2(0.0, 0.0);
      for (int c0 = 0; c0 < T.cols; c0 += ncp, ++q) {
        const int nc = min(ncp, T.cols - c0), slot = static_cast<int>(q % ns);
        wmbar_wait(full + slot, (q / ns) & 1u);
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
        if (lane == 0) wmbar_arrive(empty + slot);
      }
      if (active) {
        double2 y = acc[0];
#pragma unroll
        for (int u = 1; u < U; ++u) y = cadd(y, acc[u]);
        red[cg * (RG * 32) + rg * 32 + lane] = y;
      }
      wbar_consumers(NT);
      double2* dst = a.part + M.part[k] + static_cast<size_t>(T.cb) * M.R[k] + T.r0;
      for (int i = tid; i < rows; i += NT) {
        double2 y = red[i];
        for (int g = 1; g < CG; ++g) y = cadd(y, red[g * (RG * 32) + i]);
        __stcg(dst + i, y);
      }
    }
  }
  grid_sync(a.bar, G, NT);
  stage_writes(a, 3, b, G, tid, NT);
}

// gmres_fixed_steps (krylov.cpp:194-201) on the coarse system
// M_L = I + sum_boxes scatter(T_box) as ONE persistent cooperative launch:
// per Arnoldi step the matvec tiles (the box maps, streamed by the producer
// warp through the TMA ring -- ahead of the grid barriers, the maps are
// static), a grid barrier, the projections (classical Gram-Schmidt, as the
// other coarse kernels: the j + 1 dot products of a step reduce together),
// a grid barrier, the update and partial norm, a grid barrier.  Every CTA
// keeps the identical Hessenberg / Givens state (sums in a fixed order), so
// no broadcast is needed.  V_0 is the right-hand side itself; V_k (k >= 1)
// are stored unnormalised with their scale factors.
__device__ __forceinline__ double grid_sum_fixed(const double* v, int n, double* sh) {
  // every CTA sums the same n values in the same order (warp 0, then lane 0)
  if (threadIdx.x < 32) {
    double a = 0.0;
    for (int i = threadIdx.x; i < n; i += 32) a += __ldcg(v + i);
    a = warp_sum(a);
    if (threadIdx.x == 0) *sh = a;
  }
  return 0.0;
}

template <int CW>
__global__ void __launch_bounds__(32 * (CW + 1)) coarse_wide_kernel(const __grid_constant__ CoarseArgs a) {
  constexpr int U = 2, NT = 32 * CW;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, b = blockIdx.x, ci = a.ci;
  const int ns = kWideSlots, slot_stride = a.slot_entries + 32;
  double2* ring = reinterpret_cast<double2*>(smem_raw);
  double2* red = ring + static_cast<size_t>(ns) * slot_stride;  // [CW * 32]
  double2* xs = red + 32 * CW;                                   // [tc_max]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(xs + a.tc_max);
  unsigned long long* empty = full + kWideSlots;
  __shared__ double2 Hs[kCoarseWideMax + 1][kCoarseWideMax];  // Hessenberg (rotated), column j
  __shared__ double2 gs[kCoarseWideMax + 1], rs[kCoarseWideMax], hsum[kCoarseWideMax + 1];
  __shared__ double rcs[kCoarseWideMax], sc[kCoarseWideMax + 1], dsh[2];
  __shared__ double2 dpart[CW][kCoarseWideMax + 1];
  if (tid == 0) {
    for (int q = 0; q < ns; ++q) wmbar_init(full + q, 1), wmbar_init(empty + q, CW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int t0, t1;
  t0 = a.cta_tiles[b], t1 = a.cta_tiles[b + 1];
  if (warp == CW) {  // producer: the same tiles every step
    unsigned q = 0;
    for (int j = 0; j < ci; ++j)
      for (int t = t0; t < t1; ++t) {
        const WideTile T = a.tiles[t];
        const int ncp = max(1, a.slot_entries / T.rows);
        for (int c0 = 0; c0 < T.cols; c0 += ncp, ++q) {
          const int nc = min(ncp, T.cols - c0), slot = static_cast<int>(q % ns);
          if (q >= static_cast<unsigned>(ns)) wmbar_wait(empty + slot, (q / ns - 1) & 1u);
          const unsigned cb = static_cast<unsigned>(sizeof(double2) * T.rows);
          if (lane == 0) wmbar_expect_tx(full + slot, cb * nc);
          __syncwarp();
          double2* dst = ring + static_cast<size_t>(slot) * slot_stride;
          const double2* src = T.A + static_cast<size_t>(c0) * T.ld;
          for (int jj = lane; jj < nc; jj += 32)
            wbulk_g2s(dst + static_cast<size_t>(jj) * T.rows, src + static_cast<size_t>(jj) * T.ld, cb, full + slot);
        }
      }
    return;
  }
  pdl_wait();
  const int64_t n = a.n;
  const int64_t i0 = n * b / G, i1 = n * (b + 1) / G;  // this CTA's slice of the coarse vector
  auto Vk = [&](int k) -> const double2* { return k == 0 ? a.rhs : a.V + static_cast<int64_t>(k) * n; };
  auto block_red = [&](double v) -> double {  // consumer-block sum (fixed order)
    v = warp_sum(v);
    __shared__ double wsum[CW];
    if (lane == 0) wsum[warp] = v;
    wbar_consumers(NT);
    double t = 0.0;
    for (int w = 0; w < CW; ++w) t += wsum[w];
    wbar_consumers(NT);
    return t;
  };
  // ---- ||b||
  {
    double s2 = 0.0;
    for (int64_t i = i0 + tid; i < i1; i += NT) s2 += cabs2(__ldcg(a.rhs + i));
    s2 = block_red(s2);
    if (tid == 0) a.pn[b] = s2;
  }
  grid_sync(a.bar, G, NT);
  grid_sum_fixed(a.pn, G, dsh);
  wbar_consumers(NT);
  const double beta = sqrt(dsh[0]);
  if (tid <= ci) gs[tid] = make_double2(tid == 0 ? beta : 0.0, 0.0);
  if (tid == 0) sc[0] = beta > 0.0 ? 1.0 / beta : 0.0;
  wbar_consumers(NT);
  int ju = 0;
  unsigned q = 0;
  if (beta > 0.0) {
    for (int j = 0; j < ci; ++j) {
      const double2* Vj = Vk(j);
      const double sj = sc[j];
      // ---- matvec tiles: partial products of the box maps with x = s_j V_j
      for (int t = t0; t < t1; ++t) {
        const WideTile T = a.tiles[t];
        const WideMerge& B = a.boxes[T.m];
        for (int c = tid; c < T.cols; c += NT) {
          const double2 v = __ldcg(Vj + B.in1s[T.c0 + c]);
          xs[c] = make_double2(sj * v.x, sj * v.y);
        }
        wbar_consumers(NT);
        const int rows = T.rows, ncp = max(1, a.slot_entries / rows);
        const int RG = (rows + 31) >> 5, CG = CW / RG;
        const int rg = warp % RG, cg = warp / RG;
        const bool active = cg < CG;
        double2 acc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = make_double2(0.0, 0.0);
        for (int c0 = 0; c0 < T.cols; c0 += ncp, ++q) {
          const int nc = min(ncp, T.cols - c0), slot = static_cast<int>(q % ns);
          wmbar_wait(full + slot, (q / ns) & 1u);
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
          if (lane == 0) wmbar_arrive(empty + slot);
        }
        if (active) red[cg * (RG * 32) + rg * 32 + lane] = cadd(acc[0], acc[1]);
        wbar_consumers(NT);
        double2* dst = a.part + B.part[0] + static_cast<size_t>(T.cb) * B.R[0] + T.r0;
        for (int i = tid; i < rows; i += NT) {
          double2 y = red[i];
          for (int g = 1; g < CG; ++g) y = cadd(y, red[g * (RG * 32) + i]);
          __stcg(dst + i, y);
        }
        wbar_consumers(NT);
      }
      grid_sync(a.bar, G, NT);
      // ---- w = s_j V_j + sum of the partials (this CTA's slice), dots with V_0..V_j
      double2 dk[kCoarseWideMax + 1];
#pragma unroll
      for (int k = 0; k <= kCoarseWideMax; ++k) dk[k] = make_double2(0.0, 0.0);
      for (int64_t i = i0 + tid; i < i1; i += NT) {
        const int bx = a.inv_box[i], row = a.inv_row[i];
        const WideMerge& B = a.boxes[bx];
        const double2* pp = a.part + B.part[0] + row;
        double2 w = __ldcg(Vj + i);
        w = make_double2(sj * w.x, sj * w.y);
        for (int cb = 0; cb < B.ncb[0]; ++cb) w = cadd(w, __ldcg(pp + static_cast<size_t>(cb) * B.R[0]));
        __stcg(a.W + i, w);
#pragma unroll
        for (int k = 0; k <= kCoarseWideMax; ++k)
          if (k <= j) {
            const double2 v = __ldcg(Vk(k) + i);
            dk[k] = cfma_conj(make_double2(sc[k] * v.x, sc[k] * v.y), w, dk[k]);
          }
      }
#pragma unroll
      for (int k = 0; k <= kCoarseWideMax; ++k)
        if (k <= j) {
          double2 d = dk[k];
          d.x = warp_sum(d.x), d.y = warp_sum(d.y);
          if (lane == 0) dpart[warp][k] = d;
        }
      wbar_consumers(NT);
      if (tid <= j) {
        double2 t = make_double2(0.0, 0.0);
        for (int w = 0; w < CW; ++w) t = cadd(t, dpart[w][tid]);
        a.pd[static_cast<int64_t>(b) * (kCoarseWideMax + 1) + tid] = t;
      }
      grid_sync(a.bar, G, NT);
      // ---- h = sum of the dots (fixed order), w' = w - sum_k h_k v_k, ||w'||
      if (warp <= j) {
        double2 t = make_double2(0.0, 0.0);
        for (int c = lane; c < G; c += 32) t = cadd(t, __ldcg(a.pd + static_cast<int64_t>(c) * (kCoarseWideMax + 1) + warp));
        t.x = warp_sum(t.x), t.y = warp_sum(t.y);
        if (lane == 0) hsum[warp] = t;
      }
      wbar_consumers(NT);
      double s2 = 0.0;
      double2* Vn = a.V + static_cast<int64_t>(j + 1) * n;
      for (int64_t i = i0 + tid; i < i1; i += NT) {
        double2 w = __ldcg(a.W + i);
        for (int k = 0; k <= j; ++k) {
          const double2 v = __ldcg(Vk(k) + i);
          w = csub(w, cmul(hsum[k], make_double2(sc[k] * v.x, sc[k] * v.y)));
        }
        __stcg(Vn + i, w);
        s2 += cabs2(w);
      }
      s2 = block_red(s2);
      if (tid == 0) a.pn[b] = s2;
      grid_sync(a.bar, G, NT);
      grid_sum_fixed(a.pn, G, dsh);
      wbar_consumers(NT);
      const double hn = sqrt(dsh[0]);
      if (tid == 0) {  // Hessenberg column j, previous rotations, new rotation (krylov.cpp:110-131)
        for (int i = 0; i <= j; ++i) Hs[i][j] = hsum[i];
        Hs[j + 1][j] = make_double2(hn, 0.0);
        for (int i = 0; i < j; ++i) apply_givens_w(rcs[i], rs[i], Hs[i][j], Hs[i + 1][j]);
        double cc;
        double2 ss;
        make_givens_w(Hs[j][j], Hs[j + 1][j], cc, ss);
        rcs[j] = cc, rs[j] = ss;
        apply_givens_w(cc, ss, Hs[j][j], Hs[j + 1][j]);
        apply_givens_w(cc, ss, gs[j], gs[j + 1]);
        sc[j + 1] = hn > 0.0 ? 1.0 / hn : 0.0;
      }
      wbar_consumers(NT);
      ju = j + 1;
      if (hn <= 1e-14 * beta) break;  // happy breakdown (identical in every CTA)
    }
  }
  // ---- y = H^{-1} g, z = sum_k y_k v_k on this CTA's slice
  __shared__ double2 ys[kCoarseWideMax];
  if (tid == 0) {
    for (int i = ju - 1; i >= 0; --i) {
      double2 t = gs[i];
      for (int k = i + 1; k < ju; ++k) t = csub(t, cmul(Hs[i][k], ys[k]));
      ys[i] = cdiv(t, Hs[i][i]);
    }
  }
  wbar_consumers(NT);
  for (int64_t i = i0 + tid; i < i1; i += NT) {
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < ju; ++k) {
      const double2 v = __ldcg(Vk(k) + i);
      acc = cfma(ys[k], make_double2(sc[k] * v.x, sc[k] * v.y), acc);
    }
    a.z[i] = acc;
  }
}

}  // namespace

WideLevel::Shape wide_level_shape(int tc_max, int sms) {
  WideLevel::Shape sh;
  // 8 consumer warps + a producer per CTA, two CTAs per SM (measured at
  // cfg3 levels 9-13: 2 x 8 warps 1.04 ms, 3 x 8 1.05 ms, 1 x 16 1.20 ms)
  sh.warps = 8;
  sh.ctas_per_sm = 2;
  const size_t budget = (220u << 10) / sh.ctas_per_sm;
  const size_t fixed = sizeof(double2) * (32 * static_cast<size_t>(sh.warps) + tc_max) +
                       2 * sizeof(unsigned long long) * kWideSlots;
  const int slot = static_cast<int>((budget - fixed) / (sizeof(double2) * kWideSlots)) - 32;
  sh.slot_entries = slot;
  sh.tc_max = tc_max;
  sh.smem = fixed + sizeof(double2) * kWideSlots * (static_cast<size_t>(slot) + 32);
  sh.grid = sms * sh.ctas_per_sm;
  sh.ok = slot >= 128;
  return sh;
}

void WideLevel::run(Context* ctx, bool down, double2* r, double2* out) const {
  const Dir& d = dir[down ? 0 : 1];
  if (d.ntiles == 0) return;
  KernelScope ks(ctx, label.empty() ? (down ? "vcycle_down" : "vcycle_up") : label.c_str(), d.bytes, 0.0);
  WideArgs a = d.args;
  a.r = r, a.out = out;
  allow_smem<merge_wide_kernel<8>>(shape.smem);
  // cooperative: the grid barriers need every CTA resident, also when other
  // contexts' kernels share the GPU
  launch_k(ctx, merge_wide_kernel<8>, dim3(shape.grid), dim3(32 * (shape.warps + 1)), shape.smem, -1, a);
}

int wide_max_ctas_per_sm(size_t smem) {
  int n = 0;
  allow_smem<merge_wide_kernel<8>>(smem);
  HPSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, merge_wide_kernel<8>, 32 * 9, smem));
  return n;
}

}  // namespace hpsb

namespace hpsb {

void CoarseWide::run(Context* ctx, const double2* rhs, double2* z) const {
  KernelScope ks(ctx, "coarse_wide", bytes, 0.0);
  CoarseArgs a = args;
  a.rhs = rhs, a.z = z;
  allow_smem<coarse_wide_kernel<8>>(shape.smem);
  launch_k(ctx, coarse_wide_kernel<8>, dim3(shape.grid), dim3(32 * (shape.warps + 1)), shape.smem, -1, a);
}

int coarse_wide_max_ctas_per_sm(size_t smem) {
  int n = 0;
  allow_smem<coarse_wide_kernel<8>>(smem);
  HPSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, coarse_wide_kernel<8>, 32 * 9, smem));
  return n;
}

}  // namespace hpsb
