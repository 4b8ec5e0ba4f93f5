// Grouped complex FP64 GEMM on the FP64 tensor cores (DMMA), plus the
// batched gathers / copies / inverses the merge stage is built from.
//
// On sm_100 the tensor-core path for FP64 is the warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4); tcgen05.mma has no f64 kind.  A
// complex product is four real DMMA products on de-interleaved fragments:
//   Cr += Ar Br - Ai Bi,   Ci += Ar Bi + Ai Br.
// Tiles are 64 x 64 complex outputs per 256-thread CTA (8 warps, 32 x 16 per
// warp), K-steps of 16 staged through a 3-stage cp.async pipeline with
// padded shared-memory strides that make the 16-byte fragment loads
// bank-conflict free.  A launch covers a whole list of independent problems
// (every merge of a quadtree level): CTAs map to (problem, tile) through a
// prefix sum of tile counts, so levels with thousands of tiny merges and
// levels with two huge ones use the same kernel.
#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cooperative_groups.h>

#include "device.cuh"
#include "internal.hpp"
#include "linalg.cuh"
#include "zgemm.hpp"
#include "gj_reg.cuh"
#include "gj_dmma.cuh"

namespace hpsb {

namespace {
constexpr int BK = 16, STAGES = 3, THREADS = 256;
constexpr int SB = BK + 4;  // complex stride of a B column in smem
// Tile shapes: IM = 4 / 3 / 2 row fragments per warp (64 / 48 / 32 rows over
// 2 warp rows), JN = 2 / 1 column fragments per warp (64 / 32 columns over 4
// warp columns).  A tile's time is its busiest warp's: with 64 x 64 tiles
// only, a ragged dimension (merge sizes are multiples of N - 1: 76 = 64 + 12)
// cost a full tile and the launch times followed the tile-padded flops.
// Shapes are compile time (a run-time shape spilled registers in the main
// loop: 116.6 -> 131 ms at cfg3); GemmBatch::run launches once per shape.
template <int IM, int JN>
struct GemmTile {
  static constexpr int BM = 16 * IM, BN = 32 * JN;
  static constexpr int SA = BM + 2;  // complex stride of an A k-row in smem
  static constexpr int A_STAGE = BK * SA, B_STAGE = BN * SB;
  static constexpr size_t kSmem = sizeof(double2) * STAGES * (A_STAGE + B_STAGE);
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int IM, int JN>
__global__ void __launch_bounds__(THREADS, 2) zgemm_grouped_kernel(const GemmDesc* __restrict__ descs,
                                                                const int* __restrict__ tile_map) {
  using TS = GemmTile<IM, JN>;
  constexpr int BM = TS::BM, BN = TS::BN, SA = TS::SA, A_STAGE = TS::A_STAGE, B_STAGE = TS::B_STAGE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* As = reinterpret_cast<double2*>(smem_raw);
  double2* Bs = As + STAGES * A_STAGE;
  const int tile = blockIdx.x;
  // the problem owning this tile: one load (a binary search over the
  // thousands of problems of a low level was a chain of ~14 dependent L2
  // loads per CTA, as long as a K = 19 tile's whole main loop)
  const GemmDesc d = descs[tile_map[tile]];
  const int local = tile - d.tile_begin;
  const int tm = local % d.tiles_m, tn = local / d.tiles_m;
  const int m0 = tm * BM, n0 = tn * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;  // 2 x 4 warps of (8 IM) x (8 JN)
  const int ktiles = (d.K + BK - 1) / BK;

  auto load_stage = [&](int kt, int st) {
    const int k0 = kt * BK;
    double2* as = As + st * A_STAGE;
    double2* bs = Bs + st * B_STAGE;
#pragma unroll
    for (int r = 0; r < (BM * BK) / THREADS; ++r) {
      const int idx = tid + r * THREADS;
      const int m = idx % BM, k = idx / BM;
      const bool ok = (m0 + m < d.M) && (k0 + k < d.K);
      const double2* src = ok ? d.A + (size_t)(m0 + m) + (size_t)(k0 + k) * d.lda : d.A;
      cp_async16(as + k * SA + m, src, ok);
    }
#pragma unroll
    for (int r = 0; r < (BN * BK) / THREADS; ++r) {
      const int idx = tid + r * THREADS;
      const int k = idx % BK, n = idx / BK;
      const bool ok = (n0 + n < d.N) && (k0 + k < d.K);
      const double2* src = ok ? d.B + (size_t)(k0 + k) + (size_t)(n0 + n) * d.ldb : d.B;
      cp_async16(bs + n * SB + k, src, ok);
    }
  };

  double cr[IM][JN][2], ci[IM][JN][2];
#pragma unroll
  for (int i = 0; i < IM; ++i)
#pragma unroll
    for (int j = 0; j < JN; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_async_commit();
  }
  const int arow = wm * (8 * IM) + (lane >> 2), kq = lane & 3;
  const int bcol = wn * (8 * JN) + (lane >> 2);
  // Edge tiles: fragments wholly outside M x N and k-steps past K are
  // skipped (warp-uniform), so ragged merge dimensions (multiples of N-1,
  // e.g. 76 = 64 + 12) do not pay for a full padded tile on the DMMA pipe.
  const int ni_act = max(0, min(IM, (d.M - m0 - wm * (8 * IM) + 7) / 8));
  const int nj_act = max(0, min(JN, (d.N - n0 - wn * (8 * JN) + 7) / 8));
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (kt + STAGES - 1 < ktiles) load_stage(kt + STAGES - 1, (kt + STAGES - 1) % STAGES);
    cp_async_commit();
    const double2* as = As + (kt % STAGES) * A_STAGE;
    const double2* bs = Bs + (kt % STAGES) * B_STAGE;
    const int krem = d.K - kt * BK;
    // FULL: every fragment and k-step of this stage is inside the problem
    // (interior tiles of the large merges): no predicates, no early exit,
    // so the fragment loads of step kk + 4 are scheduled under the DMMAs of kk
    // KFULL: all BK k-values are inside K (fragment predicates only, no
    // early exit: the loads still pipeline under the DMMAs)
    auto stage = [&](auto full_tag, auto kfull_tag) {
      constexpr bool FULL = decltype(full_tag)::value, KFULL = decltype(kfull_tag)::value;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        if (!KFULL && kk >= krem) break;
        double2 a[IM], b[JN];
#pragma unroll
        for (int i = 0; i < IM; ++i) a[i] = as[(kk + kq) * SA + arow + i * 8];
#pragma unroll
        for (int j = 0; j < JN; ++j) b[j] = bs[(bcol + j * 8) * SB + kk + kq];
        // four passes over the 4 x 2 fragment grid: the two DMMAs into the
        // same accumulator are 24 issues apart instead of back to back (the
        // asm statements are volatile, so the compiler keeps this order)
#pragma unroll
        for (int i = 0; i < IM; ++i)
#pragma unroll
          for (int j = 0; j < JN; ++j)
            if (FULL || (i < ni_act && j < nj_act)) dmma(cr[i][j][0], cr[i][j][1], a[i].x, b[j].x);
#pragma unroll
        for (int i = 0; i < IM; ++i)
#pragma unroll
          for (int j = 0; j < JN; ++j)
            if (FULL || (i < ni_act && j < nj_act)) dmma(ci[i][j][0], ci[i][j][1], a[i].x, b[j].y);
#pragma unroll
        for (int i = 0; i < IM; ++i)
#pragma unroll
          for (int j = 0; j < JN; ++j)
            if (FULL || (i < ni_act && j < nj_act)) dmma(cr[i][j][0], cr[i][j][1], -a[i].y, b[j].y);
#pragma unroll
        for (int i = 0; i < IM; ++i)
#pragma unroll
          for (int j = 0; j < JN; ++j)
            if (FULL || (i < ni_act && j < nj_act)) dmma(ci[i][j][0], ci[i][j][1], a[i].y, b[j].x);
      }
    };
    if (krem >= BK) {
      if (ni_act == IM && nj_act == JN) stage(std::true_type{}, std::true_type{});
      else stage(std::false_type{}, std::true_type{});
    } else {
      stage(std::false_type{}, std::false_type{});
    }
  }
  cp_async_wait<0>();
  // epilogue: C = alpha * acc + beta * C.  All C reads are issued before
  // the first store: interleaved, every read waited for the previous store
  // (possible aliasing), 16 serial L2/HBM round trips per thread -- longer
  // than the whole main loop of the K = 19..76 merges of the low levels.
  const double2 alpha = make_double2(d.alpha_re, d.alpha_im);
  const double2 beta = make_double2(d.beta_re, d.beta_im);
  const bool use_beta = (d.beta_re != 0.0 || d.beta_im != 0.0);
  const int row0 = m0 + wm * (8 * IM) + (lane >> 2), col0 = n0 + wn * (8 * JN) + 2 * (lane & 3);
  // fragment rows two at a time: 4 JN reads in flight, no spills
#pragma unroll
  for (int half = 0; half < (IM + 1) / 2; ++half) {
    double2 cold[2][JN][2];
    if (use_beta) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < JN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = row0 + (2 * half + i) * 8, col = col0 + j * 8 + h;
            double2 cv = make_double2(0.0, 0.0);
            if (2 * half + i < IM && row < d.M && col < d.N) {
              if (!d.Cin) cv = d.C[(size_t)row + (size_t)col * d.ldc];
              else if (col >= d.cin_c0 && col < d.cin_c1)
                cv = d.Cin[(size_t)row + (size_t)(col - d.cin_c0) * d.ldcin];
            }
            cold[i][j][h] = cv;
          }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int ii = 2 * half + i, row = row0 + ii * 8;
      if (ii >= IM || row >= d.M) continue;
#pragma unroll
      for (int j = 0; j < JN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = col0 + j * 8 + h;
          if (col >= d.N) continue;
          double2 v = cmul(alpha, make_double2(cr[ii < IM ? ii : 0][j][h], ci[ii < IM ? ii : 0][j][h]));
          if (use_beta) v = cadd(v, cmul(beta, cold[i][j][h]));
          d.C[(size_t)row + (size_t)col * d.ldc] = v;
        }
    }
  }
}

// Sub-matrix copy / gather ops, tiled 8 columns per CTA.  A thread owns rows
// and walks the tile's 8 columns with all 8 loads in flight before the first
// store (row index loaded once): per-column loops with one dependent load per
// iteration ran the gathers at 4.3 TB/s.
__global__ void copy_ops_kernel(const CopyOp* __restrict__ ops, const int* __restrict__ tile_map) {
  const int tile = blockIdx.x;
  const CopyOp op = ops[tile_map[tile]];
  const int c0 = (tile - op.tile_begin) * 8;
  const int nc = min(8, op.cols - c0);
  if (op.mode != CopyOp::kCopy) {
    for (int c = c0; c < c0 + nc; ++c)
      for (int r = threadIdx.x; r < op.rows; r += blockDim.x)
        op.dst[(size_t)r + (size_t)c * op.ldd] =
            make_double2(op.mode == CopyOp::kIdentity && r == c ? 1.0 : 0.0, 0.0);
    return;
  }
  size_t scol[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = c0 + min(j, nc - 1);
    scol[j] = (size_t)(op.cidx ? op.cidx[c] : c) * op.lds;
  }
  for (int r = threadIdx.x; r < op.rows; r += blockDim.x) {
    const double2* s = op.src + (op.ridx ? op.ridx[r] : r);
    double2 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = s[scol[j]];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < nc) op.dst[(size_t)r + (size_t)(c0 + j) * op.ldd] = cscale(v[j], op.scale);
  }
}

// One CTA per matrix: complex Gauss-Jordan inverse (n <= kSmemInvMax), the
// matrix register-resident across 512 threads (gj_reg.cuh); the result is
// written back in place.  MODE 0: partial pivoting.  MODE 1: diagonal
// pivots, guarded -- written only if the guard holds, else flags[op] = 1
// (flags != null: the MODE 2 launch that follows redoes it) or guard[0] = 1.
// MODE 2: partial pivoting of the flagged matrices only.
// Diagonal pivots are safe for the merge blocks W = I - T2_ss T1_ss: ItI maps
// of passive media are contractions (unitary when lossless), so W has a
// positive definite Hermitian part, and so do its leading blocks and Schur
// complements.
template <int TR, int MODE>
__global__ void __launch_bounds__(kGjThreads) inverse_reg_kernel(const InvOp* __restrict__ ops,
                                                                 int* status, int* flags,
                                                                 int* guard) {
  constexpr int TC = (TR + 1) / 2;
  __shared__ GjShared sh;
  const InvOp op = ops[blockIdx.x];
  if (MODE == 2 && !flags[blockIdx.x]) return;
  GjReg<TR, TC> g;
  auto get = [&](int i, int j) { return op.A[(size_t)i + (size_t)j * op.lda]; };
  const int ty = threadIdx.x % kGjY, tx = threadIdx.x / kGjY;
  if (MODE == 1) {
    __shared__ unsigned long long smax;
    if (threadIdx.x == 0) smax = 0ull;
    __syncthreads();
    double m = 0.0;  // max |a_ij|^2 (order-preserving bits of a non-negative double)
    for (int idx = threadIdx.x; idx < op.n * op.n; idx += kGjThreads)
      m = fmax(m, cabs2(get(idx % op.n, idx / op.n)));
    atomicMax(&smax, static_cast<unsigned long long>(__double_as_longlong(m)));
    __syncthreads();
    const double m0 = __longlong_as_double(static_cast<long long>(smax));
    if (!gj_reg_inverse_nopiv<TR, TC>(op.n, get, g, sh, kGjTiny2 * m0, kGjHuge2 / fmax(m0, 1e-300))) {
      if (threadIdx.x == 0) {
        if (flags) flags[blockIdx.x] = 1;
        else *guard = 1;
      }
      return;
    }
#pragma unroll
    for (int a = 0; a < TR; ++a) {
      const int i = ty + kGjY * a;
      if (i >= op.n) continue;
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        const int j = tx + kGjX * b;
        if (j < op.n) op.A[(size_t)i + (size_t)j * op.lda] = g.x[a][b];
      }
    }
    return;
  }
  const bool ok = gj_reg_inverse<TR, TC>(op.n, get, g, sh);
#pragma unroll
  for (int a = 0; a < TR; ++a) {
    const int i = ty + kGjY * a;
    if (i >= op.n) continue;
    const int r = sh.step[i];
#pragma unroll
    for (int b = 0; b < TC; ++b) {
      const int j = tx + kGjX * b;
      if (j < op.n) op.A[(size_t)r + (size_t)sh.piv[j] * op.lda] = g.x[a][b];
    }
  }
  if (threadIdx.x == 0 && !ok) status[0] = op.tag + 1;
}

template <int MODE>
void launch_inverse_reg(int nmax, int grid, cudaStream_t st, const InvOp* ops, int* status,
                        int* flags, int* guard) {
  switch ((nmax + kGjY - 1) / kGjY) {
    case 0: case 1: case 2: inverse_reg_kernel<2, MODE><<<grid, kGjThreads, 0, st>>>(ops, status, flags, guard); break;
    case 3: inverse_reg_kernel<3, MODE><<<grid, kGjThreads, 0, st>>>(ops, status, flags, guard); break;
    case 4: inverse_reg_kernel<4, MODE><<<grid, kGjThreads, 0, st>>>(ops, status, flags, guard); break;
    case 5: inverse_reg_kernel<5, MODE><<<grid, kGjThreads, 0, st>>>(ops, status, flags, guard); break;
    default: inverse_reg_kernel<6, MODE><<<grid, kGjThreads, 0, st>>>(ops, status, flags, guard); break;
  }
}

// MODE 1 of inverse_reg_kernel on the FP64 tensor cores: the diagonal-pivot
// blocked Gauss-Jordan of gj_dmma.cuh, one matrix per CTA (identity padded
// to NP) in shared memory.  A guard failure (small pivot, or an inverse entry
// beyond kGjHuge2 / max|a_ij|^2) leaves the matrix untouched and flags it for
// the pivoted redo (flags) or the whole build (guard, blocked-inverse blocks).
template <int NP>
__global__ void __launch_bounds__(256) inverse_dmma_kernel(const InvOp* __restrict__ ops, int* flags,
                                                           int* guard) {
  using G = GdShape<NP>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* M = reinterpret_cast<double2*>(smem_raw);
  __shared__ double red[8];
  __shared__ int flag;
  const InvOp op = ops[blockIdx.x];
  const int n = op.n, tid = threadIdx.x;
  double m = 0.0;
  for (int j = tid / 32; j < NP; j += 8)
    for (int i = tid & 31; i < NP; i += 32) {
      double2 val = make_double2(i == j ? 1.0 : 0.0, 0.0);
      if (i < n && j < n) {
        val = op.A[(size_t)i + (size_t)j * op.lda];
        m = fmax(m, cabs2(val));
      }
      M[j * G::LD + i] = val;
    }
  m = warp_max(m);
  if ((tid & 31) == 0) red[tid >> 5] = m;
  __syncthreads();
  double m0 = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) m0 = fmax(m0, red[w]);
  bool ok = gd_inverse<NP, 8>(M, &flag, kGjTiny2 * m0);
  if (ok) {
    const double huge2 = kGjHuge2 / fmax(m0, 1e-300);
    bool bad = false;
    for (int j = tid / 32; j < n; j += 8)
      for (int i = tid & 31; i < n; i += 32) bad |= !(cabs2(M[j * G::LD + i]) <= huge2);
    ok = !__syncthreads_or(bad);
  }
  if (!ok) {
    if (tid == 0) {
      if (flags) flags[blockIdx.x] = 1;
      else *guard = 1;
    }
    return;
  }
  for (int j = tid / 32; j < n; j += 8)
    for (int i = tid & 31; i < n; i += 32) op.A[(size_t)i + (size_t)j * op.lda] = M[j * G::LD + i];
}

void launch_inverse_dmma(int nmax, int grid, cudaStream_t st, const InvOp* ops, int* flags, int* guard) {
  auto go = [&](auto np_tag) {
    constexpr int NP = decltype(np_tag)::value;
    allow_smem<inverse_dmma_kernel<NP>>(GdShape<NP>::kSmem);
    inverse_dmma_kernel<NP><<<grid, 256, GdShape<NP>::kSmem, st>>>(ops, flags, guard);
  };
  switch ((nmax + 15) / 16) {
    case 0: case 1: go(std::integral_constant<int, 16>{}); break;
    case 2: go(std::integral_constant<int, 32>{}); break;
    case 3: go(std::integral_constant<int, 48>{}); break;
    case 4: go(std::integral_constant<int, 64>{}); break;
    case 5: go(std::integral_constant<int, 80>{}); break;
    default: go(std::integral_constant<int, 96>{}); break;
  }
}

// ---- pivot selection for one panel, one thread-block CLUSTER per matrix.
// The panel rows k0..n-1 (x kw columns) are split across the C CTAs of the
// cluster and kept in shared memory; per column j: local argmax of |a_ij|
// over the unused rows, candidates pushed to every peer (DSMEM), the same
// fixed-order reduction in every CTA, the owner pushes the pivot row to every
// peer, every CTA eliminates column j from its unused rows.  Pivoting is
// implicit (used flags, no row swaps); the pivot order is converted to the
// LAPACK swap sequence ipiv[k0+j] = k0 + p at the end.  The same pivots as a
// swap-based partial-pivoting LU of the panel (ties aside); only ipiv is
// produced (the elimination proper is the GEMM sweep below).
// (Replaces a one-CTA panel LU whose rank-1 updates went through L2: up to
// 77 MB of traffic per 32-column panel of a 2432-row matrix.)
constexpr int kPivThreads = 512;
constexpr int kPivMaxCluster = 16;
constexpr int kPivMaxKb = 64;
__global__ void __launch_bounds__(kPivThreads) panel_pivot_cluster_kernel(
    const InvOp* __restrict__ ops, int k0, int kb, int chunk_max, int* ipiv_ws, int* status) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks()), crank = static_cast<int>(cl.block_rank());
  const InvOp op = ops[blockIdx.x / C];
  if (k0 >= op.n) return;  // the whole cluster (same matrix) leaves together
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = op.n, kw = min(kb, n - k0), rows = n - k0;
  const int chunk = (rows + C - 1) / C, r0 = min(rows, crank * chunk), nr = min(rows, r0 + chunk) - r0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Ps = reinterpret_cast<double2*>(smem_raw);                  // [kw][chunk_max]
  int* used = reinterpret_cast<int*>(Ps + static_cast<size_t>(kb) * chunk_max);  // [chunk_max]
  int* posof = used + chunk_max;                                        // [rows] (CTA 0)
  int* rowat = posof + n;                                               // [rows] (CTA 0)
  __shared__ double2 prow[kPivMaxKb];
  __shared__ double cand_v[kPivMaxCluster];
  __shared__ int cand_i[kPivMaxCluster];
  __shared__ double red_v[kPivThreads / 32];
  __shared__ int red_i[kPivThreads / 32];
  __shared__ int order[kPivMaxKb];
  for (int idx = tid; idx < nr * kw; idx += kPivThreads) {
    const int r = idx % nr, c = idx / nr;
    Ps[r + static_cast<size_t>(c) * chunk_max] = op.A[(size_t)(k0 + r0 + r) + (size_t)(k0 + c) * op.lda];
  }
  for (int r = tid; r < nr; r += kPivThreads) used[r] = 0;
  __syncthreads();
  for (int j = 0; j < kw; ++j) {
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int r = tid; r < nr; r += kPivThreads)
      if (!used[r]) {
        const double v = cabs2(Ps[r + static_cast<size_t>(j) * chunk_max]);
        if (v > best) best = v, bi = r0 + r;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) best = ov, bi = oi;
    }
    if (lane == 0) red_v[warp] = best, red_i[warp] = bi;
    __syncthreads();
    if (tid < C) {
      double b = -1.0;
      int p = 0x7fffffff;
      for (int w = 0; w < kPivThreads / 32; ++w)
        if (red_v[w] > b || (red_v[w] == b && red_i[w] < p)) b = red_v[w], p = red_i[w];
      *cl.map_shared_rank(&cand_v[crank], tid) = b;
      *cl.map_shared_rank(&cand_i[crank], tid) = p;
    }
    cl.sync();  // candidates of every CTA delivered
    double pv = -1.0;
    int p = 0x7fffffff;
    for (int q = 0; q < C; ++q)
      if (cand_v[q] > pv || (cand_v[q] == pv && cand_i[q] < p)) pv = cand_v[q], p = cand_i[q];
    if (!(pv > 0.0)) {
      if (tid == 0 && crank == 0) status[0] = op.tag + 1;
      p = j < rows ? p : 0;
    }
    if (p >= r0 && p < r0 + nr) {  // owner: pivot row (columns j..kw-1) to every peer
      const int lr = p - r0;
      for (int t = tid; t < C * (kw - j); t += kPivThreads) {
        const int q = t / (kw - j), c = j + t % (kw - j);
        *cl.map_shared_rank(&prow[c], q) = Ps[lr + static_cast<size_t>(c) * chunk_max];
      }
      __syncthreads();
      if (tid == 0) used[lr] = 1;
    }
    if (tid == 0) order[j] = p;
    cl.sync();  // pivot row delivered
    const double2 inv = cinv(prow[j]);
    const int cw = kw - j - 1;
    for (int idx = tid; idx < nr * cw; idx += kPivThreads) {
      const int r = idx % nr, c = j + 1 + idx / nr;
      if (used[r]) continue;
      const double2 l = cmul(Ps[r + static_cast<size_t>(j) * chunk_max], inv);
      double2& a = Ps[r + static_cast<size_t>(c) * chunk_max];
      a = csub(a, cmul(l, prow[c]));
    }
    __syncthreads();
  }
  if (crank == 0) {  // pivot order -> swap sequence over positions k0..n-1
    for (int r = tid; r < rows; r += kPivThreads) posof[r] = r, rowat[r] = r;
    __syncthreads();
    if (tid == 0)
      for (int j = 0; j < kw; ++j) {
        const int q = order[j], pos = posof[q];
        ipiv_ws[op.perm_off + k0 + j] = k0 + pos;
        const int a = rowat[j];
        rowat[j] = q, rowat[pos] = a;
        posof[a] = pos, posof[q] = j;
      }
  }
  cl.sync();  // no CTA leaves while a peer may still write its shared memory
}


// Apply the panel's row swaps to every column of A (sequential swaps per column).
__global__ void swap_rows_kernel(const InvOp* __restrict__ ops, int k0, int kb,
                                 const int* __restrict__ ipiv_ws) {
  const InvOp op = ops[blockIdx.y];
  if (k0 >= op.n) return;
  const int kw = min(kb, op.n - k0);
  const int* ipiv = ipiv_ws + op.perm_off;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < op.n; c += gridDim.x * blockDim.x) {
    double2* col = op.A + (size_t)c * op.lda;
    for (int j = 0; j < kw; ++j) {
      const int p = ipiv[k0 + j];
      if (p != k0 + j) {
        const double2 t = col[k0 + j];
        col[k0 + j] = col[p];
        col[p] = t;
      }
    }
  }
}

// Undo the row interchanges as column interchanges, in reverse order.
__global__ void unscramble_kernel(const InvOp* __restrict__ ops, const int* __restrict__ ipiv_ws) {
  const InvOp op = ops[blockIdx.y];
  const int* ipiv = ipiv_ws + op.perm_off;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < op.n; r += gridDim.x * blockDim.x)
    for (int j = op.n - 1; j >= 0; --j) {
      const int p = ipiv[j];
      if (p != j) {
        double2* a = op.A + r + (size_t)j * op.lda;
        double2* b = op.A + r + (size_t)p * op.lda;
        const double2 t = *a;
        *a = *b;
        *b = t;
      }
    }
}
}  // namespace

int GemmBatch::add(const GemmDesc& d0) {
  if (d0.M <= 0 || d0.N <= 0) return -1;
  flops += 8.0 * d0.M * d0.N * std::max(d0.K, 0);
  descs.push_back(d0);
  return static_cast<int>(descs.size()) - 1;
}

namespace {
// the largest tile, unless a smaller one cuts the padded size by more than 8%
int pick_tile(int n, std::initializer_list<int> sizes) {
  int best = *sizes.begin();
  for (int b : sizes) {
    const int pb = (n + best - 1) / best * best, pn = (n + b - 1) / b * b;
    if (pn * 100 < pb * 92) best = b;
  }
  return best;
}
template <int IM, int JN>
void launch_gemm(Context* ctx, int tiles, const GemmDesc* descs, const int* map) {
  static const bool attr = [] {  // thread-safe one-time init
    HPSB_CUDA(cudaFuncSetAttribute(zgemm_grouped_kernel<IM, JN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(GemmTile<IM, JN>::kSmem)));
    return true;
  }();
  (void)attr;
  zgemm_grouped_kernel<IM, JN><<<tiles, THREADS, GemmTile<IM, JN>::kSmem, ctx->stream>>>(descs, map);
  HPSB_LAUNCHED(ctx);
}
}  // namespace

void GemmBatch::run(Context* ctx) {
  if (descs.empty()) return;
  // K == 0 problems still apply the epilogue (C = beta C): keep them valid.
  // Problems are grouped by tile shape, one launch per shape present.
  constexpr int kShapes = 6;  // (bm, bn): 64/48/32 x 64/32
  auto shape_of = [](const GemmDesc& d) {
    return (d.bm == 64 ? 0 : d.bm == 48 ? 1 : 2) * 2 + (d.bn == 64 ? 0 : 1);
  };
  // counting sort by shape (stable: problems keep their order within a shape)
  int first[kShapes + 1] = {0}, tiles[kShapes] = {0}, map_off[kShapes + 1] = {0};
  double padded = 0;
  for (auto& d : descs) {
    d.bm = pick_tile(d.M, {64, 48, 32});
    d.bn = pick_tile(d.N, {64, 32});
    d.tiles_m = (d.M + d.bm - 1) / d.bm;
    d.tiles_n = (d.N + d.bn - 1) / d.bn;
    ++first[shape_of(d) + 1];
    padded += 8.0 * d.tiles_m * d.bm * d.tiles_n * d.bn * (((d.K + BK - 1) / BK) * BK);
  }
  for (int sh = 0; sh < kShapes; ++sh) first[sh + 1] += first[sh];
  std::vector<GemmDesc> sorted(descs.size());
  {
    int at[kShapes];
    for (int sh = 0; sh < kShapes; ++sh) at[sh] = first[sh];
    for (const auto& d0 : descs) {
      const int sh = shape_of(d0);
      GemmDesc& d = sorted[at[sh]++];
      d = d0;
      d.tile_begin = tiles[sh];
      tiles[sh] += d.tiles_m * d.tiles_n;
    }
  }
  for (int sh = 0; sh < kShapes; ++sh) map_off[sh + 1] = map_off[sh] + tiles[sh];
  total_tiles = map_off[kShapes];
  d_descs.upload(sorted, ctx->stream);
  {
    std::vector<int> map(total_tiles);
    for (int sh = 0; sh < kShapes; ++sh)
      for (int i = first[sh]; i < first[sh + 1]; ++i) {
        const GemmDesc& d = sorted[i];
        std::fill(map.begin() + map_off[sh] + d.tile_begin,
                  map.begin() + map_off[sh] + d.tile_begin + d.tiles_m * d.tiles_n, i - first[sh]);
      }
    d_map.upload(map, ctx->stream);
  }
  if (std::getenv("HPSB_TRACE")) {  // executed (tile-padded) vs useful flops per batch
    static double tu = 0, tp = 0;
    tu += flops, tp += padded;
    std::fprintf(stderr, "[gemm] descs %zu tiles %d useful %.3g padded %.3g (cum useful %.4g padded %.4g)\n",
                 descs.size(), total_tiles, flops, padded, tu, tp);
  }
  KernelScope ks(ctx, "zgemm_dmma", 0.0, flops);
  for (int sh = 0; sh < kShapes; ++sh) {
    if (!tiles[sh]) continue;
    const GemmDesc* dp = d_descs.p + first[sh];
    const int* mp = d_map.p + map_off[sh];
    switch (sh) {
      case 0: launch_gemm<4, 2>(ctx, tiles[sh], dp, mp); break;
      case 1: launch_gemm<4, 1>(ctx, tiles[sh], dp, mp); break;
      case 2: launch_gemm<3, 2>(ctx, tiles[sh], dp, mp); break;
      case 3: launch_gemm<3, 1>(ctx, tiles[sh], dp, mp); break;
      case 4: launch_gemm<2, 2>(ctx, tiles[sh], dp, mp); break;
      default: launch_gemm<2, 1>(ctx, tiles[sh], dp, mp); break;
    }
  }
}

void CopyBatch::add(const CopyOp& o0) {
  if (o0.rows <= 0 || o0.cols <= 0) return;
  ops.push_back(o0);
}

void CopyBatch::run(Context* ctx) {
  if (ops.empty()) return;
  total_tiles = 0;
  for (auto& o : ops) {
    o.tile_begin = total_tiles;
    total_tiles += (o.cols + 7) / 8;
  }
  d_ops.upload(ops, ctx->stream);
  {
    std::vector<int> map(total_tiles);
    for (size_t i = 0; i < ops.size(); ++i) {
      const int end = i + 1 < ops.size() ? ops[i + 1].tile_begin : total_tiles;
      std::fill(map.begin() + ops[i].tile_begin, map.begin() + end, static_cast<int>(i));
    }
    d_map.upload(map, ctx->stream);
  }
  double elems = 0;
  for (const auto& o : ops) elems += double(o.rows) * o.cols;
  KernelScope ks(ctx, "merge_copy", 32.0 * elems, 0.0);
  copy_ops_kernel<<<total_tiles, 128, 0, ctx->stream>>>(d_ops.p, d_map.p);
  HPSB_LAUNCHED(ctx);
}

// m0_out != null: m0_out[op] = max |a_ij|^2 of matrix op.  Else the growth
// check of a diagonal-pivot blocked inverse: any entry of A^{-1} beyond
// kGjHuge2 / m0_in[op] (or NaN) sets *guard.
// Grid (chunks, matrices): every CTA scans a contiguous slice of one
// matrix (column-major, ld >= n) and folds its max with an atomic on the
// order-preserving bits of a non-negative double (m0_out zeroed before).
// One CTA per matrix ran at 160 GB/s (a handful of CTAs per level).
__global__ void __launch_bounds__(256) absmax2_kernel(const InvOp* __restrict__ ops, double* m0_out,
                                                      const double* __restrict__ m0_in, int* guard) {
  __shared__ double red[8];
  const InvOp op = ops[blockIdx.y];
  const long long total = static_cast<long long>(op.n) * op.n;
  double m = 0.0;
  bool bad = false;
  for (long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(idx / op.n), i = static_cast<int>(idx - static_cast<long long>(j) * op.n);
    const double v = cabs2(op.A[(size_t)i + (size_t)j * op.lda]);
    m = fmax(m, v);
    bad |= !(v == v);
  }
  if (m0_out) {
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
      double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
      v = warp_max(v);
      if (threadIdx.x == 0)
        atomicMax(reinterpret_cast<unsigned long long*>(m0_out) + blockIdx.y,
                  static_cast<unsigned long long>(__double_as_longlong(v)));
    }
    return;
  }
  if (bad || !(m <= kGjHuge2 / fmax(m0_in[blockIdx.y], 1e-300))) *guard = 1;
}

dim3 absmax2_grid(size_t nmat, int nmax, int sms) {
  const long long per = static_cast<long long>(nmax) * nmax;
  const long long want = std::max<long long>(1, (4LL * sms + static_cast<long long>(nmat) - 1) / static_cast<long long>(nmat));
  return dim3(static_cast<unsigned>(std::min<long long>(want, (per + 255) / 256)), static_cast<unsigned>(nmat));
}

void InverseBatch::run(Context* ctx, int* status_dev) {
  std::vector<InvOp> small, large;
  int perm_total = 0;
  for (auto o : ops) {
    if (o.n <= kSmemInvMax) {
      small.push_back(o);
    } else {
      o.perm_off = perm_total;
      perm_total += o.n;
      large.push_back(o);
    }
  }
  if (!small.empty()) {
    int nmax = 0;
    for (const auto& o : small) nmax = std::max(nmax, o.n);
    d_small.upload(small, ctx->stream);
    double fl = 0;
    for (const auto& o : small) fl += 8.0 * o.n * double(o.n) * o.n;
    KernelScope ks(ctx, "zinverse_smem", 0.0, fl);
    const int grid = static_cast<int>(small.size());
    if (diag_pivots) {
      // per-matrix redo of guard failures; the diagonal blocks of a blocked
      // inverse cannot be redone alone and report to guard_dev instead
      int* flags = nullptr;
      if (!panel_blocks) {
        d_flags.alloc(small.size());
        HPSB_CUDA(cudaMemsetAsync(d_flags.p, 0, d_flags.bytes(), ctx->stream));
        flags = d_flags.p;
      }
      launch_inverse_dmma(nmax, grid, ctx->stream, d_small.p, flags, guard_dev);
      HPSB_LAUNCHED(ctx);
      if (flags) {
        launch_inverse_reg<2>(nmax, grid, ctx->stream, d_small.p, status_dev, flags, guard_dev);
        HPSB_LAUNCHED(ctx);
      }
    } else {
      launch_inverse_reg<0>(nmax, grid, ctx->stream, d_small.p, status_dev, nullptr, nullptr);
      HPSB_LAUNCHED(ctx);
    }
  }
  if (!large.empty()) {
    // Blocked Gauss-Jordan with partial pivoting: for each panel K of kb
    // columns, choose pivot rows by a panel LU, swap them in, invert the
    // pivot block P = A_KK^{-1} and sweep the rest of the matrix with grouped
    // DMMA GEMMs:  U = P A_KR,  A_RR -= A_RK U,  A_RK = -A_RK P,  A_KR = U.
    const int kb = kPivMaxKb;
    d_large.upload(large, ctx->stream);
    perm_ws.alloc(perm_total);
    int nmax = 0;
    for (const auto& o : large) nmax = std::max(nmax, o.n);
    // pivot-selection cluster: rows split so a CTA's panel slice fits in ~150 KB
    const int csize = std::min(kPivMaxCluster,
                               std::max(1, static_cast<int>((static_cast<size_t>(nmax) * kb * 16 + 150 * 1024 - 1) /
                                                            (150 * 1024))));
    const int chunk_max = (nmax + csize - 1) / csize;
    const size_t piv_smem = sizeof(double2) * static_cast<size_t>(kb) * chunk_max +
                            sizeof(int) * (chunk_max + 2 * static_cast<size_t>(nmax));
    static const bool piv_attr = [] {
      HPSB_CUDA(cudaFuncSetAttribute(panel_pivot_cluster_kernel,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      return true;
    }();
    (void)piv_attr;
    allow_smem<panel_pivot_cluster_kernel>(piv_smem);
    DevBuf<double2> panel(static_cast<size_t>(perm_total) * kb), U(static_cast<size_t>(perm_total) * kb),
        Q(static_cast<size_t>(perm_total) * kb);
    std::vector<InvOp> pivops(large.size());
    // diag_pivots needs a guard word for the diagonal blocks (no redo)
    const bool diag = diag_pivots && guard_dev;
    if (diag) {  // largest |a_ij|^2 of every input, for the final growth check
      d_m0.alloc(large.size());
      HPSB_CUDA(cudaMemsetAsync(d_m0.p, 0, sizeof(double) * large.size(), ctx->stream));
      KernelScope ks(ctx, "zinverse_guard", 16.0 * nmax * nmax * large.size(), 0.0);
      absmax2_kernel<<<absmax2_grid(large.size(), nmax, ctx->num_sms), 256, 0, ctx->stream>>>(
          d_large.p, d_m0.p, nullptr, nullptr);
      HPSB_LAUNCHED(ctx);
    }
    for (int k0 = 0; k0 < nmax; k0 += kb) {
      if (!diag) {
        KernelScope ks(ctx, "zinverse_panel", 0.0, 0.0);
          cudaLaunchConfig_t cfg{};
          cfg.gridDim = dim3(static_cast<unsigned>(large.size() * csize));
          cfg.blockDim = dim3(kPivThreads);
          cfg.dynamicSmemBytes = piv_smem;
          cfg.stream = ctx->stream;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = static_cast<unsigned>(csize);
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          HPSB_CUDA(cudaLaunchKernelEx(&cfg, panel_pivot_cluster_kernel, static_cast<const InvOp*>(d_large.p),
                                       k0, kb, chunk_max, perm_ws.p, status_dev));
          HPSB_LAUNCHED(ctx);
      }
      if (!diag) {
        KernelScope ks(ctx, "zinverse_swap", 0.0, 0.0);
        dim3 grid((nmax + 255) / 256, static_cast<unsigned>(large.size()));
        swap_rows_kernel<<<grid, 256, 0, ctx->stream>>>(d_large.p, k0, kb, perm_ws.p);
        HPSB_LAUNCHED(ctx);
      }
      InverseBatch piv;
      GemmBatch gu, gr;
      CopyBatch back;
      for (const auto& o : large) {
        if (k0 >= o.n) continue;
        const int n = o.n, kw = std::min(kb, n - k0), k1 = k0 + kw, tail = n - k1;
        double2* A = o.A;
        const size_t ld = o.lda;
        double2* AKK = A + k0 + k0 * ld;
        piv.ops.push_back(InvOp{AKK, kw, o.lda, o.tag, 0});
        double2* Ub = U.p + static_cast<size_t>(o.perm_off) * kb;  // kw x n, ld kw
        double2* Qb = Q.p + static_cast<size_t>(o.perm_off) * kb;  // n x kw, ld n
        // U = P A_KR (left and right column ranges)
        gu.add(AKK, o.lda, A + k0, o.lda, Ub, kw, kw, k0, kw, 1.0, 0.0);
        gu.add(AKK, o.lda, A + k0 + k1 * ld, o.lda, Ub + static_cast<size_t>(k1) * kw, kw, kw, tail,
               kw, 1.0, 0.0);
        // A_RR -= A_RK U (four blocks)
        for (int rb = 0; rb < 2; ++rb) {
          const int r0 = rb == 0 ? 0 : k1, rn = rb == 0 ? k0 : tail;
          for (int cb = 0; cb < 2; ++cb) {
            const int c0 = cb == 0 ? 0 : k1, cn = cb == 0 ? k0 : tail;
            gr.add(A + r0 + k0 * ld, o.lda, Ub + static_cast<size_t>(c0) * kw, kw,
                   A + r0 + c0 * ld, o.lda, rn, cn, kw, -1.0, 1.0);
          }
          // Q = -A_RK P (needs only P: same launch as U; both are a few dozen tiles)
          gu.add(A + r0 + k0 * ld, o.lda, AKK, o.lda, Qb + r0, n, rn, kw, kw, -1.0, 0.0);
          back.copy(Qb + r0, n, A + r0 + k0 * ld, o.lda, rn, kw, 1.0);
        }
        back.copy(Ub, kw, A + k0, o.lda, kw, k0, 1.0);
        back.copy(Ub + static_cast<size_t>(k1) * kw, kw, A + k0 + k1 * ld, o.lda, kw, tail, 1.0);
      }
      piv.diag_pivots = diag, piv.guard_dev = diag ? guard_dev : nullptr, piv.panel_blocks = true;
      piv.run(ctx, status_dev);  // in place: A_KK <- P (kw <= 32 uses the smem kernel)
      gu.run(ctx);
      gr.run(ctx);
      back.run(ctx);
    }
    if (diag) {  // no pivots, nothing to unscramble; check the inverse's growth
      KernelScope ks(ctx, "zinverse_guard", 16.0 * nmax * nmax * large.size(), 0.0);
      absmax2_kernel<<<absmax2_grid(large.size(), nmax, ctx->num_sms), 256, 0, ctx->stream>>>(
          d_large.p, nullptr, d_m0.p, guard_dev);
      HPSB_LAUNCHED(ctx);
      return;
    }
    KernelScope ks(ctx, "zinverse_swap", 0.0, 0.0);
    dim3 grid((nmax + 255) / 256, static_cast<unsigned>(large.size()));
    unscramble_kernel<<<grid, 256, 0, ctx->stream>>>(d_large.p, perm_ws.p);
    HPSB_LAUNCHED(ctx);
    // workspaces are released stream-ordered: no synchronisation needed
  }
}

}  // namespace hpsb
