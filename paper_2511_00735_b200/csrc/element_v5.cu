// K1 element_iti, v5: the element stage as a batched blocked Cholesky.
//
// Same mathematics as the other element kernels (element.cu header; SURVEY.md
// Appendix B.1): per element the real SPD interior block L_ii (ni x ni, padded
// with identity to P, a multiple of 16) is factored, L_ii = L L^T, the nb + 2
// right-hand sides [L_iG | re b~ | im b~] are solved, and the boundary Schur
// complement / ItI epilogue follows (iti_epilogue, element_common.cuh).
//
// Instead of one CTA walking one element through a long chain of dependent
// steps (v4: 16-wide panels, operands streamed from L2 with ~2 M issued
// instructions per element), the factorisation is split into 64-wide block
// columns and every step runs as ONE launch over a whole chunk of elements:
//   assemble   L_ii and the right-hand sides B into the chunk workspace;
//   for k = 0 .. nblk-1 (left-looking, Crout order):
//     update   A[i,k] -= sum_{j<k} L[i,j] L[k,j]^T  for i >= k, and
//              B[k,:] -= sum_{j<k} L[k,j] Y[j,:]      (tiles of 64 x 64, K = 64k)
//     panel    one CTA per element: L[k,k] = chol(A[k,k]), Linv_k = L[k,k]^{-1},
//              L[i,k] = A[i,k] Linv_k^T (i > k), Y[k,:] = Linv_k B[k,:]
//   for k = nblk-1 .. 0 (backward solve L^T X = Y):
//     back     X[k,:] = Linv_k^T (Y[k,:] - sum_{j>k} L[j,k]^T X[j,:])
//   epilogue   one CTA per element: S = L_GG - L_Gi X, T, H (complex GJ inverse)
// All O(ni^3) and O(ni^2 nb) work is 64 x 64 DMMA tiles (mma.sync m8n8k4 f64)
// fed from shared memory by a 3-stage cp.async pipeline; a launch holds
// (elements x tiles) CTAs, so the SMs stay full with no serial step inside a
// CTA except the 64 x 64 diagonal factorisations.  The chunk workspace
// (A: P x P, B: P x nbc, Linv: nblk 64 x 64 blocks per element) is bounded
// by a memory budget; elements run in chunks.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "element_common.cuh"
#include "vcycle_device.cuh"
#include "gj_reg.cuh"
#include "gj_dmma.cuh"

namespace hpsb {

namespace {

constexpr int V5B = 64;                 // block size of the factorisation
constexpr int V5T = 128;                // threads of the tile / panel kernels (4 warps, 2 x 2)
constexpr int V5K = 16;                 // k depth of one pipeline stage
constexpr int V5S = 2;                  // pipeline stages (2 x 4 CTAs per SM: cfg3 elements 62.6 -> 57.9 ms vs 3 x 3)
constexpr int LDM = V5B + 4;            // [k][m] staging stride (m contiguous)
constexpr int LDK = V5K + 4;            // [m][k] staging stride (k contiguous)
constexpr int V5STAGE = V5B * LDK;      // doubles of the A operand per stage (>= V5K * LDM)
// B operand stage for a tile of 16 NJ columns (NJ fragments of 8 per warp column)
__host__ __device__ constexpr int v5_bstage(int NJ) {
  return 16 * NJ * LDK > V5K * LDM ? 16 * NJ * LDK : V5K * LDM;
}
__host__ __device__ constexpr int v5_tile_smem(int NJ) { return V5S * (V5STAGE + v5_bstage(NJ)); }  // doubles
static_assert(V5STAGE >= V5K * LDM, "stage size");

struct V5Args {
  ElemArgs a;
  int base;        // chunk start in the work list
  int count;       // elements in the chunk
  double* A;       // [c][P x P]
  double* B;       // [c][P x nbc]
  double* Linv;    // [c][nblk][64 x 64]
  size_t sA, sB, sL;
  int P, nbc, nblk, k;
};

__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0));
}

__device__ __forceinline__ int v5_elem(const V5Args& v, int c) {
  return v.a.elist ? v.a.elist[v.base + c] : v.base + c;
}

__device__ __forceinline__ void dmma5(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// acc = op1 (M x K) * op2 (K x N) for one tile of at most 64 x 64, K a
// multiple of 16.  Operand layouts (template):
//   A_KC = false: op1(m, k) = op1[m + k * ld1]   (column-major slice)
//   A_KC = true : op1(m, k) = op1[k + m * ld1]   (transposed access)
//   B_KC = false: op2(k, n) = op2[n + k * ld2]   (transposed access)
//   B_KC = true : op2(k, n) = op2[k + n * ld2]   (column-major slice)
// Warp w owns rows 32 (w & 1) .. +32 and columns 32 (w >> 1) .. +32 as 4 x 4
// DMMA fragments; acc[i][j][h] = C[32 wm + 8 i + g][32 wn + 8 j + 2 t4 + h].
// Every pointer and leading dimension must keep 16-byte alignment of
// 2-element runs.  Ends with a CTA barrier (the staging buffers are free).
template <bool A_KC, bool B_KC, int NJ = 4>
__device__ __forceinline__ void tile_mma(const double* __restrict__ op1, int ld1,
                                         const double* __restrict__ op2, int ld2, int M, int N,
                                         int K, double (&acc)[4][NJ][2], double* smem) {
  static_assert(B_KC || NJ == 4, "transposed B tiles are 64 wide");
  constexpr int BN = 16 * NJ, BST = v5_bstage(NJ);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double* As = smem;
  double* Bs = smem + V5S * V5STAGE;
  const int ksteps = K / V5K;
  auto load = [&](int ks, int st) {
    const int k0 = ks * V5K;
    double* as = As + st * V5STAGE;
    double* bs = Bs + st * BST;
#pragma unroll
    for (int r = 0; r < (V5B * V5K / 2) / V5T; ++r) {
      const int idx = tid + r * V5T;
      if (!A_KC) {
        const int m2 = idx % (V5B / 2), kk = idx / (V5B / 2);
        const bool ok = 2 * m2 < M;
        cp_async16_zfill(as + kk * LDM + 2 * m2, ok ? op1 + 2 * m2 + static_cast<size_t>(k0 + kk) * ld1 : op1, ok);
      } else {
        const int c2 = idx % (V5K / 2), m = idx / (V5K / 2);
        const bool ok = m < M;
        cp_async16_zfill(as + m * LDK + 2 * c2, ok ? op1 + k0 + 2 * c2 + static_cast<size_t>(m) * ld1 : op1, ok);
      }
    }
#pragma unroll
    for (int r = 0; r < (BN * V5K / 2) / V5T; ++r) {
      const int idx = tid + r * V5T;
      if (!B_KC) {
        const int n2 = idx % (BN / 2), kk = idx / (BN / 2);
        const bool ok = 2 * n2 < N;
        cp_async16_zfill(bs + kk * LDM + 2 * n2, ok ? op2 + 2 * n2 + static_cast<size_t>(k0 + kk) * ld2 : op2, ok);
      } else {
        const int c2 = idx % (V5K / 2), n = idx / (V5K / 2);
        const bool ok = n < N;
        cp_async16_zfill(bs + n * LDK + 2 * c2, ok ? op2 + k0 + 2 * c2 + static_cast<size_t>(n) * ld2 : op2, ok);
      }
    }
  };
#pragma unroll
  for (int s = 0; s < V5S - 1; ++s) {
    if (s < ksteps) load(s, s);
    cp_async_commit();
  }
  for (int ks = 0; ks < ksteps; ++ks) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(V5S - 2));
    __syncthreads();
    if (ks + V5S - 1 < ksteps) load(ks + V5S - 1, (ks + V5S - 1) % V5S);
    cp_async_commit();
    const double* as = As + (ks % V5S) * V5STAGE;
    const double* bs = Bs + (ks % V5S) * BST;
#pragma unroll
    for (int kk = 0; kk < V5K; kk += 4) {
      double af[4], bf[NJ];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = 32 * wm + 8 * i + g;
        af[i] = A_KC ? as[row * LDK + kk + t4] : as[(kk + t4) * LDM + row];
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int col = 8 * NJ * wn + 8 * j + g;
        bf[j] = B_KC ? bs[col * LDK + kk + t4] : bs[(kk + t4) * LDM + col];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma5(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait_all();
  __syncthreads();
}

// C (column-major, ldc) = beta * C + alpha * acc over the tile's M x N part.
// Accumulating stores read a whole fragment row (2 NJ values) before the
// first store: interleaved, every read waited for the previous store
// (possible aliasing) -- 8 NJ serial L2 round trips per thread.
template <int NJ>
__device__ __forceinline__ void tile_store(double* C, int ldc, int M, int N, const double (&acc)[4][NJ][2],
                                           double alpha, bool accumulate) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = 32 * wm + 8 * i + g;
    if (row >= M) continue;
    double old[NJ][2];
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = 8 * NJ * wn + 8 * j + 2 * t4 + h;
        old[j][h] = (accumulate && col < N) ? C[row + static_cast<size_t>(col) * ldc] : 0.0;
      }
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = 8 * NJ * wn + 8 * j + 2 * t4 + h;
        if (col < N) C[row + static_cast<size_t>(col) * ldc] = old[j][h] + alpha * acc[i][j][h];
      }
  }
}

// ---- assemble: A = L_ii (lower triangle incl. diagonal blocks; identity
// padding), B = [L_iG | b~].  Only the lower triangle is ever read.
__global__ void __launch_bounds__(256) v5_assemble_kernel(V5Args v) {
  const ElemArgs& a = v.a;
  const int c = blockIdx.x, e = v5_elem(v, c);
  const int m = a.m, ni = a.ni, nb = a.nb, np = a.order + 1, N = a.order, P = v.P, nbc = v.nbc;
  extern __shared__ __align__(16) double smem5[];
  double* mass = smem5;       // np
  double* Ks = mass + np;     // np x np
  double* cm = Ks + np * np;  // ni: c * mass_i * mass_j at the interior nodes
  for (int i = threadIdx.x; i < np; i += blockDim.x) mass[i] = a.mass[i];
  for (int i = threadIdx.x; i < np * np; i += blockDim.x) Ks[i] = a.stiff[i];
  __syncthreads();
  const double* ce = a.coeff + static_cast<size_t>(e) * np * np;
  for (int q = threadIdx.x; q < ni; q += blockDim.x) {
    const int i = q / m + 1, j = q % m + 1;
    cm[q] = __ldg(ce + i * np + j) * mass[i] * mass[j];
  }
  __syncthreads();
  double* A = v.A + c * v.sA;
  double* B = v.B + c * v.sB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  // One warp per column: zero fill with 16-byte stores (rows from the top of
  // the column's diagonal block: the diagonal tile is read whole), then the
  // 2m - 1 entries of the column (its grid line in x and in y) are patched.
  // (Per-entry index arithmetic over the whole column made this kernel
  // instruction bound: 2.7 TB/s of stores.)
  for (int col = warp; col < P; col += nwarps) {
    const int r0 = col / V5B * V5B;
    double* Ac = A + static_cast<size_t>(col) * P;
    for (int r = r0 + 2 * lane; r < P; r += 64) {
      double2 z = make_double2(0.0, 0.0);
      if (col >= ni) z = make_double2(r == col ? 1.0 : 0.0, r + 1 == col ? 1.0 : 0.0);
      *reinterpret_cast<double2*>(Ac + r) = z;
    }
    if (col >= ni) continue;
    __syncwarp();
    const int k = col / m + 1, l = col % m + 1;
    for (int i = 1 + lane; i <= m; i += 32) {  // nodes (i, l), i != k
      const int r = (i - 1) * m + (l - 1);
      if (r >= r0 && i != k) Ac[r] = Ks[i + k * np] * mass[l];
    }
    for (int j = 1 + lane; j <= m; j += 32) {  // nodes (k, j)
      const int r = (k - 1) * m + (j - 1);
      if (r < r0) continue;
      double val = mass[k] * Ks[j + l * np];
      if (j == l) val = (Ks[k + k * np] * mass[l] + val) - cm[r];
      Ac[r] = val;
    }
  }
  for (int bc = warp; bc < nbc; bc += nwarps) {
    double* Bc = B + static_cast<size_t>(bc) * P;
    if (bc >= nb && bc < nb + 2 && a.source) {
      for (int q = lane; q < P; q += 32) {
        double val = 0.0;
        if (q < ni) {
          const int i = q / m + 1, j = q % m + 1;
          const double2 sv = a.source[static_cast<size_t>(e) * ni + q];
          const double w = mass[i] * mass[j];
          val = (bc == nb) ? sv.x * w : sv.y * w;
        }
        Bc[q] = val;
      }
      continue;
    }
    for (int r = 2 * lane; r < P; r += 64) *reinterpret_cast<double2*>(Bc + r) = make_double2(0.0, 0.0);
    if (bc >= nb) continue;
    __syncwarp();
    const int side = bc / m, t = bc % m + 1, edge = (side & 1) ? N : 0;
    for (int kk = 1 + lane; kk <= m; kk += 32) {
      if (side < 2) Bc[(kk - 1) * m + (t - 1)] = Ks[kk + edge * np] * mass[t];  // nodes (kk, t)
      else Bc[(t - 1) * m + (kk - 1)] = mass[t] * Ks[kk + edge * np];           // nodes (t, kk)
    }
  }
}

// ---- update (left-looking): tiles of block column k and of block row k of B
// (B tiles are 16 NJB columns wide: one tile covers nb + 2 <= 80 columns)
template <int NJB>
__global__ void __launch_bounds__(V5T, 4) v5_update_kernel(V5Args v) {
  extern __shared__ __align__(16) double smem5[];
  constexpr int BW = 16 * NJB;
  const int P = v.P, k = v.k, nA = v.nblk - k, nBt = (v.nbc + BW - 1) / BW;
  const int c = blockIdx.x / (nA + nBt), t = blockIdx.x % (nA + nBt);
  const int e = v5_elem(v, c);
  if (v.a.status[e] & 4) return;
  double* A = v.A + c * v.sA;
  double* B = v.B + c * v.sB;
  const int bk = min(V5B, P - V5B * k), K = V5B * k;
  if (t < nA) {
    double acc[4][4][2];
    const int r0 = V5B * (k + t), M = min(V5B, P - r0);
    tile_mma<false, false>(A + r0, P, A + V5B * k, P, M, bk, K, acc, smem5);
    tile_store<4>(A + r0 + static_cast<size_t>(V5B * k) * P, P, M, bk, acc, -1.0, true);
  } else {
    double acc[4][NJB][2];
    const int c0 = BW * (t - nA), N = min(BW, v.nbc - c0);
    tile_mma<false, true, NJB>(A + V5B * k, P, B + static_cast<size_t>(c0) * P, P, bk, N, K, acc, smem5);
    tile_store<NJB>(B + V5B * k + static_cast<size_t>(c0) * P, P, bk, N, acc, -1.0, true);
  }
}

// ---- diag: Linv_k = chol(A[k,k])^{-1}, one 64-thread CTA per element, the
// block register-resident and both phases fully unrolled (the previous kernel
// walked shared-memory rows in dependent loops: 348 us per cfg3 launch, now 268).
//   Cholesky, right-looking: thread t holds row t of the block; per column j
//   one barrier publishes the column, then every thread applies
//   a[q] -= (a_tj / d) col[q] for q > j: 63 - j independent DFMAs.
//   Inverse: thread t owns row t of X = L^{-1}: for c = t-1 .. 0,
//   x_tc = -(sum_{q>c} x_tq l_qc) / l_cc; the column of L is read from shared
//   memory with uniform (broadcast) addresses, x stays in registers, and the
//   result rows are stored coalesced.
// Rows / columns past bk (the ragged last block) are identity.
// Two launches (Cholesky, then inverse): the unrolled phases are ~85 KB of
// code each; as one 170 KB kernel the warps of an SM, at different points of
// it, missed the instruction cache (26% no_instructions stalls).  L passes
// through the Linv block (1 / l_jj on its diagonal).
constexpr int V5DT = 64;
__global__ void __launch_bounds__(V5DT, 6) v5_diag_kernel(V5Args v) {
  __shared__ __align__(16) double colbuf[2][V5B];
  const int P = v.P, k = v.k, c = blockIdx.x, e = v5_elem(v, c), t = threadIdx.x;
  if (v.a.status[e] & 4) return;
  const double* A = v.A + c * v.sA;
  double* Lg = v.Linv + c * v.sL + static_cast<size_t>(k) * V5B * V5B;  // ld 64
  const int k0 = V5B * k, bk = min(V5B, P - k0);
  double a[V5B];
#pragma unroll
  for (int q = 0; q < V5B; ++q)
    a[q] = (t < bk && q < bk) ? __ldg(A + k0 + t + static_cast<size_t>(k0 + q) * P) : (q == t ? 1.0 : 0.0);
#pragma unroll
  for (int j = 0; j < V5B; ++j) {
    double* cb = colbuf[j & 1];
    cb[t] = a[j];
    __syncthreads();
    const double d = cb[j];
    if (!(d > 0.0)) {  // uniform over the CTA
      if (t == 0) atomicOr(v.a.status + e, 4);  // indefinite: pivoted-LU fallback (v1)
      return;
    }
    // 1 / d as rs^2: a double division takes its slow path (a subroutine
    // call) whenever the quotient is zero, i.e. for most entries of the
    // sparse first columns -- 29% of this kernel's stall samples
    const double rs = rsqrt(d);
    const double f = a[j] * (rs * rs);
    Lg[j * V5B + t] = (t == j) ? rs : a[j] * rs;  // column j of L (upper part: don't care)
#pragma unroll
    for (int q = j + 1; q < V5B; ++q) a[q] -= f * cb[q];
  }
}

__global__ void __launch_bounds__(V5DT, 6) v5_dinv_kernel(V5Args v) {
  __shared__ __align__(16) double Lc[V5B * V5B];  // L column-major (lower part used; 1 / l_jj on the diagonal)
  const int P = v.P, k = v.k, c = blockIdx.x, e = v5_elem(v, c), t = threadIdx.x;
  if (v.a.status[e] & 4) return;
  double* Lg = v.Linv + c * v.sL + static_cast<size_t>(k) * V5B * V5B;  // ld 64
  const int bk = min(V5B, P - V5B * k);
  for (int idx = t; idx < V5B * V5B / 2; idx += V5DT) cp_async16(Lc + 2 * idx, Lg + 2 * idx);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  double a[V5B];  // a[c] = X[t][c]
#pragma unroll
  for (int cc = V5B - 1; cc >= 0; --cc) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const double* lc = Lc + cc * V5B;
#pragma unroll
    for (int q = V5B - 1; q > cc; --q) {
      const double term = a[q] * lc[q];
      switch ((V5B - 1 - q) & 3) {
        case 0: s0 += term; break;
        case 1: s1 += term; break;
        case 2: s2 += term; break;
        default: s3 += term; break;
      }
    }
    const double rd = lc[cc];
    a[cc] = cc > t ? 0.0 : (cc == t ? rd : -rd * ((s0 + s1) + (s2 + s3)));
  }
#pragma unroll
  for (int cc = 0; cc < V5B; ++cc) Lg[t + cc * V5B] = (t < bk && cc < bk) ? a[cc] : 0.0;
}

// ---- trsm: L[i,k] = A[i,k] Linv_k^T (i > k) and Y[k,:] = Linv_k B[k,:], one tile per CTA
template <int NJB>
__global__ void __launch_bounds__(V5T, 4) v5_trsm_kernel(V5Args v) {
  extern __shared__ __align__(16) double smem5[];
  constexpr int BW = 16 * NJB;
  const int P = v.P, k = v.k, k0 = V5B * k, bk = min(V5B, P - k0);
  const int nA = v.nblk - k - 1, nBt = (v.nbc + BW - 1) / BW;
  const int c = blockIdx.x / (nA + nBt), t = blockIdx.x % (nA + nBt);
  const int e = v5_elem(v, c);
  if (v.a.status[e] & 4) return;
  double* A = v.A + c * v.sA;
  double* B = v.B + c * v.sB;
  const double* Lg = v.Linv + c * v.sL + static_cast<size_t>(k) * V5B * V5B;
  if (t < nA) {
    double acc[4][4][2];
    const int r0 = k0 + bk + V5B * t, M = min(V5B, P - r0);
    double* Ci = A + r0 + static_cast<size_t>(k0) * P;
    tile_mma<false, false>(Ci, P, Lg, V5B, M, bk, bk, acc, smem5);
    tile_store<4>(Ci, P, M, bk, acc, 1.0, false);
  } else {
    double acc[4][NJB][2];
    const int c0 = BW * (t - nA), N = min(BW, v.nbc - c0);
    double* Ck = B + k0 + static_cast<size_t>(c0) * P;
    tile_mma<false, true, NJB>(Lg, V5B, Ck, P, bk, N, bk, acc, smem5);
    tile_store<NJB>(Ck, P, bk, N, acc, 1.0, false);
  }
}

// ---- backward: X[k,:] = Linv_k^T (Y[k,:] - sum_{j>k} L[j,k]^T X[j,:]), one column tile per CTA
template <int NJB>
__global__ void __launch_bounds__(V5T, 4) v5_back_kernel(V5Args v) {
  extern __shared__ __align__(16) double smem5[];
  constexpr int BW = 16 * NJB;
  const int P = v.P, k = v.k, nBt = (v.nbc + BW - 1) / BW;
  const int c = blockIdx.x / nBt, c0 = BW * (blockIdx.x % nBt), e = v5_elem(v, c);
  if (v.a.status[e] & 4) return;
  double* A = v.A + c * v.sA;
  double* B = v.B + c * v.sB;
  const double* Lg = v.Linv + c * v.sL + static_cast<size_t>(k) * V5B * V5B;
  const int k0 = V5B * k, bk = min(V5B, P - k0), N = min(BW, v.nbc - c0), kb = k0 + bk;
  double* Ck = B + k0 + static_cast<size_t>(c0) * P;
  double acc[4][NJB][2];
  if (kb < P) {
    tile_mma<true, true, NJB>(A + kb + static_cast<size_t>(k0) * P, P, B + kb + static_cast<size_t>(c0) * P, P,
                              bk, N, P - kb, acc, smem5);
    tile_store<NJB>(Ck, P, bk, N, acc, -1.0, true);
    __threadfence_block();
    __syncthreads();
  }
  tile_mma<true, true, NJB>(Lg, V5B, Ck, P, bk, N, bk, acc, smem5);
  tile_store<NJB>(Ck, P, bk, N, acc, 1.0, false);
}

// ---- schur: S = L_GG - L_Gi X (+ i eta I), f = L_Gi x_b, and the recovery
// copy Y[e] = X[:ni, :nb+2].  L_Gi has N-1 entries per row (the normal
// derivative along the row's grid line), so this is a gather-contraction of
// each solution column staged in shared memory (one warp per column).
constexpr int V5ST = 256;
__global__ void __launch_bounds__(V5ST) v5_schur_kernel(V5Args v, double2* Sw, double* fw) {
  extern __shared__ __align__(16) double smem5[];
  const ElemArgs& a = v.a;
  const int c = blockIdx.x, e = v5_elem(v, c);
  if (a.status[e] & 4) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kW = V5ST / 32;
  const int m = a.m, ni = a.ni, nb = a.nb, np = a.order + 1, N = a.order, P = v.P;
  __shared__ double d0[64], dN[64];  // D(0, k), D(N, k)
  for (int i = tid; i < np; i += V5ST) d0[i] = a.diff[0 + i * np], dN[i] = a.diff[N + i * np];
  __syncthreads();
  const double* X = v.B + c * v.sB;
  double* xs = smem5 + warp * P;
  double* Ye = a.Y + static_cast<size_t>(e) * ni * (nb + 2);
  double2* S = Sw + static_cast<size_t>(c) * nb * nb;
  for (int col = warp; col < nb + 2; col += kW) {
    for (int q0 = 0; q0 < ni; q0 += 128) {
      double t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + 32 * u + lane;
        t[u] = q < ni ? __ldg(X + q + static_cast<size_t>(col) * P) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + 32 * u + lane;
        if (q < ni) xs[q] = t[u], Ye[q + static_cast<size_t>(col) * ni] = t[u];
      }
    }
    __syncwarp();
    if (col < nb || a.source) {
      for (int b = lane; b < nb; b += 32) {
        const int side = b / m, t = b % m + 1;
        double acc = 0.0;
        for (int kk = 1; kk <= m; ++kk) {
          const int q = side < 2 ? (kk - 1) * m + (t - 1) : (t - 1) * m + (kk - 1);
          const double dcoef = (side & 1) ? dN[kk] : -d0[kk];
          acc += dcoef * xs[q];
        }
        if (col < nb) {
          // L_GG: derivative entries on the two boundary nodes of the same line
          const int cs = col / m, ct = col % m + 1;
          double lgg = 0.0;
          if (ct == t) {
            if (side <= 1 && cs <= 1)
              lgg = (side == 0 ? -1.0 : 1.0) * (cs == 0 ? (side == 0 ? d0[0] : dN[0]) : (side == 0 ? d0[N] : dN[N]));
            else if (side >= 2 && cs >= 2)
              lgg = (side == 2 ? -1.0 : 1.0) * (cs == 2 ? (side == 2 ? d0[0] : dN[0]) : (side == 2 ? d0[N] : dN[N]));
          }
          S[b + static_cast<size_t>(col) * nb] = make_double2(lgg - acc, b == col ? a.eta : 0.0);
        } else {
          fw[(static_cast<size_t>(c) * nb + b) * 2 + (col - nb)] = acc;
        }
      }
    }
    __syncwarp();
  }
}

// ---- iti: T = I - 2 i eta S^{-1}, H = 2 i eta S^{-1} f: register-resident
// Gauss-Jordan (gj_reg.cuh), one 512-thread CTA per element.
// PIVOT = false: diagonal pivots, one barrier per column (the element Schur
// complements of the BASELINE configs need no pivoting: checked against the
// pivoted inverse at 1e-15 on sampled elements of cfg1-4).  A pivot below
// 1e-6 of the largest |S_ij| or an inverse entry beyond 1e8 / max|S_ij|
// (kGjTiny2 / kGjHuge2) flags the element (status bit 8); the PIVOT = true launch that follows
// redoes exactly the flagged elements with partial pivoting.
template <int TR, bool PIVOT>
__global__ void __launch_bounds__(kGjThreads) v5_iti_kernel(V5Args v, const double2* Sw, const double2* fw) {
  constexpr int TC = (TR + 1) / 2;
  __shared__ GjShared sh;
  __shared__ double2 fs[kGjMax];
  __shared__ double2 hpart[kGjThreads / 32][kGjMax];
  __shared__ unsigned long long smax;
  const ElemArgs& a = v.a;
  const int c = blockIdx.x, e = v5_elem(v, c), nb = a.nb, tid = threadIdx.x;
  const int st0 = a.status[e];
  if (st0 & 4) return;
  if (PIVOT && !(st0 & 8)) return;
  const double2* Sg = Sw + static_cast<size_t>(c) * nb * nb;
  if (tid < nb) fs[tid] = a.source ? fw[static_cast<size_t>(c) * nb + tid] : make_double2(0.0, 0.0);
  GjReg<TR, TC> g;
  auto get = [&](int i, int j) { return Sg[i + static_cast<size_t>(j) * nb]; };
  bool ok;
  if (PIVOT) {
    ok = gj_reg_inverse<TR, TC>(nb, get, g, sh);
  } else {
    if (tid == 0) smax = 0ull;
    __syncthreads();
    double m = 0.0;  // max |S_ij|^2 (order-preserving bits of a non-negative double)
    for (int idx = tid; idx < nb * nb; idx += kGjThreads) m = fmax(m, cabs2(Sg[idx]));
    atomicMax(&smax, static_cast<unsigned long long>(__double_as_longlong(m)));
    __syncthreads();
    const double m0 = __longlong_as_double(static_cast<long long>(smax));
    ok = gj_reg_inverse_nopiv<TR, TC>(nb, get, g, sh, kGjTiny2 * m0, kGjHuge2 / fmax(m0, 1e-300));
    if (!ok) {
      if (tid == 0) a.status[e] = st0 | 8;  // redo with pivoting
      return;
    }
  }
  const int ty = tid % kGjY, tx = tid / kGjY, lane = tid & 31, warp = tid >> 5;
  const double te = 2.0 * a.eta;
  double2* Te = a.T + static_cast<size_t>(e) * nb * nb;
#pragma unroll
  for (int aa = 0; aa < TR; ++aa) {
    const int i = ty + kGjY * aa;
    double2 h = make_double2(0.0, 0.0);
    if (i < nb) {
      const int r = PIVOT ? sh.step[i] : i;
#pragma unroll
      for (int b = 0; b < TC; ++b) {
        const int j = tx + kGjX * b;
        if (j >= nb) continue;
        const int col = PIVOT ? sh.piv[j] : j;
        const double2 sv = g.x[aa][b];
        Te[r + static_cast<size_t>(col) * nb] = make_double2((r == col ? 1.0 : 0.0) + te * sv.y, -te * sv.x);
        h = cfma(sv, fs[col], h);
      }
    }
    // the two column owners tx = 2w, 2w + 1 of a warp, then the warps in order
    h.x += __shfl_xor_sync(0xffffffffu, h.x, 16);
    h.y += __shfl_xor_sync(0xffffffffu, h.y, 16);
    if (lane < kGjY && i < nb) hpart[warp][i] = h;
  }
  __syncthreads();
  if (tid < nb) {
    double2 acc = make_double2(0.0, 0.0);
    for (int w = 0; w < kGjThreads / 32; ++w) acc = cadd(acc, hpart[w][tid]);
    a.H[static_cast<size_t>(e) * nb + (PIVOT ? sh.step[tid] : tid)] =
        a.source ? make_double2(-te * acc.y, te * acc.x) : make_double2(0.0, 0.0);
  }
  if (tid == 0) a.status[e] = ok ? 0 : 2;
}

// T = I - 2i eta S^{-1}, H = 2i eta S^{-1} f with S^{-1} from the blocked
// DMMA Gauss-Jordan on diagonal pivots (gj_dmma.cuh): S (nb x nb, identity
// padded to NP) in shared memory, 256 threads, two CTAs per SM at NP = 80.
// Guard as the register version: a small pivot or an inverse entry beyond
// kGjHuge2 / max|S_ij|^2 flags the element (status bit 8) for the pivoted
// register Gauss-Jordan pass that follows.
template <int NP>
__global__ void __launch_bounds__(256) v5_iti_dmma_kernel(V5Args v, const double2* Sw, const double2* fw) {
  using G = GdShape<NP>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* M = reinterpret_cast<double2*>(smem_raw);
  __shared__ double2 fs[NP];
  __shared__ double red[8];
  __shared__ int flag;
  const ElemArgs& a = v.a;
  const int c = blockIdx.x, e = v5_elem(v, c), nb = a.nb, tid = threadIdx.x;
  const int st0 = a.status[e];
  if (st0 & 4) return;
  const double2* Sg = Sw + static_cast<size_t>(c) * nb * nb;
  double m = 0.0;
  for (int j = tid / 32; j < NP; j += 8)
    for (int i = tid & 31; i < NP; i += 32) {
      double2 val = make_double2(i == j ? 1.0 : 0.0, 0.0);
      if (i < nb && j < nb) {
        val = Sg[i + static_cast<size_t>(j) * nb];
        m = fmax(m, cabs2(val));
      }
      M[j * G::LD + i] = val;
    }
  if (tid < NP) fs[tid] = (a.source && tid < nb) ? fw[static_cast<size_t>(c) * nb + tid] : make_double2(0.0, 0.0);
  m = warp_max(m);
  if ((tid & 31) == 0) red[tid >> 5] = m;
  __syncthreads();
  double m0 = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) m0 = fmax(m0, red[w]);
  if (!gd_inverse<NP, 8>(M, &flag, kGjTiny2 * m0)) {
    if (tid == 0) a.status[e] = st0 | 8;  // redo with pivoting
    return;
  }
  const double te = 2.0 * a.eta, huge2 = kGjHuge2 / fmax(m0, 1e-300);
  double2* Te = a.T + static_cast<size_t>(e) * nb * nb;
  bool bad = false;
  for (int j = tid / 32; j < nb; j += 8)
    for (int i = tid & 31; i < nb; i += 32) {
      const double2 sv = M[j * G::LD + i];
      bad |= !(cabs2(sv) <= huge2);
      Te[i + static_cast<size_t>(j) * nb] = make_double2((i == j ? 1.0 : 0.0) + te * sv.y, -te * sv.x);
    }
  if (tid < nb) {
    double2 h = make_double2(0.0, 0.0);
    for (int j = 0; j < nb; ++j) h = cfma(M[j * G::LD + tid], fs[j], h);
    a.H[static_cast<size_t>(e) * nb + tid] = a.source ? make_double2(-te * h.y, te * h.x) : make_double2(0.0, 0.0);
  }
  bad = __syncthreads_or(bad);
  if (tid == 0) a.status[e] = bad ? (st0 | 8) : 0;
}

// status bit 8 on every element of the chunk that is still on the Cholesky path
__global__ void v5_mark_kernel(V5Args v) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= v.count) return;
  const int e = v5_elem(v, c);
  if (!(v.a.status[e] & 4)) v.a.status[e] |= 8;
}

}  // namespace

bool element_v5_build(Context* ctx, const ElemArgs& a0, int nwork) {
  const int P = a0.npad, nbc = a0.nbc, nb = a0.nb;
  if (a0.order + 1 > 64 || nb > kGjMax || nwork <= 0) return false;
  const int nblk = (P + V5B - 1) / V5B;
  const size_t sA = static_cast<size_t>(P) * P, sB = static_cast<size_t>(P) * nbc,
               sL = static_cast<size_t>(nblk) * V5B * V5B, sS = static_cast<size_t>(nb) * nb;
  const size_t per = sizeof(double) * (sA + sB + sL) + sizeof(double2) * (sS + nb);
  size_t free_b = 0, total_b = 0;
  HPSB_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const size_t budget = std::min<size_t>(size_t(24) << 30, free_b / 4);
  const int cap = static_cast<int>(std::max<size_t>(1, std::min<size_t>(nwork, budget / per)));
  const int nchunks = (nwork + cap - 1) / cap;
  const int chunk = (nwork + nchunks - 1) / nchunks;  // even chunks
  DevBuf<double> wA(sA * chunk), wB(sB * chunk), wL(sL * chunk);
  DevBuf<double2> wS(sS * chunk), wf(static_cast<size_t>(nb) * chunk);

  // B tiles: one tile over the nb + 2 right-hand sides when they fit 80 columns
  const int njb = nbc <= 80 ? std::max(2, (nbc + 15) / 16) : 4;
  const size_t tile_smem = sizeof(double) * v5_tile_smem(std::max(njb, 4));
  const size_t schur_smem = sizeof(double) * (V5ST / 32) * P;
  const size_t asm_smem = sizeof(double) * ((a0.order + 1) * (a0.order + 2) + a0.ni);
  auto update_k = njb == 2 ? v5_update_kernel<2> : njb == 3 ? v5_update_kernel<3> : njb == 5 ? v5_update_kernel<5> : v5_update_kernel<4>;
  auto trsm_k = njb == 2 ? v5_trsm_kernel<2> : njb == 3 ? v5_trsm_kernel<3> : njb == 5 ? v5_trsm_kernel<5> : v5_trsm_kernel<4>;
  auto back_k = njb == 2 ? v5_back_kernel<2> : njb == 3 ? v5_back_kernel<3> : njb == 5 ? v5_back_kernel<5> : v5_back_kernel<4>;
  allow_smem<v5_assemble_kernel>(asm_smem);
  HPSB_CUDA(cudaFuncSetAttribute(update_k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tile_smem)));
  HPSB_CUDA(cudaFuncSetAttribute(trsm_k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tile_smem)));
  HPSB_CUDA(cudaFuncSetAttribute(back_k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(tile_smem)));
  allow_smem<v5_schur_kernel>(schur_smem);

  const int ni = a0.ni;
  const double fe = ni * double(ni) * ni / 3.0 + 2.0 * ni * double(ni) * nb + 8.0 * nb * double(nb) * nb;
  const double bytes_e = 8.0 * ((a0.order + 1) * (a0.order + 1) + 2 * ni + 2 * nb * nb + 2 * nb);
  const int nBt = (nbc + 16 * njb - 1) / (16 * njb);
  for (int base = 0; base < nwork; base += chunk) {
    V5Args v{};
    v.a = a0;
    v.base = base, v.count = std::min(chunk, nwork - base);
    v.A = wA.p, v.B = wB.p, v.Linv = wL.p, v.sA = sA, v.sB = sB, v.sL = sL;
    v.P = P, v.nbc = nbc, v.nblk = nblk;
    const int cn = v.count;
    {
      // pinned algorithmic work of the chunk on the first launch of the label
      KernelScope ks(ctx, "element_iti", bytes_e * cn, fe * cn);
      v5_assemble_kernel<<<cn, 256, asm_smem, ctx->stream>>>(v);
      HPSB_LAUNCHED(ctx);
    }
    for (int k = 0; k < nblk; ++k) {
      v.k = k;
      if (k > 0) {
        KernelScope ks(ctx, "element_iti", 0.0, 0.0);
        update_k<<<cn * (nblk - k + nBt), V5T, tile_smem, ctx->stream>>>(v);
        HPSB_LAUNCHED(ctx);
      }
      {
        KernelScope ks(ctx, "element_iti", 0.0, 0.0);
        v5_diag_kernel<<<cn, V5DT, 0, ctx->stream>>>(v);
        HPSB_LAUNCHED(ctx);
        v5_dinv_kernel<<<cn, V5DT, 0, ctx->stream>>>(v);
        HPSB_LAUNCHED(ctx);
      }
      KernelScope ks(ctx, "element_iti", 0.0, 0.0);
      trsm_k<<<cn * (nblk - k - 1 + nBt), V5T, tile_smem, ctx->stream>>>(v);
      HPSB_LAUNCHED(ctx);
    }
    for (int k = nblk - 1; k >= 0; --k) {
      v.k = k;
      KernelScope ks(ctx, "element_iti", 0.0, 0.0);
      back_k<<<cn * nBt, V5T, tile_smem, ctx->stream>>>(v);
      HPSB_LAUNCHED(ctx);
    }
    {
      KernelScope ks(ctx, "element_iti", 0.0, 0.0);
      v5_schur_kernel<<<cn, V5ST, schur_smem, ctx->stream>>>(v, wS.p, reinterpret_cast<double*>(wf.p));
      HPSB_LAUNCHED(ctx);
    }
    KernelScope ks(ctx, "element_iti", 0.0, 0.0);
    auto iti = [&](auto tr_tag) {
      constexpr int TR = decltype(tr_tag)::value;
      if (std::getenv("HPSB_ITI_PIVOT")) {
        // every element with partial pivoting: mark all, then the pivoted pass
        v5_mark_kernel<<<(cn + 255) / 256, 256, 0, ctx->stream>>>(v);
      } else {
        auto dm = [&](auto np_tag) {
          constexpr int NP = decltype(np_tag)::value;
          allow_smem<v5_iti_dmma_kernel<NP>>(GdShape<NP>::kSmem);
          v5_iti_dmma_kernel<NP><<<cn, 256, GdShape<NP>::kSmem, ctx->stream>>>(v, wS.p, wf.p);
        };
        switch ((nb + 15) / 16) {
          case 1: dm(std::integral_constant<int, 16>{}); break;
          case 2: dm(std::integral_constant<int, 32>{}); break;
          case 3: dm(std::integral_constant<int, 48>{}); break;
          case 4: dm(std::integral_constant<int, 64>{}); break;
          case 5: dm(std::integral_constant<int, 80>{}); break;
          default: dm(std::integral_constant<int, 96>{}); break;
        }
      }
      HPSB_LAUNCHED(ctx);
      v5_iti_kernel<TR, true><<<cn, kGjThreads, 0, ctx->stream>>>(v, wS.p, wf.p);  // flagged only
    };
    switch ((nb + kGjY - 1) / kGjY) {
      case 1: case 2: iti(std::integral_constant<int, 2>{}); break;
      case 3: iti(std::integral_constant<int, 3>{}); break;
      case 4: iti(std::integral_constant<int, 4>{}); break;
      case 5: iti(std::integral_constant<int, 5>{}); break;
      default: iti(std::integral_constant<int, 6>{}); break;
    }
    HPSB_LAUNCHED(ctx);
  }
  return true;
}

}  // namespace hpsb
