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

#include "device.cuh"
#include "internal.hpp"
#include "linalg.cuh"
#include "zgemm.hpp"

namespace hpsb {

namespace {
constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3, THREADS = 256;
constexpr int SA = BM + 2;  // complex stride of an A k-row in smem
constexpr int SB = BK + 4;  // complex stride of a B column in smem
constexpr int A_STAGE = BK * SA, B_STAGE = BN * SB;
constexpr size_t GEMM_SMEM = sizeof(double2) * STAGES * (A_STAGE + B_STAGE);

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

__global__ void __launch_bounds__(THREADS) zgemm_grouped_kernel(const GemmDesc* __restrict__ descs,
                                                                int ndesc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* As = reinterpret_cast<double2*>(smem_raw);
  double2* Bs = As + STAGES * A_STAGE;
  const int tile = blockIdx.x;
  // locate the problem owning this tile
  int lo = 0, hi = ndesc - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (descs[mid].tile_begin <= tile) lo = mid;
    else hi = mid - 1;
  }
  const GemmDesc d = descs[lo];
  const int local = tile - d.tile_begin;
  const int tm = local % d.tiles_m, tn = local / d.tiles_m;
  const int m0 = tm * BM, n0 = tn * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;  // 2 x 4 warps
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

  double cr[4][2][2], ci[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_async_commit();
  }
  const int arow = wm * 32 + (lane >> 2), kq = lane & 3;
  const int bcol = wn * 16 + (lane >> 2);
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (kt + STAGES - 1 < ktiles) load_stage(kt + STAGES - 1, (kt + STAGES - 1) % STAGES);
    cp_async_commit();
    const double2* as = As + (kt % STAGES) * A_STAGE;
    const double2* bs = Bs + (kt % STAGES) * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double2 a[4], b[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = as[(kk + kq) * SA + arow + i * 8];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = bs[(bcol + j * 8) * SB + kk + kq];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double nai = -a[i].y;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma(cr[i][j][0], cr[i][j][1], a[i].x, b[j].x);
          dmma(cr[i][j][0], cr[i][j][1], nai, b[j].y);
          dmma(ci[i][j][0], ci[i][j][1], a[i].x, b[j].y);
          dmma(ci[i][j][0], ci[i][j][1], a[i].y, b[j].x);
        }
      }
    }
  }
  cp_async_wait<0>();
  // epilogue: C = alpha * acc + beta * C
  const double2 alpha = make_double2(d.alpha_re, d.alpha_im);
  const double2 beta = make_double2(d.beta_re, d.beta_im);
  const bool use_beta = (d.beta_re != 0.0 || d.beta_im != 0.0);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + (lane >> 2);
    if (row >= d.M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * 16 + j * 8 + 2 * (lane & 3) + h;
        if (col >= d.N) continue;
        double2* c = d.C + (size_t)row + (size_t)col * d.ldc;
        double2 v = cmul(alpha, make_double2(cr[i][j][h], ci[i][j][h]));
        if (use_beta) v = cadd(v, cmul(beta, *c));
        *c = v;
      }
  }
}

// Sub-matrix copy / gather ops, tiled 8 columns per CTA.
__global__ void copy_ops_kernel(const CopyOp* __restrict__ ops, int nops) {
  const int tile = blockIdx.x;
  int lo = 0, hi = nops - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ops[mid].tile_begin <= tile) lo = mid;
    else hi = mid - 1;
  }
  const CopyOp op = ops[lo];
  const int c0 = (tile - op.tile_begin) * 8;
  const int c1 = min(c0 + 8, op.cols);
  for (int c = c0; c < c1; ++c) {
    const int sc = op.cidx ? op.cidx[c] : c;
    for (int r = threadIdx.x; r < op.rows; r += blockDim.x) {
      double2 v;
      if (op.mode == CopyOp::kIdentity) {
        v = make_double2(r == c ? 1.0 : 0.0, 0.0);
      } else if (op.mode == CopyOp::kZero) {
        v = make_double2(0.0, 0.0);
      } else {
        const int sr = op.ridx ? op.ridx[r] : r;
        v = cscale(op.src[(size_t)sr + (size_t)sc * op.lds], op.scale);
      }
      op.dst[(size_t)r + (size_t)c * op.ldd] = v;
    }
  }
}

// One CTA per matrix: complex Gauss-Jordan inverse (n <= kSmemInvMax in smem).
__global__ void __launch_bounds__(256) inverse_smem_kernel(const InvOp* __restrict__ ops,
                                                           int* status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const InvOp op = ops[blockIdx.x];
  double2* A = reinterpret_cast<double2*>(smem_raw);
  int* perm = reinterpret_cast<int*>(A + op.n * op.n);
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  for (int idx = threadIdx.x; idx < op.n * op.n; idx += blockDim.x) {
    const int r = idx % op.n, c = idx / op.n;
    A[idx] = op.A[(size_t)r + (size_t)c * op.lda];
  }
  __syncthreads();
  const bool ok = gj_inverse_cta(A, op.n, perm, red_v, red_i);
  for (int idx = threadIdx.x; idx < op.n * op.n; idx += blockDim.x) {
    const int r = idx % op.n, c = idx / op.n;
    op.A[(size_t)r + (size_t)c * op.lda] = A[idx];
  }
  if (threadIdx.x == 0 && !ok) status[0] = op.tag + 1;
}

// Large matrices: the same algorithm on global memory (ld == n required).
__global__ void __launch_bounds__(1024) inverse_global_kernel(const InvOp* __restrict__ ops,
                                                              int* perm_ws, int* status) {
  const InvOp op = ops[blockIdx.x];
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  const bool ok = gj_inverse_cta(op.A, op.n, perm_ws + op.perm_off, red_v, red_i);
  if (threadIdx.x == 0 && !ok) status[0] = op.tag + 1;
}
}  // namespace

int GemmBatch::add(const GemmDesc& d0) {
  if (d0.M <= 0 || d0.N <= 0) return -1;
  GemmDesc d = d0;
  d.tiles_m = (d.M + BM - 1) / BM;
  d.tiles_n = (d.N + BN - 1) / BN;
  d.tile_begin = total_tiles;
  total_tiles += d.tiles_m * d.tiles_n;
  flops += 8.0 * d.M * d.N * std::max(d.K, 0);
  descs.push_back(d);
  return static_cast<int>(descs.size()) - 1;
}

void GemmBatch::run(Context* ctx) {
  if (descs.empty()) return;
  // K == 0 problems still apply the epilogue (C = beta C): keep them valid.
  d_descs.upload(descs, ctx->stream);
  static bool attr = false;
  if (!attr) {
    HPSB_CUDA(cudaFuncSetAttribute(zgemm_grouped_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(GEMM_SMEM)));
    attr = true;
  }
  KernelScope ks(ctx, "zgemm_dmma", 0.0, flops);
  zgemm_grouped_kernel<<<total_tiles, THREADS, GEMM_SMEM, ctx->stream>>>(
      d_descs.p, static_cast<int>(descs.size()));
  HPSB_LAUNCHED(ctx);
}

void CopyBatch::add(const CopyOp& o0) {
  if (o0.rows <= 0 || o0.cols <= 0) return;
  CopyOp o = o0;
  o.tile_begin = total_tiles;
  total_tiles += (o.cols + 7) / 8;
  ops.push_back(o);
}

void CopyBatch::run(Context* ctx) {
  if (ops.empty()) return;
  d_ops.upload(ops, ctx->stream);
  double elems = 0;
  for (const auto& o : ops) elems += double(o.rows) * o.cols;
  KernelScope ks(ctx, "merge_copy", 32.0 * elems, 0.0);
  copy_ops_kernel<<<total_tiles, 128, 0, ctx->stream>>>(d_ops.p, static_cast<int>(ops.size()));
  HPSB_LAUNCHED(ctx);
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
    const size_t smem = sizeof(double2) * nmax * nmax + sizeof(int) * nmax + 16;
    HPSB_CUDA(cudaFuncSetAttribute(inverse_smem_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    d_small.upload(small, ctx->stream);
    double fl = 0;
    for (const auto& o : small) fl += 8.0 * o.n * double(o.n) * o.n;
    KernelScope ks(ctx, "zinverse_smem", 0.0, fl);
    inverse_smem_kernel<<<static_cast<int>(small.size()), 256, smem, ctx->stream>>>(d_small.p,
                                                                                 status_dev);
    HPSB_LAUNCHED(ctx);
  }
  if (!large.empty()) {
    d_large.upload(large, ctx->stream);
    perm_ws.alloc(perm_total);
    double fl = 0;
    for (const auto& o : large) fl += 8.0 * o.n * double(o.n) * o.n;
    KernelScope ks(ctx, "zinverse_global", 0.0, fl);
    inverse_global_kernel<<<static_cast<int>(large.size()), 1024, 0, ctx->stream>>>(
        d_large.p, perm_ws.p, status_dev);
    HPSB_LAUNCHED(ctx);
  }
}

}  // namespace hpsb
