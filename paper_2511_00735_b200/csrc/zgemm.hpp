// Batched dense complex kernels used by the merge stage (csrc/zgemm.cu).
#pragma once

#include <vector>

#include "internal.hpp"

namespace hpsb {

// C = alpha * A * B + beta * C, all column-major complex.  With Cin != null
// the beta term reads Cin (ld ldcin) on the column window [cin_c0, cin_c1)
// and zero outside it instead of C, and C is write-only: the merges take
// their additive terms from the child blocks where they lie, with no staging
// copy into C.
struct GemmDesc {
  const double2* A;
  const double2* B;
  double2* C;
  int M, N, K;
  int lda, ldb, ldc;
  double alpha_re, alpha_im, beta_re, beta_im;
  int tiles_m, tiles_n, tile_begin, ldcin;
  const double2* Cin;
  int cin_c0, cin_c1;
  int bm, bn;  // tile shape, chosen per problem by GemmBatch::run (64 / 48 / 32 rows, 64 / 32 columns)
};

struct GemmBatch {
  std::vector<GemmDesc> descs;
  int total_tiles = 0;
  double flops = 0;
  DevBuf<GemmDesc> d_descs;
  DevBuf<int> d_map;  // tile -> problem (one load per CTA instead of a binary search)
  int add(const GemmDesc& d);
  int add(const double2* A, int lda, const double2* B, int ldb, double2* C, int ldc, int M, int N,
          int K, double alpha, double beta) {
    GemmDesc d{};
    d.A = A, d.B = B, d.C = C, d.M = M, d.N = N, d.K = K, d.lda = lda, d.ldb = ldb, d.ldc = ldc;
    d.alpha_re = alpha, d.beta_re = beta;
    return add(d);
  }
  void run(Context* ctx);
};

// dst[r, c] = scale * src[ridx[r], cidx[c]] (identity / zero fills by mode).
struct CopyOp {
  enum Mode : int { kCopy = 0, kIdentity = 1, kZero = 2 };
  const double2* src;
  double2* dst;
  const int* ridx;
  const int* cidx;
  int lds, ldd, rows, cols;
  double scale;
  int mode, tile_begin;
};

struct CopyBatch {
  std::vector<CopyOp> ops;
  int total_tiles = 0;
  DevBuf<CopyOp> d_ops;
  DevBuf<int> d_map;  // tile -> op
  void add(const CopyOp& o);
  void copy(const double2* src, int lds, double2* dst, int ldd, int rows, int cols, double scale) {
    add(CopyOp{src, dst, nullptr, nullptr, lds, ldd, rows, cols, scale, CopyOp::kCopy, 0});
  }
  void gather(const double2* src, int lds, const int* ridx, const int* cidx, double2* dst, int ldd,
              int rows, int cols) {
    add(CopyOp{src, dst, ridx, cidx, lds, ldd, rows, cols, 1.0, CopyOp::kCopy, 0});
  }
  void identity(double2* dst, int ldd, int n) {
    add(CopyOp{nullptr, dst, nullptr, nullptr, 0, ldd, n, n, 1.0, CopyOp::kIdentity, 0});
  }
  void zero(double2* dst, int ldd, int rows, int cols) {
    add(CopyOp{nullptr, dst, nullptr, nullptr, 0, ldd, rows, cols, 1.0, CopyOp::kZero, 0});
  }
  void run(Context* ctx);
};

// In-place inverse of an n x n complex matrix (ld == n for the large path).
struct InvOp {
  double2* A;
  int n, lda, tag, perm_off;
};
constexpr int kSmemInvMax = 96;

// In-place complex inverses.  Default: partial pivoting.  diag_pivots:
// Gauss-Jordan on the diagonal (no pivot search, one barrier per column;
// blocked panels without pivot selection or row swaps), guarded: a pivot
// below 1e-10 max|a_ij| or an inverse entry beyond 1e10 / max|a_ij| marks
// the matrix.  Marked matrices of <= kSmemInvMax are redone with partial
// pivoting in the same call; a marked diagonal block of a blocked inverse
// sets guard_dev[0] = 1 instead (its caller redoes the whole build with
// pivoting, see build_hierarchy).
// Batched complex inverses in place.  diag_pivots: Gauss-Jordan on the
// diagonal (merge blocks W = I - T2_ss T1_ss), guarded (gj_reg.cuh):
//   register-resident matrices (n <= 96) that fail the guard are redone with
//   partial pivoting in the same call;
//   blocked matrices (n > 96) are checked per diagonal block and, at the end,
//   on every entry of the inverse against the input's largest entry; a
//   failure sets *guard_dev (the caller rebuilds with pivoting).
struct InverseBatch {
  std::vector<InvOp> ops;
  bool diag_pivots = false;
  bool panel_blocks = false;  // internal: the diagonal blocks of a blocked inverse
  int* guard_dev = nullptr;
  DevBuf<InvOp> d_small, d_large;
  DevBuf<int> perm_ws, d_flags;
  DevBuf<double> d_m0;
  void run(Context* ctx, int* status_dev);
};

}  // namespace hpsb
