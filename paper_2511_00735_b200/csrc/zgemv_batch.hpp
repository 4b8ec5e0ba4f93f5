// Multi-RHS ("block") application of the per-iteration operators
// (csrc/zgemv_batch.cu).  With R right-hand sides every GEMV item of the
// single-RHS work lists -- y[yi] = beta y[yi] + gamma z[zi] + alpha A x[xi]
// -- becomes a complex GEMM with gathered B rows and scattered C rows,
//     Y[yi, :] = beta Y[yi, :] + gamma Z[zi, :] + alpha A X[xi, :],
// where X / Y / Z hold the R vectors column-wise (leading dimensions ldb /
// ldc / ldz).  Each operator element is then used R times (8R flops per 16
// bytes): the apply is FP64 compute bound and runs on the DMMA tensor cores.
#pragma once

#include <string>
#include <vector>

#include "internal.hpp"

namespace hpsb {

struct BDesc {
  const double2* A;  // M x K column-major (null: K == 0)
  const double2* B;  // rows bidx[k] (or k) of the R columns, ld ldb
  const int* bidx;
  double2* C;        // rows cidx[m] (or m), ld ldc
  const int* cidx;
  const double2* Z;  // rows zidx[m] (or m), ld ldz
  const int* zidx;
  int lda, M, K, ldb, ldc, ldz;
  double alpha, beta, gamma;
  int tiles_m, tile_begin, pad;
};

// Run-time rebinding: descriptors built on `from` address `to` instead
// (the caller's output block), so no copies are needed around a run.
struct BBind {
  const double2* from[2] = {nullptr, nullptr};
  double2* to[2] = {nullptr, nullptr};
};

// One launch: every descriptor's row tiles, R <= 32 right-hand sides.
struct BPhase {
  std::vector<BDesc> descs;
  int total_tiles = 0;
  int bm = 64;  // tile rows, chosen in finalize(): 32 when 64-row tiles would not fill the SMs
  double flops = 0, bytes = 0;
  std::string label;  // profiling name (overrides run()'s)
  DevBuf<BDesc> d;
  DevBuf<int> d_map;  // tile -> desc
  void add(const BDesc& x);
  void finalize(cudaStream_t s);
  void run(Context* ctx, int R, const char* label, BBind bind = {}) const;
};

constexpr int kBatchMaxRhs = 32;

}  // namespace hpsb
