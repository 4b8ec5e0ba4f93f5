// Fused small-merge V-cycle step (csrc/vcycle_small.cu).
#pragma once

#include <string>

#include "internal.hpp"

namespace hpsb {

struct SmallMerge {
  const double2 *T1, *T2, *W;  // [p | s]-permuted child maps (ld P1 / P2), W (ld s)
  const int *in1s, *in2s, *in1p, *in2p, *out1p, *out2p;
  int s, p1, p2, P1, P2, pad;
};

// Shared memory one merge needs (operators + vectors).
size_t small_merge_smem(int s, int p1, int p2);

size_t small_merge_batch_smem(int s, int p1, int p2, int R);
size_t small_merge_batch_vec(int s, int p1, int p2, bool down);  // vector entries per RHS and direction
struct SmallLevel {
  int level = 0, count = 0;
  int max_s = 0;  // largest separator of the level (multi-RHS: DMMA tiles from 16 nodes up)
  size_t smem = 0;
  size_t batch_ops = 0, batch_vec = 0;  // multi-RHS smem: operators + per-RHS vectors (larger direction)
  size_t batch_vec_down = 0, batch_vec_up = 0;  // vector entries per RHS of each direction
  size_t batch_smem(int R) const { return batch_ops + static_cast<size_t>(R) * batch_vec; }
  double bytes_down = 0, bytes_up = 0;
  std::string label;
  DevBuf<SmallMerge> d;
  void run(Context* ctx, bool down, double2* r, double2* out) const;
  // R right-hand sides, vectors with RHS stride ld
  void run_batch(Context* ctx, bool down, double2* r, double2* out, int R, int64_t ld) const;
};

// One thread-block cluster of `csize` CTAs per merge (csrc/vcycle_cluster.cu).
size_t cluster_merge_smem(int s, int p1, int p2, int csize);
// Can a cluster of csize CTAs with this much shared memory each be resident?
bool cluster_merge_fits(size_t smem, int csize);
struct ClusterLevel {
  int level = 0, count = 0, csize = 1;
  size_t smem = 0;
  double bytes_down = 0, bytes_up = 0;
  std::string label;
  DevBuf<SmallMerge> d;
  void run(Context* ctx, bool down, double2* r, double2* out) const;
};

// One CTA per merge (persistent over the level), operators streamed through
// a TMA bulk-copy ring by a producer warp (csrc/vcycle_stream.cu): levels
// with >= one merge per SM whose child maps have at most 512 rows.
struct StreamLevel {
  struct Shape {
    bool ok = false;
    int rpl = 0;  // CTAs per SM
    bool pre_out = false;  // prefetch the epilogue's output bases with the inputs
    int warps = 0, ns = 0, slot_entries = 0, vec_entries = 0;  // consumer warps
    size_t smem = 0;
  };
  int level = 0, count = 0;
  Shape shape;
  double bytes_down = 0, bytes_up = 0;
  std::string label;
  DevBuf<SmallMerge> d;
  void run(Context* ctx, bool down, double2* r, double2* out) const;
};
// rows_max: largest child perimeter P; vec_in: max(5 s, p1 + p2 + 3 s) (the vector
// scratch), vec_all: 5 s + p1 + p2 (with the epilogue's output bases).
StreamLevel::Shape stream_level_shape(int rows_max, int vec_in, int vec_all, int merges, int sms);

// Independent streamed GEMVs y[yi] = x[yi] + A x[xi] (csrc/vcycle_stream.cu):
// the interface matvec over the element maps.
struct GemvItem {
  const double2* A;  // rows x cols, contiguous column-major
  const int* xi;     // [cols] (< 0: zero)
  const int* yi;     // [rows] (< 0: no output)
  int rows, cols;
};
struct GemvStream {
  struct Shape {
    bool ok = false;
    int warps = 0, ctas_per_sm = 0, ns = 0, slot_entries = 0, xs_entries = 0;
    size_t smem = 0;
  };
  Shape shape;
  int count = 0;
  double bytes = 0;
  std::string label = "skeleton_matvec";
  DevBuf<GemvItem> d;
  void run(Context* ctx, const double2* x, double2* y) const;
};
GemvStream::Shape gemv_stream_shape(int rows_max, int cols_max);

// Few-merge levels: one persistent launch per level step, the four stages
// separated by grid barriers (csrc/vcycle_wide.cu).
struct WideTile {
  const double2* A;  // operator origin of the tile (row r0, column c0)
  int rows, cols, ld, m, r0, c0, cb;
};
struct WideMerge {
  const int *in1s, *in2s, *in1p, *in2p, *out1p, *out2p;
  int s, p1, p2, pad;
  int R[4], ncb[4];  // per stage: output rows, column blocks
  long long part[4];  // per stage: offset of the [ncb][R] partial product
};
struct WideArgs {
  const WideTile* tiles;
  const int* cta_tiles;  // [4][grid + 1]: CTA b's tiles of stage k
  const WideMerge* merges;
  int nm;
  const int* row_prefix;  // [4][nm + 1] output-row prefix per stage
  double2* part;
  unsigned* bar;          // grid barrier: count, generation
  double2* r;
  double2* out;
  int down, slot_entries, tc_max, pad;
};
struct WideLevel {
  struct Shape {
    bool ok = false;
    int warps = 0, ctas_per_sm = 0, grid = 0, slot_entries = 0, tc_max = 0;
    size_t smem = 0;
  };
  struct Dir {
    WideArgs args{};
    int ntiles = 0;
    double bytes = 0;
    DevBuf<WideTile> tiles;
    DevBuf<WideMerge> merges;
    DevBuf<int> prefix, cta_tiles;
  };
  int level = 0;
  Shape shape;
  Dir dir[2];  // down, up
  DevBuf<double2> part;
  DevBuf<unsigned> bar;
  std::string label;
  void run(Context* ctx, bool down, double2* r, double2* out) const;
};
WideLevel::Shape wide_level_shape(int tc_max, int sms);

// The coarse gmres_fixed_steps as one persistent cooperative launch
// (csrc/vcycle_wide.cu); coarse_iters <= kCoarseWideMax.
constexpr int kCoarseWideMax = 8;
struct CoarseArgs {
  const WideTile* tiles;  // matvec tiles of the coarse box maps (m = box)
  const int* cta_tiles;   // [grid + 1]
  const WideMerge* boxes; // in1s = box input indices, R[0] / ncb[0] / part[0]
  const int* inv_box;     // coarse index -> (box, row of its map)
  const int* inv_row;
  double2* part;
  double2* V;             // (ci + 1) x n; V_0 is the right-hand side
  double2* W;             // n
  double2* pd;            // [grid][kCoarseWideMax + 1] partial dots
  double* pn;             // [grid] partial squared norms
  unsigned* bar;
  const double2* rhs;
  double2* z;
  int64_t n;
  int ci, slot_entries, tc_max, pad;
};
struct CoarseWide {
  WideLevel::Shape shape;
  CoarseArgs args{};
  double bytes = 0;
  DevBuf<WideTile> tiles;
  DevBuf<WideMerge> boxes;
  DevBuf<int> cta_tiles, inv_box, inv_row;
  DevBuf<double2> part, pd;
  DevBuf<double> pn;
  DevBuf<unsigned> bar;
  void run(Context* ctx, const double2* rhs, double2* z) const;
};
int coarse_wide_max_ctas_per_sm(size_t smem);
int wide_max_ctas_per_sm(size_t smem);

}  // namespace hpsb
