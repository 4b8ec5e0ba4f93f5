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
struct SmallLevel {
  int level = 0, count = 0;
  size_t smem = 0;
  size_t batch_ops = 0, batch_vec = 0;  // multi-RHS smem: operators + per-RHS vectors
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
// rows_max: largest child perimeter P; vec_max: max(5 s, p1 + p2 + 3 s).
StreamLevel::Shape stream_level_shape(int rows_max, int s_max, int vec_max, int merges, int sms);

}  // namespace hpsb
