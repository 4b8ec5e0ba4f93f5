// Level structures of the merge hierarchy (shared by hierarchy.cu / precond.cu).
#pragma once

#include <vector>

#include "internal.hpp"

namespace hpsb {

// One perimeter node of a box: global skeleton index of the box's own
// incoming datum (`in`) and of the neighbour's incoming datum across the same
// face node (`out`, the row its outgoing datum feeds).  -1 on physical sides.
struct BoxPos {
  int in, out;
};

// A box entering a level (a child of one of the level's merges), stored as
// its ItI map permuted to [perimeter | separator] order:
//   T = [[T_pp, T_ps], [T_sp, T_ss]],  P = p + s.
struct ChildBox {
  int P = 0, p = 0, s = 0;
  size_t t_off = 0;               // offset of the P x P map in LevelOps::tperm
  std::vector<BoxPos> pos;        // perm order
};

// One merge (group) of the level: child 2g (left / bottom box, holds the
// faces' e1) and child 2g+1.  W = (I - T2_ss T1_ss)^{-1}.
struct MergeRec {
  int c1 = 0, c2 = 0;
  int s = 0, p1 = 0, p2 = 0;
  int group = 0;  // group index within the level (face-graph order)
  // merges of the previous level that produced child 1 / child 2 (-1: an
  // element at level 1, or another rank's box)
  int src1 = -1, src2 = -1;
  size_t w_off = 0;
  // offsets (in ints) into LevelOps::idx of the V-cycle index lists
  size_t in1_sep = 0, in2_sep = 0, in1_per = 0, out1_per = 0, in2_per = 0, out2_per = 0;
};

struct LevelOps {
  int level = 0, first_face = 0, nfaces = 0;
  bool coarse = false;            // level == depth: boxes only, no merges
  std::vector<ChildBox> children;
  std::vector<MergeRec> merges;
  DevBuf<double2> tperm;
  DevBuf<double2> w;
  DevBuf<int> idx;
  std::vector<int> h_idx;
  double merge_flops = 0;
};

}  // namespace hpsb
