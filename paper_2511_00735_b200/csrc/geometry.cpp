// Host-side integer structure of the HPS discretisation: GLL rule, element
// index sets and the quadtree merge order of the interior faces.  These are
// tiny 1-D / integer computations done once per problem; they must be
// bit-identical to the reference, so they follow its exact sequences.
#include <cmath>
#include <cstring>

#include "internal.hpp"

namespace hpsb {

// GLL nodes, weights and barycentric differentiation matrix
// (proj/src/spectral.cpp:26-87).  The floating-point sequence (Newton from
// Chebyshev-Lobatto guesses, symmetrisation, pinned endpoints, normalised
// barycentric weights, negative-sum diagonal) is kept so that the nodes are
// bit-identical to the reference's.
Gll gll_rule(int order) {
  if (order < 1) throw InvalidArgument("gll_rule: order must be >= 1");
  const int np = order + 1;
  auto legendre = [order](double x, double& p_prev, double& p) {
    p_prev = 1.0;
    p = x;
    for (int k = 1; k < order; ++k) {
      const double next = ((2.0 * k + 1.0) * x * p - k * p_prev) / (k + 1.0);
      p_prev = p;
      p = next;
    }
  };
  Gll g;
  g.nodes.resize(np);
  g.weights.resize(np);
  for (int i = 0; i < np; ++i) {
    double x = -std::cos(M_PI * i / order);
    for (int it = 0; it < 100; ++it) {
      double a, b;
      legendre(x, a, b);
      const double step = (x * b - a) / (np * b);
      x -= step;
      if (std::abs(step) <= 1e-15) break;
    }
    g.nodes[i] = x;
  }
  for (int i = 0; i <= order / 2; ++i) {
    const double half = 0.5 * (g.nodes[i] - g.nodes[order - i]);
    g.nodes[i] = half;
    g.nodes[order - i] = -half;
  }
  g.nodes.front() = -1.0;
  g.nodes.back() = 1.0;
  if (order % 2 == 0) g.nodes[order / 2] = 0.0;
  for (int i = 0; i < np; ++i) {
    double a, b;
    legendre(g.nodes[i], a, b);
    g.weights[i] = 2.0 / (order * np * b * b);
  }
  std::vector<double> bw(np);
  double scale = 0.0;
  for (int i = 0; i < np; ++i) {
    double prod = 1.0;
    for (int j = 0; j < np; ++j)
      if (j != i) prod *= g.nodes[i] - g.nodes[j];
    bw[i] = 1.0 / prod;
    scale = std::max(scale, std::abs(bw[i]));
  }
  for (double& w : bw) w /= scale;
  g.diff.assign(static_cast<std::size_t>(np) * np, 0.0);
  for (int i = 0; i < np; ++i) {
    double acc = 0.0;
    for (int j = 0; j < np; ++j) {
      if (j == i) continue;
      const double d = (bw[j] / bw[i]) / (g.nodes[i] - g.nodes[j]);
      g.diff[i + static_cast<std::size_t>(j) * np] = d;
      acc += d;
    }
    g.diff[i + static_cast<std::size_t>(i) * np] = -acc;
  }
  return g;
}

// Corner-free index bookkeeping (proj/src/element.cpp:22-55): node (i, j)
// -> i (N+1) + j, sides ascending along the side, interior i-major.
IndexSets build_index_sets(int order) {
  if (order < 2) throw InvalidArgument("build_index_sets: order must be >= 2");
  const int np = order + 1;
  IndexSets s;
  s.order = order;
  for (int t = 1; t < order; ++t) {
    s.left.push_back(t);
    s.right.push_back(order * np + t);
    s.bottom.push_back(t * np);
    s.top.push_back(t * np + order);
  }
  for (auto* side : {&s.left, &s.right, &s.bottom, &s.top})
    s.boundary.insert(s.boundary.end(), side->begin(), side->end());
  for (int i = 1; i < order; ++i)
    for (int j = 1; j < order; ++j) s.interior.push_back(i * np + j);
  s.comp_of_full.assign(np * np, -1);
  for (int idx = 0, k = 0; idx < np * np; ++idx) {
    const int i = idx / np, j = idx % np;
    if ((i == 0 || i == order) && (j == 0 || j == order)) continue;
    s.noncorner.push_back(idx);
    s.comp_of_full[idx] = k++;
  }
  return s;
}

// Merge order of the interior faces (proj/src/skeleton.cpp:20-78): level
// 2k+1 joins 2^k x 2^k squares left-right (groups row-major), level 2k+2
// joins 2^{k+1} x 2^k boxes bottom-top (groups column-major).
FaceGraph build_face_graph(int n) {
  if (n < 2 || (n & (n - 1)) != 0)
    throw InvalidArgument("build_face_graph: n must be a power of two >= 2");
  int lg = 0;
  while ((1 << lg) < n) ++lg;
  FaceGraph g;
  g.n = n;
  g.face_of_element.assign(static_cast<std::size_t>(n) * n, {-1, -1, -1, -1});
  g.groups.resize(2 * lg);
  for (int level = 1; level <= 2 * lg; ++level) {
    const int first = g.num_faces();
    auto& lvl_groups = g.groups[level - 1];
    const bool across_x = (level & 1) == 1;
    const int k = across_x ? (level - 1) / 2 : level / 2;
    const int boxes_x = across_x ? (n >> (k + 1)) : (n >> k);
    const int boxes_y = n >> k;
    lvl_groups.resize(static_cast<std::size_t>(boxes_x) * boxes_y);
    const int faces_per_group = across_x ? (1 << k) : (1 << k);
    for (int gi = 0; gi < boxes_x * boxes_y; ++gi) {
      // x-merges enumerate groups row-major, y-merges column-major.
      const int a = across_x ? gi / boxes_x : gi % boxes_y;  // row index
      const int b = across_x ? gi % boxes_x : gi / boxes_y;  // column index
      for (int t = 0; t < faces_per_group; ++t) {
        int e1, e2, s1, s2;
        if (across_x) {
          const int line = (2 * b + 1) << k;  // vertical grid line
          const int row = (a << k) + t;
          e1 = row * n + line - 1, e2 = e1 + 1, s1 = 1, s2 = 0;
        } else {
          const int line = (2 * a + 1) << (k - 1);  // horizontal grid line
          const int col = (b << k) + t;
          e1 = (line - 1) * n + col, e2 = e1 + n, s1 = 3, s2 = 2;
        }
        const int id = g.num_faces();
        g.faces.push_back({e1, e2, s1, s2, level, gi});
        g.face_of_element[e1][s1] = id;
        g.face_of_element[e2][s2] = id;
        lvl_groups[gi].push_back(id);
      }
    }
    g.level_range.emplace_back(first, g.num_faces());
  }
  return g;
}

Partition make_partition(const FaceGraph& g, int G, int rank) {
  if (G < 1 || (G & (G - 1)) != 0) throw InvalidArgument("partition: ranks must be a power of two");
  if (rank < 0 || rank >= G) throw InvalidArgument("partition: rank out of range");
  Partition p;
  p.G = G, p.rank = rank, p.L = g.num_levels();
  while ((1 << p.g) < G) ++p.g;
  if (G > 1 && p.g > p.L - 1)
    throw InvalidArgument("partition: too many ranks for the mesh (need at least one local level)");
  p.last_local = p.L - p.g;
  const int ne = g.n * g.n;
  // Follow the merges of levels 1..last_local: after level l an element's
  // box is identified by the level-l group that produced it.
  std::vector<int> box(ne);
  for (int e = 0; e < ne; ++e) box[e] = e;
  std::vector<int> elem_first_box(ne);
  for (int level = 1; level <= p.last_local; ++level) {
    const auto& groups = g.groups[level - 1];
    std::vector<int> merged(ne, -1);  // old box id -> group id at this level
    for (int gi = 0; gi < static_cast<int>(groups.size()); ++gi) {
      const Face& f = g.faces[groups[gi][0]];
      merged[box[f.e1]] = gi;
      merged[box[f.e2]] = gi;
    }
    for (int e = 0; e < ne; ++e) box[e] = merged[box[e]];
  }
  p.elem_owner.resize(ne);
  for (int e = 0; e < ne; ++e) {
    p.elem_owner[e] = G == 1 ? 0 : box[e];
    if (p.elem_owner[e] == rank) p.own_elems.push_back(e);
  }
  p.face_owner.resize(g.num_faces());
  for (int f = 0; f < g.num_faces(); ++f)
    p.face_owner[f] = g.faces[f].level <= p.last_local ? p.elem_owner[g.faces[f].e1] : -1;
  if (G == 1) p.last_local = p.L;
  return p;
}

// Owner-computes rule of the sharded merges: a level's group (merge) runs on
// the rank holding its first child -- the box with the faces' e1 -- and the
// box it produces stays there.  Level 1's children are elements (their
// owners); the boxes entering a level are the previous level's groups.
std::vector<std::vector<int>> merge_owners(const FaceGraph& g, const Partition& part) {
  const int ne = g.n * g.n;
  std::vector<int> box(ne), box_owner(ne);
  for (int e = 0; e < ne; ++e) box[e] = e, box_owner[e] = part.elem_owner[e];
  std::vector<std::vector<int>> owners(g.num_levels());
  for (int level = 1; level <= g.num_levels(); ++level) {
    const auto& groups = g.groups[level - 1];
    std::vector<int>& own = owners[level - 1];
    own.resize(groups.size());
    std::vector<int> merged(ne, -1);
    for (size_t gi = 0; gi < groups.size(); ++gi) {
      const Face& f = g.faces[groups[gi][0]];
      own[gi] = box_owner[box[f.e1]];
      merged[box[f.e1]] = static_cast<int>(gi);
      merged[box[f.e2]] = static_cast<int>(gi);
    }
    for (int e = 0; e < ne; ++e) box[e] = merged[box[e]];
    box_owner = own;
  }
  return owners;
}

}  // namespace hpsb
