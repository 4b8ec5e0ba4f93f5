// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp for the parity status).
// Restatement of the reference hps2d hot path; each function cites the
// reference file:line it follows (paths relative to the reference root).
#include "oracle.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <limits>
#include <set>
#include <thread>

namespace oracle {

namespace {
int g_threads = 1;             // host threads for the per-iteration operators (set_threads)
bool g_lean_elements = false;  // set_lean_elements
}  // namespace

// ===================== dense helpers ======================================
double CMat::max_abs() const {
  double m = 0.0;
  for (const auto& x : v) m = std::max(m, std::abs(x));
  return m;
}

CMat CMat::block(int r0, int c0, int nr, int nc) const {
  CMat out(nr, nc);
  for (int j = 0; j < nc; ++j)
    for (int i = 0; i < nr; ++i) out(i, j) = (*this)(r0 + i, c0 + j);
  return out;
}

void CMat::set_block(int r0, int c0, const CMat& b) {
  for (int j = 0; j < b.cols; ++j)
    for (int i = 0; i < b.rows; ++i) (*this)(r0 + i, c0 + j) = b(i, j);
}

void CMat::add_block(int r0, int c0, const CMat& b, cplx scale) {
  for (int j = 0; j < b.cols; ++j)
    for (int i = 0; i < b.rows; ++i) (*this)(r0 + i, c0 + j) += scale * b(i, j);
}

CMat matmul(const CMat& A, const CMat& B) {
  if (A.cols != B.rows) throw std::invalid_argument("matmul: shape mismatch");
  CMat C(A.rows, B.cols);
  for (int j = 0; j < B.cols; ++j) {
    cplx* c = C.col(j);
    for (int k = 0; k < A.cols; ++k) {
      const cplx b = B(k, j);
      if (b == cplx(0.0, 0.0)) continue;
      const cplx* a = A.col(k);
      for (int i = 0; i < A.rows; ++i) c[i] += a[i] * b;
    }
  }
  return C;
}

void gemv_acc(const CMat& A, const cplx* x, cplx* y, cplx alpha) {
  for (int k = 0; k < A.cols; ++k) {
    const cplx b = alpha * x[k];
    const cplx* a = A.col(k);
    for (int i = 0; i < A.rows; ++i) y[i] += a[i] * b;
  }
}

double norm2(const CVec& x) {
  double s = 0.0;
  for (const auto& z : x) s += std::norm(z);
  return std::sqrt(s);
}

cplx dotc(const CVec& a, const CVec& b) {
  cplx s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += std::conj(a[i]) * b[i];
  return s;
}

// Eigen::PartialPivLU semantics: P A = L U, unit lower L, largest-magnitude
// pivot in the current column.
PivLU::PivLU(const CMat& A) : lu(A) {
  if (A.rows != A.cols) throw std::invalid_argument("PivLU: square matrix required");
  const int n = A.rows;
  perm.resize(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::norm(lu(k, k));
    for (int i = k + 1; i < n; ++i) {
      const double s = std::norm(lu(i, k));
      if (s > best) best = s, p = i;
    }
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(lu(k, j), lu(p, j));
      std::swap(perm[k], perm[p]);
    }
    const cplx piv = lu(k, k);
    if (piv == cplx(0.0, 0.0)) continue;  // singular: left for min_abs_pivot
    const cplx inv = 1.0 / piv;
    cplx* ck = lu.col(k);
    for (int i = k + 1; i < n; ++i) ck[i] *= inv;
    for (int j = k + 1; j < n; ++j) {
      cplx* cj = lu.col(j);
      const cplx u = cj[k];
      if (u == cplx(0.0, 0.0)) continue;
      for (int i = k + 1; i < n; ++i) cj[i] -= ck[i] * u;
    }
  }
}

double PivLU::min_abs_pivot() const {
  double m = INFINITY;
  for (int i = 0; i < lu.rows; ++i) m = std::min(m, std::abs(lu(i, i)));
  return lu.rows ? m : 0.0;
}

void PivLU::solve_inplace(cplx* b, int nrhs, int ldb) const {
  const int n = lu.rows;
  CVec tmp(n);
  for (int r = 0; r < nrhs; ++r) {
    cplx* x = b + static_cast<std::size_t>(r) * ldb;
    for (int i = 0; i < n; ++i) tmp[i] = x[perm[i]];
    for (int k = 0; k < n; ++k) {  // L y = P b
      const cplx t = tmp[k];
      if (t == cplx(0.0, 0.0)) continue;
      const cplx* ck = lu.col(k);
      for (int i = k + 1; i < n; ++i) tmp[i] -= ck[i] * t;
    }
    for (int k = n - 1; k >= 0; --k) {  // U x = y
      tmp[k] /= lu(k, k);
      const cplx t = tmp[k];
      if (t == cplx(0.0, 0.0)) continue;
      const cplx* ck = lu.col(k);
      for (int i = 0; i < k; ++i) tmp[i] -= ck[i] * t;
    }
    for (int i = 0; i < n; ++i) x[i] = tmp[i];
  }
}

CMat PivLU::solve(const CMat& B) const {
  CMat X = B;
  solve_inplace(X.v.data(), X.cols, X.rows);
  return X;
}

CVec PivLU::solve(const CVec& b) const {
  CVec x = b;
  solve_inplace(x.data(), 1, static_cast<int>(x.size()));
  return x;
}

// ===================== spectral (spectral.cpp:12-98) =====================
namespace {
// P_{N-1}(x), P_N(x) by the three-term recurrence (spectral.cpp:12-21).
void legendre(int order, double x, double& pm, double& p) {
  pm = 1.0;
  p = x;
  for (int k = 1; k < order; ++k) {
    const double pn = ((2.0 * k + 1.0) * x * p - k * pm) / (k + 1.0);
    pm = p;
    p = pn;
  }
}
}  // namespace

Gll gll_rule(int order) {
  if (order < 1) throw std::invalid_argument("gll_rule: order must be >= 1");
  const int np = order + 1;
  Gll r;
  r.order = order;
  r.nodes.resize(np);
  r.weights.resize(np);
  // Newton on (1-x^2) P_N' from Chebyshev-Lobatto guesses (spectral.cpp:35-46).
  for (int i = 0; i < np; ++i) {
    double x = -std::cos(M_PI * i / order);
    for (int it = 0; it < 100; ++it) {
      double pm, p;
      legendre(order, x, pm, p);
      const double dx = (x * p - pm) / (np * p);
      x -= dx;
      if (std::abs(dx) <= 1e-15) break;
    }
    r.nodes[i] = x;
  }
  // Symmetrize, pin endpoints / centre (spectral.cpp:47-55).
  for (int i = 0; i <= order / 2; ++i) {
    const double s = 0.5 * (r.nodes[i] - r.nodes[order - i]);
    r.nodes[i] = s;
    r.nodes[order - i] = -s;
  }
  r.nodes[0] = -1.0;
  r.nodes[order] = 1.0;
  if (order % 2 == 0) r.nodes[order / 2] = 0.0;
  for (int i = 0; i < np; ++i) {  // spectral.cpp:57-61
    double pm, p;
    legendre(order, r.nodes[i], pm, p);
    r.weights[i] = 2.0 / (order * np * p * p);
  }
  // Barycentric differentiation matrix (spectral.cpp:63-86).
  std::vector<double> bary(np);
  double bmax = 0.0;
  for (int i = 0; i < np; ++i) {
    double w = 1.0;
    for (int j = 0; j < np; ++j)
      if (j != i) w *= r.nodes[i] - r.nodes[j];
    bary[i] = 1.0 / w;
    bmax = std::max(bmax, std::abs(bary[i]));
  }
  for (auto& b : bary) b /= bmax;
  r.diff.assign(static_cast<std::size_t>(np) * np, 0.0);
  for (int i = 0; i < np; ++i) {
    double rowsum = 0.0;
    for (int j = 0; j < np; ++j) {
      if (j == i) continue;
      const double d = (bary[j] / bary[i]) / (r.nodes[i] - r.nodes[j]);
      r.diff[i + static_cast<std::size_t>(j) * np] = d;
      rowsum += d;
    }
    r.diff[i + static_cast<std::size_t>(i) * np] = -rowsum;
  }
  return r;
}

Ops1D scale_to_element(const Gll& rule, double h) {  // spectral.cpp:89-98
  if (!(h > 0.0)) throw std::invalid_argument("scale_to_element: h must be > 0");
  const int np = rule.order + 1;
  Ops1D o;
  o.order = rule.order;
  o.h = h;
  o.mass.resize(np);
  o.diff.resize(static_cast<std::size_t>(np) * np);
  o.stiff.assign(static_cast<std::size_t>(np) * np, 0.0);
  for (int i = 0; i < np; ++i) o.mass[i] = (0.5 * h) * rule.weights[i];
  for (std::size_t k = 0; k < o.diff.size(); ++k) o.diff[k] = (2.0 / h) * rule.diff[k];
  // stiff = diff^T diag(mass) diff
  for (int j = 0; j < np; ++j)
    for (int i = 0; i < np; ++i) {
      double s = 0.0;
      for (int m = 0; m < np; ++m) s += (o.Dm(m, i) * o.mass[m]) * o.Dm(m, j);
      o.stiff[i + static_cast<std::size_t>(j) * np] = s;
    }
  return o;
}

// ===================== element (element.cpp:22-188) ======================
IndexSets build_index_sets(int order) {  // element.cpp:22-55
  if (order < 2) throw std::invalid_argument("build_index_sets: order must be >= 2");
  const int np = order + 1;
  IndexSets s;
  s.order = order;
  auto lin = [np](int i, int j) { return i * np + j; };
  for (int j = 1; j < order; ++j) s.left.push_back(lin(0, j));
  for (int j = 1; j < order; ++j) s.right.push_back(lin(order, j));
  for (int i = 1; i < order; ++i) s.bottom.push_back(lin(i, 0));
  for (int i = 1; i < order; ++i) s.top.push_back(lin(i, order));
  for (const auto* side : {&s.left, &s.right, &s.bottom, &s.top})
    s.boundary.insert(s.boundary.end(), side->begin(), side->end());
  for (int i = 1; i < order; ++i)
    for (int j = 1; j < order; ++j) s.interior.push_back(lin(i, j));
  s.comp_of_full.assign(np * np, -1);
  int pos = 0;
  for (int i = 0; i < np; ++i)
    for (int j = 0; j < np; ++j) {
      const bool corner = (i == 0 || i == order) && (j == 0 || j == order);
      if (corner) continue;
      s.noncorner.push_back(lin(i, j));
      s.comp_of_full[lin(i, j)] = pos++;
    }
  return s;
}

CMat assemble_local_pde(const Ops1D& ox, const Ops1D& oy, const CVec& coeff,
                        const IndexSets& sets) {  // element.cpp:57-90
  const int np = sets.order + 1;
  if (ox.order != sets.order || oy.order != sets.order)
    throw std::invalid_argument("assemble_local_pde: rule/order mismatch");
  if (static_cast<int>(coeff.size()) != np * np)
    throw std::invalid_argument("assemble_local_pde: coefficient grid mismatch");
  CMat L(sets.total(), sets.total());
  const auto& comp = sets.comp_of_full;
  for (int i = 0; i < np; ++i)
    for (int j = 0; j < np; ++j) {
      const int r = comp[i * np + j];
      if (r < 0) continue;
      for (int k = 0; k < np; ++k) {
        const int c = comp[k * np + j];
        if (c >= 0) L(r, c) += ox.K(i, k) * oy.mass[j];
      }
      for (int k = 0; k < np; ++k) {
        const int c = comp[i * np + k];
        if (c >= 0) L(r, c) += ox.mass[i] * oy.K(j, k);
      }
      L(r, r) -= coeff[i * np + j] * ox.mass[i] * oy.mass[j];
    }
  return L;
}

std::pair<CMat, CMat> impedance_operators(const IndexSets& sets, const Ops1D& ox,
                                          const Ops1D& oy, double eta) {  // element.cpp:92-125
  if (!(eta > 0.0)) throw std::invalid_argument("impedance: eta must be > 0");
  const int np = sets.order + 1;
  const int nb = static_cast<int>(sets.boundary.size());
  const auto& comp = sets.comp_of_full;
  CMat out(nb, sets.total()), in(nb, sets.total());
  for (int r = 0; r < nb; ++r) {
    const int full = sets.boundary[r];
    const int i = full / np, j = full % np;
    auto put = [&](int col, double d) { out(r, col) = d; in(r, col) = d; };
    if (i == 0) {
      for (int k = 0; k < np; ++k) put(comp[k * np + j], -ox.Dm(0, k));
    } else if (i == sets.order) {
      for (int k = 0; k < np; ++k) put(comp[k * np + j], ox.Dm(i, k));
    } else if (j == 0) {
      for (int k = 0; k < np; ++k) put(comp[i * np + k], -oy.Dm(0, k));
    } else {
      for (int k = 0; k < np; ++k) put(comp[i * np + k], oy.Dm(j, k));
    }
    const int c = comp[full];
    out(r, c) -= kI * eta;
    in(r, c) += kI * eta;
  }
  return {std::move(out), std::move(in)};
}

Element::Element(const Gll& rule, double h_, double eta_, const CVec& coeff_full)
    : order(rule.order), h(h_), eta(eta_), sets(build_index_sets(rule.order)) {
  // element.cpp:127-160
  ops = scale_to_element(rule, h);
  pde = assemble_local_pde(ops, ops, coeff_full, sets);
  std::tie(imp_out, imp_in) = impedance_operators(sets, ops, ops, eta);
  op = pde;
  const int nb = static_cast<int>(sets.boundary.size());
  for (int r = 0; r < nb; ++r) {
    const int row = sets.comp_of_full[sets.boundary[r]];
    for (int c = 0; c < sets.total(); ++c) op(row, c) = imp_in(r, c);
  }
  factor = PivLU(op);
  if (!(factor.min_abs_pivot() > 0.0))
    throw std::runtime_error("ElementOperators: singular local operator");
  CMat rhs(sets.total(), nb);
  for (int r = 0; r < nb; ++r) rhs(sets.comp_of_full[sets.boundary[r]], r) = 1.0;
  iti = matmul(imp_out, factor.solve(rhs));
  const int np = order + 1;
  mass2d.resize(sets.total());
  for (int k = 0; k < sets.total(); ++k) {
    const int full = sets.noncorner[k];
    mass2d[k] = ops.mass[full / np] * ops.mass[full % np];
  }
}

CVec Element::source_to_outgoing(const CVec& src) const {  // element.cpp:167-174
  if (src.size() != sets.interior.size())
    throw std::invalid_argument("source_to_outgoing: interior size mismatch");
  CVec b(sets.total());
  for (std::size_t k = 0; k < sets.interior.size(); ++k)
    b[sets.comp_of_full[sets.interior[k]]] = src[k];
  const CVec u = factor.solve(b);
  CVec out(imp_out.rows);
  gemv_acc(imp_out, u.data(), out.data(), 1.0);
  return out;
}

CVec Element::solve(const CVec& g, const CVec& src) const {  // element.cpp:176-188
  CVec b(sets.total());
  for (std::size_t r = 0; r < sets.boundary.size(); ++r) b[sets.comp_of_full[sets.boundary[r]]] = g[r];
  for (std::size_t k = 0; k < sets.interior.size(); ++k)
    b[sets.comp_of_full[sets.interior[k]]] = src[k];
  return factor.solve(b);
}

// ===================== mesh (mesh.cpp:36-109) ============================
namespace {
template <class F>
void parallel_for(int count, int threads, F&& fn) {
  if (threads <= 1 || count <= 1) {
    for (int i = 0; i < count; ++i) fn(i);
    return;
  }
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::atomic<bool> failed{false};
  for (int t = 0; t < std::min(threads, count); ++t)
    pool.emplace_back([&] {
      for (int i = next++; i < count && !failed; i = next++) {
        try {
          fn(i);
        } catch (...) {
          if (!failed.exchange(true)) err = std::current_exception();
        }
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}
}  // namespace

std::vector<ElementRecord> build_elements(const Mesh& mesh, const Gll& rule, int threads) {
  const int np = mesh.order + 1, m = mesh.order - 1;
  const double h = mesh.h();
  const IndexSets sets = build_index_sets(mesh.order);
  const int ne = mesh.n * mesh.n;
  std::vector<ElementRecord> recs(ne);
  // The reference shares factorizations between elements with bit-identical
  // coefficient samples (mesh.cpp:66-87); that cache changes no value, so the
  // oracle builds every element.
  parallel_for(ne, threads, [&](int e) {
    ElementRecord& rec = recs[e];
    rec.ox = h * (e % mesh.n);
    rec.oy = h * (e / mesh.n);
    CVec coeff(np * np);
    for (int k = 0; k < np * np; ++k) coeff[k] = mesh.coeff[static_cast<std::size_t>(e) * np * np + k];
    try {
      rec.ops = std::make_shared<Element>(rule, h, mesh.eta, coeff);
    } catch (const std::runtime_error& ex) {
      throw std::runtime_error("element " + std::to_string(e) + ": " + ex.what());
    }
    rec.interior_source.resize(m * m);
    bool zero = true;
    for (std::size_t k = 0; k < sets.interior.size(); ++k) {
      const cplx s = mesh.source[static_cast<std::size_t>(e) * m * m + k];
      rec.interior_source[k] = s * rec.ops->mass2d[sets.comp_of_full[sets.interior[k]]];
      if (s != cplx(0.0, 0.0)) zero = false;
    }
    rec.outgoing_source =
        zero ? CVec(4 * m, cplx(0.0, 0.0)) : rec.ops->source_to_outgoing(rec.interior_source);
    if (g_lean_elements) {
      // keep T (and mass2d) only: the t x t operators and the LU factor are
      // ~10 MB per element at N = 20 (160 GB for cfg3) and only the solution
      // recovery needs them
      Element& el = *rec.ops;
      el.pde = CMat(), el.op = CMat(), el.imp_out = CMat(), el.imp_in = CMat();
      el.factor = PivLU();
    }
  });
  return recs;
}

// ===================== face graph / skeleton (skeleton.cpp) ==============
FaceGraph build_face_graph(int n) {  // skeleton.cpp:20-78
  if (n < 2 || (n & (n - 1)) != 0)
    throw std::invalid_argument("build_face_graph: n must be a power of two >= 2");
  int m = 0;
  while ((1 << m) < n) ++m;
  FaceGraph g;
  g.n = n;
  g.face_of_element.assign(n * n, {-1, -1, -1, -1});
  g.groups.resize(2 * m);
  auto add = [&](int level, int group, int e1, int e2, int s1, int s2) {
    const int id = static_cast<int>(g.faces.size());
    g.faces.push_back({e1, e2, s1, s2, level, group});
    g.face_of_element[e1][s1] = id;
    g.face_of_element[e2][s2] = id;
    g.groups[level - 1][group].push_back(id);
  };
  for (int level = 1; level <= 2 * m; ++level) {
    const int begin = static_cast<int>(g.faces.size());
    if (level % 2 == 1) {  // merges across vertical grid lines
      const int k = (level - 1) / 2, half = 1 << k;
      const int cols = n >> (k + 1), rows = n >> k;
      g.groups[level - 1].resize(cols * rows);
      int group = 0;
      for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c, ++group)
          for (int t = 0; t < half; ++t) {
            const int fx = (2 * c + 1) * half, fy = r * half + t;
            add(level, group, fy * n + fx - 1, fy * n + fx, kRight, kLeft);
          }
    } else {  // merges across horizontal grid lines, column-major groups
      const int k = level / 2, wide = 1 << k, half = 1 << (k - 1);
      const int cols = n >> k, rows = n >> k;
      g.groups[level - 1].resize(cols * rows);
      int group = 0;
      for (int c = 0; c < cols; ++c)
        for (int r = 0; r < rows; ++r, ++group)
          for (int t = 0; t < wide; ++t) {
            const int fy = (2 * r + 1) * half, fx = c * wide + t;
            add(level, group, (fy - 1) * n + fx, fy * n + fx, kTop, kBottom);
          }
    }
    g.level_range.emplace_back(begin, static_cast<int>(g.faces.size()));
  }
  return g;
}

CMat& BlockMatrix::block(int r, int c) {  // block_matrix.cpp:9-16
  if (r < 0 || r >= nblocks || c < 0 || c >= nblocks)
    throw std::out_of_range("BlockMatrix::block: index out of range");
  auto it = blocks.find({r, c});
  if (it == blocks.end()) it = blocks.emplace(std::make_pair(r, c), CMat(bs, bs)).first;
  return it->second;
}

const CMat* BlockMatrix::find(int r, int c) const {
  auto it = blocks.find({r, c});
  return it == blocks.end() ? nullptr : &it->second;
}

namespace {

// fn(key, block) for every stored block with block row in [r0, r1), block
// rows split into contiguous chunks over the threads.  Each block row is
// visited by one thread in the map's (column-ascending) order, so the
// accumulation order per row -- and every result bit -- equals the serial
// loop's.
template <class F>
void for_block_rows(const BlockMatrix& M, int r0, int r1, F&& fn) {
  const int rows = r1 - r0;
  const int chunks = (g_threads <= 1 || M.blocks.size() < 2048) ? 1 : 8 * g_threads;
  const int per = std::max(1, (rows + chunks - 1) / chunks);
  const int nchunk = (rows + per - 1) / per;
  parallel_for(nchunk, g_threads, [&](int k) {
    const int a = r0 + k * per, b = std::min(r1, a + per);
    auto it = M.blocks.lower_bound({a, std::numeric_limits<int>::min()});
    const auto end = M.blocks.lower_bound({b, std::numeric_limits<int>::min()});
    for (; it != end; ++it) fn(it->first, it->second);
  });
}
}  // namespace

void set_threads(int threads) { g_threads = std::max(1, threads); }
void set_lean_elements(bool lean) { g_lean_elements = lean; }

CVec BlockMatrix::apply(const CVec& v) const {  // block_matrix.cpp:23-31
  if (v.size() != dim()) throw std::invalid_argument("BlockMatrix::apply: size mismatch");
  CVec y(dim());
  for_block_rows(*this, 0, nblocks, [&](const std::pair<int, int>& key, const CMat& blk) {
    gemv_acc(blk, v.data() + static_cast<std::size_t>(key.second) * bs,
             y.data() + static_cast<std::size_t>(key.first) * bs, 1.0);
  });
  return y;
}

CMat BlockMatrix::to_dense_sub(int r0, int r1, int c0, int c1) const {
  CMat out((r1 - r0) * bs, (c1 - c0) * bs);
  for (const auto& [key, blk] : blocks) {
    if (key.first < r0 || key.first >= r1 || key.second < c0 || key.second >= c1) continue;
    out.set_block((key.first - r0) * bs, (key.second - c0) * bs, blk);
  }
  return out;
}

CMat BlockMatrix::to_dense() const { return to_dense_sub(0, nblocks, 0, nblocks); }

std::size_t BlockMatrix::storage_bytes() const {
  std::size_t b = 0;
  for (const auto& kv : blocks) b += sizeof(cplx) * kv.second.v.size();
  return b;
}

SkeletonSystem assemble_skeleton(const Mesh& mesh, const std::vector<ElementRecord>& elements) {
  // skeleton.cpp:88-137
  if (static_cast<int>(elements.size()) != mesh.n * mesh.n)
    throw std::invalid_argument("assemble_skeleton: element operators missing");
  SkeletonSystem sys;
  sys.graph = build_face_graph(mesh.n);
  sys.side_len = mesh.order - 1;
  const int bs = sys.block_size(), sl = sys.side_len;
  sys.M = BlockMatrix(sys.graph.num_faces(), bs);
  sys.rhs.assign(sys.M.dim(), cplx(0.0, 0.0));
  for (int f = 0; f < sys.graph.num_faces(); ++f) {
    const Face& face = sys.graph.faces[f];
    for (int slot = 0; slot < 2; ++slot) {
      const int eid = slot == 0 ? face.e1 : face.e2;
      const int alpha = slot == 0 ? face.s1 : face.s2;
      const ElementRecord& rec = elements[eid];
      CMat& diag = sys.M.block(f, f);
      for (int k = 0; k < sl; ++k) diag(slot * sl + k, slot * sl + k) = 1.0;
      cplx* rhs = sys.rhs.data() + static_cast<std::size_t>(f) * bs + slot * sl;
      for (int k = 0; k < sl; ++k) rhs[k] = -rec.outgoing_source[alpha * sl + k];
      for (int gamma = 0; gamma < 4; ++gamma) {
        const CMat tb = rec.ops->iti_block(alpha, gamma);
        const int fg = sys.graph.face_of_element[eid][gamma];
        if (fg >= 0) {
          const int cslot = sys.graph.faces[fg].e1 == eid ? 1 : 0;
          sys.M.block(f, fg).add_block(slot * sl, cslot * sl, tb);
        } else {
          const cplx* t = mesh.tside.data() + (static_cast<std::size_t>(eid) * 4 + gamma) * sl;
          gemv_acc(tb, t, rhs, -1.0);
        }
      }
    }
  }
  return sys;
}

LevelPartition partition_level(const FaceGraph& g, int first_face, int level) {
  // skeleton.cpp:139-158
  if (level < 1 || level > g.num_levels())
    throw std::invalid_argument("partition_level: level out of range");
  const auto [begin, end] = g.level_range[level - 1];
  if (begin != first_face)
    throw std::logic_error("partition_level: level's faces are not leading in this system");
  LevelPartition p;
  p.level = level;
  p.a_faces = end - begin;
  for (const auto& grp : g.groups[level - 1]) {
    std::vector<int> local;
    for (int f : grp) local.push_back(f - first_face);
    p.groups.push_back(std::move(local));
  }
  return p;
}

// ===================== dissection (dissection.cpp) =======================
int FusedPair::side_position(int element, int side, int alpha, int beta) {
  // dissection.cpp:11-21
  const int skip = element == 0 ? alpha : beta;
  if (side == skip) return -1;
  int pos = 0;
  for (int s = 0; s < 4; ++s) {
    if (s == skip) continue;
    if (s == side) return (element == 0 ? 0 : 3) + pos;
    ++pos;
  }
  return -1;
}

FusedPair merge_pair(const CMat& T1, const CVec& H1, const CMat& T2, const CVec& H2,
                     int alpha, int beta, int m) {  // dissection.cpp:23-82
  if (T1.rows != 4 * m || T2.rows != 4 * m || T1.cols != 4 * m || T2.cols != 4 * m ||
      static_cast<int>(H1.size()) != 4 * m || static_cast<int>(H2.size()) != 4 * m)
    throw std::invalid_argument("merge_pair: operator dimensions mismatch");
  auto blk = [m](const CMat& T, int a, int b) { return T.block(a * m, b * m, m, m); };
  std::vector<int> ext1, ext2;
  for (int s = 0; s < 4; ++s) {
    if (s != alpha) ext1.push_back(s);
    if (s != beta) ext2.push_back(s);
  }
  CMat A = CMat::identity(2 * m);
  A.set_block(0, m, blk(T1, alpha, alpha));
  A.set_block(m, 0, blk(T2, beta, beta));
  CMat B(2 * m, 6 * m), C(6 * m, 2 * m), D(6 * m, 6 * m);
  CVec hext(6 * m), hface(2 * m);
  for (int k = 0; k < 3; ++k) {
    B.add_block(0, k * m, blk(T1, alpha, ext1[k]), -1.0);
    B.add_block(m, (3 + k) * m, blk(T2, beta, ext2[k]), -1.0);
    C.set_block(k * m, m, blk(T1, ext1[k], alpha));
    C.set_block((3 + k) * m, 0, blk(T2, ext2[k], beta));
    for (int l = 0; l < 3; ++l) {
      D.set_block(k * m, l * m, blk(T1, ext1[k], ext1[l]));
      D.set_block((3 + k) * m, (3 + l) * m, blk(T2, ext2[k], ext2[l]));
    }
    for (int i = 0; i < m; ++i) {
      hext[k * m + i] = H1[ext1[k] * m + i];
      hext[(3 + k) * m + i] = H2[ext2[k] * m + i];
    }
  }
  for (int i = 0; i < m; ++i) {
    hface[i] = -H1[alpha * m + i];
    hface[m + i] = -H2[beta * m + i];
  }
  const PivLU lu(A);
  if (!(lu.min_abs_pivot() > 0.0)) throw std::runtime_error("merge_pair: singular face block");
  FusedPair fp;
  fp.iti = D;
  fp.iti.add_block(0, 0, matmul(C, lu.solve(B)));
  fp.source = hext;
  const CVec x = lu.solve(hface);
  gemv_acc(C, x.data(), fp.source.data(), 1.0);
  return fp;
}

namespace {
struct GroupIndex {
  std::vector<int> group_of, pos_of;
};
GroupIndex index_groups(const LevelPartition& p) {  // dissection.cpp:92-104
  GroupIndex gi;
  gi.group_of.assign(p.a_faces, -1);
  gi.pos_of.assign(p.a_faces, -1);
  for (std::size_t g = 0; g < p.groups.size(); ++g)
    for (std::size_t i = 0; i < p.groups[g].size(); ++i) {
      gi.group_of[p.groups[g][i]] = static_cast<int>(g);
      gi.pos_of[p.groups[g][i]] = static_cast<int>(i);
    }
  return gi;
}

std::vector<CVec> solve_groups(const LevelPartition& p, const std::vector<PivLU>& lus,
                               const CVec& lead, int bs) {  // dissection.cpp:136-150
  std::vector<CVec> x(p.groups.size());
  for (std::size_t g = 0; g < p.groups.size(); ++g) {
    const auto& grp = p.groups[g];
    CVec hg(grp.size() * bs);
    for (std::size_t i = 0; i < grp.size(); ++i)
      std::copy_n(lead.begin() + static_cast<std::size_t>(grp[i]) * bs, bs, hg.begin() + i * bs);
    x[g] = lus[g].solve(hg);
  }
  return x;
}
}  // namespace

BlockMatrix eliminate_level(const BlockMatrix& parent, const LevelPartition& part,
                            std::vector<PivLU>& group_lu, int threads) {
  // dissection.cpp:106-133 (factor_groups) and 153-198
  const int bs = parent.bs, na = part.a_faces;
  const GroupIndex gidx = index_groups(part);
  for (const auto& kv : parent.blocks) {
    const auto [r, c] = kv.first;
    if (r < na && c < na && gidx.group_of[r] != gidx.group_of[c])
      throw std::logic_error("eliminate_level: leading block couples faces " + std::to_string(r) +
                             " and " + std::to_string(c) + " across merge groups");
  }
  const int ng = static_cast<int>(part.groups.size());
  group_lu.assign(ng, PivLU());
  parallel_for(ng, threads, [&](int g) {
    const auto& grp = part.groups[g];
    const int gsz = static_cast<int>(grp.size());
    CMat A(gsz * bs, gsz * bs);
    for (int i = 0; i < gsz; ++i)
      for (int j = 0; j < gsz; ++j)
        if (const CMat* b = parent.find(grp[i], grp[j])) A.set_block(i * bs, j * bs, *b);
    group_lu[g] = PivLU(A);
    if (!(group_lu[g].min_abs_pivot() > 0.0))
      throw std::runtime_error("eliminate_level: singular merge block at face " +
                               std::to_string(grp.front()));
  });
  BlockMatrix next(parent.nblocks - na, bs);
  std::vector<std::set<int>> bcols(ng), crows(ng);
  for (const auto& kv : parent.blocks) {
    const auto [r, c] = kv.first;
    if (r >= na && c >= na)
      next.block(r - na, c - na) = kv.second;
    else if (r < na && c >= na)
      bcols[gidx.group_of[r]].insert(c);
    else if (r >= na && c < na)
      crows[gidx.group_of[c]].insert(r);
  }
  // Per-(group, column) updates, computed in parallel into private lists and
  // merged afterwards in the serial loop's order (group, then column, then
  // row), so every next(r, c) accumulates its terms in the same order.
  std::vector<std::pair<int, int>> work;  // (group, column)
  for (int g = 0; g < ng; ++g)
    for (int c : bcols[g]) work.push_back({g, c});
  std::vector<std::vector<std::pair<std::pair<int, int>, CMat>>> upd(work.size());
  parallel_for(static_cast<int>(work.size()), threads, [&](int w) {
    const auto [g, c] = work[w];
    const auto& grp = part.groups[g];
    const int gsz = static_cast<int>(grp.size());
    CMat Bg(gsz * bs, bs);
    for (int i = 0; i < gsz; ++i)
      if (const CMat* b = parent.find(grp[i], c)) Bg.set_block(i * bs, 0, *b);
    const CMat X = group_lu[g].solve(Bg);
    for (int r : crows[g]) {
      CMat u(bs, bs);
      bool touched = false;
      for (int i = 0; i < gsz; ++i)
        if (const CMat* b = parent.find(r, grp[i])) {
          u.add_block(0, 0, matmul(*b, X.block(i * bs, 0, bs, bs)));
          touched = true;
        }
      if (touched) upd[w].push_back({{r - na, c - na}, std::move(u)});
    }
  });
  for (auto& lst : upd)
    for (auto& [key, u] : lst) next.block(key.first, key.second).add_block(0, 0, u, -1.0);
  return next;
}

MergeHierarchy build_hierarchy(const SkeletonSystem& sys, int depth, bool factor_coarse,
                               int threads) {  // dissection.cpp:200-227
  MergeHierarchy h;
  h.graph = sys.graph;
  h.side_len = sys.side_len;
  const int total = h.total_levels();
  if (depth == 0) depth = total;
  if (depth < 1 || depth > total) throw std::invalid_argument("build_hierarchy: depth out of range");
  h.depth = depth;
  BlockMatrix current = sys.M;
  int first = 0;
  for (int level = 1; level <= depth; ++level) {
    HierarchyLevel hl;
    hl.level = level;
    hl.first_face = first;
    hl.partition = partition_level(h.graph, first, level);
    hl.M = std::move(current);
    if (level < depth) {
      current = eliminate_level(hl.M, hl.partition, hl.group_lu, threads);
      first += hl.partition.a_faces;
    }
    h.levels.push_back(std::move(hl));
  }
  if (factor_coarse) h.coarse_lu.emplace(h.levels.back().M.to_dense());
  return h;
}

std::size_t MergeHierarchy::storage_bytes() const {  // dissection.cpp:229-238
  std::size_t b = 0;
  for (const auto& hl : levels) {
    b += hl.M.storage_bytes();
    for (const auto& lu : hl.group_lu) b += sizeof(cplx) * lu.entries();
  }
  if (coarse_lu) b += sizeof(cplx) * coarse_lu->entries();
  return b;
}

CVec direct_solve(const MergeHierarchy& h, const CVec& rhs) {  // dissection.cpp:240-292
  if (h.depth != h.total_levels() || !h.coarse_lu)
    throw std::logic_error("direct_solve: hierarchy not built to full depth");
  if (rhs.size() != h.levels.front().M.dim())
    throw std::invalid_argument("direct_solve: rhs size mismatch");
  const int bs = h.block_size();
  std::vector<CVec> lead(h.levels.size());
  CVec cur = rhs;
  for (std::size_t li = 0; li + 1 < h.levels.size(); ++li) {
    const HierarchyLevel& hl = h.levels[li];
    const int na = hl.partition.a_faces;
    const GroupIndex gidx = index_groups(hl.partition);
    const std::size_t nl = static_cast<std::size_t>(na) * bs;
    lead[li].assign(cur.begin(), cur.begin() + nl);
    CVec tail(cur.begin() + nl, cur.end());
    const auto x = solve_groups(hl.partition, hl.group_lu, lead[li], bs);
    for (const auto& [key, blk] : hl.M.blocks) {
      const auto [r, c] = key;
      if (r < na || c >= na) continue;
      gemv_acc(blk, x[gidx.group_of[c]].data() + static_cast<std::size_t>(gidx.pos_of[c]) * bs,
               tail.data() + static_cast<std::size_t>(r - na) * bs, -1.0);
    }
    cur = std::move(tail);
  }
  CVec x = h.coarse_lu->solve(cur);
  for (auto li = static_cast<std::ptrdiff_t>(h.levels.size()) - 2; li >= 0; --li) {
    const HierarchyLevel& hl = h.levels[li];
    const int na = hl.partition.a_faces;
    const GroupIndex gidx = index_groups(hl.partition);
    CVec top = lead[li];
    for (const auto& [key, blk] : hl.M.blocks) {
      const auto [r, c] = key;
      if (r < na && c >= na)
        gemv_acc(blk, x.data() + static_cast<std::size_t>(c - na) * bs,
                 top.data() + static_cast<std::size_t>(r) * bs, -1.0);
    }
    const auto xg = solve_groups(hl.partition, hl.group_lu, top, bs);
    CVec merged(static_cast<std::size_t>(na) * bs + x.size());
    for (int f = 0; f < na; ++f)
      std::copy_n(xg[gidx.group_of[f]].begin() + static_cast<std::size_t>(gidx.pos_of[f]) * bs, bs,
                  merged.begin() + static_cast<std::size_t>(f) * bs);
    std::copy(x.begin(), x.end(), merged.begin() + static_cast<std::size_t>(na) * bs);
    x = std::move(merged);
  }
  return x;
}

// ===================== krylov (krylov.cpp:12-202) ========================
namespace {
struct Givens {
  double c = 1.0;
  cplx s{0.0, 0.0};
};
Givens make_givens(cplx a, cplx b) {  // krylov.cpp:17-31
  Givens g;
  const double na = std::abs(a), nb = std::abs(b);
  if (nb == 0.0) return g;
  const double r = std::hypot(na, nb);
  if (na == 0.0) {
    g.c = 0.0;
    g.s = std::conj(b) / nb;
  } else {
    g.c = na / r;
    g.s = (a / na) * std::conj(b) / r;
  }
  return g;
}
void apply_givens(const Givens& g, cplx& a, cplx& b) {  // krylov.cpp:33-37
  const cplx t = g.c * a + g.s * b;
  b = -std::conj(g.s) * a + g.c * b;
  a = t;
}
enum class Mode { kNone, kRight, kFlexible };

std::pair<CVec, SolveReport> gmres_driver(const LinOp& op, const CVec& rhs,
                                          const KrylovConfig& cfg, Mode mode,
                                          const LinOp* precond, int fixed_steps) {
  // krylov.cpp:45-178
  if (cfg.restart < 1) throw std::invalid_argument("gmres: restart must be >= 1");
  if (fixed_steps == 0 && !(cfg.tol > 0.0 && cfg.tol < 1.0))
    throw std::invalid_argument("gmres: tol must lie in (0, 1)");
  const std::size_t n = rhs.size();
  SolveReport rep;
  CVec x(n);
  const double bnorm = norm2(rhs);
  if (bnorm == 0.0) {
    rep.converged = true;
    return {x, rep};
  }
  const int restart = fixed_steps > 0 ? fixed_steps : cfg.restart;
  const int max_iters = fixed_steps > 0 ? fixed_steps : cfg.max_iters;
  std::vector<CVec> V, Z;
  CMat H(restart + 1, restart);
  std::vector<Givens> rot(restart);
  CVec gv(restart + 1);
  auto residual = [&](const CVec& xx) {
    CVec r = op(xx);
    for (std::size_t i = 0; i < n; ++i) r[i] = rhs[i] - r[i];
    return r;
  };
  int total = 0;
  bool converged = false;
  while (total < max_iters && !converged) {
    const CVec r0 = total == 0 ? rhs : residual(x);
    const double beta = norm2(r0);
    if (fixed_steps == 0 && beta / bnorm <= cfg.tol) {
      converged = true;
      break;
    }
    V.assign(1, r0);
    for (auto& z : V[0]) z /= beta;
    Z.clear();
    std::fill(gv.begin(), gv.end(), cplx(0.0, 0.0));
    std::fill(H.v.begin(), H.v.end(), cplx(0.0, 0.0));
    gv[0] = beta;
    int j = 0;
    bool breakdown = false;
    for (; j < restart && total < max_iters; ++j, ++total) {
      CVec w;
      if (mode == Mode::kFlexible) {
        Z.push_back((*precond)(V[j]));
        w = op(Z.back());
      } else if (mode == Mode::kRight) {
        w = op((*precond)(V[j]));
      } else {
        w = op(V[j]);
      }
      for (int i = 0; i <= j; ++i) {
        H(i, j) = dotc(V[i], w);
        for (std::size_t k = 0; k < n; ++k) w[k] -= H(i, j) * V[i][k];
      }
      if (cfg.reorthogonalize)
        for (int i = 0; i <= j; ++i) {
          const cplx corr = dotc(V[i], w);
          H(i, j) += corr;
          for (std::size_t k = 0; k < n; ++k) w[k] -= corr * V[i][k];
        }
      const double hnext = norm2(w);
      H(j + 1, j) = hnext;
      for (int i = 0; i < j; ++i) apply_givens(rot[i], H(i, j), H(i + 1, j));
      rot[j] = make_givens(H(j, j), H(j + 1, j));
      apply_givens(rot[j], H(j, j), H(j + 1, j));
      apply_givens(rot[j], gv[j], gv[j + 1]);
      const double rel = std::abs(gv[j + 1]) / bnorm;
      if (cfg.record_history) rep.residual_history.push_back(rel);
      if (hnext <= 1e-14 * bnorm) {
        breakdown = true;
        ++j;
        ++total;
        break;
      }
      V.push_back(w);
      for (auto& z : V.back()) z /= hnext;
      if (fixed_steps == 0 && rel <= cfg.tol) {
        ++j;
        ++total;
        break;
      }
    }
    if (j > 0) {  // upper-triangular solve H y = g, then expand
      CVec y(j);
      for (int i = j - 1; i >= 0; --i) {
        cplx s = gv[i];
        for (int k = i + 1; k < j; ++k) s -= H(i, k) * y[k];
        y[i] = s / H(i, i);
      }
      CVec upd(n);
      const auto& basis = mode == Mode::kFlexible ? Z : V;
      for (int i = 0; i < j; ++i)
        for (std::size_t k = 0; k < n; ++k) upd[k] += y[i] * basis[i][k];
      if (mode == Mode::kRight) upd = (*precond)(upd);
      for (std::size_t k = 0; k < n; ++k) x[k] += upd[k];
    }
    if (cfg.record_history) {
      const std::size_t used = std::min<std::size_t>(j, V.size());
      double dev = 0.0;
      for (std::size_t a = 0; a < used; ++a)
        for (std::size_t b = 0; b <= a; ++b)
          dev = std::max(dev, std::abs(std::abs(dotc(V[a], V[b])) - (a == b ? 1.0 : 0.0)));
      rep.basis_orthogonality = std::max(rep.basis_orthogonality, dev);
    }
    if (fixed_steps > 0) break;
    const double true_rel = norm2(residual(x)) / bnorm;
    rep.final_residual = true_rel;
    if (true_rel <= cfg.tol) converged = true;
    if (breakdown && !converged && true_rel > cfg.tol)
      throw std::runtime_error("gmres: numerical breakdown before convergence");
  }
  rep.iterations = total;
  if (fixed_steps == 0) {
    rep.final_residual = norm2(residual(x)) / bnorm;
    rep.converged = rep.final_residual <= cfg.tol;
  } else {
    rep.converged = true;
  }
  return {x, rep};
}
}  // namespace

std::pair<CVec, SolveReport> gmres(const LinOp& op, const CVec& rhs, const KrylovConfig& cfg,
                                   const LinOp* right_precond) {
  return gmres_driver(op, rhs, cfg, right_precond ? Mode::kRight : Mode::kNone, right_precond, 0);
}

std::pair<CVec, SolveReport> fgmres(const LinOp& op, const CVec& rhs, const LinOp& precond,
                                    const KrylovConfig& cfg) {
  return gmres_driver(op, rhs, cfg, Mode::kFlexible, &precond, 0);
}

CVec gmres_fixed_steps(const LinOp& op, const CVec& rhs, int steps) {
  if (steps < 1) throw std::invalid_argument("gmres_fixed_steps: steps must be >= 1");
  KrylovConfig cfg;
  cfg.record_history = false;
  return gmres_driver(op, rhs, cfg, Mode::kNone, nullptr, steps).first;
}

// ===================== multigrid (multigrid.cpp) ==========================
MgPreconditioner::MgPreconditioner(const MergeHierarchy& hh, const MgConfig& c) : h(&hh), cfg(c) {
  // multigrid.cpp:9-28
  if (cfg.depth < 2) throw std::invalid_argument("MgPreconditioner: depth must be >= 2");
  if (cfg.depth > hh.depth)
    throw std::invalid_argument("MgPreconditioner: depth exceeds the built hierarchy");
  if (!cfg.exact_coarse && cfg.gamma < 1)
    throw std::invalid_argument("MgPreconditioner: gamma must be >= 1");
  if (!cfg.exact_coarse && cfg.coarse_iters < 1)
    throw std::invalid_argument("MgPreconditioner: coarse_iters must be >= 1");
  if (cfg.exact_coarse) {
    if (cfg.depth == hh.depth && hh.coarse_lu)
      exact_lu = *hh.coarse_lu;
    else
      exact_lu.emplace(hh.levels[cfg.depth - 1].M.to_dense());
  }
}

namespace {
struct BlockOp : LinOp {
  const BlockMatrix* M;
  explicit BlockOp(const BlockMatrix& m) : M(&m) {}
  CVec operator()(const CVec& v) const override { return M->apply(v); }
};
}  // namespace

CVec MgPreconditioner::apply_level(const CVec& v, int level) const {  // multigrid.cpp:30-100
  if (level < 1 || level > cfg.depth)
    throw std::invalid_argument("MgPreconditioner: level out of range");
  const HierarchyLevel& hl = h->levels[level - 1];
  if (v.size() != hl.M.dim()) throw std::invalid_argument("MgPreconditioner: vector size mismatch");
  if (level == cfg.depth) {
    if (cfg.exact_coarse) return exact_lu->solve(v);
    return gmres_fixed_steps(BlockOp(hl.M), v, cfg.coarse_iters);
  }
  const int bs = h->block_size(), na = hl.partition.a_faces;
  const std::size_t lead = static_cast<std::size_t>(na) * bs;
  CVec w(v.size());
  const int ng = static_cast<int>(hl.partition.groups.size());
  parallel_for(ng, ng >= 64 ? g_threads : 1, [&](int g) {  // F (groups are independent)
    const auto& grp = hl.partition.groups[g];
    CVec hg(grp.size() * bs);
    for (std::size_t i = 0; i < grp.size(); ++i)
      std::copy_n(v.begin() + static_cast<std::size_t>(grp[i]) * bs, bs, hg.begin() + i * bs);
    const CVec xg = hl.group_lu[g].solve(hg);
    for (std::size_t i = 0; i < grp.size(); ++i)
      std::copy_n(xg.begin() + i * bs, bs, w.begin() + static_cast<std::size_t>(grp[i]) * bs);
  });
  const CVec mw = hl.M.apply(w);  // R (v - M F v)
  CVec rc(v.size() - lead);
  for (std::size_t k = 0; k < rc.size(); ++k) rc[k] = v[lead + k] - mw[lead + k];
  const HierarchyLevel& next = h->levels[level];
  const int gamma = cfg.exact_coarse ? 1 : cfg.gamma;
  CVec z(rc.size());
  for (int step = 0; step < gamma; ++step) {
    CVec inner = rc;
    if (step > 0) {
      const CVec mz = next.M.apply(z);
      for (std::size_t k = 0; k < inner.size(); ++k) inner[k] -= mz[k];
    }
    const CVec dz = apply_level(inner, level + 1);
    for (std::size_t k = 0; k < z.size(); ++k) z[k] += dz[k];
  }
  CVec bz(lead);  // P z = [-A^{-1} B z; z]
  for_block_rows(hl.M, 0, na, [&](const std::pair<int, int>& key, const CMat& blk) {
    const auto [r, c] = key;
    if (c >= na)
      gemv_acc(blk, z.data() + static_cast<std::size_t>(c - na) * bs,
               bz.data() + static_cast<std::size_t>(r) * bs, 1.0);
  });
  CVec out = w;
  parallel_for(ng, ng >= 64 ? g_threads : 1, [&](int g) {
    const auto& grp = hl.partition.groups[g];
    CVec hg(grp.size() * bs);
    for (std::size_t i = 0; i < grp.size(); ++i)
      std::copy_n(bz.begin() + static_cast<std::size_t>(grp[i]) * bs, bs, hg.begin() + i * bs);
    const CVec xg = hl.group_lu[g].solve(hg);
    for (std::size_t i = 0; i < grp.size(); ++i)
      for (int k = 0; k < bs; ++k) out[static_cast<std::size_t>(grp[i]) * bs + k] -= xg[i * bs + k];
  });
  for (std::size_t k = 0; k < z.size(); ++k) out[lead + k] += z[k];
  return out;
}

std::size_t MgPreconditioner::memory_bytes() const {  // multigrid.cpp:102-113
  std::size_t b = 0;
  for (int level = 1; level <= cfg.depth; ++level) {
    const HierarchyLevel& hl = h->levels[level - 1];
    if (level > 1) b += hl.M.storage_bytes();
    if (level < cfg.depth)
      for (const auto& lu : hl.group_lu) b += sizeof(cplx) * lu.entries();
  }
  if (exact_lu) b += sizeof(cplx) * exact_lu->entries();
  return b;
}

// ===================== recovery (problems.cpp:60-92) ======================
std::vector<CVec> recover_solution(const Mesh& mesh, const std::vector<ElementRecord>& elements,
                                   const FaceGraph& graph, const CVec& g) {
  const int sl = mesh.order - 1, bs = 2 * sl;
  std::vector<CVec> values(elements.size());
  for (std::size_t e = 0; e < elements.size(); ++e) {
    CVec gb(4 * sl);
    for (int s = 0; s < 4; ++s) {
      const int f = graph.face_of_element[e][s];
      for (int k = 0; k < sl; ++k) {
        if (f >= 0) {
          const int slot = graph.faces[f].e1 == static_cast<int>(e) ? 1 : 0;
          gb[s * sl + k] = g[static_cast<std::size_t>(f) * bs + slot * sl + k];
        } else {
          gb[s * sl + k] = mesh.tside[(e * 4 + s) * sl + k];
        }
      }
    }
    values[e] = elements[e].ops->solve(gb, elements[e].interior_source);
  }
  return values;
}

}  // namespace oracle
