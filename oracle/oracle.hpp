// CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain-C++ (no Eigen) restatement of the reference hps2d solver's hot path,
// used as the parity checker for the B200 library and as the bench's CPU
// baseline ("port").  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it; the product library never
// links or calls it.
//
// Parity status: the reference cannot be built here (Eigen3 is required by
// proj/CMakeLists.txt:10 and is absent on both this container and the GPU
// box), so no reference-produced numbers exist.  This oracle is pinned by
// restating every known-answer test the reference holds for the path
// (GLL closed forms, index-set counts, face enumeration, level sizes, the
// M2/M3/M4 block-sparsity patterns, identity/own-map diagonal blocks) and its
// numerical property tests (ItI closure, PairProbe, Schur blocks,
// associativity, direct = dense, MG exact inverse, plane-wave accuracy); see
// tests/test_oracle_*.py.  Numeric values are therefore "pinned by property",
// structure is pinned bit-exactly.
//
// Every function cites the reference file:line it follows.  Matrices are
// column-major complex<double>, the reference's Eigen layout (types.hpp:11-17).
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace oracle {

using cplx = std::complex<double>;
inline constexpr cplx kI{0.0, 1.0};

// Dense column-major complex matrix.
struct CMat {
  int rows = 0, cols = 0;
  std::vector<cplx> v;
  CMat() = default;
  CMat(int r, int c) : rows(r), cols(c), v(static_cast<std::size_t>(r) * c) {}
  cplx& operator()(int i, int j) { return v[i + static_cast<std::size_t>(j) * rows]; }
  const cplx& operator()(int i, int j) const {
    return v[i + static_cast<std::size_t>(j) * rows];
  }
  cplx* col(int j) { return v.data() + static_cast<std::size_t>(j) * rows; }
  const cplx* col(int j) const { return v.data() + static_cast<std::size_t>(j) * rows; }
  static CMat identity(int n) {
    CMat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
  double max_abs() const;
  CMat block(int r0, int c0, int nr, int nc) const;
  void set_block(int r0, int c0, const CMat& b);
  void add_block(int r0, int c0, const CMat& b, cplx scale = 1.0);
};

using CVec = std::vector<cplx>;

// Host threads used by the per-iteration operators (BlockMatrix::apply, the
// multigrid group solves); every result is bit-identical for any count.
void set_threads(int threads);
// Drop each element's dense t x t operators and LU after its T and H are
// formed (the solution recovery then fails): for the full-size golden runs.
void set_lean_elements(bool lean);

CMat matmul(const CMat& A, const CMat& B);           // A * B
void gemv_acc(const CMat& A, const cplx* x, cplx* y, cplx alpha);  // y += alpha A x
double norm2(const CVec& x);
cplx dotc(const CVec& a, const CVec& b);              // sum conj(a) b

// Partial-pivoting LU (the reference's Eigen::PartialPivLU).
struct PivLU {
  CMat lu;
  std::vector<int> perm;  // row i of P*A is row perm[i] of A
  explicit PivLU(const CMat& A);
  PivLU() = default;
  double min_abs_pivot() const;
  void solve_inplace(cplx* b, int nrhs, int ldb) const;
  CMat solve(const CMat& B) const;
  CVec solve(const CVec& b) const;
  std::size_t entries() const { return lu.v.size(); }
};

// ---- spectral (spectral.cpp:12-98) -------------------------------------
struct Gll {
  int order = 0;
  std::vector<double> nodes, weights;
  std::vector<double> diff;  // (N+1)^2 column-major
  double D(int i, int j) const { return diff[i + static_cast<std::size_t>(j) * (order + 1)]; }
};
Gll gll_rule(int order);

struct Ops1D {
  int order = 0;
  double h = 2.0;
  std::vector<double> mass;  // N+1
  std::vector<double> diff;  // (N+1)^2 col-major
  std::vector<double> stiff;
  double Dm(int i, int j) const { return diff[i + static_cast<std::size_t>(j) * (order + 1)]; }
  double K(int i, int j) const { return stiff[i + static_cast<std::size_t>(j) * (order + 1)]; }
};
Ops1D scale_to_element(const Gll& rule, double h);

// ---- element (element.cpp:22-188) ---------------------------------------
enum Side : int { kLeft = 0, kRight = 1, kBottom = 2, kTop = 3 };

struct IndexSets {
  int order = 0;
  std::vector<int> left, right, bottom, top, boundary, interior, noncorner, comp_of_full;
  int total() const { return (order + 1) * (order + 1) - 4; }
  int side_len() const { return order - 1; }
};
IndexSets build_index_sets(int order);

struct Element {
  int order = 0;
  double h = 0, eta = 0;
  IndexSets sets;
  Ops1D ops;
  CMat pde, op, imp_out, imp_in, iti;
  std::vector<double> mass2d;
  PivLU factor;
  Element(const Gll& rule, double h, double eta, const CVec& coeff_full);
  CMat iti_block(int a, int b) const { const int m = sets.side_len(); return iti.block(a * m, b * m, m, m); }
  CVec source_to_outgoing(const CVec& interior_src) const;
  CVec solve(const CVec& g, const CVec& interior_src) const;
};
CMat assemble_local_pde(const Ops1D& ox, const Ops1D& oy, const CVec& coeff, const IndexSets& sets);
std::pair<CMat, CMat> impedance_operators(const IndexSets& sets, const Ops1D& ox, const Ops1D& oy, double eta);

// ---- face graph / skeleton (skeleton.cpp:20-158) ------------------------
struct Face {
  int e1 = -1, e2 = -1, s1 = kRight, s2 = kLeft, level = 0, group = 0;
};
struct FaceGraph {
  int n = 0;
  std::vector<Face> faces;
  std::vector<std::pair<int, int>> level_range;
  std::vector<std::vector<std::vector<int>>> groups;
  std::vector<std::array<int, 4>> face_of_element;
  int num_levels() const { return static_cast<int>(level_range.size()); }
  int num_faces() const { return static_cast<int>(faces.size()); }
};
FaceGraph build_face_graph(int n);

// Block-sparse matrix keyed by (block row, block column) (block_matrix.cpp).
struct BlockMatrix {
  int nblocks = 0, bs = 0;
  std::map<std::pair<int, int>, CMat> blocks;
  BlockMatrix() = default;
  BlockMatrix(int nb, int b) : nblocks(nb), bs(b) {}
  std::size_t dim() const { return static_cast<std::size_t>(nblocks) * bs; }
  CMat& block(int r, int c);
  const CMat* find(int r, int c) const;
  CVec apply(const CVec& v) const;
  CMat to_dense() const;
  CMat to_dense_sub(int r0, int r1, int c0, int c1) const;
  std::size_t storage_bytes() const;
};

struct LevelPartition {
  int level = 0, a_faces = 0;
  std::vector<std::vector<int>> groups;
};
LevelPartition partition_level(const FaceGraph& g, int first_face, int level);

// ---- problem-level state (mesh.cpp, skeleton.cpp, problems.cpp) ----------
struct ElementRecord {
  double ox = 0, oy = 0;
  std::shared_ptr<Element> ops;
  CVec interior_source;  // b~ = s * mass2d
  CVec outgoing_source;  // H
};

// Inputs are the sampled problem (see paper_2511_00735_b200/csrc/problem.hpp).
struct Mesh {
  int n = 0, order = 0;
  double kappa = 0, eta = 0;
  std::vector<double> coeff;   // [e][(N+1)^2], real
  std::vector<cplx> source;    // [e][(N-1)^2]
  std::vector<cplx> tside;     // [e][4][N-1]
  double h() const { return 1.0 / n; }
};

std::vector<ElementRecord> build_elements(const Mesh& mesh, const Gll& rule, int threads);

struct SkeletonSystem {
  FaceGraph graph;
  int side_len = 0;
  BlockMatrix M;
  CVec rhs;
  int block_size() const { return 2 * side_len; }
};
SkeletonSystem assemble_skeleton(const Mesh& mesh, const std::vector<ElementRecord>& elements);

// ---- dissection (dissection.cpp:11-292) --------------------------------
struct FusedPair {
  CMat iti;
  CVec source;
  static int side_position(int element, int side, int alpha, int beta);
};
FusedPair merge_pair(const CMat& T1, const CVec& H1, const CMat& T2, const CVec& H2,
                     int alpha, int beta, int m);

struct HierarchyLevel {
  int level = 0, first_face = 0;
  LevelPartition partition;
  BlockMatrix M;
  std::vector<PivLU> group_lu;
};
struct MergeHierarchy {
  FaceGraph graph;
  int side_len = 0, depth = 0;
  std::vector<HierarchyLevel> levels;
  std::optional<PivLU> coarse_lu;
  int block_size() const { return 2 * side_len; }
  int total_levels() const { return graph.num_levels(); }
  std::size_t storage_bytes() const;
};
BlockMatrix eliminate_level(const BlockMatrix& parent, const LevelPartition& part,
                            std::vector<PivLU>& group_lu, int threads);
MergeHierarchy build_hierarchy(const SkeletonSystem& sys, int depth, bool factor_coarse,
                               int threads);
CVec direct_solve(const MergeHierarchy& h, const CVec& rhs);

// ---- krylov (krylov.cpp:12-202) ----------------------------------------
struct KrylovConfig {
  int restart = 60;
  double tol = 1e-8;
  int max_iters = 2000;
  bool record_history = true;
  bool reorthogonalize = false;
};
struct SolveReport {
  int iterations = 0;
  std::vector<double> residual_history;
  bool converged = false;
  double final_residual = 0.0;
  double basis_orthogonality = 0.0;
};
struct LinOp {
  virtual ~LinOp() = default;
  virtual CVec operator()(const CVec& v) const = 0;
};
std::pair<CVec, SolveReport> gmres(const LinOp& op, const CVec& rhs, const KrylovConfig& cfg,
                                   const LinOp* right_precond);
std::pair<CVec, SolveReport> fgmres(const LinOp& op, const CVec& rhs, const LinOp& precond,
                                    const KrylovConfig& cfg);
CVec gmres_fixed_steps(const LinOp& op, const CVec& rhs, int steps);

// ---- multigrid (multigrid.cpp:9-118) -----------------------------------
struct MgConfig {
  int depth = 2, gamma = 1, coarse_iters = 4;
  bool exact_coarse = false;
};
struct MgPreconditioner {
  const MergeHierarchy* h = nullptr;
  MgConfig cfg;
  std::optional<PivLU> exact_lu;
  MgPreconditioner(const MergeHierarchy& h, const MgConfig& cfg);
  CVec apply(const CVec& v) const { return apply_level(v, 1); }
  CVec apply_level(const CVec& v, int level) const;
  std::size_t memory_bytes() const;
};

// ---- recovery (problems.cpp:60-92) --------------------------------------
std::vector<CVec> recover_solution(const Mesh& mesh, const std::vector<ElementRecord>& elements,
                                   const FaceGraph& graph, const CVec& g);

}  // namespace oracle
