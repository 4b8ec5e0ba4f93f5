// CPU ORACLE — TEST INFRASTRUCTURE ONLY.  C entry points for ctypes (tests,
// smoke(), bench.py's cpu_baseline).  Complex arrays are interleaved
// (re, im) doubles; matrices column-major, as in the reference.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>

#include "../paper_2511_00735_b200/csrc/problem.hpp"
#include "oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

void put(const CVec& v, double* out) { std::memcpy(out, v.data(), v.size() * sizeof(cplx)); }
CVec get(const double* in, std::size_t n) {
  CVec v(n);
  std::memcpy(static_cast<void*>(v.data()), in, n * sizeof(cplx));
  return v;
}

struct Session {
  Mesh mesh;
  Gll rule;
  std::vector<ElementRecord> elements;
  SkeletonSystem sys;
  std::unique_ptr<MergeHierarchy> hier;
  std::unique_ptr<MgPreconditioner> mg;
  int threads = 1;
  double t_elements = 0, t_skeleton = 0, t_hierarchy = 0;
  std::vector<double> history;  // residual history of the last solve (record_history)
};

struct MOp : LinOp {
  const BlockMatrix* M;
  explicit MOp(const BlockMatrix& m) : M(&m) {}
  CVec operator()(const CVec& v) const override { return M->apply(v); }
};
struct POp : LinOp {
  const MgPreconditioner* P;
  explicit POp(const MgPreconditioner& p) : P(&p) {}
  CVec operator()(const CVec& v) const override { return P->apply(v); }
};

double secs(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

void oracle_set_lean_elements(int lean) { set_lean_elements(lean != 0); }

int oracle_gll_rule(int order, double* nodes, double* weights, double* diff) {
  return guarded([&] {
    const Gll r = gll_rule(order);
    std::memcpy(nodes, r.nodes.data(), r.nodes.size() * 8);
    std::memcpy(weights, r.weights.data(), r.weights.size() * 8);
    std::memcpy(diff, r.diff.data(), r.diff.size() * 8);
  });
}

// Writes left|right|bottom|top|interior|noncorner|comp_of_full back to back.
int oracle_index_sets(int order, int* out) {
  return guarded([&] {
    const IndexSets s = build_index_sets(order);
    int* p = out;
    for (const auto* v : {&s.left, &s.right, &s.bottom, &s.top, &s.interior, &s.noncorner,
                          &s.comp_of_full}) {
      std::memcpy(p, v->data(), v->size() * sizeof(int));
      p += v->size();
    }
  });
}

// faces[f*6 + {e1,e2,s1,s2,level,group}], level_range[2L], face_of_element[4 n^2]
int oracle_face_graph(int n, int* faces, int* level_range, int* face_of_element) {
  return guarded([&] {
    const FaceGraph g = build_face_graph(n);
    for (int f = 0; f < g.num_faces(); ++f) {
      const Face& x = g.faces[f];
      const int row[6] = {x.e1, x.e2, x.s1, x.s2, x.level, x.group};
      std::memcpy(faces + 6 * f, row, sizeof(row));
    }
    for (int l = 0; l < g.num_levels(); ++l) {
      level_range[2 * l] = g.level_range[l].first;
      level_range[2 * l + 1] = g.level_range[l].second;
    }
    for (int e = 0; e < n * n; ++e)
      for (int s = 0; s < 4; ++s) face_of_element[4 * e + s] = g.face_of_element[e][s];
  });
}

// One element with a (possibly complex) coefficient on all (N+1)^2 nodes.
int oracle_element(int order, double h, double eta, const double* coeff_full,
                   const double* interior_src, double* T, double* H, double* pde, double* iout) {
  return guarded([&] {
    const Gll r = gll_rule(order);
    const Element el(r, h, eta, get(coeff_full, (order + 1) * (order + 1)));
    put(el.iti.v, T);
    if (H) put(el.source_to_outgoing(get(interior_src, (order - 1) * (order - 1))), H);
    if (pde) put(el.pde.v, pde);
    if (iout) put(el.imp_out.v, iout);
  });
}

int oracle_merge_pair(int m, const double* T1, const double* H1, const double* T2,
                      const double* H2, int alpha, int beta, double* T, double* H) {
  return guarded([&] {
    CMat a(4 * m, 4 * m), b(4 * m, 4 * m);
    a.v = get(T1, a.v.size());
    b.v = get(T2, b.v.size());
    const FusedPair fp = merge_pair(a, get(H1, 4 * m), b, get(H2, 4 * m), alpha, beta, m);
    put(fp.iti.v, T);
    put(fp.source, H);
  });
}

// Seeded sample generation through the shared problem definitions.
// kind: 0 reference bump, 1 reference plane wave, 2 BASELINE config.
int oracle_sample(int kind, int config, unsigned long long seed, int n, int order, double kappa,
                  double* coeff, double* source, double* tside, int* source_zero) {
  return guarded([&] {
    hpsb::problem::Spec spec;
    if (kind == 0) spec = hpsb::problem::reference_bump(n, order, kappa);
    else if (kind == 1) spec = hpsb::problem::reference_planewave(n, order, kappa);
    else spec = hpsb::problem::baseline_config(config, seed, n, order, kappa);
    const Gll r = gll_rule(spec.order);
    const auto s = hpsb::problem::sample(spec, r.nodes.data());
    std::memcpy(coeff, s.coeff.data(), s.coeff.size() * 8);
    std::memcpy(source, s.source.data(), s.source.size() * 16);
    std::memcpy(tside, s.tside.data(), s.tside.size() * 16);
    *source_zero = s.source_is_zero ? 1 : 0;
  });
}

void* oracle_session_create(int n, int order, double kappa, double eta, const double* coeff,
                            const double* source, const double* tside, int threads) {
  auto* S = new Session;
  const int rc = guarded([&] {
    S->threads = threads;
    set_threads(threads);
    Mesh& m = S->mesh;
    if (n < 2 || (n & (n - 1))) throw std::invalid_argument("Mesh: n must be a power of two >= 2");
    m.n = n, m.order = order, m.kappa = kappa, m.eta = eta;
    const std::size_t ne = static_cast<std::size_t>(n) * n, np = order + 1, sl = order - 1;
    m.coeff.assign(coeff, coeff + ne * np * np);
    m.source = get(source, ne * sl * sl);
    m.tside = get(tside, ne * 4 * sl);
    S->rule = gll_rule(order);
    auto t0 = std::chrono::steady_clock::now();
    S->elements = build_elements(m, S->rule, threads);
    S->t_elements = secs(t0);
    t0 = std::chrono::steady_clock::now();
    S->sys = assemble_skeleton(m, S->elements);
    S->t_skeleton = secs(t0);
  });
  if (rc) {
    delete S;
    return nullptr;
  }
  return S;
}

void oracle_session_destroy(void* s) { delete static_cast<Session*>(s); }

long long oracle_dim(void* s) { return static_cast<long long>(static_cast<Session*>(s)->sys.M.dim()); }

int oracle_get_element(void* s, int e, double* T, double* H) {
  return guarded([&] {
    auto* S = static_cast<Session*>(s);
    const auto& rec = S->elements.at(e);
    put(rec.ops->iti.v, T);
    put(rec.outgoing_source, H);
  });
}

int oracle_get_rhs(void* s, double* rhs) {
  return guarded([&] { put(static_cast<Session*>(s)->sys.rhs, rhs); });
}

// The skeleton right-hand side of another impedance datum t on the same
// elements (the rhs part of assemble_skeleton, skeleton.cpp:121-132):
// rhs slot = -H_alpha - sum_{gamma physical} T_{alpha gamma} t_gamma.
int oracle_rhs_for_tside(void* s, const double* tside, double* out) {
  return guarded([&] {
    auto* S = static_cast<Session*>(s);
    const Mesh& mesh = S->mesh;
    const FaceGraph& graph = S->sys.graph;
    const int sl = mesh.order - 1, bs = 2 * sl;
    const std::size_t ne = static_cast<std::size_t>(mesh.n) * mesh.n;
    const CVec t = get(tside, ne * 4 * sl);
    CVec rhs(S->sys.M.dim());
    for (int f = 0; f < graph.num_faces(); ++f) {
      const Face& face = graph.faces[f];
      for (int slot = 0; slot < 2; ++slot) {
        const int eid = slot == 0 ? face.e1 : face.e2;
        const int alpha = slot == 0 ? face.s1 : face.s2;
        const ElementRecord& rec = S->elements[eid];
        cplx* r = rhs.data() + static_cast<std::size_t>(f) * bs + slot * sl;
        for (int k = 0; k < sl; ++k) r[k] = -rec.outgoing_source[alpha * sl + k];
        for (int gamma = 0; gamma < 4; ++gamma)
          if (graph.face_of_element[eid][gamma] < 0)
            gemv_acc(rec.ops->iti_block(alpha, gamma),
                     t.data() + (static_cast<std::size_t>(eid) * 4 + gamma) * sl, r, -1.0);
      }
    }
    put(rhs, out);
  });
}

int oracle_apply_M(void* s, const double* x, double* y) {
  return guarded([&] {
    auto* S = static_cast<Session*>(s);
    put(S->sys.M.apply(get(x, S->sys.M.dim())), y);
  });
}

int oracle_build_hierarchy(void* s, int depth, int factor_coarse) {
  return guarded([&] {
    auto* S = static_cast<Session*>(s);
    S->mg.reset();
    const auto t0 = std::chrono::steady_clock::now();
    S->hier = std::make_unique<MergeHierarchy>(
        build_hierarchy(S->sys, depth, factor_coarse != 0, S->threads));
    S->t_hierarchy = secs(t0);
  });
}

// Number of stored blocks of level l's system (1-based), and its first face.
int oracle_level_info(void* s, int level, int* nblocks_stored, int* first_face, int* nfaces) {
  return guarded([&] {
    auto* S = static_cast<Session*>(s);
    if (!S->hier) throw std::logic_error("no hierarchy");
    const auto& hl = S->hier->levels.at(level - 1);
    *nblocks_stored = static_cast<int>(hl.M.blocks.size());
    *first_face = hl.first_face;
    *nfaces = hl.M.nblocks;
  });
}

// keys[2k] = (row, col) block index (local to the level system), data = bs*bs complex each.
int oracle_level_blocks(void* s, int level, int* keys, double* data) {
  return guarded([&] {
    auto* S = static_cast<Session*>(s);
    const auto& hl = S->hier->levels.at(level - 1);
    std::size_t k = 0;
    const std::size_t bb = static_cast<std::size_t>(hl.M.bs) * hl.M.bs;
    for (const auto& [key, blk] : hl.M.blocks) {
      keys[2 * k] = key.first;
      keys[2 * k + 1] = key.second;
      std::memcpy(data + 2 * bb * k, blk.v.data(), bb * sizeof(cplx));
      ++k;
    }
  });
}

// y = M_l x for level l's system (faces [first_face, total), the level's
// HierarchyLevel::M, BlockMatrix::apply of block_matrix.cpp:23-31).
int oracle_level_apply(void* s, int level, const double* x, double* y) {
  return guarded([&] {
    auto* S = static_cast<Session*>(s);
    if (!S->hier) throw std::logic_error("no hierarchy");
    const auto& M = S->hier->levels.at(level - 1).M;
    put(M.apply(get(x, M.dim())), y);
  });
}

int oracle_precond_create(void* s, int depth, int gamma, int coarse_iters, int exact) {
  return guarded([&] {
    auto* S = static_cast<Session*>(s);
    if (!S->hier) throw std::logic_error("no hierarchy");
    MgConfig c;
    c.depth = depth, c.gamma = gamma, c.coarse_iters = coarse_iters, c.exact_coarse = exact != 0;
    S->mg = std::make_unique<MgPreconditioner>(*S->hier, c);
  });
}

int oracle_precond_apply(void* s, const double* v, double* z) {
  return guarded([&] {
    auto* S = static_cast<Session*>(s);
    put(S->mg->apply(get(v, S->sys.M.dim())), z);
  });
}

long long oracle_precond_memory(void* s) {
  auto* S = static_cast<Session*>(s);
  return S->mg ? static_cast<long long>(S->mg->memory_bytes()) : -1;
}

long long oracle_hierarchy_storage(void* s) {
  auto* S = static_cast<Session*>(s);
  return S->hier ? static_cast<long long>(S->hier->storage_bytes()) : -1;
}

// mode 0: gmres (no preconditioner), 1: fgmres with the session preconditioner,
// 2: gmres with the session preconditioner on the right (krylov.cpp:180-186).
// stats[0]=iterations, stats[1]=converged, stats[2]=final residual, stats[3]=seconds,
// stats[4]=basis orthogonality
int oracle_solve(void* s, int mode, const double* rhs, double* x, int restart, double tol,
                 int max_iters, int reorth, int record_history, double* stats) {
  return guarded([&] {
    auto* S = static_cast<Session*>(s);
    KrylovConfig k;
    k.restart = restart, k.tol = tol, k.max_iters = max_iters;
    k.reorthogonalize = reorth != 0, k.record_history = record_history != 0;
    const MOp op(S->sys.M);
    const CVec b = get(rhs, S->sys.M.dim());
    const auto t0 = std::chrono::steady_clock::now();
    std::pair<CVec, SolveReport> res;
    if (mode == 1) {
      if (!S->mg) throw std::logic_error("no preconditioner");
      res = fgmres(op, b, POp(*S->mg), k);
    } else if (mode == 2) {
      if (!S->mg) throw std::logic_error("no preconditioner");
      const POp pc(*S->mg);
      res = gmres(op, b, k, &pc);
    } else {
      res = gmres(op, b, k, nullptr);
    }
    stats[3] = secs(t0);
    put(res.first, x);
    stats[0] = res.second.iterations;
    stats[1] = res.second.converged ? 1.0 : 0.0;
    stats[2] = res.second.final_residual;
    stats[4] = res.second.basis_orthogonality;
    S->history = res.second.residual_history;
  });
}

// Residual history of the last oracle_solve with record_history (length returned).
long long oracle_history(void* s, double* out, long long cap) {
  auto* S = static_cast<Session*>(s);
  const long long n = static_cast<long long>(S->history.size());
  if (out)
    for (long long i = 0; i < std::min(n, cap); ++i) out[i] = S->history[i];
  return n;
}

int oracle_direct_solve(void* s, const double* rhs, double* x) {
  return guarded([&] {
    auto* S = static_cast<Session*>(s);
    put(direct_solve(*S->hier, get(rhs, S->sys.M.dim())), x);
  });
}

// field[e][total] complex in the corner-free node order.
int oracle_recover(void* s, const double* g, double* field) {
  return guarded([&] {
    auto* S = static_cast<Session*>(s);
    const auto vals = recover_solution(S->mesh, S->elements, S->sys.graph, get(g, S->sys.M.dim()));
    std::size_t off = 0;
    for (const auto& v : vals) {
      std::memcpy(field + 2 * off, v.data(), v.size() * sizeof(cplx));
      off += v.size();
    }
  });
}

// Dense M (for tiny systems only).
int oracle_dense_M(void* s, double* out) {
  return guarded([&] { put(static_cast<Session*>(s)->sys.M.to_dense().v, out); });
}

void oracle_timings(void* s, double* t) {
  auto* S = static_cast<Session*>(s);
  t[0] = S->t_elements, t[1] = S->t_skeleton, t[2] = S->t_hierarchy;
}

}  // extern "C"
