// C ABI of the hps_b200 library (include/hps_b200.h).  Mirrors the
// reference C API's conventions: statuses instead of exceptions, a
// thread-local last-error string, create/destroy ownership
// (proj/src/capi.cpp:13-24,109-137).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/hps_b200.h"
#include "internal.hpp"
#include "problem.hpp"

struct hpsb_context_s {
  hpsb::Context c;
};
struct hpsb_elements_s {
  std::unique_ptr<hpsb::Elements> e;
};
struct hpsb_skeleton_s {
  std::unique_ptr<hpsb::Skeleton> s;
};
struct hpsb_hierarchy_s {
  std::unique_ptr<hpsb::Hierarchy> h;
  // factor_coarse: the exact (dense-inverse) coarse solve at the built depth,
  // used by direct_solve (dissection.cpp:225, :240-292).
  hpsb::Precond* direct = nullptr;
  // The reference driver's default preconditioner (MgConfig defaults:
  // depth = L, gamma = 1, coarse_iters = 4; multigrid.hpp:12-18,
  // driver.hpp:30-32), planned on the host while the device finishes the
  // merges; handed out by precond_create for that configuration.
  hpsb::Precond* pending = nullptr;
  ~hpsb_hierarchy_s() {
    hpsb::destroy_precond(direct);
    hpsb::destroy_precond(pending);
  }
};
struct hpsb_precond_s {
  hpsb::Precond* p = nullptr;
  ~hpsb_precond_s() { hpsb::destroy_precond(p); }
};
struct hpsb_local_group_s {
  std::shared_ptr<hpsb::LocalGroup> g;
};

namespace hpsb {
void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                           cudaGetErrorString(e) + ") at " + file + ":" + std::to_string(line) +
                           ": " + what);
}
}  // namespace hpsb

namespace {
thread_local std::string g_last_error;

template <class F>
hpsb_status guarded(F&& f) {
  try {
    return f();
  } catch (const hpsb::InvalidArgument& e) {
    g_last_error = e.what();
    return HPSB_INVALID_ARGUMENT;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return HPSB_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HPSB_INTERNAL;
  } catch (...) {
    g_last_error = "unknown error";
    return HPSB_INTERNAL;
  }
}

hpsb::Context* ctx_of(hpsb_context c) { return c ? &c->c : nullptr; }
hpsb::Context* ctx_of(hpsb_elements e) { return e && e->e ? e->e->ctx : nullptr; }
hpsb::Context* ctx_of(hpsb_skeleton s) { return s && s->s ? s->s->ctx : nullptr; }
hpsb::Context* ctx_of(hpsb_hierarchy h) { return h && h->h ? h->h->ctx : nullptr; }
hpsb::Context* ctx_of(hpsb_precond p) { return p ? hpsb::precond_context(p->p) : nullptr; }
void ctx_retain(hpsb::Context* c) {
  if (c) c->refs.fetch_add(1);
}
// Drop one reference; the last one tears the context down in dependency
// order: its communicator's buffers are freed on the stream before the
// stream itself goes.
void ctx_release(hpsb::Context* c) {
  if (!c || c->refs.fetch_sub(1) != 1) return;
  hpsb::ContextBind bind(c);
  cudaStreamSynchronize(c->stream);
  c->comm.reset();
  c->collect();
  cudaStreamSynchronize(c->stream);
  for (auto& e : c->ev) cudaEventDestroy(e);
  for (auto& e : c->timer)
    if (e) cudaEventDestroy(e);
  c->pending.clear();
  for (auto& e : c->event_pool) cudaEventDestroy(e);
  cudaStreamDestroy(c->stream);
  c->stream = nullptr;
  delete static_cast<hpsb_context_s*>(c->owner);
}
// Device allocations and staged uploads of the call go to the stream of the
// handle's own context (internal.hpp, ContextBind).
#define BIND(h) hpsb::ContextBind bind_ctx_(ctx_of(h))

#define REQUIRE(cond, msg) \
  do {                     \
    if (!(cond)) throw hpsb::InvalidArgument(msg); \
  } while (0)

hpsb::problem::Spec make_spec(int kind, int config, uint64_t seed, int n, int order, double kappa) {
  if (kind == 0) return hpsb::problem::reference_bump(n, order, kappa);
  if (kind == 1) return hpsb::problem::reference_planewave(n, order, kappa);
  if (kind == 2) return hpsb::problem::baseline_config(config, seed, n, order, kappa);
  throw hpsb::InvalidArgument("problem kind must be 0, 1 or 2");
}
}  // namespace

extern "C" {

const char* hpsb_last_error(void) { return g_last_error.c_str(); }
const char* hpsb_version(void) { return "hps_b200 0.1.0 (sm_100a)"; }

hpsb_status hpsb_context_create(int device, hpsb_context* out) {
  return guarded([&] {
    REQUIRE(out, "context_create: null output");
    int count = 0;
    HPSB_CUDA(cudaGetDeviceCount(&count));
    REQUIRE(device >= 0 && device < count, "context_create: no such CUDA device");
    cudaDeviceProp prop{};
    HPSB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      throw std::runtime_error("context_create: hps_b200 needs an sm_100 (B200) device");
    auto ctx = std::make_unique<hpsb_context_s>();
    ctx->c.owner = ctx.get();
    ctx->c.device = device;
    HPSB_CUDA(cudaSetDevice(device));
    ctx->c.num_sms = prop.multiProcessorCount;
    ctx->c.pdl = std::getenv("HPSB_NO_PDL") == nullptr;
    HPSB_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
    for (auto& e : ctx->c.ev) HPSB_CUDA(cudaEventCreate(&e));
    cudaMemPool_t pool;
    HPSB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    HPSB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    // Map pool memory once, here, instead of inside the first setups: growing
    // a stream-ordered pool maps physical pages (~60 ms/GB measured), which
    // would otherwise land inside build_hierarchy.  HPSB_POOL_RESERVE_GB
    // overrides the default (min(48 GB, 40% of free memory)).
    {
      size_t free_b = 0, total_b = 0;
      HPSB_CUDA(cudaMemGetInfo(&free_b, &total_b));
      double gb = std::min(48.0, 0.4 * free_b / double(1 << 30));
      if (const char* env = std::getenv("HPSB_POOL_RESERVE_GB")) gb = std::atof(env);
      uint64_t used = 0;
      HPSB_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &used));
      const size_t want = static_cast<size_t>(gb * double(1 << 30));
      if (want > used) {
        void* p = nullptr;
        if (cudaMallocAsync(&p, want - used, ctx->c.stream) == cudaSuccess)
          HPSB_CUDA(cudaFreeAsync(p, ctx->c.stream));
        else
          cudaGetLastError();  // best effort
        HPSB_CUDA(cudaStreamSynchronize(ctx->c.stream));
      }
    }
    *out = ctx.release();
    return HPSB_OK;
  });
}

hpsb_status hpsb_context_destroy(hpsb_context ctx) {
  return guarded([&] {
    if (ctx) ctx_release(&ctx->c);  // the handle's reference (objects hold theirs)
    return HPSB_OK;
  });
}

hpsb_status hpsb_context_synchronize(hpsb_context ctx) {
  return guarded([&] {
    BIND(ctx);
    HPSB_CUDA(cudaStreamSynchronize(ctx->c.stream));
    return HPSB_OK;
  });
}

int64_t hpsb_context_launches(hpsb_context ctx) { return ctx ? ctx->c.launches : -1; }

int64_t hpsb_context_residual_history(hpsb_context ctx, double* out, int64_t cap) {
  if (!ctx) return -1;
  const auto& hst = ctx->c.history;
  const int64_t n = static_cast<int64_t>(hst.size());
  if (out)
    for (int64_t i = 0; i < std::min(n, cap); ++i) out[i] = hst[i];
  return n;
}

hpsb_status hpsb_context_timer_start(hpsb_context ctx) {
  return guarded([&] {
    BIND(ctx);
    REQUIRE(ctx, "timer: null context");
    for (auto& e : ctx->c.timer)
      if (!e) HPSB_CUDA(cudaEventCreate(&e));
    HPSB_CUDA(cudaEventRecord(ctx->c.timer[0], ctx->c.stream));
    return HPSB_OK;
  });
}

hpsb_status hpsb_context_timer_stop(hpsb_context ctx, double* seconds) {
  return guarded([&] {
    BIND(ctx);
    REQUIRE(ctx && seconds && ctx->c.timer[0], "timer: not started");
    HPSB_CUDA(cudaEventRecord(ctx->c.timer[1], ctx->c.stream));
    HPSB_CUDA(cudaEventSynchronize(ctx->c.timer[1]));
    float ms = 0;
    HPSB_CUDA(cudaEventElapsedTime(&ms, ctx->c.timer[0], ctx->c.timer[1]));
    *seconds = ms * 1e-3;
    return HPSB_OK;
  });
}

hpsb_status hpsb_context_profile(hpsb_context ctx, int enable) {
  return guarded([&] {
    BIND(ctx);
    REQUIRE(ctx, "profile: null context");
    ctx->c.collect();
    ctx->c.profile = enable != 0;
    return HPSB_OK;
  });
}

int hpsb_context_profile_count(hpsb_context ctx) {
  if (!ctx) return -1;
  try {
    ctx->c.collect();
  } catch (...) {
    return -1;
  }
  return static_cast<int>(ctx->c.agg.size());
}

hpsb_status hpsb_context_profile_entry(hpsb_context ctx, int i, char* name, int name_len,
                                       int64_t* launches, double* ms, double* bytes,
                                       double* flops) {
  return guarded([&] {
    BIND(ctx);
    REQUIRE(ctx, "profile: null context");
    ctx->c.collect();
    REQUIRE(i >= 0 && i < static_cast<int>(ctx->c.agg.size()), "profile: index out of range");
    const auto& kv = ctx->c.agg[i];
    if (name && name_len > 0) {
      std::strncpy(name, kv.first.c_str(), name_len - 1);
      name[name_len - 1] = 0;
    }
    if (launches) *launches = kv.second.launches;
    if (ms) *ms = kv.second.ms;
    if (bytes) *bytes = kv.second.bytes;
    if (flops) *flops = kv.second.flops;
    return HPSB_OK;
  });
}

hpsb_status hpsb_context_profile_reset(hpsb_context ctx) {
  return guarded([&] {
    BIND(ctx);
    REQUIRE(ctx, "profile: null context");
    ctx->c.collect();
    ctx->c.agg.clear();
    return HPSB_OK;
  });
}

int64_t hpsb_precond_bytes(hpsb_precond p) { return p ? hpsb::precond_bytes(p->p) : -1; }

hpsb_status hpsb_hierarchy_pinned_flops(hpsb_hierarchy h, double* element_flops,
                                        double* merge_flops) {
  return guarded([&] {
    BIND(h);
    REQUIRE(h, "hierarchy_pinned_flops: null handle");
    double fe = 0, fm = 0;
    hpsb::hierarchy_pinned(h->h.get(), &fe, &fm, nullptr);
    if (element_flops) *element_flops = fe;
    if (merge_flops) *merge_flops = fm;
    return HPSB_OK;
  });
}

double hpsb_precond_pinned_bytes(hpsb_precond p) {
  if (!p) return -1.0;
  try {
    return hpsb::precond_pinned_bytes(p->p);
  } catch (...) {
    return -1.0;
  }
}

hpsb_status hpsb_nccl_unique_id(unsigned char id[128]) {
  return guarded([&] {
    REQUIRE(id, "nccl_unique_id: null output");
    hpsb::nccl_unique_id(id);
    return HPSB_OK;
  });
}

hpsb_status hpsb_context_attach_nccl(hpsb_context ctx, const unsigned char id[128], int rank,
                                     int world) {
  return guarded([&] {
    BIND(ctx);
    REQUIRE(ctx && id && world >= 1 && rank >= 0 && rank < world, "attach_nccl: bad argument");
    ctx->c.comm = hpsb::make_nccl_comm(id, rank, world, ctx->c.device);
    return HPSB_OK;
  });
}

hpsb_status hpsb_local_group_create(int world, hpsb_local_group* out) {
  return guarded([&] {
    REQUIRE(out && world >= 1, "local_group_create: bad argument");
    *out = new hpsb_local_group_s{hpsb::make_local_group(world)};
    return HPSB_OK;
  });
}

hpsb_status hpsb_local_group_destroy(hpsb_local_group g) {
  delete g;
  return HPSB_OK;
}

hpsb_status hpsb_context_attach_local(hpsb_context ctx, hpsb_local_group g, int rank) {
  return guarded([&] {
    BIND(ctx);
    REQUIRE(ctx && g, "attach_local: null argument");
    ctx->c.comm = hpsb::make_thread_comm(g->g, rank);
    return HPSB_OK;
  });
}

hpsb_status hpsb_context_comm_info(hpsb_context ctx, int* rank, int* world) {
  return guarded([&] {
    BIND(ctx);
    REQUIRE(ctx, "comm_info: null context");
    if (rank) *rank = ctx->c.rank();
    if (world) *world = ctx->c.world();
    return HPSB_OK;
  });
}

hpsb_status hpsb_partition(int n, int world, int rank, int* elem_owner, int* face_owner,
                           int* last_local_level) {
  return guarded([&] {
    const hpsb::Partition p = hpsb::make_partition(hpsb::build_face_graph(n), world, rank);
    if (elem_owner) std::memcpy(elem_owner, p.elem_owner.data(), p.elem_owner.size() * sizeof(int));
    if (face_owner) std::memcpy(face_owner, p.face_owner.data(), p.face_owner.size() * sizeof(int));
    if (last_local_level) *last_local_level = p.last_local;
    return HPSB_OK;
  });
}

hpsb_status hpsb_merge_owners(int n, int world, int level, int* owners) {
  return guarded([&] {
    const hpsb::FaceGraph g = hpsb::build_face_graph(n);
    REQUIRE(level >= 1 && level <= g.num_levels(), "merge_owners: level out of range");
    const auto all = hpsb::merge_owners(g, hpsb::make_partition(g, world, 0));
    const auto& o = all[level - 1];
    if (owners) std::memcpy(owners, o.data(), o.size() * sizeof(int));
    return HPSB_OK;
  });
}

hpsb_status hpsb_gll_rule(int order, double* nodes, double* weights, double* diff) {
  return guarded([&] {
    const hpsb::Gll g = hpsb::gll_rule(order);
    std::memcpy(nodes, g.nodes.data(), g.nodes.size() * sizeof(double));
    std::memcpy(weights, g.weights.data(), g.weights.size() * sizeof(double));
    std::memcpy(diff, g.diff.data(), g.diff.size() * sizeof(double));
    return HPSB_OK;
  });
}

hpsb_status hpsb_index_sets(int order, int* out) {
  return guarded([&] {
    const hpsb::IndexSets s = hpsb::build_index_sets(order);
    int* p = out;
    for (const auto* v : {&s.left, &s.right, &s.bottom, &s.top, &s.interior, &s.noncorner,
                          &s.comp_of_full}) {
      std::memcpy(p, v->data(), v->size() * sizeof(int));
      p += v->size();
    }
    return HPSB_OK;
  });
}

hpsb_status hpsb_face_graph(int n, int* faces, int* level_range, int* face_of_element) {
  return guarded([&] {
    const hpsb::FaceGraph g = hpsb::build_face_graph(n);
    for (int f = 0; f < g.num_faces(); ++f) {
      const auto& x = g.faces[f];
      const int row[6] = {x.e1, x.e2, x.s1, x.s2, x.level, x.group};
      std::memcpy(faces + 6 * f, row, sizeof(row));
    }
    for (int l = 0; l < g.num_levels(); ++l) {
      level_range[2 * l] = g.level_range[l].first;
      level_range[2 * l + 1] = g.level_range[l].second;
    }
    for (int e = 0; e < n * n; ++e)
      for (int s = 0; s < 4; ++s) face_of_element[4 * e + s] = g.face_of_element[e][s];
    return HPSB_OK;
  });
}

hpsb_status hpsb_problem_dims(int kind, int config, int n, int order, int* n_out, int* order_out,
                              int* nrhs_out, double* kappa_out, int* restart_out,
                              double* tol_out) {
  return guarded([&] {
    const auto spec = make_spec(kind, config, 0, n, order, kind == 2 ? 0.0 : 1.0);
    *n_out = spec.n, *order_out = spec.order, *nrhs_out = static_cast<int>(spec.angles.size());
    if (kappa_out) *kappa_out = spec.kappa;
    if (restart_out) *restart_out = spec.restart;
    if (tol_out) *tol_out = spec.tol;
    return HPSB_OK;
  });
}

hpsb_status hpsb_problem_sample(int kind, int config, uint64_t seed, int n, int order, double kappa,
                                double* coeff, double* source, double* tside, int* source_zero) {
  return guarded([&] {
    const auto spec = make_spec(kind, config, seed, n, order, kappa);
    const hpsb::Gll g = hpsb::gll_rule(spec.order);
    const auto s = hpsb::problem::sample(spec, g.nodes.data());
    std::memcpy(coeff, s.coeff.data(), s.coeff.size() * sizeof(double));
    std::memcpy(source, s.source.data(), s.source.size() * 2 * sizeof(double));
    std::memcpy(tside, s.tside.data(), s.tside.size() * 2 * sizeof(double));
    if (source_zero) *source_zero = s.source_is_zero ? 1 : 0;
    return HPSB_OK;
  });
}

hpsb_status hpsb_elements_build_dev(hpsb_context ctx, int n, int order, double eta,
                                    const double* coeff_dev, const double* source_dev,
                                    hpsb_elements* out) {
  return guarded([&] {
    BIND(ctx);
    REQUIRE(ctx && out && coeff_dev, "elements_build: null argument");
    auto h = std::make_unique<hpsb_elements_s>();
    h->e = hpsb::build_elements(&ctx->c, n, order, eta, coeff_dev,
                                reinterpret_cast<const double2*>(source_dev));
    ctx_retain(ctx_of(h.get()));  // the object holds its context
    *out = h.release();
    return HPSB_OK;
  });
}

hpsb_status hpsb_elements_build(hpsb_context ctx, int n, int order, double eta, const double* coeff,
                                const double* source, hpsb_elements* out) {
  return guarded([&] {
    BIND(ctx);
    REQUIRE(ctx && out && coeff, "elements_build: null argument");
    REQUIRE(n >= 2 && order >= 2, "elements_build: bad mesh");
    const size_t ne = static_cast<size_t>(n) * n, np = order + 1, m = order - 1;
    hpsb::DevBuf<double> c(ne * np * np);
    hpsb::DevBuf<double2> s(source ? ne * m * m : 0);
    HPSB_CUDA(cudaMemcpyAsync(c.p, coeff, c.bytes(), cudaMemcpyHostToDevice, ctx->c.stream));
    if (source)
      HPSB_CUDA(cudaMemcpyAsync(s.p, source, s.bytes(), cudaMemcpyHostToDevice, ctx->c.stream));
    auto h = std::make_unique<hpsb_elements_s>();
    h->e = hpsb::build_elements(&ctx->c, n, order, eta, c.p, source ? s.p : nullptr);
    ctx_retain(ctx_of(h.get()));  // the object holds its context
    *out = h.release();
    return HPSB_OK;
  });
}

hpsb_status hpsb_elements_destroy(hpsb_elements el) {
  hpsb::Context* c = ctx_of(el);
  {
    BIND(el);
    delete el;
  }
  ctx_release(c);
  return HPSB_OK;
}

hpsb_status hpsb_elements_fallbacks(hpsb_elements el, int* count) {
  return guarded([&] {
    BIND(el);
    REQUIRE(el && count, "elements_fallbacks: null argument");
    hpsb::elements_wait(el->e.get());
    *count = el->e->fallbacks;
    return HPSB_OK;
  });
}

hpsb_status hpsb_elements_get(hpsb_elements el, int e0, int count, double* T, double* H) {
  return guarded([&] {
    BIND(el);
    hpsb::elements_wait(el ? el->e.get() : nullptr);
    const auto& E = *el->e;
    const int ne = E.n * E.n;
    REQUIRE(e0 >= 0 && count >= 0 && e0 + count <= ne, "elements_get: range out of bounds");
    const size_t nb = E.nb;
    if (T)
      HPSB_CUDA(cudaMemcpy(T, E.T.p + e0 * nb * nb, count * nb * nb * sizeof(double2),
                           cudaMemcpyDeviceToHost));
    if (H)
      HPSB_CUDA(cudaMemcpy(H, E.H.p + e0 * nb, count * nb * sizeof(double2), cudaMemcpyDeviceToHost));
    return HPSB_OK;
  });
}

hpsb_status hpsb_skeleton_create(hpsb_elements el, const double* tside, int nrhs,
                                 hpsb_skeleton* out) {
  return guarded([&] {
    BIND(el);
    REQUIRE(el && out && tside && nrhs >= 1, "skeleton_create: bad argument");
    auto h = std::make_unique<hpsb_skeleton_s>();
    h->s = hpsb::build_skeleton(el->e.get(), reinterpret_cast<const double2*>(tside), nrhs);
    ctx_retain(ctx_of(h.get()));  // the object holds its context
    *out = h.release();
    return HPSB_OK;
  });
}

hpsb_status hpsb_skeleton_create_boundary(hpsb_elements el, const double* tbnd, int nrhs,
                                          hpsb_skeleton* out) {
  return guarded([&] {
    BIND(el);
    REQUIRE(el && out && tbnd && nrhs >= 1, "skeleton_create_boundary: bad argument");
    auto h = std::make_unique<hpsb_skeleton_s>();
    h->s = hpsb::build_skeleton(el->e.get(), reinterpret_cast<const double2*>(tbnd), nrhs, true);
    ctx_retain(ctx_of(h.get()));  // the object holds its context
    *out = h.release();
    return HPSB_OK;
  });
}

hpsb_status hpsb_skeleton_destroy(hpsb_skeleton sk) {
  hpsb::Context* c = ctx_of(sk);
  {
    BIND(sk);
    delete sk;
  }
  ctx_release(c);
  return HPSB_OK;
}

int64_t hpsb_skeleton_dim(hpsb_skeleton sk) { return sk ? sk->s->dim : -1; }

const double* hpsb_skeleton_rhs_dev(hpsb_skeleton sk, int r) {
  if (!sk || r < 0 || r >= sk->s->nrhs) return nullptr;
  return reinterpret_cast<const double*>(sk->s->rhs.p + static_cast<size_t>(r) * sk->s->dim);
}

hpsb_status hpsb_skeleton_rhs(hpsb_skeleton sk, int r, double* rhs) {
  return guarded([&] {
    BIND(sk);
    REQUIRE(sk && rhs && r >= 0 && r < sk->s->nrhs, "skeleton_rhs: bad argument");
    hpsb::elements_wait(sk->s->el);  // element-stage errors surface here at the latest
    // the skeleton build returns without synchronising; cudaMemcpy runs on
    // the legacy stream, which does not wait for the context's stream
    HPSB_CUDA(cudaStreamSynchronize(sk->s->ctx->stream));
    HPSB_CUDA(cudaMemcpy(rhs, sk->s->rhs.p + static_cast<size_t>(r) * sk->s->dim,
                         sk->s->dim * sizeof(double2), cudaMemcpyDeviceToHost));
    return HPSB_OK;
  });
}

hpsb_status hpsb_skeleton_apply_dev(hpsb_skeleton sk, const double* x, double* y) {
  return guarded([&] {
    BIND(sk);
    REQUIRE(sk && x && y, "skeleton_apply: null argument");
    hpsb::elements_wait(sk->s->el);  // element-stage errors surface here at the latest
    hpsb::skeleton_apply(sk->s.get(), reinterpret_cast<const double2*>(x),
                         reinterpret_cast<double2*>(y));
    return HPSB_OK;
  });
}

hpsb_status hpsb_skeleton_apply(hpsb_skeleton sk, const double* x, double* y) {
  return guarded([&] {
    BIND(sk);
    REQUIRE(sk && x && y, "skeleton_apply: null argument");
    hpsb::elements_wait(sk->s->el);  // element-stage errors surface here at the latest
    auto* S = sk->s.get();
    cudaStream_t st = S->ctx->stream;
    HPSB_CUDA(cudaMemcpyAsync(S->x_buf.p, x, S->dim * sizeof(double2), cudaMemcpyHostToDevice, st));
    hpsb::skeleton_apply(S, S->x_buf.p, S->y_buf.p);
    HPSB_CUDA(cudaMemcpyAsync(y, S->y_buf.p, S->dim * sizeof(double2), cudaMemcpyDeviceToHost, st));
    HPSB_CUDA(cudaStreamSynchronize(st));
    return HPSB_OK;
  });
}

hpsb_status hpsb_recover_dev(hpsb_skeleton sk, const double* x, int r, double* field) {
  return guarded([&] {
    BIND(sk);
    REQUIRE(sk && x && field, "recover: null argument");
    hpsb::elements_wait(sk->s->el);  // element-stage errors surface here at the latest
    hpsb::recover_field(sk->s.get(), reinterpret_cast<const double2*>(x), r,
                        reinterpret_cast<double2*>(field));
    return HPSB_OK;
  });
}

hpsb_status hpsb_recover(hpsb_skeleton sk, const double* x, int r, double* field) {
  return guarded([&] {
    BIND(sk);
    REQUIRE(sk && x && field, "recover: null argument");
    hpsb::elements_wait(sk->s->el);  // element-stage errors surface here at the latest
    auto* S = sk->s.get();
    cudaStream_t st = S->ctx->stream;
    const auto* el = S->el;
    const size_t nf = static_cast<size_t>(el->n) * el->n * ((el->order + 1) * (el->order + 1) - 4);
    hpsb::DevBuf<double2> d_f(nf);
    HPSB_CUDA(cudaMemcpyAsync(S->x_buf.p, x, S->dim * sizeof(double2), cudaMemcpyHostToDevice, st));
    hpsb::recover_field(S, S->x_buf.p, r, d_f.p);
    HPSB_CUDA(cudaMemcpyAsync(field, d_f.p, nf * sizeof(double2), cudaMemcpyDeviceToHost, st));
    HPSB_CUDA(cudaStreamSynchronize(st));
    return HPSB_OK;
  });
}

hpsb_status hpsb_hierarchy_build(hpsb_skeleton sk, int depth, int factor_coarse,
                                 hpsb_hierarchy* out) {
  return guarded([&] {
    BIND(sk);
    REQUIRE(sk && out, "hierarchy_build: null argument");
    auto h = std::make_unique<hpsb_hierarchy_s>();
    auto* hs = h.get();
    h->h = hpsb::build_hierarchy(sk->s.get(), depth, [hs](hpsb::Hierarchy* hh) {
      if (hh->depth < 2 || hh->ctx->profile) return;
      hpsb_mg_config c{};
      c.depth = hh->depth, c.gamma = 1, c.coarse_iters = 4, c.exact_coarse = 0;
      hpsb::destroy_precond(hs->pending);  // a discarded first pass (pivot redo)
      hs->pending = nullptr;
      try {
        hs->pending = hpsb::create_precond(hh, c);
      } catch (...) {
        hs->pending = nullptr;  // built on demand by precond_create instead
      }
    });
    if (factor_coarse && h->h->depth >= 2) {
      hpsb_mg_config c{};
      c.depth = h->h->depth, c.gamma = 1, c.coarse_iters = 0, c.exact_coarse = 1;
      h->direct = hpsb::create_precond(h->h.get(), c);
    }
    ctx_retain(ctx_of(h.get()));  // the object holds its context
    *out = h.release();
    return HPSB_OK;
  });
}

hpsb_status hpsb_hierarchy_destroy(hpsb_hierarchy h) {
  hpsb::Context* c = ctx_of(h);
  {
    BIND(h);
    delete h;
  }
  ctx_release(c);
  return HPSB_OK;
}

hpsb_status hpsb_hierarchy_info(hpsb_hierarchy h, int* depth, int* total_levels,
                                int64_t* device_bytes, double* build_seconds) {
  return guarded([&] {
    BIND(h);
    REQUIRE(h, "hierarchy_info: null handle");
    if (depth) *depth = h->h->depth;
    if (total_levels) *total_levels = h->h->total_levels;
    if (device_bytes) *device_bytes = h->h->device_bytes;
    if (build_seconds) *build_seconds = h->h->build_seconds;
    return HPSB_OK;
  });
}

hpsb_status hpsb_hierarchy_level_blocks(hpsb_hierarchy h, int level, int* nblocks, int* first_face,
                                        int* keys, double* data) {
  return guarded([&] {
    BIND(h);
    REQUIRE(h && nblocks && first_face, "hierarchy_level_blocks: null argument");
    hpsb::hierarchy_level_blocks(h->h.get(), level, nblocks, first_face, keys, data);
    return HPSB_OK;
  });
}

hpsb_status hpsb_hierarchy_level_apply(hpsb_hierarchy h, int level, const double* x, double* y) {
  return guarded([&] {
    BIND(h);
    REQUIRE(h && x && y, "hierarchy_level_apply: null argument");
    auto* H = h->h.get();
    REQUIRE(level >= 1 && level <= H->depth, "hierarchy_level_apply: level out of range");
    const auto& g = H->sk->graph;
    const size_t n = static_cast<size_t>(g.num_faces() - g.level_range[level - 1].first) * H->sk->bs;
    cudaStream_t st = H->ctx->stream;
    hpsb::DevBuf<double2> xd(n), yd(n);
    HPSB_CUDA(cudaMemcpyAsync(xd.p, x, xd.bytes(), cudaMemcpyHostToDevice, st));
    hpsb::hierarchy_level_apply(H, level, xd.p, yd.p);
    HPSB_CUDA(cudaMemcpyAsync(y, yd.p, yd.bytes(), cudaMemcpyDeviceToHost, st));
    HPSB_CUDA(cudaStreamSynchronize(st));
    return HPSB_OK;
  });
}

hpsb_status hpsb_merge_pair(hpsb_context ctx, int side_len, const double* T1, const double* H1,
                            const double* T2, const double* H2, int alpha, int beta, double* T,
                            double* H) {
  return guarded([&] {
    BIND(ctx);
    REQUIRE(ctx && T1 && H1 && T2 && H2 && T && H, "merge_pair: null argument");
    REQUIRE(side_len >= 1 && alpha >= 0 && alpha < 4 && beta >= 0 && beta < 4,
            "merge_pair: bad sides");
    hpsb::merge_pair(&ctx->c, side_len, reinterpret_cast<const double2*>(T1),
                     reinterpret_cast<const double2*>(H1), reinterpret_cast<const double2*>(T2),
                     reinterpret_cast<const double2*>(H2), alpha, beta,
                     reinterpret_cast<double2*>(T), reinterpret_cast<double2*>(H));
    return HPSB_OK;
  });
}

hpsb_status hpsb_precond_create(hpsb_hierarchy h, hpsb_mg_config cfg, hpsb_precond* out) {
  return guarded([&] {
    BIND(h);
    REQUIRE(h && out, "precond_create: null argument");
    auto p = std::make_unique<hpsb_precond_s>();
    if (h->pending && cfg.depth == h->h->depth && cfg.gamma == 1 && cfg.coarse_iters == 4 &&
        cfg.exact_coarse == 0) {
      p->p = h->pending;  // planned during hierarchy_build (same configuration)
      h->pending = nullptr;
    } else {
      p->p = hpsb::create_precond(h->h.get(), cfg);
    }
    ctx_retain(ctx_of(p.get()));  // the object holds its context
    *out = p.release();
    return HPSB_OK;
  });
}

hpsb_status hpsb_direct_solve_dev(hpsb_hierarchy h, const double* rhs, double* x) {
  return guarded([&] {
    BIND(h);
    REQUIRE(h && rhs && x, "direct_solve: null argument");
    REQUIRE(h->direct && h->h->depth == h->h->total_levels,
            "direct_solve: hierarchy not built to full depth");
    hpsb::precond_apply(h->direct, reinterpret_cast<const double2*>(rhs), reinterpret_cast<double2*>(x));
    return HPSB_OK;
  });
}

hpsb_status hpsb_direct_solve(hpsb_hierarchy h, const double* rhs, double* x) {
  return guarded([&] {
    BIND(h);
    REQUIRE(h && rhs && x, "direct_solve: null argument");
    REQUIRE(h->direct && h->h->depth == h->h->total_levels,
            "direct_solve: hierarchy not built to full depth");
    hpsb::precond_apply_host(h->direct, reinterpret_cast<const double2*>(rhs),
                             reinterpret_cast<double2*>(x));
    return HPSB_OK;
  });
}

hpsb_status hpsb_precond_destroy(hpsb_precond p) {
  hpsb::Context* c = ctx_of(p);
  {
    BIND(p);
    delete p;
  }
  ctx_release(c);
  return HPSB_OK;
}

hpsb_status hpsb_precond_apply_dev(hpsb_precond p, const double* v, double* z) {
  return guarded([&] {
    BIND(p);
    REQUIRE(p && v && z, "precond_apply: null argument");
    hpsb::precond_apply(p->p, reinterpret_cast<const double2*>(v), reinterpret_cast<double2*>(z));
    return HPSB_OK;
  });
}

hpsb_status hpsb_precond_apply(hpsb_precond p, const double* v, double* z) {
  return guarded([&] {
    BIND(p);
    REQUIRE(p && v && z, "precond_apply: null argument");
    hpsb::precond_apply_host(p->p, reinterpret_cast<const double2*>(v),
                             reinterpret_cast<double2*>(z));
    return HPSB_OK;
  });
}

hpsb_status hpsb_fgmres_dev(hpsb_skeleton sk, hpsb_precond precond, const double* rhs, double* x,
                            hpsb_krylov_config cfg, hpsb_solve_report* report) {
  return guarded([&] {
    BIND(sk);
    REQUIRE(sk && rhs && x && report, "fgmres: null argument");
    hpsb::elements_wait(sk->s->el);  // element-stage errors surface here at the latest
    return hpsb::fgmres(sk->s.get(), precond ? precond->p : nullptr,
                        reinterpret_cast<const double2*>(rhs), reinterpret_cast<double2*>(x), cfg,
                        report);
  });
}

hpsb_status hpsb_fgmres(hpsb_skeleton sk, hpsb_precond precond, const double* rhs, double* x,
                        hpsb_krylov_config cfg, hpsb_solve_report* report) {
  return guarded([&] {
    BIND(sk);
    REQUIRE(sk && rhs && x && report, "fgmres: null argument");
    hpsb::elements_wait(sk->s->el);  // element-stage errors surface here at the latest
    auto* S = sk->s.get();
    cudaStream_t st = S->ctx->stream;
    hpsb::DevBuf<double2> b(S->dim), xd(S->dim);
    HPSB_CUDA(cudaMemcpyAsync(b.p, rhs, b.bytes(), cudaMemcpyHostToDevice, st));
    const hpsb_status rc =
        hpsb::fgmres(S, precond ? precond->p : nullptr, b.p, xd.p, cfg, report);
    HPSB_CUDA(cudaMemcpyAsync(x, xd.p, xd.bytes(), cudaMemcpyDeviceToHost, st));
    HPSB_CUDA(cudaStreamSynchronize(st));
    return rc;
  });
}

hpsb_status hpsb_gmres_dev(hpsb_skeleton sk, hpsb_precond precond, const double* rhs, double* x,
                           hpsb_krylov_config cfg, hpsb_solve_report* report) {
  return guarded([&] {
    BIND(sk);
    REQUIRE(sk && rhs && x && report, "gmres: null argument");
    hpsb::elements_wait(sk->s->el);
    return hpsb::fgmres(sk->s.get(), precond ? precond->p : nullptr,
                        reinterpret_cast<const double2*>(rhs), reinterpret_cast<double2*>(x), cfg,
                        report, /*right=*/true);
  });
}

hpsb_status hpsb_gmres(hpsb_skeleton sk, hpsb_precond precond, const double* rhs, double* x,
                       hpsb_krylov_config cfg, hpsb_solve_report* report) {
  return guarded([&] {
    BIND(sk);
    REQUIRE(sk && rhs && x && report, "gmres: null argument");
    hpsb::elements_wait(sk->s->el);
    auto* S = sk->s.get();
    cudaStream_t st = S->ctx->stream;
    hpsb::DevBuf<double2> b(S->dim), xd(S->dim);
    HPSB_CUDA(cudaMemcpyAsync(b.p, rhs, b.bytes(), cudaMemcpyHostToDevice, st));
    const hpsb_status rc =
        hpsb::fgmres(S, precond ? precond->p : nullptr, b.p, xd.p, cfg, report, /*right=*/true);
    HPSB_CUDA(cudaMemcpyAsync(x, xd.p, xd.bytes(), cudaMemcpyDeviceToHost, st));
    HPSB_CUDA(cudaStreamSynchronize(st));
    return rc;
  });
}

hpsb_status hpsb_skeleton_apply_batch_dev(hpsb_skeleton sk, const double* x, double* y, int nrhs) {
  return guarded([&] {
    BIND(sk);
    REQUIRE(sk && x && y, "skeleton_apply: null argument");
    hpsb::elements_wait(sk->s->el);  // element-stage errors surface here at the latest
    hpsb::skeleton_apply_batch(sk->s.get(), reinterpret_cast<const double2*>(x),
                               reinterpret_cast<double2*>(y), nrhs);
    return HPSB_OK;
  });
}

hpsb_status hpsb_precond_apply_batch_dev(hpsb_precond p, const double* v, double* z, int nrhs) {
  return guarded([&] {
    BIND(p);
    REQUIRE(p && v && z, "precond_apply: null argument");
    hpsb::precond_apply_batch(p->p, reinterpret_cast<const double2*>(v),
                              reinterpret_cast<double2*>(z), nrhs);
    return HPSB_OK;
  });
}

hpsb_status hpsb_fgmres_batch_dev(hpsb_skeleton sk, hpsb_precond precond, const double* rhs,
                                  double* x, int nrhs, hpsb_krylov_config cfg,
                                  hpsb_solve_report* reports) {
  return guarded([&] {
    BIND(sk);
    REQUIRE(sk && rhs && x && reports, "fgmres: null argument");
    hpsb::elements_wait(sk->s->el);  // element-stage errors surface here at the latest
    return hpsb::fgmres_batch(sk->s.get(), precond ? precond->p : nullptr,
                              reinterpret_cast<const double2*>(rhs), reinterpret_cast<double2*>(x),
                              nrhs, cfg, reports);
  });
}

hpsb_status hpsb_fgmres_batch(hpsb_skeleton sk, hpsb_precond precond, const double* rhs, double* x,
                              int nrhs, hpsb_krylov_config cfg, hpsb_solve_report* reports) {
  return guarded([&] {
    BIND(sk);
    REQUIRE(sk && rhs && x && reports, "fgmres: null argument");
    hpsb::elements_wait(sk->s->el);  // element-stage errors surface here at the latest
    REQUIRE(nrhs >= 1 && nrhs <= 32, "fgmres: 1 <= nrhs <= 32");
    auto* S = sk->s.get();
    cudaStream_t st = S->ctx->stream;
    const size_t count = static_cast<size_t>(nrhs) * S->dim;
    hpsb::DevBuf<double2> b(count), xd(count);
    HPSB_CUDA(cudaMemcpyAsync(b.p, rhs, b.bytes(), cudaMemcpyHostToDevice, st));
    const hpsb_status rc = hpsb::fgmres_batch(S, precond ? precond->p : nullptr, b.p, xd.p, nrhs,
                                              cfg, reports);
    HPSB_CUDA(cudaMemcpyAsync(x, xd.p, xd.bytes(), cudaMemcpyDeviceToHost, st));
    HPSB_CUDA(cudaStreamSynchronize(st));
    return rc;
  });
}

}  // extern "C"
