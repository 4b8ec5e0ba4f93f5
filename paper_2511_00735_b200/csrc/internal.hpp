// Internal host-side structures of the hps_b200 library.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <functional>
#include <utility>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hps_b200.h"

namespace hpsb {

// ---------------------------------------------------------------- errors
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NoConvergence : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_fail(cudaError_t e, const char* what, const char* file, int line);
#define HPSB_CUDA(x)                                              \
  do {                                                            \
    cudaError_t e_ = (x);                                         \
    if (e_ != cudaSuccess) ::hpsb::cuda_fail(e_, #x, __FILE__, __LINE__); \
  } while (0)
// Raise a kernel's dynamic shared-memory cap once, to the device maximum.
// The attribute is process-wide, so per-launch values would race between
// host threads driving different contexts (the emulated ranks).
// The cap only ever grows (under a lock), so a concurrent launch that needs
// less shared memory is never invalidated by another thread's setting.
template <auto Kernel>
void allow_smem(size_t bytes) {
  static std::mutex mu;
  static int cap = 0;  // the default limit is 48 KB minus the kernel's static smem
  if (static_cast<int>(bytes) <= cap) return;
  std::lock_guard<std::mutex> lk(mu);
  if (static_cast<int>(bytes) > cap) {
    const cudaError_t e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(bytes));
    if (e != cudaSuccess) cuda_fail(e, "cudaFuncSetAttribute", __FILE__, __LINE__);
    cap = static_cast<int>(bytes);
  }
}

// After a kernel launch: catch launch-configuration errors immediately.
#define HPSB_LAUNCHED(ctx)                 \
  do {                                     \
    HPSB_CUDA(cudaGetLastError());         \
    ++(ctx)->launches;                     \
  } while (0)

// ---------------------------------------------------------------- device memory
// Device buffers come from the stream-ordered pool (cudaMallocAsync with an
// unbounded release threshold): the merge stage allocates and frees per
// level, and pooled allocations keep that off the critical path (no implicit
// device synchronisation as in cudaFree).  Allocations are ordered on the
// stream of the context BOUND to the calling host thread (every ABI entry
// point binds the context of the handle it works on, ContextBind); a buffer
// remembers that stream and is freed on it, so its release is ordered after
// every kernel of its own context whatever context is bound at that point.
struct Context;
Context*& bound_context();
cudaStream_t alloc_stream();  // the bound context's stream, or null (plain cudaMalloc)
struct ContextBind {
  Context* prev;
  explicit ContextBind(Context* c) : prev(bound_context()) { bound_context() = c; }
  ~ContextBind() { bound_context() = prev; }
  ContextBind(const ContextBind&) = delete;
  ContextBind& operator=(const ContextBind&) = delete;
};

// Pinned staging ring for host->device descriptor uploads, one per context
// (from a process-wide pool, gemv.cu): a cudaMemcpyAsync from pageable memory
// waits for the stream to drain, which would serialise every batched launch
// of the merge stage with the host.  Uploads are copied into the ring and
// issued from pinned memory on the context's stream; when the ring wraps,
// the stream is synchronised (every earlier staged copy has landed).
struct Staging {
  unsigned char* base = nullptr;
  size_t size = 0, head = 0;
  ~Staging();
};
constexpr size_t kStagingMax = size_t(512) << 20;
void staged_upload(void* dst, const void* src, size_t bytes, cudaStream_t s);

template <class T>
struct DevBuf {
  T* p = nullptr;
  std::size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(std::size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  cudaStream_t s = nullptr;  // stream the buffer was allocated on (null: cudaMalloc)
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr, o.n = 0, o.s = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p, n = o.n, s = o.s;
      o.p = nullptr, o.n = 0, o.s = nullptr;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(std::size_t count) {
    release();
    if (count) {
      s = alloc_stream();
      if (s)
        HPSB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
      else
        HPSB_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), count * sizeof(T)));
    }
    n = count;
  }
  void release() {
    if (p) {
      if (s) cudaFreeAsync(p, s);
      else cudaFree(p);
    }
    p = nullptr, n = 0, s = nullptr;
  }
  std::size_t bytes() const { return n * sizeof(T); }
  void upload(const std::vector<T>& v, cudaStream_t s) {
    if (v.size() != n) alloc(v.size());
    if (n) staged_upload(p, v.data(), bytes(), s);
  }
};

// ---------------------------------------------------------------- communication
struct Context;
// Collectives used by the sharded path (one rank per GPU).  NcclComm runs
// them with NCCL over NVLink / NVSwitch; ThreadComm is the single-process
// emulation used to test the sharded path with several ranks on one GPU
// (host barriers only -- no kernel ever waits on another rank's kernel).
struct Comm {
  int rank = 0, size = 1;
  virtual ~Comm() = default;
  // In-place sum over ranks of n complex values on the context stream.
  virtual void allreduce_sum(double2* buf, size_t n, Context* ctx) = 0;
  virtual void broadcast(void* buf, size_t bytes, int root, Context* ctx) = 0;
  // Point-to-point transfers of one step (every rank calls it; the sends and
  // receives of all ranks must match pairwise): ncclSend / ncclRecv in one
  // NCCL group.
  struct Xfer {
    int peer;
    void* buf;
    size_t bytes;
  };
  virtual void exchange(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                        Context* ctx) = 0;
};
// One segment of a sharded exchange: rows [0, n) of `cols` columns of a
// (column stride lda), against the baseline `base` (stride ldb; null = 0).
struct DeltaSeg {
  double2* a;
  const double2* base;
  int64_t n;
  int cols = 1;
  int64_t lda = 0, ldb = 0;
};
// Every row of the segments changed on at most one rank: one allreduce
// makes a = base + sum_ranks (a_rank - base) on every rank (buf: workspace).
void exchange_deltas(Context* ctx, DevBuf<double2>& buf, const std::vector<DeltaSeg>& segs);
std::unique_ptr<Comm> make_nccl_comm(const unsigned char id[128], int rank, int size, int device);
struct LocalGroup;
std::shared_ptr<LocalGroup> make_local_group(int size);
std::unique_ptr<Comm> make_thread_comm(std::shared_ptr<LocalGroup> group, int rank);
void nccl_unique_id(unsigned char id[128]);

// ---------------------------------------------------------------- context
struct ProfAgg {
  int64_t launches = 0;
  double ms = 0, bytes = 0, flops = 0;
};
struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
  double bytes, flops;
};
struct Context {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t timer[2] = {nullptr, nullptr};
  // Per-kernel CUDA-event profiling (off by default; see KernelScope).
  bool profile = false;
  std::vector<ProfRec> pending;
  std::vector<cudaEvent_t> event_pool;
  std::vector<std::pair<std::string, ProfAgg>> agg;
  void collect();
  std::unique_ptr<Comm> comm;  // null: single GPU
  int rank() const { return comm ? comm->rank : 0; }
  int world() const { return comm ? comm->size : 1; }
  // Programmatic dependent launch for the per-iteration kernels (off while
  // profiling, so each kernel's events bracket only its own work).
  bool pdl = true;
  bool use_pdl() const { return pdl && !profile; }
  // residual history of the last single-RHS (F)GMRES with record_history
  // (gmres_driver's report.residual_history, krylov.cpp:118)
  std::vector<double> history;
  Staging staging;  // pinned upload ring of this context's stream
  // Lifetime: the ABI handle holds one reference and every object built on
  // the context holds one; the stream and the context's buffers are released
  // with the last reference (capi.cpp), so an object may outlive
  // hpsb_context_destroy of its context.
  std::atomic<int> refs{1};
  void* owner = nullptr;  // the hpsb_context_s that embeds this context
};

// Brackets one kernel launch with CUDA events when profiling is enabled and
// attributes its algorithmic bytes / flops (the roofline numerators).
struct KernelScope {
  Context* c;
  int idx = -1;
  KernelScope(Context* ctx, const char* name, double bytes, double flops);
  ~KernelScope();
};

// Launch on the context stream with programmatic dependent launch (PDL) and
// an optional thread-block cluster.  A PDL kernel may start while its
// predecessor drains: it must execute pdl_wait() (device.cuh) before it reads
// or writes anything a predecessor produces or consumes; only prefetches of
// data written before the previous host synchronisation may precede it.
#ifdef __CUDACC__
// cluster < 0: a cooperative launch (every CTA co-resident; the kernel
// synchronises its grid) instead of a cluster.
template <typename... KArgs, typename... Args>
void launch_k(Context* ctx, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
              int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[3];
  unsigned na = 0;
  if (cluster < 0) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  if (ctx->use_pdl()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = static_cast<unsigned>(cluster);
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  HPSB_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
  ++ctx->launches;
}
#endif

// ---------------------------------------------------------------- host structure
struct IndexSets {
  int order = 0;
  std::vector<int> left, right, bottom, top, boundary, interior, noncorner, comp_of_full;
};
IndexSets build_index_sets(int order);

struct Face {
  int e1, e2, s1, s2, level, group;
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

struct Gll {
  std::vector<double> nodes, weights, diff;  // diff col-major (N+1)^2
};
Gll gll_rule(int order);

// Quadtree-subtree sharding over G = 2^g ranks: levels
// 1..last_local of the merge tree are eliminated inside each rank's box (the
// box produced by group `rank` of level last_local = L - g); the top g
// levels are global.  Faces of local levels belong to one rank; faces of
// global levels (the cuts between rank boxes) are shared.
struct Partition {
  int G = 1, g = 0, rank = 0, L = 0, last_local = 0;
  std::vector<int> elem_owner;  // [n^2]
  std::vector<int> face_owner;  // [faces], -1 on global-level faces
  std::vector<int> own_elems;
  bool owns_elem(int e) const { return elem_owner[e] == rank; }
};
Partition make_partition(const FaceGraph& g, int G, int rank);
// owners[l - 1][group]: the rank that runs merge `group` of level l
// (owner-computes: the holder of its first child, geometry.cpp).
std::vector<std::vector<int>> merge_owners(const FaceGraph& g, const Partition& part);

// ---------------------------------------------------------------- GEMV work lists
// y[yi] = beta * y[yi] + gamma * z[zi] + alpha * A x[xi]   (complex, A col-major)
// Negative indices: x entries read as 0, y entries are skipped.
struct VItem {
  const double2* A;
  const double2* x;
  const double2* z;
  double2* y;
  const int* xi;
  const int* zi;
  const int* yi;
  int lda, rows, cols, flags;
  double alpha, beta, gamma, pad2;
  static constexpr int kPhaseEnd = 1;  // cluster barrier after this item
};
// A unit is a chain of items executed in order by one CTA.
struct VUnit {
  int first, count;
};
// One kernel launch: a set of independent units.
struct VPhase {
  int unit_begin = 0, unit_count = 0;
  int max_cols = 0;
  int csize = 1;  // CTAs per unit (thread-block cluster)
  double bytes = 0;
  size_t stage = 0;  // operator bytes per CTA staged in smem (0: streamed)
  std::string label;  // profiling name (defaults to the plan's name)
};
struct VPlan {
  std::vector<VItem> items;
  std::vector<VUnit> units;
  std::vector<VPhase> phases;
  DevBuf<VItem> d_items;
  DevBuf<VUnit> d_units;
  int64_t bytes_per_run = 0;  // algorithmic operator bytes streamed per run
  const char* name = "vplan";
  DevBuf<int> idx_store;  // index lists owned by the plan (optional)
  // Start a new phase (one launch, csize CTAs per unit); returns its index.
  int begin_phase(int csize = 1);
  void add_unit(const std::vector<VItem>& chain);
  // Adds A (rows x cols) split into row blocks as independent units.
  void add_split(const VItem& it, int row_block);
  void finalize(cudaStream_t s);
  // Run all phases; vectors `from*` the plan was built on are replaced by `to*`.
  void run(Context* ctx, const double2* from0 = nullptr, double2* to0 = nullptr,
           const double2* from1 = nullptr, double2* to1 = nullptr) const;
  void run_phase(Context* ctx, int p, const double2* from0 = nullptr, double2* to0 = nullptr,
                 const double2* from1 = nullptr, double2* to1 = nullptr) const;
};

// ---------------------------------------------------------------- objects
struct Elements {
  Context* ctx = nullptr;
  int n = 0, order = 0, m = 0, nb = 0;
  double eta = 0, h = 0;
  DevBuf<double2> T;  // [e][nb*nb]
  DevBuf<double2> H;  // [e][nb]
  DevBuf<int> status; // per-element failure flags
  DevBuf<double> Y;   // [e][nb+2][ni] L_ii^{-1}[L_iG | re b~ | im b~] (solution recovery)
  double build_seconds = 0;
  Partition part;     // sharding of the elements over the context's ranks
  // The element stage returns without waiting for the device: the status
  // copy lands in h_status (pinned) behind `done`, and elements_wait checks
  // it at the first call that needs the stage finished (the host builds the
  // skeleton and the merge plans meanwhile).
  int* h_status = nullptr;
  size_t h_status_cap = 0;
  cudaEvent_t done = nullptr;
  bool pending = false;
  int fallbacks = 0;  // elements redone by the pivoted-LU fallback (v1)
  ~Elements();
};
int* pinned_ints_acquire(size_t n, size_t* cap);  // recycled pinned host ints
// Wait for the element stage and raise its per-element errors (mesh.cpp:82-84).
void elements_wait(Elements* el);

struct GemvStream;
struct Skeleton {
  Context* ctx = nullptr;
  Elements* el = nullptr;
  FaceGraph graph;
  int m = 0, bs = 0;
  int64_t dim = 0;
  int nrhs = 1;
  DevBuf<double2> rhs;  // [nrhs][dim]
  // Element-level in/out skeleton indices: [e][nb] (-1 on physical sides).
  std::vector<int> h_in, h_out;
  DevBuf<int> d_in, d_out;
  DevBuf<double2> tside;  // [nrhs][e][nb] physical-side impedance data
  VPlan apply_plan;      // y = x + sum_e scatter(T_e gather(x))
  DevBuf<double2> x_buf, y_buf;  // plan endpoints
  std::shared_ptr<GemvStream> apply_stream;  // the same matvec, TMA-streamed (vcycle_stream.cu)
  std::shared_ptr<void> batch;   // multi-RHS matvec phase (skeleton.cu), built on first use
  // Sharded layout of the solver's vectors: every rank keeps full-length
  // buffers but owns only its subtree's local-face rows; the global rows
  // (faces of the levels above the subtrees: the tail [tail_off, dim)) are
  // replicated.  dist_rows lists the owned rows, then the tail rows encoded
  // as -(row + 1) on ranks other than 0 (updated everywhere, counted in the
  // dot products once).
  int64_t tail_off = 0;
  DevBuf<int> dist_rows;
  int64_t n_dist_rows = 0;
  DevBuf<int> keep_face;  // faces whose rows this rank contributes to a gathered vector
  DevBuf<double2> gather_buf;
};
// Full vector on every rank from a distributed one (owned rows from their
// owner, global rows from rank 0): one allreduce.
void gather_distributed(const Skeleton* sk, double2* v, int R = 1);

struct LevelOps;
struct Hierarchy {
  Context* ctx = nullptr;
  Skeleton* sk = nullptr;
  int depth = 0, total_levels = 0;
  std::vector<std::unique_ptr<LevelOps>> levels;  // levels[l-1], l = 1..depth
  double build_seconds = 0;
  int64_t device_bytes = 0;
  bool pivot_redone = false;  // diagonal-pivot guard tripped: rebuilt with partial pivoting
  ~Hierarchy();
};

struct Precond;

// ---------------------------------------------------------------- entry points
std::unique_ptr<Elements> build_elements(Context* ctx, int n, int order, double eta,
                                         const double* coeff_dev, const double2* source_dev);
// tside_host: [nrhs][e][4][N-1] (boundary_only false) or the physical sides
// only, [nrhs][4][n][N-1] (boundary_only true).
std::unique_ptr<Skeleton> build_skeleton(Elements* el, const double2* tside_host, int nrhs,
                                         bool boundary_only = false);
// distributed (sharded): y valid on the owned and global rows only (one
// allreduce of the global rows) -- the sharded FGMRES's layout; else full.
void skeleton_apply(const Skeleton* sk, const double2* x_dev, double2* y_dev,
                    bool distributed = false);
// Multi-RHS: R <= 32 vectors stored column-wise with leading dimension dim.
void precond_apply_batch(Precond* p, const double2* v, double2* z, int R,
                         bool distributed = false);
void skeleton_apply_batch(const Skeleton* sk, const double2* x, double2* y, int R,
                          bool distributed = false);
hpsb_status fgmres_batch(Skeleton* sk, Precond* pc, const double2* rhs, double2* x, int R,
                         const hpsb_krylov_config& cfg, hpsb_solve_report* reports);
void recover_field(const Skeleton* sk, const double2* x_dev, int rhs_index, double2* field_dev);
// before_wait runs on the host once every device operation of the build is
// enqueued, before the final synchronisation (host work that only needs the
// host-side structure overlaps the device's merge tail).
std::unique_ptr<Hierarchy> build_hierarchy(Skeleton* sk, int depth,
                                           const std::function<void(Hierarchy*)>& before_wait = {});
void hierarchy_level_blocks(const Hierarchy* h, int level, int* nblocks, int* first_face,
                            int* keys, double* data);
// y = M_l x on level l's system (device vectors of the level's length).
void hierarchy_level_apply(Hierarchy* h, int level, const double2* x_dev, double2* y_dev);
Precond* create_precond(Hierarchy* h, const hpsb_mg_config& cfg);
void destroy_precond(Precond* p);
Context* precond_context(const Precond* p);
// Sharded contexts: distributed = true leaves z valid on this rank's own
// (subtree-local) rows and the global rows only, as the sharded FGMRES keeps
// its vectors; false returns the full vector on every rank.
void precond_apply(Precond* p, const double2* v_dev, double2* z_dev, bool distributed = false);
// precond_apply is a fixed launch sequence (single GPU, gamma == 1 or exact
// coarse): it can be captured into a CUDA graph
bool precond_graph_safe(const Precond* p);
void precond_apply_host(Precond* p, const double2* v_host, double2* z_host);
int64_t precond_bytes(const Precond* p);
// Pinned SURVEY §8(d) work: element flops, merge flops (all merges of the
// problem), and per-level operator entries used by precond_pinned_bytes.
void hierarchy_pinned(const Hierarchy* h, double* elem_flops, double* merge_flops,
                      double* level_entries);
double precond_pinned_bytes(const Precond* p);
void merge_pair(Context* ctx, int m, const double2* T1, const double2* H1, const double2* T2,
                const double2* H2, int alpha, int beta, double2* T, double2* H);
hpsb_status fgmres(Skeleton* sk, Precond* pc, const double2* rhs_dev, double2* x_dev,
                   const hpsb_krylov_config& cfg, hpsb_solve_report* rep, bool right = false);
// MgPreconditioner::memory_bytes (multigrid.cpp:102-113) on the device layout
// (box maps of levels 2..depth, merge factors of levels < depth, dense coarse
// inverse), and the device build time of the hierarchy behind it.
int64_t precond_memory(const Precond* p);
double precond_build_seconds(const Precond* p);

// Small device kernels shared between modules (csrc/blas.cu).
void zfill(Context* ctx, double2* p, std::size_t n, double2 v);
void zcopy(Context* ctx, double2* dst, const double2* src, std::size_t n);

}  // namespace hpsb
