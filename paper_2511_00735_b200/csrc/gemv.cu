// Batched complex GEMV work lists: the memory-bound per-iteration engine.
//
// Every per-iteration operator of the hot path is a set of dense complex
// matrix blocks applied to gathered vector entries and scattered back:
//   - the global ItI interface matvec (BlockMatrix::apply on the skeleton,
//     proj/src/block_matrix.cpp:23-31): y = x + sum_e scatter(T_e gather(x));
//   - the multigrid sweeps (MgPreconditioner::apply_level,
//     proj/src/multigrid.cpp:47-98): group solves, restriction C_l w and
//     prolongation B_l z, all expressed on the stored box maps;
//   - the coarse-level matvec inside gmres_fixed_steps.
// A plan is a list of phases (kernel launches); a phase is a list of units;
// a unit is a chain of items run in order by one thread-block cluster of
// `csize` CTAs (csize = 1: a single CTA).  The CTAs of a cluster split the
// rows of every item; items flagged kPhaseEnd are followed by a cluster
// barrier (barrier.cluster release/acquire), so a whole merge's dependent
// GEMV chain runs in one launch on up to 16 SMs.  Each item streams its
// matrix once with coalesced 16-byte loads (threads map to rows of the
// column-major block, column groups split the K loop, shared-memory
// reduction); vector traffic goes through L2 (ld/st .cg) so the cluster
// barrier is the only ordering needed.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <tuple>

#include "device.cuh"
#include "gemv_device.cuh"
#include "internal.hpp"

namespace cg = cooperative_groups;

namespace hpsb {

namespace {
constexpr int kThreads = kGemvThreads;

// Pointer rebinding: vectors a plan was built on (bind.from[k]) are replaced
// at run time by the caller's buffers (bind.to[k]), so no copies are needed
// around a plan run.
struct Rebind {
  const double2* from[2];
  double2* to[2];
};
__device__ __forceinline__ const double2* rebind(const double2* p, const Rebind& b) {
  return p == b.from[0] ? b.to[0] : p == b.from[1] ? b.to[1] : p;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

// kStage: every item's operator rows for this CTA are copied into shared
// memory before the PDL wait -- operators never depend on the vectors, so
// the copies overlap the previous kernel's tail and the chain below then
// runs on on-chip operands (the small / medium levels are latency bound).
// Otherwise the first 32 KB of the CTA's operator rows are prefetched into L2.
template <bool kCluster, bool kStage>
__global__ void __launch_bounds__(kThreads) vplan_kernel(const VItem* __restrict__ items,
                                                         const VUnit* __restrict__ units,
                                                         int unit_begin, int csize, int xs_cols,
                                                         Rebind bind) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* xs = reinterpret_cast<double2*>(smem_raw);
  double2* stage = xs + xs_cols;
  __shared__ double2 red[kThreads];
  pdl_trigger();
  const int crank = kCluster ? static_cast<int>(blockIdx.x % csize) : 0;
  const VUnit u = units[unit_begin + (kCluster ? blockIdx.x / csize : blockIdx.x)];
  auto rows_of = [&](const VItem& I, int& rb, int& re) {
    const int chunk = kCluster ? cluster_chunk(I.rows, csize) : I.rows;
    rb = crank * chunk;
    re = min(I.rows, rb + chunk);
  };
  if (kStage) {
    size_t off = 0;
    for (int it = u.first; it < u.first + u.count; ++it) {
      const VItem I = items[it];
      int rb, re;
      rows_of(I, rb, re);
      if (!I.A || rb >= re) continue;
      const int nr = re - rb;
      for (int k = threadIdx.x; k < nr * I.cols; k += kThreads)
        cp_async16(stage + off + k, I.A + rb + (k % nr) + static_cast<size_t>(k / nr) * I.lda);
      off += static_cast<size_t>(nr) * I.cols;
    }
    asm volatile("cp.async.commit_group;\n" ::);
  } else {
    int budget = 256;  // 128-byte lines per CTA
    for (int it = u.first; it < u.first + u.count && budget > 0; ++it) {
      const VItem I = items[it];
      int rb, re;
      rows_of(I, rb, re);
      if (!I.A || rb >= re) continue;
      const int lines = ((re - rb) * 16 + 127) / 128;
      const int n = min(budget, lines * I.cols);
      for (int k = threadIdx.x; k < n; k += kThreads)
        prefetch_l2(I.A + rb + (k % lines) * 8 + static_cast<size_t>(k / lines) * I.lda);
      budget -= n;
    }
  }
  pdl_wait();
  if (kStage) {
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();  // every thread's copies visible before any operand read
  }
  size_t off = 0;
  for (int it = u.first; it < u.first + u.count; ++it) {
    const VItem I = items[it];
    int rb, re;
    rows_of(I, rb, re);
    if (rb < re) {
      if (kStage) {
        gemv_item_rows<true>(I, rb, re, rebind(I.x, bind), rebind(I.z, bind),
                             const_cast<double2*>(rebind(I.y, bind)), xs, red, stage + off, re - rb);
        if (I.A) off += static_cast<size_t>(re - rb) * I.cols;
      } else {
        gemv_item_rows<false>(I, rb, re, rebind(I.x, bind), rebind(I.z, bind),
                              const_cast<double2*>(rebind(I.y, bind)), xs, red);
      }
    }
    if (kCluster && (I.flags & VItem::kPhaseEnd)) cg::this_cluster().sync();
    else __syncthreads();
  }
}

template <auto Kernel, typename Tuple>
void launch_plan(Context* ctx, int grid, size_t smem, int csize, const Tuple& args) {
  allow_smem<Kernel>(smem);
  std::apply([&](auto... a) { launch_k(ctx, Kernel, dim3(grid), dim3(kThreads), smem, csize, a...); },
             args);
}

__global__ void fill_kernel(double2* p, size_t n, double2 v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}
}  // namespace

int VPlan::begin_phase(int csize) {
  VPhase ph;
  ph.unit_begin = static_cast<int>(units.size());
  ph.csize = csize;
  phases.push_back(ph);
  return static_cast<int>(phases.size()) - 1;
}

void VPlan::add_unit(const std::vector<VItem>& chain) {
  VUnit u{static_cast<int>(items.size()), static_cast<int>(chain.size())};
  for (const auto& it : chain) {
    items.push_back(it);
    phases.back().max_cols = std::max(phases.back().max_cols, it.cols);
    if (it.A) {
      bytes_per_run += int64_t(16) * it.rows * it.cols;
      phases.back().bytes += 16.0 * it.rows * it.cols;
    }
  }
  units.push_back(u);
  phases.back().unit_count++;
}

void VPlan::add_split(const VItem& it, int row_block) {
  for (int r0 = 0; r0 < it.rows; r0 += row_block) {
    VItem s = it;
    s.rows = std::min(row_block, it.rows - r0);
    if (s.A) s.A += r0;
    if (s.yi) s.yi += r0;
    else s.y += r0;
    if (s.zi) s.zi += r0;
    else if (s.z) s.z += r0;
    add_unit({s});
  }
}

void VPlan::finalize(cudaStream_t s) {
  // Stage a phase's operators in shared memory when every CTA's share fits
  // (default 96 KB: two CTAs per SM).
  constexpr size_t limit = 96 * 1024;
  for (VPhase& ph : phases) {
    size_t worst = 0;
    for (int ui = ph.unit_begin; ui < ph.unit_begin + ph.unit_count; ++ui) {
      const VUnit& u = units[ui];
      for (int rank = 0; rank < ph.csize; ++rank) {
        size_t b = 0;
        for (int it = u.first; it < u.first + u.count; ++it) {
          const VItem& I = items[it];
          if (!I.A) continue;
          const int chunk = ph.csize > 1 ? cluster_chunk(I.rows, ph.csize) : I.rows;
          const int rb = rank * chunk, re = std::min(I.rows, rb + chunk);
          if (re > rb) b += sizeof(double2) * static_cast<size_t>(re - rb) * I.cols;
        }
        worst = std::max(worst, b);
      }
    }
    // Staging serialises each CTA's load and compute and (at up to 96 KB a
    // CTA) caps residency at ~2 CTAs/SM: it pays for latency-bound phases of
    // a few MB, not for streaming phases (ncu, cfg3: staged 47 MB phases ran
    // at 1.7-2.1 TB/s, streamed ones at 2.3-4.7).
    ph.stage = (worst <= limit && ph.bytes <= 16e6) ? worst : 0;
  }
  d_items.upload(items, s);
  d_units.upload(units, s);
}

void VPlan::run_phase(Context* ctx, int p, const double2* from0, double2* to0,
                      const double2* from1, double2* to1) const {
  const VPhase& ph = phases[p];
  if (ph.unit_count == 0) return;
  Rebind bind{{from0, from1}, {to0, to1}};
  const int xs_cols = std::max(ph.max_cols, 1);
  const size_t smem = sizeof(double2) * xs_cols + ph.stage;
  KernelScope ks(ctx, ph.label.empty() ? name : ph.label.c_str(), ph.bytes, 0.0);
  const int grid = ph.unit_count * std::max(ph.csize, 1);
  auto args = std::make_tuple(d_items.p, d_units.p, ph.unit_begin, ph.csize, xs_cols, bind);
  if (ph.csize <= 1) {
    if (ph.stage) launch_plan<vplan_kernel<false, true>>(ctx, grid, smem, 1, args);
    else launch_plan<vplan_kernel<false, false>>(ctx, grid, smem, 1, args);
  } else {
    static const bool nonportable = [] {  // thread-safe one-time init
      HPSB_CUDA(cudaFuncSetAttribute(vplan_kernel<true, true>,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      HPSB_CUDA(cudaFuncSetAttribute(vplan_kernel<true, false>,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      return true;
    }();
    (void)nonportable;
    if (ph.stage) launch_plan<vplan_kernel<true, true>>(ctx, grid, smem, ph.csize, args);
    else launch_plan<vplan_kernel<true, false>>(ctx, grid, smem, ph.csize, args);
  }
  HPSB_CUDA(cudaGetLastError());
}

void VPlan::run(Context* ctx, const double2* from0, double2* to0, const double2* from1,
                double2* to1) const {
  for (int p = 0; p < static_cast<int>(phases.size()); ++p)
    run_phase(ctx, p, from0, to0, from1, to1);
}

KernelScope::KernelScope(Context* ctx, const char* name, double bytes, double flops) : c(ctx) {
  if (!c->profile) return;
  cudaEvent_t e[2];
  for (auto& ev : e) {
    if (c->event_pool.empty()) {
      HPSB_CUDA(cudaEventCreate(&ev));
    } else {
      ev = c->event_pool.back();
      c->event_pool.pop_back();
    }
  }
  HPSB_CUDA(cudaEventRecord(e[0], c->stream));
  c->pending.push_back({name, e[0], e[1], bytes, flops});
  idx = static_cast<int>(c->pending.size()) - 1;
}

KernelScope::~KernelScope() {
  if (idx >= 0) cudaEventRecord(c->pending[idx].b, c->stream);
}

void Context::collect() {
  if (pending.empty()) return;
  HPSB_CUDA(cudaStreamSynchronize(stream));
  for (auto& r : pending) {
    float ms = 0;
    HPSB_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    ProfAgg* a = nullptr;
    for (auto& kv : agg)
      if (kv.first == r.name) a = &kv.second;
    if (!a) {
      agg.emplace_back(r.name, ProfAgg{});
      a = &agg.back().second;
    }
    a->launches += 1, a->ms += ms, a->bytes += r.bytes, a->flops += r.flops;
    event_pool.push_back(r.a);
    event_pool.push_back(r.b);
  }
  pending.clear();
}

Context*& bound_context() {
  thread_local Context* c = nullptr;
  return c;
}
cudaStream_t alloc_stream() {
  const Context* c = bound_context();
  return c ? c->stream : nullptr;
}

// Pinned rings are recycled process-wide: cudaMallocHost of a 512 MB ring
// costs ~0.1-0.5 s (page pinning) and cudaFreeHost synchronises the device,
// so a context takes a ring from the pool at its first staged upload and
// returns it when it is destroyed (its stream drained by then).
namespace {
std::mutex g_ring_mu;
std::vector<std::pair<unsigned char*, size_t>> g_rings;
}  // namespace

Staging::~Staging() {
  if (!base) return;
  std::lock_guard<std::mutex> lk(g_ring_mu);
  g_rings.emplace_back(base, size);
}

void staged_upload(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  Context* c = bound_context();
  if (!c || c->stream != s || bytes > kStagingMax / 2) {
    HPSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  Staging& st = c->staging;
  if (!st.base) {
    {
      std::lock_guard<std::mutex> lk(g_ring_mu);
      if (!g_rings.empty()) {
        st.base = g_rings.back().first, st.size = g_rings.back().second;
        g_rings.pop_back();
      }
    }
    if (!st.base) {
      HPSB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&st.base), kStagingMax));
      st.size = kStagingMax;
    }
    st.head = 0;
  }
  const size_t need = (bytes + 255) & ~size_t(255);
  if (st.head + need > st.size) {
    HPSB_CUDA(cudaStreamSynchronize(s));  // all earlier staged copies have completed
    st.head = 0;
  }
  std::memcpy(st.base + st.head, src, bytes);
  HPSB_CUDA(cudaMemcpyAsync(dst, st.base + st.head, bytes, cudaMemcpyHostToDevice, s));
  st.head += need;
}

void zfill(Context* ctx, double2* p, std::size_t n, double2 v) {
  if (!n) return;
  const int blocks = static_cast<int>(std::min<std::size_t>((n + 255) / 256, 4 * 148));
  KernelScope ks(ctx, "fill", 16.0 * n, 0.0);
  fill_kernel<<<blocks, 256, 0, ctx->stream>>>(p, n, v);
  HPSB_LAUNCHED(ctx);
}

void zcopy(Context* ctx, double2* dst, const double2* src, std::size_t n) {
  if (!n) return;
  HPSB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double2), cudaMemcpyDeviceToDevice, ctx->stream));
}

}  // namespace hpsb
