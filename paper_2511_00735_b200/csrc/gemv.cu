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
#include <cstring>

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

template <bool kCluster>
__global__ void __launch_bounds__(kThreads) vplan_kernel(const VItem* __restrict__ items,
                                                         const VUnit* __restrict__ units,
                                                         int unit_begin, int csize, Rebind bind) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* xs = reinterpret_cast<double2*>(smem_raw);
  __shared__ double2 red[kThreads];
  const int crank = kCluster ? static_cast<int>(blockIdx.x % csize) : 0;
  const VUnit u = units[unit_begin + (kCluster ? blockIdx.x / csize : blockIdx.x)];
  for (int it = u.first; it < u.first + u.count; ++it) {
    const VItem I = items[it];
    const int chunk = kCluster ? (((I.rows + csize - 1) / csize + 31) & ~31) : I.rows;
    const int rb = crank * chunk, re = min(I.rows, rb + chunk);
    if (rb < re)
      gemv_item_rows(I, rb, re, rebind(I.x, bind), rebind(I.z, bind),
                     const_cast<double2*>(rebind(I.y, bind)), xs, red);
    if (kCluster && (I.flags & VItem::kPhaseEnd)) cg::this_cluster().sync();
    else __syncthreads();
  }
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
  d_items.upload(items, s);
  d_units.upload(units, s);
}

void VPlan::run_phase(Context* ctx, int p, const double2* from0, double2* to0,
                      const double2* from1, double2* to1) const {
  const VPhase& ph = phases[p];
  if (ph.unit_count == 0) return;
  Rebind bind{{from0, from1}, {to0, to1}};
  const size_t smem = sizeof(double2) * std::max(ph.max_cols, 1);
  KernelScope ks(ctx, ph.label.empty() ? name : ph.label.c_str(), ph.bytes, 0.0);
  if (ph.csize <= 1) {
    allow_smem<vplan_kernel<false>>(smem);
    vplan_kernel<false><<<ph.unit_count, kThreads, smem, ctx->stream>>>(d_items.p, d_units.p,
                                                                         ph.unit_begin, 1, bind);
  } else {
    static const bool nonportable = [] {  // thread-safe one-time init
      HPSB_CUDA(cudaFuncSetAttribute(vplan_kernel<true>,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      return true;
    }();
    (void)nonportable;
    allow_smem<vplan_kernel<true>>(smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ph.unit_count * ph.csize);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ph.csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HPSB_CUDA(cudaLaunchKernelEx(&cfg, vplan_kernel<true>, d_items.p, d_units.p, ph.unit_begin,
                                 ph.csize, bind));
  }
  HPSB_LAUNCHED(ctx);
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

void staged_upload(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  Staging& st = staging();
  if (!st.base || st.stream != s || bytes > st.size / 2) {
    HPSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
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
