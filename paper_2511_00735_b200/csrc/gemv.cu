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
// A plan is a list of phases (kernel launches); a phase is a list of units
// (one CTA each); a unit is a chain of items run in order by its CTA.  Each
// item streams its matrix once with coalesced 16-byte loads (threads map to
// rows of the column-major block, column groups split the K loop) and
// reduces the column groups through shared memory.
#include <algorithm>

#include "device.cuh"
#include "internal.hpp"

namespace hpsb {

namespace {
constexpr int kThreads = 256;

__device__ __forceinline__ double2 ld_vec(const double2* base, const int* idx, int j) {
  if (idx) {
    const int k = idx[j];
    return k >= 0 ? base[k] : make_double2(0.0, 0.0);
  }
  return base[j];
}

__global__ void __launch_bounds__(kThreads) vplan_kernel(const VItem* __restrict__ items,
                                                         const VUnit* __restrict__ units,
                                                         int unit_begin) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* xs = reinterpret_cast<double2*>(smem_raw);
  __shared__ double2 red[kThreads];
  const int tid = threadIdx.x;
  const VUnit u = units[unit_begin + blockIdx.x];
  for (int it = u.first; it < u.first + u.count; ++it) {
    const VItem I = items[it];
    for (int j = tid; j < I.cols; j += kThreads) xs[j] = ld_vec(I.x, I.xi, j);
    __syncthreads();
    for (int r0 = 0; r0 < I.rows; r0 += kThreads) {
      const int rows = min(I.rows - r0, kThreads);
      const int rpad = (rows + 31) & ~31;
      const int groups = kThreads / rpad;
      const int r = tid % rpad, g = tid / rpad;
      double2 acc = make_double2(0.0, 0.0);
      if (I.A && g < groups && r < rows) {
        const double2* Ar = I.A + r0 + r;
        const size_t lda = I.lda;
        int j = g;
        double2 a0, a1, a2, a3;
        for (; j + 3 * groups < I.cols; j += 4 * groups) {
          a0 = ldg2(Ar + j * lda);
          a1 = ldg2(Ar + (j + groups) * lda);
          a2 = ldg2(Ar + (j + 2 * groups) * lda);
          a3 = ldg2(Ar + (j + 3 * groups) * lda);
          acc = cfma(a0, xs[j], acc);
          acc = cfma(a1, xs[j + groups], acc);
          acc = cfma(a2, xs[j + 2 * groups], acc);
          acc = cfma(a3, xs[j + 3 * groups], acc);
        }
        for (; j < I.cols; j += groups) acc = cfma(ldg2(Ar + j * lda), xs[j], acc);
      }
      red[tid] = acc;
      __syncthreads();
      if (tid < rows) {
        double2 s = red[tid];
        for (int gg = 1; gg < groups; ++gg) s = cadd(s, red[tid + gg * rpad]);
        const int row = r0 + tid;
        const int yk = I.yi ? I.yi[row] : row;
        if (yk >= 0) {
          double2 v = cscale(s, I.alpha);
          if (I.gamma != 0.0) v = cadd(v, cscale(ld_vec(I.z, I.zi, row), I.gamma));
          if (I.beta != 0.0) v = cadd(v, cscale(I.y[yk], I.beta));
          I.y[yk] = v;
        }
      }
      __syncthreads();
    }
  }
}

__global__ void fill_kernel(double2* p, size_t n, double2 v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}
}  // namespace

int VPlan::begin_phase() {
  VPhase ph;
  ph.unit_begin = static_cast<int>(units.size());
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

void VPlan::run_phase(Context* ctx, int p) const {
  const VPhase& ph = phases[p];
  if (ph.unit_count == 0) return;
  const size_t smem = sizeof(double2) * std::max(ph.max_cols, 1);
  if (smem > 48 * 1024)
    HPSB_CUDA(cudaFuncSetAttribute(vplan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  KernelScope ks(ctx, name, ph.bytes, 0.0);
  vplan_kernel<<<ph.unit_count, kThreads, smem, ctx->stream>>>(d_items.p, d_units.p,
                                                                  ph.unit_begin);
  HPSB_LAUNCHED(ctx);
}

void VPlan::run(Context* ctx) const {
  for (int p = 0; p < static_cast<int>(phases.size()); ++p) run_phase(ctx, p);
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
