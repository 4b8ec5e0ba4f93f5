// Fused V-cycle step for medium merges: one thread-block cluster per merge.
//
// The middle levels of the hierarchy have too few merges to fill the GPU with
// one CTA each, and a merge's operators are too large for one CTA's shared
// memory, but small enough to be split across a cluster of C <= 16 CTAs.
// Every CTA owns a row slice of each operator block of the step and copies
// all of them into its shared memory in ONE cp.async burst issued before the
// PDL wait (operators never depend on the vectors, so the copies overlap the
// previous kernel).  The dependent chain of multigrid.cpp:47-98 then runs
// on-chip: each GEMV produces the CTA's slice of its output vector, the
// slices are exchanged through distributed shared memory (DSMEM) after a
// cluster barrier, and only the level's inputs / outputs touch global memory:
//   down: t = r1 - T2_ss r2,  x1 = W t,  x2 = r2 - T1_ss x1,
//         out[s] = (x1, x2),  r[out_k,p] -= T_k,ps x_k
//   up:   b1 = T2_sp u2, b2 = T1_sp u1, t = b1 - T2_ss b2, y1 = W t,
//         out[s2] += T1_ss y1 - b2,  out[s1] -= y1
#include <cooperative_groups.h>

#include <algorithm>

#include "device.cuh"
#include "gemv_device.cuh"
#include "vcycle_device.cuh"
#include "vcycle_small.hpp"

namespace cg = cooperative_groups;

namespace hpsb {

namespace {
constexpr int kThreads = 256;

struct Slices {
  int cs, s0, ns;    // rows of the s-blocks
  int cp1, a0, na;   // rows of T1_ps
  int cp2, b0, nb;   // rows of T2_ps
};
__host__ __device__ inline Slices slices(int s, int p1, int p2, int C, int c) {
  Slices q;
  q.cs = cluster_chunk(s, C);
  q.s0 = min(s, c * q.cs);
  q.ns = max(0, min(s, q.s0 + q.cs) - q.s0);
  q.cp1 = cluster_chunk(max(p1, 1), C);
  q.a0 = min(p1, c * q.cp1);
  q.na = max(0, min(p1, q.a0 + q.cp1) - q.a0);
  q.cp2 = cluster_chunk(max(p2, 1), C);
  q.b0 = min(p2, c * q.cp2);
  q.nb = max(0, min(p2, q.b0 + q.cp2) - q.b0);
  return q;
}

// Shared-memory footprint (double2 units) of one CTA; the same layout is used
// by every CTA of the cluster (DSMEM addresses must match).
__host__ __device__ inline size_t cluster_layout(int s, int p1, int p2, int C, bool down,
                                                 size_t* off /* 12 offsets or null */) {
  const Slices q = slices(s, p1, p2, C, 0);  // rank 0 has the largest slices
  const size_t ops = down ? 3ull * q.cs * s + static_cast<size_t>(q.cp1) * s + static_cast<size_t>(q.cp2) * s
                          : static_cast<size_t>(q.cs) * (p1 + p2) + 3ull * q.cs * s;
  size_t o = 0;
  size_t v[12];
  v[0] = o; o += ops;                               // operator slices
  v[1] = o; o += std::max(std::max(s, p1), 1);      // full vector A
  v[2] = o; o += std::max(std::max(s, p2), 1);      // full vector B
  v[3] = o; o += q.cs;                              // exchange slice 1
  v[4] = o; o += q.cs;                              // exchange slice 2
  v[5] = o; o += q.cs;                              // exchange slice 3
  if (off)
    for (int k = 0; k < 6; ++k) off[k] = v[k];
  return o;
}

__device__ __forceinline__ void stage_rows(double2* dst, const double2* A, int lda, int r0, int nr,
                                           int ncols) {
  // column segments of nr rows; warps over columns, lanes over rows (no division)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = warp; c < ncols; c += kThreads / 32)
    for (int r = lane; r < nr; r += 32)
      cp_async16(dst + r + static_cast<size_t>(c) * nr, A + r0 + r + static_cast<size_t>(c) * lda);
}

// full[j] = slice_owner(j)[j - owner * cs] for j < n (DSMEM gather)
__device__ __forceinline__ void gather_full(cg::cluster_group& cl, double2* ex, int cs, int n,
                                            double2* full) {
  for (int j = threadIdx.x; j < n; j += kThreads) {
    const int owner = j / cs;
    full[j] = cl.map_shared_rank(ex, owner)[j - owner * cs];
  }
  __syncthreads();
}

// rows >= kThreads are processed in passes of kThreads rows
template <class F>
__device__ __forceinline__ void gemv_rows(const double2* A, int nr, int ncols, const double2* x,
                                          double2* red, F&& emit) {
  for (int r0 = 0; r0 < nr; r0 += kThreads) {
    const int rows = min(nr - r0, kThreads);
    const double2 y = smem_gemv<kThreads>(A + r0, nr, rows, ncols, x, red);
    if (threadIdx.x < rows) emit(r0 + threadIdx.x, y);
  }
}

__global__ void __launch_bounds__(kThreads) merge_cluster_kernel(const SmallMerge* __restrict__ ms,
                                                                 int down, double2* r,
                                                                 double2* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double2 red[kThreads];
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks()), c = static_cast<int>(cl.block_rank());
  const SmallMerge M = ms[blockIdx.x / C];
  const int tid = threadIdx.x, s = M.s, p1 = M.p1, p2 = M.p2, P1 = M.P1, P2 = M.P2;
  const Slices q = slices(s, p1, p2, C, c);
  size_t off[6];
  cluster_layout(s, p1, p2, C, down != 0, off);
  double2* base = reinterpret_cast<double2*>(smem_raw);
  double2* fa = base + off[1];
  double2* fb = base + off[2];
  double2* ex1 = base + off[3];
  double2* ex2 = base + off[4];
  double2* ex3 = base + off[5];
  pdl_trigger();

  const double2 *T1ss = M.T1 + p1 + static_cast<size_t>(p1) * P1,
                *T2ss = M.T2 + p2 + static_cast<size_t>(p2) * P2;
  double2* A_t2ss = base;
  double2* A_w = A_t2ss + static_cast<size_t>(q.ns) * s;
  double2* A_t1ss = A_w + static_cast<size_t>(q.ns) * s;
  if (down) {
    double2* A_t1ps = A_t1ss + static_cast<size_t>(q.ns) * s;
    double2* A_t2ps = A_t1ps + static_cast<size_t>(q.na) * s;
    stage_rows(A_t2ss, T2ss, P2, q.s0, q.ns, s);
    stage_rows(A_w, M.W, s, q.s0, q.ns, s);
    stage_rows(A_t1ss, T1ss, P1, q.s0, q.ns, s);
    stage_rows(A_t1ps, M.T1 + static_cast<size_t>(p1) * P1, P1, q.a0, q.na, s);
    stage_rows(A_t2ps, M.T2 + static_cast<size_t>(p2) * P2, P2, q.b0, q.nb, s);
    cp_async_commit();
    pdl_wait();
    for (int j = tid; j < s; j += kThreads) fa[j] = __ldcg(r + M.in2s[j]);  // r2 (full)
    double2 v1 = make_double2(0.0, 0.0);
    if (tid < q.ns) v1 = __ldcg(r + M.in1s[q.s0 + tid]);
    cp_async_wait_all();
    __syncthreads();
    // t = r1 - T2_ss r2
    gemv_rows(A_t2ss, q.ns, s, fa, red, [&](int i, double2 y) { ex1[i] = csub(v1, y); });
    cl.sync();
    gather_full(cl, ex1, q.cs, s, fb);
    // x1 = W t
    gemv_rows(A_w, q.ns, s, fb, red, [&](int i, double2 y) {
      ex2[i] = y;
      __stcg(out + M.in1s[q.s0 + i], y);
    });
    cl.sync();
    gather_full(cl, ex2, q.cs, s, fb);  // fb = x1 (full)
    // x2 = r2 - T1_ss x1
    gemv_rows(A_t1ss, q.ns, s, fb, red, [&](int i, double2 y) {
      const double2 x2 = csub(fa[q.s0 + i], y);
      ex3[i] = x2;
      __stcg(out + M.in2s[q.s0 + i], x2);
    });
    // r[out1_p] -= T1_ps x1
    gemv_rows(A_t1ps, q.na, s, fb, red, [&](int i, double2 y) {
      const int o = M.out1p[q.a0 + i];
      __stcg(r + o, csub(__ldcg(r + o), y));
    });
    cl.sync();
    gather_full(cl, ex3, q.cs, s, fa);  // fa = x2 (full)
    // r[out2_p] -= T2_ps x2
    gemv_rows(A_t2ps, q.nb, s, fa, red, [&](int i, double2 y) {
      const int o = M.out2p[q.b0 + i];
      __stcg(r + o, csub(__ldcg(r + o), y));
    });
  } else {
    double2* A_t2sp = A_t1ss + static_cast<size_t>(q.ns) * s;
    double2* A_t1sp = A_t2sp + static_cast<size_t>(q.ns) * p2;
    stage_rows(A_t2ss, T2ss, P2, q.s0, q.ns, s);
    stage_rows(A_w, M.W, s, q.s0, q.ns, s);
    stage_rows(A_t1ss, T1ss, P1, q.s0, q.ns, s);
    stage_rows(A_t2sp, M.T2 + p2, P2, q.s0, q.ns, p2);
    stage_rows(A_t1sp, M.T1 + p1, P1, q.s0, q.ns, p1);
    cp_async_commit();
    pdl_wait();
    for (int j = tid; j < p1; j += kThreads) fa[j] = __ldcg(out + M.in1p[j]);  // u1
    for (int j = tid; j < p2; j += kThreads) fb[j] = __ldcg(out + M.in2p[j]);  // u2
    cp_async_wait_all();
    __syncthreads();
    double2 b1 = make_double2(0.0, 0.0), b2 = make_double2(0.0, 0.0);
    // b1 = T2_sp u2, b2 = T1_sp u1 (ns <= kThreads rows)
    {
      const double2 y1 = q.ns ? smem_gemv<kThreads>(A_t2sp, q.ns, q.ns, p2, fb, red) : b1;
      const double2 y2 = q.ns ? smem_gemv<kThreads>(A_t1sp, q.ns, q.ns, p1, fa, red) : b2;
      if (tid < q.ns) b1 = y1, b2 = y2, ex1[tid] = y2;
    }
    cl.sync();
    gather_full(cl, ex1, q.cs, s, fb);  // fb = b2 (full)
    // t = b1 - T2_ss b2
    gemv_rows(A_t2ss, q.ns, s, fb, red, [&](int i, double2 y) { ex2[i] = csub(b1, y); });
    cl.sync();
    gather_full(cl, ex2, q.cs, s, fa);  // fa = t (full)
    // y1 = W t;  out[s1] -= y1
    gemv_rows(A_w, q.ns, s, fa, red, [&](int i, double2 y) {
      ex3[i] = y;
      const int o = M.in1s[q.s0 + i];
      __stcg(out + o, csub(__ldcg(out + o), y));
    });
    cl.sync();
    gather_full(cl, ex3, q.cs, s, fb);  // fb = y1 (full)
    // out[s2] += T1_ss y1 - b2
    gemv_rows(A_t1ss, q.ns, s, fb, red, [&](int i, double2 y) {
      const int o = M.in2s[q.s0 + i];
      __stcg(out + o, cadd(__ldcg(out + o), csub(y, b2)));
    });
  }
  cl.sync();  // no CTA exits while another still reads its shared memory
}
}  // namespace

size_t cluster_merge_smem(int s, int p1, int p2, int C) {
  const size_t d = cluster_layout(s, p1, p2, C, true, nullptr);
  const size_t u = cluster_layout(s, p1, p2, C, false, nullptr);
  return sizeof(double2) * std::max(d, u);
}

bool cluster_merge_fits(size_t smem, int csize) {
  static const bool attr = [] {
    HPSB_CUDA(cudaFuncSetAttribute(merge_cluster_kernel,
                                   cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    return true;
  }();
  (void)attr;
  allow_smem<merge_cluster_kernel>(smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(csize);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, merge_cluster_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return n > 0;
}

void ClusterLevel::run(Context* ctx, bool down, double2* r, double2* out) const {
  if (!count) return;
  allow_smem<merge_cluster_kernel>(smem);
  KernelScope ks(ctx, label.empty() ? (down ? "vcycle_down" : "vcycle_up") : label.c_str(),
                 down ? bytes_down : bytes_up, 0.0);
  launch_k(ctx, merge_cluster_kernel, dim3(count * csize), dim3(kThreads), smem, csize,
           static_cast<const SmallMerge*>(d.p), down ? 1 : 0, r, out);
}

}  // namespace hpsb
