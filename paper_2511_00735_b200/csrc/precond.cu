#include <chrono>
// K4/K5: the HPS-multigrid preconditioner apply on the stored box maps.
//
// MgPreconditioner::apply_level (proj/src/multigrid.cpp:30-100) with gamma = 1
// is a V-cycle over the merge hierarchy.  On the B200 it runs in place on two
// skeleton-length vectors r (residual, initialised with v) and out:
//   down, level l = 1 .. depth-1, per merge (A_g x = v_g solved through
//   W = (I - T2_ss T1_ss)^{-1}):
//     D1  t          = r[in1_s] - T2_ss r[in2_s]
//     D2  out[in1_s] = W t                                  (x1)
//     D3  out[in2_s] = r[in2_s] - T1_ss out[in1_s]          (x2)
//     D4  r[out_k_p] -= T_k,ps out[ink_s]   (k = 1, 2)      (restriction, C_l w)
//   coarse, level depth: gmres_fixed_steps(M_depth, r_tail, coarse_iters)
//     (multigrid.cpp:37-41), M_depth = I + sum_boxes scatter(T_box);
//   up, level l = depth-1 .. 1 (prolongation, B_l z then A_g^{-1}):
//     U1  b1 = T2_sp out[in2_p],  b2 = T1_sp out[in1_p]
//     U2  t  = b1 - T2_ss b2
//     U3  y1 = W t
//     U4  out[in2_s] += T1_ss y1 - b2,   out[in1_s] -= y1
// R (v - M F v) only needs C_l w, so no full M_l
// apply is ever streamed.  Levels with many merges run one CTA per merge
// (a chained unit); levels with few, large merges split every phase over
// row blocks so the whole GPU streams the maps.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "device.cuh"
#include "gemv_device.cuh"
#include "hierarchy.hpp"
#include "vcycle_device.cuh"
#include "vcycle_small.hpp"
#include "zgemm.hpp"
#include "zgemv_batch.hpp"

namespace hpsb {

struct Precond {
  Hierarchy* h = nullptr;
  hpsb_mg_config cfg{};
  Context* ctx = nullptr;
  int64_t dim = 0, off_d = 0, dim_d = 0;
  DevBuf<double2> r, out, tmp;
  VPlan down, up, coarse_mv;
  // sharded: levels above the subtree boxes (replicated on every rank)
  VPlan down_g, up_g;
  DevBuf<int> keep_face;  // faces whose result this rank contributes to z
  DevBuf<int> coarse_idx;
  DevBuf<double2> V, cv, cw, Hm, gv, rs;
  DevBuf<double> rc, state;
  int64_t bytes_per_apply = 0;
  // fused coarse solve (one cluster launch)
  bool coarse_fused = false;
  bool coarse_cluster = false;  // on-chip variant (coarse_cluster_kernel)
  std::unique_ptr<CoarseWide> coarse_wide;  // persistent grid variant (large coarse systems)
  int coarse_slice = 0;
  size_t coarse_smem = 0, coarse_stage = 0;
  int coarse_xs = 0;
  DevBuf<VItem> coarse_items;
  int coarse_nitems = 0, coarse_max_cols = 0, coarse_csize = 16;
  // exact coarse (MgConfig.exact_coarse): dense inverse of M_depth + one GEMV
  DevBuf<double2> cinv;
  DevBuf<int> exact_yi;
  VPlan exact_mv;
  // per-level execution order of the sweeps
  struct Step {
    int level = 0, small = -1, cluster = -1, stream = -1, wide = -1;
    const VPlan* plan = nullptr;
    int p0 = 0, p1 = 0;
  };
  std::vector<Step> down_steps, up_steps;
  std::vector<std::unique_ptr<SmallLevel>> smalls;
  std::vector<std::unique_ptr<ClusterLevel>> clusters;
  std::vector<std::unique_ptr<StreamLevel>> streams;
  std::vector<std::unique_ptr<WideLevel>> wides;
  std::vector<int> small_level_of;  // level -> smalls index (-1: none)
  // fused-operator levels: per level, the folded down / up operators of every
  // merge, their index lists and the plan items that apply them
  struct FusedOps {
    DevBuf<double2> K;
    DevBuf<int> idx;
    std::vector<VItem> down, up;
  };
  std::vector<std::unique_ptr<FusedOps>> fused;
  // gamma > 1: level systems M_l on faces >= first_face(l) (global indices),
  // and per-level saved residual / accumulated correction
  std::vector<VPlan> level_mv;  // [l], l = 2..depth
  DevBuf<double2> gam_rc, gam_z, gam_t;
  double bytes_small = 0;
  // ---- multi-RHS (built on first use, capacity kBatchMaxRhs)
  // stage_items[dir][l][k]: items of every merge of level l in stage k
  std::vector<std::vector<std::vector<VItem>>> stage_items[2];
  size_t tmp_total = 0;
  bool batch_ready = false;
  DevBuf<double2> rB, tmpB, VB, cvB, cwB, HmB, gvB, rsB;
  DevBuf<double> rcB, stateB;
  std::vector<BPhase> bdown, bup;
  BPhase bcoarse;              // coarse matvec of the batched gmres_fixed_steps
  std::vector<BPhase> bexact;  // exact coarse: one phase per column chunk
  // sharded: the global rows (faces of the levels above the subtrees) form
  // the tail [tail_off, dim) of every skeleton vector; exchange buffers
  int64_t tail_off = 0;
  DevBuf<double2> xbuf, xsave;
  void run_step(const Step& st, bool down, double2* z) const {
    if (st.stream >= 0) streams[st.stream]->run(ctx, down, r.p, z);
    else if (st.wide >= 0) wides[st.wide]->run(ctx, down, r.p, z);
    else if (st.small >= 0) smalls[st.small]->run(ctx, down, r.p, z);
    else if (st.cluster >= 0) clusters[st.cluster]->run(ctx, down, r.p, z);
    else
      for (int q = st.p0; q < st.p1; ++q) st.plan->run_phase(ctx, q, out.p, z);
  }
  void run_steps(bool down, bool global, double2* z) const {
    const int last_local = h->sk->el->part.last_local;
    for (const Step& st : down ? down_steps : up_steps)
      if ((st.level > last_local) == global) run_step(st, down, z);
  }
  void run_global_sharded(bool down, double2* z);
  void run_global_level(const Step& st, bool down, double2* z);
};

constexpr int kMaxCoarseIters = 30;    // fused / on-chip coarse kernels
constexpr int kCoarseItersMax = 512;   // MgConfig.coarse_iters (coarse_finish_kernel's y)
constexpr int64_t kExactCoarseMax = 24576;  // dense coarse inverse: <= 9.7 GB
constexpr size_t kSmallMergeSmemMax = 160 * 1024;
constexpr size_t kClusterMergeSmemMax = 200 * 1024;

namespace {
constexpr int kCoarseThreads = 1024;
constexpr int kCoarseRowsReg = 8;  // coarse_step_kernel keeps <= 8 rows of w per thread in registers

// Dense M_depth = I + sum_boxes scatter(T_box): box b writes rows out_b (its
// outgoing slots, owned by b alone) and columns in_b; the identity was
// written beforehand and no box touches a diagonal entry (in != out).
__global__ void coarse_densify_kernel(const double2* __restrict__ tperm, const int64_t* __restrict__ toff,
                                      const int* __restrict__ P, const int* __restrict__ idx,
                                      const int64_t* __restrict__ at, double2* M, int64_t ld) {
  const int b = blockIdx.y;
  const int n = P[b];
  const double2* T = tperm + toff[b];
  const int* in = idx + at[2 * b];
  const int* out = idx + at[2 * b + 1];
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < int64_t(n) * n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(k % n), j = static_cast<int>(k / n);
    M[out[i] + in[j] * ld] = T[k];
  }
}
namespace cg = cooperative_groups;
__device__ void make_givens(double2 a, double2 b, double& c, double2& s);
__device__ void apply_givens(double c, double2 s, double2& a, double2& b);

// gmres_fixed_steps (krylov.cpp:194-201, driver 45-178 with fixed_steps) on
// the coarse system in ONE launch: a cluster of CTAs owns contiguous slices
// of the Krylov vectors; the matvec rows are split across the cluster; dot
// products reduce through distributed shared memory; the tiny Hessenberg /
// Givens state is kept (identically) by every CTA, so no broadcast is needed.
__global__ void __launch_bounds__(kGemvThreads) coarse_fused_kernel(
    const VItem* __restrict__ items, int nitems, int64_t n, int ci, double2* V, double2* w,
    const double2* rd, double2* outd, int max_cols) {
  pdl_trigger();
  pdl_wait();
  cg::cluster_group cl = cg::this_cluster();
  const int cs = static_cast<int>(cl.num_blocks()), rank = static_cast<int>(cl.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* xs = reinterpret_cast<double2*>(smem_raw);
  __shared__ double2 red[kGemvThreads];
  __shared__ double2 part[kMaxCoarseIters + 2];
  __shared__ double2 Hs[(kMaxCoarseIters + 1) * kMaxCoarseIters];
  __shared__ double2 gs[kMaxCoarseIters + 1], rs[kMaxCoarseIters], ys[kMaxCoarseIters];
  __shared__ double rcs[kMaxCoarseIters];
  const int64_t s0 = n * rank / cs, s1 = n * (rank + 1) / cs;
  const int ldh = ci + 1;

  auto cluster_sum = [&](double2 v, int slot) {
    v.x = warp_sum(v.x);
    v.y = warp_sum(v.y);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double2 t = make_double2(0.0, 0.0);
      for (int q = 0; q < kGemvThreads / 32; ++q) t = cadd(t, red[q]);
      part[slot] = t;
    }
    cl.sync();
    double2 t = make_double2(0.0, 0.0);
    for (int q = 0; q < cs; ++q) t = cadd(t, *cl.map_shared_rank(&part[slot], q));
    return t;
  };

  double2 loc = make_double2(0.0, 0.0);
  for (int64_t k = s0 + tid; k < s1; k += kGemvThreads) loc.x += cabs2(__ldcg(rd + k));
  const double beta = sqrt(cluster_sum(loc, 0).x);
  if (beta == 0.0) {
    for (int64_t k = s0 + tid; k < s1; k += kGemvThreads) outd[k] = make_double2(0.0, 0.0);
    cl.sync();  // no CTA may exit while others still read its shared memory
    return;
  }
  for (int64_t k = s0 + tid; k < s1; k += kGemvThreads) {
    const double2 v = __ldcg(rd + k);
    __stcg(V + k, make_double2(v.x / beta, v.y / beta));
  }
  if (tid <= ci) gs[tid] = make_double2(tid == 0 ? beta : 0.0, 0.0);
  cl.sync();
  int jused = 0;
  for (int j = 0; j < ci; ++j) {
    const double2* Vj = V + j * n;
    for (int it = 0; it < nitems; ++it) {
      const VItem I = items[it];
      const int chunk = cluster_chunk(I.rows, cs);
      const int rb = rank * chunk, re = min(I.rows, rb + chunk);
      if (rb < re) gemv_item_rows(I, rb, re, Vj, Vj, w, xs, red);
      __syncthreads();
    }
    cl.sync();
    for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt
      const double2* Vi = V + i * n;
      double2 d = make_double2(0.0, 0.0);
      for (int64_t k = s0 + tid; k < s1; k += kGemvThreads)
        d = cfma_conj(__ldcg(Vi + k), __ldcg(w + k), d);
      const double2 h = cluster_sum(d, 1 + i);
      for (int64_t k = s0 + tid; k < s1; k += kGemvThreads)
        __stcg(w + k, csub(__ldcg(w + k), cmul(h, __ldcg(Vi + k))));
      if (tid == 0) Hs[i + j * ldh] = h;
    }
    double2 nn = make_double2(0.0, 0.0);
    for (int64_t k = s0 + tid; k < s1; k += kGemvThreads) nn.x += cabs2(__ldcg(w + k));
    const double hnext = sqrt(cluster_sum(nn, j + 2).x);
    if (tid == 0) {
      Hs[j + 1 + j * ldh] = make_double2(hnext, 0.0);
      for (int i = 0; i < j; ++i) apply_givens(rcs[i], rs[i], Hs[i + j * ldh], Hs[i + 1 + j * ldh]);
      double c;
      double2 s;
      make_givens(Hs[j + j * ldh], Hs[j + 1 + j * ldh], c, s);
      rcs[j] = c, rs[j] = s;
      apply_givens(c, s, Hs[j + j * ldh], Hs[j + 1 + j * ldh]);
      apply_givens(c, s, gs[j], gs[j + 1]);
    }
    __syncthreads();
    jused = j + 1;
    if (hnext <= 1e-14 * beta) break;  // happy breakdown
    double2* Vn = V + (j + 1) * n;
    for (int64_t k = s0 + tid; k < s1; k += kGemvThreads) {
      const double2 v = __ldcg(w + k);
      __stcg(Vn + k, make_double2(v.x / hnext, v.y / hnext));
    }
    cl.sync();
  }
  cl.sync();  // all DSMEM reads of this step are done before any CTA can exit
  if (tid == 0)
    for (int i = jused - 1; i >= 0; --i) {
      double2 s = gs[i];
      for (int k = i + 1; k < jused; ++k) s = csub(s, cmul(Hs[i + k * ldh], ys[k]));
      ys[i] = cdiv(s, Hs[i + i * ldh]);
    }
  __syncthreads();
  for (int64_t k = s0 + tid; k < s1; k += kGemvThreads) {
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < jused; ++i) acc = cfma(ys[i], __ldcg(V + i * n + k), acc);
    outd[k] = acc;
  }
}

// gmres_fixed_steps on a small coarse system, fully on-chip in ONE cluster
// launch (used when every CTA's rows of the coarse box maps fit in shared
// memory).  Each of the C CTAs
//   - stages its row slice of every coarse box map (column-major) and the
//     index maps in shared memory once, before the PDL wait; the ci matvecs
//     reuse them;
//   - owns a contiguous slice (<= one row per thread) of the Krylov vectors
//     and keeps a full copy of the current basis vector, which every CTA
//     fills by pushing its new slice into all peers (DSMEM stores);
//   - scatters each product row to the owner of its output index (remote
//     store), so w lands slice-wise.
// Orthogonalisation is classical Gram-Schmidt: the j+1 projections of a step
// reduce together, so a step costs four cluster barriers instead of one per
// basis vector (MGS, krylov.cpp:98-101, equal in exact arithmetic; the
// parity tests bound the difference).  Partial sums are pushed to every peer
// and summed in rank order, so all CTAs hold identical Hessenberg / Givens
// state without a broadcast.
constexpr int kCoarseCThreads = 256;
constexpr int kCoarseClusterItems = 8;
constexpr int kCoarseMaxCluster = 16;
__global__ void __launch_bounds__(kCoarseCThreads) coarse_cluster_kernel(
    const VItem* __restrict__ gitems, int nitems, int n, int slice, int ci, int max_cols,
    size_t stage_elems, const double2* rd, double2* outd) {
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks()), crank = static_cast<int>(cl.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kWarps = kCoarseCThreads / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* vfull = reinterpret_cast<double2*>(smem_raw);   // n: current basis vector (full)
  double2* Vs = vfull + n;                                  // (ci+1) x slice
  double2* ws = Vs + static_cast<size_t>(ci + 1) * slice;   // slice
  double2* xs = ws + slice;                                 // max_cols
  double2* As = xs + max_cols;                              // staged rows, column-major
  int* Ix = reinterpret_cast<int*>(As + stage_elems);       // staged gather / scatter indices
  __shared__ double2 red[kCoarseCThreads];
  __shared__ double2 wred[kWarps][kMaxCoarseIters + 1];
  __shared__ double2 part[kCoarseMaxCluster][kMaxCoarseIters + 1];  // pushed by rank
  __shared__ double pnorm[kCoarseMaxCluster];
  __shared__ double2 hsum[kMaxCoarseIters + 1];
  __shared__ VItem items[kCoarseClusterItems];  // item descriptors read once
  __shared__ double2 Hs[(kMaxCoarseIters + 1) * kMaxCoarseIters];
  __shared__ double2 gs[kMaxCoarseIters + 1], rs[kMaxCoarseIters], ys[kMaxCoarseIters];
  __shared__ double rcs[kMaxCoarseIters];
  const int s0 = min(n, crank * slice), s1 = min(n, s0 + slice), ns = s1 - s0;
  const bool own = tid < ns;  // this thread's row of the slice
  const int ldh = ci + 1;
  pdl_trigger();
  {
    const int words = nitems * static_cast<int>(sizeof(VItem) / sizeof(int));
    for (int w = tid; w < words; w += kCoarseCThreads)
      reinterpret_cast<int*>(items)[w] = __ldg(reinterpret_cast<const int*>(gitems) + w);
    __syncthreads();
  }
  // ---- stage this CTA's rows of every item (operators are static)
  {
    size_t off = 0;
    for (int it = 0; it < nitems; ++it) {
      const VItem I = items[it];
      const int chunk = cluster_chunk(I.rows, C);
      const int rb = min(I.rows, crank * chunk), nr = max(0, min(I.rows, rb + chunk) - rb);
      for (int k = tid; k < nr * I.cols; k += kCoarseCThreads)
        cp_async16(As + off + k, I.A + rb + (k % nr) + static_cast<size_t>(k / nr) * I.lda);
      off += static_cast<size_t>(nr) * I.cols;
    }
    cp_async_commit();
    int io = 0;  // index maps are static too: [xi (cols) | own rows of yi] per item
    for (int it = 0; it < nitems; ++it) {
      const VItem I = items[it];
      const int chunk = cluster_chunk(I.rows, C);
      const int rb = min(I.rows, crank * chunk), nr = max(0, min(I.rows, rb + chunk) - rb);
      for (int c = tid; c < I.cols; c += kCoarseCThreads) Ix[io + c] = __ldg(I.xi + c);
      for (int r = tid; r < nr; r += kCoarseCThreads) Ix[io + I.cols + r] = __ldg(I.yi + rb + r);
      io += I.cols + nr;
    }
  }
  // block-reduce one value per thread, push the CTA's sum to every peer's
  // pnorm[crank]; after the next cluster barrier all CTAs sum in rank order
  auto push_norm = [&](double v) {
    v = warp_sum(v);
    if (lane == 0) red[warp].x = v;
    __syncthreads();
    if (tid < C) {
      double t = 0.0;
      for (int q = 0; q < kWarps; ++q) t += red[q].x;
      *cl.map_shared_rank(&pnorm[crank], tid) = t;
    }
  };
  auto sum_norm = [&]() {
    double t = 0.0;
    for (int q = 0; q < C; ++q) t += pnorm[q];
    return t;
  };
  // V_j slice -> every peer's vfull
  auto push_basis = [&](double2 v) {
    if (own)
      for (int q = 0; q < C; ++q) cl.map_shared_rank(vfull, q)[s0 + tid] = v;
  };
  pdl_wait();
  double2 wv = own ? __ldcg(rd + s0 + tid) : make_double2(0.0, 0.0);
  push_norm(cabs2(wv));
  cp_async_wait_all();
  cl.sync();
  const double beta = sqrt(sum_norm());
  if (beta == 0.0) {
    if (own) outd[s0 + tid] = make_double2(0.0, 0.0);
    cl.sync();
    return;
  }
  {
    const double2 v0 = make_double2(wv.x / beta, wv.y / beta);
    if (own) Vs[tid] = v0;
    push_basis(v0);
  }
  if (tid <= ci) gs[tid] = make_double2(tid == 0 ? beta : 0.0, 0.0);
  cl.sync();  // vfull = V_0 in every CTA
  int jused = 0;
  for (int j = 0; j < ci; ++j) {
    // (A) w = v_j + sum_boxes scatter(T gather(v_j)); rows go to their owner
    {
      int io = 0, xo = 0;
      for (int it = 0; it < nitems; ++it) {
        const VItem I = items[it];
        const int chunk = cluster_chunk(I.rows, C);
        const int rb = min(I.rows, crank * chunk), nr = max(0, min(I.rows, rb + chunk) - rb);
        for (int c = tid; c < I.cols; c += kCoarseCThreads) xs[xo + c] = vfull[Ix[io + c]];
        io += I.cols + nr;
        xo += I.cols;
      }
      __syncthreads();
      size_t off = 0;
      io = 0, xo = 0;
      for (int it = 0; it < nitems; ++it) {
        const VItem I = items[it];
        const int chunk = cluster_chunk(I.rows, C);
        const int rb = min(I.rows, crank * chunk), nr = max(0, min(I.rows, rb + chunk) - rb);
        for (int r0 = 0; r0 < nr; r0 += kCoarseCThreads) {
          const int rows = min(nr - r0, kCoarseCThreads);
          const double2 y = smem_gemv<kCoarseCThreads>(As + off + r0, nr, rows, I.cols, xs + xo, red);
          if (tid < rows) {
            const int k = Ix[io + I.cols + r0 + tid];
            const int o = k / slice;
            cl.map_shared_rank(ws, o)[k - o * slice] = cadd(y, vfull[k]);
          }
        }
        off += static_cast<size_t>(nr) * I.cols;
        io += I.cols + nr;
        xo += I.cols;
      }
    }
    cl.sync();  // (1) w slices complete
    // (B) the j+1 projections V_i^H w, reduced together
    wv = own ? ws[tid] : make_double2(0.0, 0.0);
    for (int i = 0; i <= j; ++i) {
      double2 d = own ? cmul(make_double2(Vs[i * slice + tid].x, -Vs[i * slice + tid].y), wv)
                      : make_double2(0.0, 0.0);
      d.x = warp_sum(d.x);
      d.y = warp_sum(d.y);
      if (lane == 0) wred[warp][i] = d;
    }
    __syncthreads();
    if (tid <= j) {
      double2 t = make_double2(0.0, 0.0);
      for (int q = 0; q < kWarps; ++q) t = cadd(t, wred[q][tid]);
      for (int q = 0; q < C; ++q) *cl.map_shared_rank(&part[crank][tid], q) = t;
    }
    cl.sync();  // (2) partial projections of every CTA delivered
    if (tid <= j) {
      double2 t = make_double2(0.0, 0.0);
      for (int q = 0; q < C; ++q) t = cadd(t, part[q][tid]);
      hsum[tid] = t;
    }
    __syncthreads();
    // (C) w -= V h, ||w||^2
    if (own)
      for (int i = 0; i <= j; ++i) wv = csub(wv, cmul(hsum[i], Vs[i * slice + tid]));
    push_norm(cabs2(wv));
    cl.sync();  // (3) norm partials delivered
    const double hnext = sqrt(sum_norm());
    if (tid == 0) {
      for (int i = 0; i <= j; ++i) Hs[i + j * ldh] = hsum[i];
      Hs[j + 1 + j * ldh] = make_double2(hnext, 0.0);
      for (int i = 0; i < j; ++i) apply_givens(rcs[i], rs[i], Hs[i + j * ldh], Hs[i + 1 + j * ldh]);
      double c;
      double2 sg;
      make_givens(Hs[j + j * ldh], Hs[j + 1 + j * ldh], c, sg);
      rcs[j] = c, rs[j] = sg;
      apply_givens(c, sg, Hs[j + j * ldh], Hs[j + 1 + j * ldh]);
      apply_givens(c, sg, gs[j], gs[j + 1]);
    }
    jused = j + 1;
    if (hnext <= 1e-14 * beta) break;  // happy breakdown (identical in all CTAs)
    // (D) V_{j+1} = w / hnext, pushed to every peer's vfull
    const double2 vn = make_double2(wv.x / hnext, wv.y / hnext);
    if (own) Vs[(j + 1) * slice + tid] = vn;
    push_basis(vn);
    cl.sync();  // (4) vfull = V_{j+1}; w and partial slots free again
  }
  __syncthreads();
  if (tid == 0)
    for (int i = jused - 1; i >= 0; --i) {
      double2 sum = gs[i];
      for (int k = i + 1; k < jused; ++k) sum = csub(sum, cmul(Hs[i + k * ldh], ys[k]));
      ys[i] = cdiv(sum, Hs[i + i * ldh]);
    }
  __syncthreads();
  if (own) {
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < jused; ++i) acc = cfma(ys[i], Vs[static_cast<size_t>(i) * slice + tid], acc);
    outd[s0 + tid] = acc;
  }
  cl.sync();  // no CTA exits while a peer may still write its shared memory
}

bool coarse_cluster_fits(size_t smem, int csize) {
  static const bool attr = [] {
    HPSB_CUDA(cudaFuncSetAttribute(coarse_cluster_kernel,
                                   cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    return true;
  }();
  (void)attr;
  allow_smem<coarse_cluster_kernel>(smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(csize);
  cfg.blockDim = dim3(kCoarseCThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, coarse_cluster_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return nclusters > 0;
}

__device__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

// y += s x
__global__ void axpy_vec_kernel(double2* y, const double2* __restrict__ x, double s, int64_t n) {
  pdl_trigger();
  pdl_wait();
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[k] = make_double2(y[k].x + s * x[k].x, y[k].y + s * x[k].y);
}

__global__ void copy_vec_kernel(double2* y, const double2* __restrict__ x, int64_t n) {
  pdl_trigger();
  pdl_wait();
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[k] = x[k];
}

// state: [0] bnorm, [1] done, [2] jused, [3] zero-rhs
// Multi-RHS: CTA b works on right-hand side b (rd / outd stride ldr, the
// Krylov state of each RHS packed behind the previous one's).
__global__ void __launch_bounds__(kCoarseThreads) coarse_init_kernel(const double2* rd, int64_t n,
                                                                     double2* V, double2* cv,
                                                                     double2* gv, int ci,
                                                                     double* state, int64_t ldr) {
  pdl_trigger();
  pdl_wait();
  {
    const int b = blockIdx.x;
    rd += b * ldr, V += static_cast<int64_t>(b) * (ci + 1) * n, cv += b * n;
    gv += b * (ci + 1), state += b * 4;
  }
  __shared__ double sh[33];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += cabs2(rd[i]);
  const double beta = sqrt(block_sum(s, sh));
  const double inv = beta > 0.0 ? 1.0 / beta : 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 v = make_double2(rd[i].x * inv, rd[i].y * inv);
    V[i] = v;
    cv[i] = v;
  }
  if (threadIdx.x <= ci) gv[threadIdx.x] = make_double2(threadIdx.x == 0 ? beta : 0.0, 0.0);
  if (threadIdx.x == 0) {
    state[0] = beta;
    state[1] = beta == 0.0 ? 1.0 : 0.0;
    state[2] = 0.0;
    state[3] = beta == 0.0 ? 1.0 : 0.0;
  }
}

__device__ void make_givens(double2 a, double2 b, double& c, double2& s) {
  // krylov.cpp:17-31
  c = 1.0;
  s = make_double2(0.0, 0.0);
  const double na = hypot(a.x, a.y), nb = hypot(b.x, b.y);
  if (nb == 0.0) return;
  const double r = hypot(na, nb);
  const double2 cb = make_double2(b.x, -b.y);
  if (na == 0.0) {
    c = 0.0;
    s = make_double2(cb.x / nb, cb.y / nb);
  } else {
    c = na / r;
    const double2 an = make_double2(a.x / na, a.y / na);
    s = cmul(an, make_double2(cb.x / r, cb.y / r));
  }
}

__device__ void apply_givens(double c, double2 s, double2& a, double2& b) {
  // krylov.cpp:33-37
  const double2 t = cadd(cscale(a, c), cmul(s, b));
  b = cadd(cmul(make_double2(-s.x, s.y), a), cscale(b, c));
  a = t;
}

// One MGS Arnoldi step of gmres_fixed_steps (no reorthogonalisation, as
// KrylovConfig's default, krylov.cpp:194-201).  Hm is (ci+1) x ci col-major.
__global__ void __launch_bounds__(kCoarseThreads) coarse_step_kernel(
    int j, int64_t n, int ci, double2* V, double2* cv, double2* cw, double2* Hm, double2* gv,
    double* rc, double2* rs, double* state, int64_t ldr) {
  pdl_trigger();
  pdl_wait();
  {
    const int b = blockIdx.x;
    (void)ldr;
    V += static_cast<int64_t>(b) * (ci + 1) * n, cv += b * n, cw += b * n;
    Hm += static_cast<int64_t>(b) * (ci + 1) * ci, gv += b * (ci + 1), rc += b * ci, rs += b * ci;
    state += b * 4;
  }
  __shared__ double sh[33];
  if (state[1] != 0.0) return;
  const int ldh = ci + 1;
  double hnext;
  if (n <= static_cast<int64_t>(kCoarseRowsReg) * kCoarseThreads && j < kMaxCoarseIters) {
    // Classical Gram-Schmidt with w's rows in registers: the j+1 projections
    // reduce together (one block reduction instead of j+1; equal to the
    // modified form of krylov.cpp:98-101 in exact arithmetic, as in the
    // cluster coarse kernel), then w -= V h and ||w|| in one pass.
    __shared__ double2 wpart[kCoarseThreads / 32][kMaxCoarseIters + 1];
    __shared__ double2 hsum[kMaxCoarseIters + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double2 wr[kCoarseRowsReg];
#pragma unroll
    for (int q = 0; q < kCoarseRowsReg; ++q) {
      const int64_t k = threadIdx.x + static_cast<int64_t>(q) * kCoarseThreads;
      wr[q] = k < n ? cw[k] : make_double2(0.0, 0.0);
    }
    for (int i = 0; i <= j; ++i) {
      const double2* Vi = V + i * n;
      double2 d = make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < kCoarseRowsReg; ++q) {
        const int64_t k = threadIdx.x + static_cast<int64_t>(q) * kCoarseThreads;
        if (k < n) d = cfma_conj(Vi[k], wr[q], d);
      }
      d.x = warp_sum(d.x);
      d.y = warp_sum(d.y);
      if (lane == 0) wpart[warp][i] = d;
    }
    __syncthreads();
    if (threadIdx.x <= j) {
      double2 t = make_double2(0.0, 0.0);
      for (int w = 0; w < kCoarseThreads / 32; ++w) t = cadd(t, wpart[w][threadIdx.x]);
      hsum[threadIdx.x] = t;
      Hm[threadIdx.x + j * ldh] = t;
    }
    __syncthreads();
    double s2 = 0.0;
#pragma unroll
    for (int q = 0; q < kCoarseRowsReg; ++q) {
      const int64_t k = threadIdx.x + static_cast<int64_t>(q) * kCoarseThreads;
      if (k < n) {
        double2 w = wr[q];
        for (int i = 0; i <= j; ++i) w = csub(w, cmul(hsum[i], V[i * n + k]));
        wr[q] = w;
        cw[k] = w;
        s2 += cabs2(w);
      }
    }
    hnext = sqrt(block_sum(s2, sh));
  } else {
    for (int i = 0; i <= j; ++i) {
      const double2* Vi = V + i * n;
      double sr = 0.0, si = 0.0;
      for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        const double2 a = Vi[k], b = cw[k];
        sr += a.x * b.x + a.y * b.y;
        si += a.x * b.y - a.y * b.x;
      }
      const double hr = block_sum(sr, sh);
      const double hi = block_sum(si, sh);
      for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        const double2 a = Vi[k];
        double2 w = cw[k];
        w.x -= hr * a.x - hi * a.y;
        w.y -= hr * a.y + hi * a.x;
        cw[k] = w;
      }
      if (threadIdx.x == 0) Hm[i + j * ldh] = make_double2(hr, hi);
      __syncthreads();
    }
    double s2 = 0.0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) s2 += cabs2(cw[k]);
    hnext = sqrt(block_sum(s2, sh));
  }
  if (threadIdx.x == 0) {
    Hm[j + 1 + j * ldh] = make_double2(hnext, 0.0);
    for (int i = 0; i < j; ++i)
      apply_givens(rc[i], rs[i], Hm[i + j * ldh], Hm[i + 1 + j * ldh]);
    double c;
    double2 s;
    make_givens(Hm[j + j * ldh], Hm[j + 1 + j * ldh], c, s);
    rc[j] = c, rs[j] = s;
    apply_givens(c, s, Hm[j + j * ldh], Hm[j + 1 + j * ldh]);
    apply_givens(c, s, gv[j], gv[j + 1]);
    state[2] = j + 1;
    if (hnext <= 1e-14 * state[0]) state[1] = 1.0;  // happy breakdown
  }
  __syncthreads();
  if (hnext <= 1e-14 * state[0]) return;
  const double inv = 1.0 / hnext;
  double2* Vn = V + (j + 1) * n;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    const double2 v = make_double2(cw[k].x * inv, cw[k].y * inv);
    Vn[k] = v;
    cv[k] = v;
  }
}

// y = H^{-1} g (upper triangular), out = sum_i y_i V_i (krylov.cpp:133-145).
__global__ void __launch_bounds__(kCoarseThreads) coarse_finish_kernel(int64_t n, int ci,
                                                                       const double2* V,
                                                                       const double2* Hm,
                                                                       const double2* gv,
                                                                       const double* state,
                                                                       double2* outd, int64_t ldr) {
  pdl_trigger();
  pdl_wait();
  {
    const int b = blockIdx.x;
    V += static_cast<int64_t>(b) * (ci + 1) * n, Hm += static_cast<int64_t>(b) * (ci + 1) * ci;
    gv += b * (ci + 1), state += b * 4, outd += b * ldr;
  }
  __shared__ double2 y[kCoarseItersMax];
  const int ju = static_cast<int>(state[2]);
  const int ldh = ci + 1;
  if (threadIdx.x == 0) {
    for (int i = ju - 1; i >= 0; --i) {
      double2 s = gv[i];
      for (int k = i + 1; k < ju; ++k) s = csub(s, cmul(Hm[i + k * ldh], y[k]));
      y[i] = cdiv(s, Hm[i + i * ldh]);
    }
  }
  __syncthreads();
  const bool zero = state[3] != 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    if (!zero)
      for (int i = 0; i < ju; ++i) acc = cfma(y[i], V[i * n + k], acc);
    outd[k] = acc;
  }
}

// Row-block size for a split phase: enough units for ~2 CTAs per SM,
// 8 / 16 / multiple-of-32 rows (the shapes the GEMV item kernel maps well).
int split_rows(int total_rows, int sms) {
  // ~8 units per SM: small units balance the SMs (no tail wave) at the cost
  // of re-gathering x per unit (a few % of the matrix bytes at these sizes).
  const int want = (total_rows + 8 * sms - 1) / (8 * sms);
  int rb = want <= 8 ? 8 : want <= 16 ? 16 : std::min(256, (want + 31) & ~31);
  // Avoid a sparse second wave: the plan kernel holds 4 CTAs per SM, and
  // e.g. 4864 rows in 8-row units (608 units for 592 slots) ran as a full
  // wave plus 16 lone CTAs (ncu, cfg3 coarse matvec: 2.8 TB/s).  Take the
  // next row block when it fits one wave.
  const int slots = 4 * sms, units = (total_rows + rb - 1) / rb;
  if (units > slots && units < 2 * slots) {
    const int rb2 = rb < 16 ? 16 : std::min(256, (2 * rb + 31) & ~31);
    if ((total_rows + rb2 - 1) / rb2 <= slots) rb = rb2;
  }
  return rb;
}

VItem item(const double2* A, int lda, int rows, int cols, const double2* x, const int* xi,
           const double2* z, const int* zi, double2* y, const int* yi, double alpha, double beta,
           double gamma) {
  VItem it{};
  it.A = A, it.lda = lda, it.rows = rows, it.cols = cols;
  it.x = x, it.xi = xi, it.z = z, it.zi = zi, it.y = y, it.yi = yi;
  it.alpha = alpha, it.beta = beta, it.gamma = gamma;
  return it;
}
}  // namespace

Context* precond_context(const Precond* p) { return p ? p->ctx : nullptr; }

int64_t precond_memory(const Precond* p) {
  int64_t b = 0;
  for (int l = 1; l <= p->cfg.depth; ++l) {
    const LevelOps& L = *p->h->levels[l - 1];
    if (l > 1) b += static_cast<int64_t>(L.tperm.bytes());  // M_l as box maps
    if (l < p->cfg.depth) b += static_cast<int64_t>(L.w.bytes());  // merge factors
  }
  return b + static_cast<int64_t>(p->cinv.bytes());
}

double precond_build_seconds(const Precond* p) { return p->h->build_seconds; }

// y = M_l x on level l's system (HierarchyLevel::M.apply, block_matrix.cpp:23-31;
// the level system over faces [first_face, total), dissection.hpp:35-41):
// M_l = I + sum_{boxes b entering level l} scatter_out(T_b gather_in(x)).  Every
// slot of the level is the outgoing row of exactly one box, so the items
// write disjoint rows (y = x there, plus the box's contribution).
void hierarchy_level_apply(Hierarchy* h, int level, const double2* x, double2* y) {
  if (level < 1 || level > h->depth) throw InvalidArgument("level_apply: level out of range");
  if (h->ctx->world() > 1) throw InvalidArgument("level_apply: single-GPU hierarchies only");
  Context* ctx = h->ctx;
  const LevelOps& Lv = *h->levels[level - 1];
  const int off = Lv.first_face * h->sk->bs;
  std::vector<int> gidx;
  std::vector<size_t> in_at, out_at;
  int rows = 0;
  for (const ChildBox& c : Lv.children) {
    in_at.push_back(gidx.size());
    for (const auto& q : c.pos) gidx.push_back(q.in - off);
    out_at.push_back(gidx.size());
    for (const auto& q : c.pos) gidx.push_back(q.out - off);
    rows += c.P;
  }
  VPlan mv;
  mv.idx_store.upload(gidx, ctx->stream);
  const int rb = split_rows(std::max(rows, 1), ctx->num_sms);
  mv.begin_phase();
  for (size_t k = 0; k < Lv.children.size(); ++k) {
    const ChildBox& c = Lv.children[k];
    const int* gi = mv.idx_store.p + in_at[k];
    const int* go = mv.idx_store.p + out_at[k];
    mv.add_split(item(Lv.tperm.p + c.t_off, c.P, c.P, c.P, x, gi, x, go, y, go, 1.0, 0.0, 1.0), rb);
  }
  mv.name = "level_matvec";
  mv.finalize(ctx->stream);
  mv.run(ctx);
  HPSB_CUDA(cudaStreamSynchronize(ctx->stream));  // the plan's buffers die here
}

Precond* create_precond(Hierarchy* h, const hpsb_mg_config& cfg) {
  // multigrid.cpp:9-28
  if (cfg.depth < 2) throw InvalidArgument("MgPreconditioner: depth must be >= 2");
  if (cfg.depth > h->depth) throw InvalidArgument("MgPreconditioner: depth exceeds the built hierarchy");
  if (!cfg.exact_coarse && cfg.gamma < 1) throw InvalidArgument("MgPreconditioner: gamma must be >= 1");
  if (!cfg.exact_coarse && cfg.coarse_iters < 1)
    throw InvalidArgument("MgPreconditioner: coarse_iters must be >= 1");
  // multigrid.cpp:71: the exact coarse mode runs gamma = 1.  gamma > 1
  // (W- / gamma-cycles) runs host-recursively (apply_level_gamma), sharded too.
  // A preconditioner shallower than the hierarchy uses levels 1..depth of it
  // (multigrid.cpp:13-16,24-26).  Sharded, the coarse level must be a global
  // one: the local levels hold this rank's boxes only.
  if (h->ctx->world() > 1 && cfg.depth <= h->sk->el->part.last_local)
    throw InvalidArgument("MgPreconditioner: a sharded preconditioner's depth must exceed the last "
                          "subtree level " + std::to_string(h->sk->el->part.last_local));
  if (!cfg.exact_coarse && cfg.coarse_iters > kCoarseItersMax)
    throw InvalidArgument("MgPreconditioner: coarse_iters must be <= " + std::to_string(kCoarseItersMax));
  Context* ctx = h->ctx;
  // HPSB_TRACE=1: host wall time per creation phase (stderr)
  const bool trace = std::getenv("HPSB_TRACE") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  std::string trace_line;
  auto mark = [&](const char* name) {
    if (!trace) return;
    const auto now = std::chrono::steady_clock::now();
    trace_line += std::string(" ") + name + "=" +
                  std::to_string(std::chrono::duration<double, std::milli>(now - t_last).count()).substr(0, 6) + "ms";
    t_last = now;
  };
  auto p = std::make_unique<Precond>();
  p->h = h, p->cfg = cfg, p->ctx = ctx;
  const Skeleton* sk = h->sk;
  p->dim = sk->dim;
  p->r.alloc(p->dim);
  p->out.alloc(p->dim);
  const int sms = ctx->num_sms;

  size_t tmp_total = 0;
  for (int l = 1; l < cfg.depth; ++l)
    for (const auto& mr : h->levels[l - 1]->merges) tmp_total += 3 * static_cast<size_t>(mr.s);
  p->tmp.alloc(std::max<size_t>(tmp_total, 1));

  // ---- down / up sweeps
  size_t toff = 0;
  std::vector<size_t> level_tmp(cfg.depth, 0);
  for (int l = 1; l < cfg.depth; ++l) {
    level_tmp[l] = toff;
    for (const auto& mr : h->levels[l - 1]->merges) toff += 3 * static_cast<size_t>(mr.s);
  }
  double2* r = p->r.p;
  double2* out = p->out.p;
  // The items of one level step, per merge and dependent stage (the same
  // lists feed the single-RHS plans and the multi-RHS batch phases):
  // out[gi][k] = stage k of merge gi (multigrid.cpp:47-98 on box maps).
  auto level_stages = [&](int l, bool downward) {
    const LevelOps& L = *h->levels[l - 1];
    const int ng = static_cast<int>(L.merges.size());
    std::vector<std::vector<std::vector<VItem>>> res(ng);
    size_t t = level_tmp[l];
    for (int gi = 0; gi < ng; ++gi) {
      const MergeRec& mr = L.merges[gi];
      const ChildBox& c1 = L.children[mr.c1];
      const ChildBox& c2 = L.children[mr.c2];
      const int s = mr.s, p1 = mr.p1, p2 = mr.p2, P1 = c1.P, P2 = c2.P;
      const double2* T1 = L.tperm.p + c1.t_off;
      const double2* T2 = L.tperm.p + c2.t_off;
      const double2 *T1ps = T1 + static_cast<size_t>(p1) * P1, *T1sp = T1 + p1,
                    *T1ss = T1 + p1 + static_cast<size_t>(p1) * P1;
      const double2 *T2ps = T2 + static_cast<size_t>(p2) * P2, *T2sp = T2 + p2,
                    *T2ss = T2 + p2 + static_cast<size_t>(p2) * P2;
      const double2* W = L.w.p + mr.w_off;
      const int* ix = L.idx.p;
      const int *in1s = ix + mr.in1_sep, *in2s = ix + mr.in2_sep, *in1p = ix + mr.in1_per,
                *in2p = ix + mr.in2_per, *out1p = ix + mr.out1_per, *out2p = ix + mr.out2_per;
      double2* t1 = p->tmp.p + t;
      double2* t2 = t1 + s;
      double2* t3 = t2 + s;
      t += 3 * static_cast<size_t>(s);
      std::vector<std::vector<VItem>>& st = res[gi];
      st.resize(4);
      if (downward) {
        st[0].push_back(item(T2ss, P2, s, s, r, in2s, r, in1s, t3, nullptr, -1.0, 0.0, 1.0));
        st[1].push_back(item(W, s, s, s, t3, nullptr, nullptr, nullptr, out, in1s, 1.0, 0.0, 0.0));
        st[2].push_back(item(T1ss, P1, s, s, out, in1s, r, in2s, out, in2s, -1.0, 0.0, 1.0));
        if (p1) st[3].push_back(item(T1ps, P1, p1, s, out, in1s, nullptr, nullptr, r, out1p, -1.0, 1.0, 0.0));
        if (p2) st[3].push_back(item(T2ps, P2, p2, s, out, in2s, nullptr, nullptr, r, out2p, -1.0, 1.0, 0.0));
      } else {
        if (p2) st[0].push_back(item(T2sp, P2, s, p2, out, in2p, nullptr, nullptr, t1, nullptr, 1.0, 0.0, 0.0));
        else st[0].push_back(item(nullptr, 0, s, 0, nullptr, nullptr, nullptr, nullptr, t1, nullptr, 0.0, 0.0, 0.0));
        if (p1) st[0].push_back(item(T1sp, P1, s, p1, out, in1p, nullptr, nullptr, t2, nullptr, 1.0, 0.0, 0.0));
        else st[0].push_back(item(nullptr, 0, s, 0, nullptr, nullptr, nullptr, nullptr, t2, nullptr, 0.0, 0.0, 0.0));
        st[1].push_back(item(T2ss, P2, s, s, t2, nullptr, t1, nullptr, t3, nullptr, -1.0, 0.0, 1.0));
        st[2].push_back(item(W, s, s, s, t3, nullptr, nullptr, nullptr, t1, nullptr, 1.0, 0.0, 0.0));
        st[3].push_back(item(T1ss, P1, s, s, t1, nullptr, t2, nullptr, out, in2s, 1.0, 1.0, -1.0));
        st[3].push_back(item(nullptr, 0, s, 0, nullptr, nullptr, t1, nullptr, out, in1s, 0.0, 1.0, -1.0));
      }
    }
    return res;
  };
  auto build_level = [&](int l, bool downward) {
    const LevelOps& L = *h->levels[l - 1];
    const int ng = static_cast<int>(L.merges.size());
    // Execution mode of the level (one launch unless the maps are huge):
    //  - one CTA per merge when there are enough merges to fill the GPU;
    //  - a cluster of up to 16 CTAs per merge otherwise (row-split items,
    //    cluster barriers between the dependent phases);
    //  - separate row-split launches per phase when a few merges carry
    //    tens of MB each (top levels of the large configs), so every SM streams.
    double bytes = 0;
    int smin = 1 << 30;
    for (const auto& mr : L.merges) {
      bytes += 16.0 * (3.0 * mr.s * mr.s + static_cast<double>(mr.s) * (mr.p1 + mr.p2));
      smin = std::min(smin, mr.s);
    }
    const double per_merge = bytes / std::max(ng, 1);
    int csize = 1;
    while (csize < 16 && csize * ng < 2 * sms && 8 * csize < smin + 8) csize *= 2;
    const bool split = per_merge > 8e6 && ng * 16 < sms;
    const bool chain = !split;
    int total_rows = 0;
    for (const auto& mr : L.merges) total_rows += mr.s + mr.p1 + mr.p2;
    int rb = ((total_rows / (2 * sms)) + 31) & ~31;
    rb = std::max(32, std::min(256, rb));
    std::vector<std::vector<VItem>> stages(downward ? 4 : 4);
    std::vector<std::vector<VItem>> chains(ng);
    auto per_merge_stages = level_stages(l, downward);
    for (int gi = 0; gi < ng; ++gi) {
      auto& st = per_merge_stages[gi];
      for (int k = 0; k < 4; ++k) {
        if (!st[k].empty()) st[k].back().flags |= VItem::kPhaseEnd;
        for (auto& it : st[k]) {
          if (chain) chains[gi].push_back(it);
          else stages[k].push_back(it);
        }
      }
    }
    const bool global_level = l > h->sk->el->part.last_local;
    VPlan& plan = downward ? (global_level ? p->down_g : p->down) : (global_level ? p->up_g : p->up);
    const std::string label = std::string(downward ? "vcycle_down" : "vcycle_up") +
                              (std::getenv("HPSB_PROFILE_LEVELS") ? "_L" + std::to_string(l) : "");
    if (chain) {
      plan.phases[plan.begin_phase(csize)].label = label;
      for (auto& c : chains) plan.add_unit(c);
    } else {
      for (auto& stg : stages) {
        plan.phases[plan.begin_phase()].label = label;
        int rows = 0;
        for (auto& it : stg) rows += it.rows;
        for (auto& it : stg) plan.add_split(it, split_rows(rows, sms));
      }
    }
  };
  mark("items");
  // Per level: the fused small-merge kernel when every merge's operators fit
  // in shared memory, else the work-list plan phases.
  auto small_level = [&](int l) -> int {
    const LevelOps& L = *h->levels[l - 1];
    if (L.merges.empty()) return -1;
    auto sl = std::make_unique<SmallLevel>();
    std::vector<SmallMerge> v;
    const int* ix = L.idx.p;
    for (const MergeRec& mr : L.merges) {
      const ChildBox& c1 = L.children[mr.c1];
      const ChildBox& c2 = L.children[mr.c2];
      const size_t need = small_merge_smem(mr.s, mr.p1, mr.p2);
      if (need > kSmallMergeSmemMax) return -1;
      sl->smem = std::max(sl->smem, need);
      sl->max_s = std::max(sl->max_s, mr.s);
      sl->batch_vec_down = std::max(sl->batch_vec_down, small_merge_batch_vec(mr.s, mr.p1, mr.p2, true));
      sl->batch_vec_up = std::max(sl->batch_vec_up, small_merge_batch_vec(mr.s, mr.p1, mr.p2, false));
      sl->batch_ops = std::max(sl->batch_ops, small_merge_batch_smem(mr.s, mr.p1, mr.p2, 0));
      sl->batch_vec = std::max(sl->batch_vec, small_merge_batch_smem(mr.s, mr.p1, mr.p2, 1) -
                                                  small_merge_batch_smem(mr.s, mr.p1, mr.p2, 0));
      SmallMerge m{};
      m.T1 = L.tperm.p + c1.t_off, m.T2 = L.tperm.p + c2.t_off, m.W = L.w.p + mr.w_off;
      m.in1s = ix + mr.in1_sep, m.in2s = ix + mr.in2_sep, m.in1p = ix + mr.in1_per;
      m.in2p = ix + mr.in2_per, m.out1p = ix + mr.out1_per, m.out2p = ix + mr.out2_per;
      m.s = mr.s, m.p1 = mr.p1, m.p2 = mr.p2, m.P1 = c1.P, m.P2 = c2.P;
      v.push_back(m);
      const double ss = 16.0 * mr.s * mr.s, sp = 16.0 * mr.s * (mr.p1 + mr.p2);
      sl->bytes_down += 3 * ss + sp;
      sl->bytes_up += 3 * ss + sp;
    }
    sl->level = l;
    sl->count = static_cast<int>(v.size());
    if (std::getenv("HPSB_PROFILE_LEVELS")) sl->label = "vcycle_small_L" + std::to_string(l);
    sl->d.upload(v, ctx->stream);
    p->smalls.push_back(std::move(sl));
    return static_cast<int>(p->smalls.size()) - 1;
  };
  // Per level, next choice: one thread-block cluster per merge with every
  // CTA's operator slices staged in shared memory (vcycle_cluster.cu).
  auto cluster_level = [&](int l) -> int {
    const LevelOps& L = *h->levels[l - 1];
    const int ng = static_cast<int>(L.merges.size());
    if (!ng) return -1;
    // Only for latency-bound levels: few merges (>= 4 CTAs each within ~2
    // CTAs per SM) and a few MB of operators.  With many merges, one CTA per
    // SM holding a whole staged slice serialises load and compute, and the
    // streaming work lists are faster (measured at cfg3 levels 2-3: 3x).
    int C = 1;
    while (C < 16 && 2 * C * ng <= 2 * sms) C *= 2;
    if (C < 4) return -1;
    auto cl = std::make_unique<ClusterLevel>();
    for (const MergeRec& mr : L.merges) {
      if (cluster_chunk(mr.s, C) > 256) return -1;  // one row pass per CTA for the s-blocks
      cl->smem = std::max(cl->smem, cluster_merge_smem(mr.s, mr.p1, mr.p2, C));
      const double ss = 16.0 * mr.s * mr.s, sp = 16.0 * mr.s * (mr.p1 + mr.p2);
      cl->bytes_down += 3 * ss + sp;
      cl->bytes_up += 3 * ss + sp;
    }
    if (cl->smem > kClusterMergeSmemMax || cl->bytes_down > 32e6) return -1;
    if (!cluster_merge_fits(cl->smem, C)) return -1;
    std::vector<SmallMerge> v;
    const int* ix = L.idx.p;
    for (const MergeRec& mr : L.merges) {
      const ChildBox& c1 = L.children[mr.c1];
      const ChildBox& c2 = L.children[mr.c2];
      SmallMerge m{};
      m.T1 = L.tperm.p + c1.t_off, m.T2 = L.tperm.p + c2.t_off, m.W = L.w.p + mr.w_off;
      m.in1s = ix + mr.in1_sep, m.in2s = ix + mr.in2_sep, m.in1p = ix + mr.in1_per;
      m.in2p = ix + mr.in2_per, m.out1p = ix + mr.out1_per, m.out2p = ix + mr.out2_per;
      m.s = mr.s, m.p1 = mr.p1, m.p2 = mr.p2, m.P1 = c1.P, m.P2 = c2.P;
      v.push_back(m);
    }
    cl->level = l;
    cl->count = ng;
    cl->csize = C;
    if (std::getenv("HPSB_PROFILE_LEVELS")) cl->label = "vcycle_cluster_L" + std::to_string(l);
    cl->d.upload(v, ctx->stream);
    p->clusters.push_back(std::move(cl));
    return static_cast<int>(p->clusters.size()) - 1;
  };
  // Fused-operator levels.  The down and up chains of multigrid.cpp:47-98
  // are linear in the level's inputs, so for latency-bound levels they are
  // folded at setup (DMMA GEMMs) into one operator per merge and direction:
  //   down: [x1; x2; dr_p1; dr_p2] = Kd [r1; r2],  X = [W, -W T2ss],
  //         Y = [0, I] - T1ss X,  Kd = [X; Y; -T1ps X; -T2ps Y]
  //         (x -> out[s], dr -> r[p] +=);
  //   up:   [ds1; ds2] = Ku [u1; u2],  Ku_1 = [W T2ss T1sp, -W T2sp],
  //         Ku_2 = -T1ss Ku_1 - [T1sp, 0]  (ds -> out[s] +=).
  // A level step is then ONE launch of independent row blocks -- no chain of
  // dependent GEMVs, no barriers -- for up to ~1.7x the chain's operator
  // bytes.  Used where the level's folded operators are small (latency
  // bound): folded operators of at most 24 MB per level.
  constexpr double fused_max = 24e6;
  auto fused_level = [&](int l) -> int {
    const LevelOps& L = *h->levels[l - 1];
    if (L.merges.empty() || fused_max <= 0.0) return -1;
    size_t kn = 0, nidx = 0;
    for (const MergeRec& mr : L.merges) {
      const size_t s2 = 2 * static_cast<size_t>(mr.s), pp = mr.p1 + mr.p2;
      kn += (s2 + pp) * s2 + s2 * pp;
      nidx += s2 + 2 * pp;
    }
    if (16.0 * static_cast<double>(kn) > fused_max) return -1;
    auto f = std::make_unique<Precond::FusedOps>();
    f->K.alloc(kn);
    f->idx.alloc(nidx);
    std::vector<int> hidx(nidx);
    CopyBatch c0;
    GemmBatch g1, g2, g3;
    size_t ko = 0, io = 0;
    const int* hx = L.h_idx.data();
    for (const MergeRec& mr : L.merges) {
      const ChildBox& c1 = L.children[mr.c1];
      const ChildBox& c2 = L.children[mr.c2];
      const int s = mr.s, p1 = mr.p1, p2 = mr.p2, P1 = c1.P, P2 = c2.P, pp = p1 + p2;
      const int Rd = 2 * s + pp, s2 = 2 * s;
      const double2* T1 = L.tperm.p + c1.t_off;
      const double2* T2 = L.tperm.p + c2.t_off;
      const double2 *T1ps = T1 + static_cast<size_t>(p1) * P1, *T1sp = T1 + p1,
                    *T1ss = T1 + p1 + static_cast<size_t>(p1) * P1;
      const double2 *T2ps = T2 + static_cast<size_t>(p2) * P2, *T2sp = T2 + p2,
                    *T2ss = T2 + p2 + static_cast<size_t>(p2) * P2;
      const double2* W = L.w.p + mr.w_off;
      double2* Kd = f->K.p + ko;
      double2* Ku = Kd + static_cast<size_t>(Rd) * s2;
      ko += static_cast<size_t>(Rd) * s2 + static_cast<size_t>(s2) * pp;
      // index lists: [in1s; in2s], [out1p; out2p], [in1p; in2p]
      int* hs = hidx.data() + io;
      int* hpo = hs + s2;
      int* hpi = hpo + pp;
      for (int i = 0; i < s; ++i) hs[i] = hx[mr.in1_sep + i], hs[s + i] = hx[mr.in2_sep + i];
      for (int i = 0; i < p1; ++i) hpo[i] = hx[mr.out1_per + i], hpi[i] = hx[mr.in1_per + i];
      for (int i = 0; i < p2; ++i) hpo[p1 + i] = hx[mr.out2_per + i], hpi[p1 + i] = hx[mr.in2_per + i];
      const int* ds = f->idx.p + io;
      const int* dpo = ds + s2;
      const int* dpi = dpo + pp;
      io += s2 + 2 * static_cast<size_t>(pp);
      // round 0: X_1 = W, Y = [0, I], Ku_2 = [-T1sp, 0]
      c0.copy(W, s, Kd, Rd, s, s, 1.0);
      c0.zero(Kd + s, Rd, s, s);
      c0.identity(Kd + s + static_cast<size_t>(s) * Rd, Rd, s);
      if (p1) c0.copy(T1sp, P1, Ku + s, s2, s, p1, -1.0);
      if (p2) c0.zero(Ku + s + static_cast<size_t>(p1) * s2, s2, s, p2);
      // round 1: X_2 = -W T2ss
      g1.add(W, s, T2ss, P2, Kd + static_cast<size_t>(s) * Rd, Rd, s, s, s, -1.0, 0.0);
      // round 2: Y -= T1ss X, -T1ps X, Ku_1
      g2.add(T1ss, P1, Kd, Rd, Kd + s, Rd, s, s2, s, -1.0, 1.0);
      if (p1) {
        g2.add(T1ps, P1, Kd, Rd, Kd + s2, Rd, p1, s2, s, -1.0, 0.0);
        g2.add(Kd + static_cast<size_t>(s) * Rd, Rd, T1sp, P1, Ku, s2, s, p1, s, -1.0, 0.0);
      }
      if (p2) g2.add(W, s, T2sp, P2, Ku + static_cast<size_t>(p1) * s2, s2, s, p2, s, -1.0, 0.0);
      // round 3: -T2ps Y, Ku_2 -= T1ss Ku_1
      if (p2) g3.add(T2ps, P2, Kd + s, Rd, Kd + s2 + p1, Rd, p2, s2, s, -1.0, 0.0);
      if (pp) g3.add(T1ss, P1, Ku, s2, Ku + s, s2, s, pp, s, -1.0, 1.0);
      f->down.push_back(item(Kd, Rd, s2, s2, r, ds, nullptr, nullptr, out, ds, 1.0, 0.0, 0.0));
      if (pp) {
        f->down.push_back(item(Kd + s2, Rd, pp, s2, r, ds, nullptr, nullptr, r, dpo, 1.0, 1.0, 0.0));
        f->up.push_back(item(Ku, s2, s2, pp, out, dpi, nullptr, nullptr, out, ds, 1.0, 1.0, 0.0));
      }
    }
    f->idx.upload(hidx, ctx->stream);
    c0.run(ctx);
    g1.run(ctx);
    g2.run(ctx);
    g3.run(ctx);
    p->fused.push_back(std::move(f));
    return static_cast<int>(p->fused.size()) - 1;
  };
  // Levels of many merges with child maps of <= 320 rows: one warp per merge
  // streaming its operators through a TMA ring (vcycle_stream.cu).  The
  // small-level object is still built for the multi-RHS path.
  auto stream_level = [&](int l) -> int {
    const LevelOps& L = *h->levels[l - 1];
    const int ng = static_cast<int>(L.merges.size());
    int rows_max = 0, vec_in = 0, vec_all = 0;
    for (const MergeRec& mr : L.merges) {
      rows_max = std::max({rows_max, L.children[mr.c1].P, L.children[mr.c2].P});
      vec_in = std::max({vec_in, 5 * mr.s, mr.p1 + mr.p2 + 3 * mr.s});
      vec_all = std::max(vec_all, 5 * mr.s + mr.p1 + mr.p2);  // with the output bases
    }
    {
      // merges of < 48 KB per step: the one-CTA small kernel (cfg2 level 1,
      // 32 KB merges: solve 39.2 -> 38.7 ms)
      double mb = 0;
      for (const MergeRec& mr : L.merges) mb += 16.0 * (3.0 * mr.s * mr.s + static_cast<double>(mr.s) * (mr.p1 + mr.p2));
      if (mb < 48e3 * ng) return -1;
    }
    const StreamLevel::Shape shp = stream_level_shape(rows_max, vec_in, vec_all, ng, sms);
    if (!shp.ok) return -1;
    auto sl = std::make_unique<StreamLevel>();
    std::vector<SmallMerge> v;
    const int* ix = L.idx.p;
    for (const MergeRec& mr : L.merges) {
      const ChildBox& c1 = L.children[mr.c1];
      const ChildBox& c2 = L.children[mr.c2];
      SmallMerge m{};
      m.T1 = L.tperm.p + c1.t_off, m.T2 = L.tperm.p + c2.t_off, m.W = L.w.p + mr.w_off;
      m.in1s = ix + mr.in1_sep, m.in2s = ix + mr.in2_sep, m.in1p = ix + mr.in1_per;
      m.in2p = ix + mr.in2_per, m.out1p = ix + mr.out1_per, m.out2p = ix + mr.out2_per;
      m.s = mr.s, m.p1 = mr.p1, m.p2 = mr.p2, m.P1 = c1.P, m.P2 = c2.P;
      v.push_back(m);
      const double ss = 16.0 * mr.s * mr.s, sp = 16.0 * mr.s * (mr.p1 + mr.p2);
      sl->bytes_down += 3 * ss + sp;
      sl->bytes_up += 3 * ss + sp;
    }
    sl->level = l;
    sl->count = ng;
    sl->shape = shp;
    if (std::getenv("HPSB_PROFILE_LEVELS")) sl->label = "vcycle_stream_L" + std::to_string(l);
    sl->d.upload(v, ctx->stream);
    p->streams.push_back(std::move(sl));
    return static_cast<int>(p->streams.size()) - 1;
  };
  // Levels of few, large merges (local ones; a sharded run's global levels
  // keep their owner-computes plans): one persistent launch per level step,
  // stages separated by grid barriers (vcycle_wide.cu).
  auto wide_level = [&](int l) -> int {
    const LevelOps& L = *h->levels[l - 1];
    const int ng = static_cast<int>(L.merges.size());
    // (levels of >= 64 merges stream faster as cluster chains; levels of
    // < 150 MB per step are bound by the grid barriers: cfg2 levels 7-11,
    // 37-88 MB, ran at 0.6-1.6 TB/s as wide levels)
    if (!ng || ng >= 64 || l > h->sk->el->part.last_local) return -1;
    {
      double lb = 0;
      for (const MergeRec& mr : L.merges) lb += 16.0 * (3.0 * mr.s * mr.s + static_cast<double>(mr.s) * (mr.p1 + mr.p2));
      if (lb < 150e6) return -1;
    }
    constexpr int kTcCap = 1024;  // tile columns (the x slice in shared memory)
    auto wl = std::make_unique<WideLevel>();
    wl->shape = wide_level_shape(kTcCap, sms);
    const int occ = wl->shape.ok ? wide_max_ctas_per_sm(wl->shape.smem) : 0;
    if (trace) std::fprintf(stderr, "[hpsb] level %d wide: shape ok %d, smem %zu, %d CTAs/SM\n", l,
                            wl->shape.ok ? 1 : 0, wl->shape.smem, occ);
    if (occ < 1) return -1;
    if (occ < wl->shape.ctas_per_sm) wl->shape.ctas_per_sm = occ, wl->shape.grid = sms * occ;
    const int G = wl->shape.grid;
    size_t part_max = 0;
    const int* ix = L.idx.p;
    for (int dir = 0; dir < 2; ++dir) {
      const bool downward = dir == 0;
      WideLevel::Dir& D = wl->dir[dir];
      std::vector<WideMerge> wm(ng);
      std::vector<WideTile> tiles;
      std::vector<int> prefix(4 * static_cast<size_t>(ng + 1), 0);
      struct OpD {
        const double2* src;
        int R, C, ld;
      };
      auto op_of = [&](int gi, int k) -> OpD {
        const MergeRec& mr = L.merges[gi];
        const ChildBox& c1 = L.children[mr.c1];
        const ChildBox& c2 = L.children[mr.c2];
        const int s = mr.s, p1 = mr.p1, p2 = mr.p2, P1 = c1.P, P2 = c2.P;
        const double2* T1 = L.tperm.p + c1.t_off;
        const double2* T2 = L.tperm.p + c2.t_off;
        const double2* W = L.w.p + mr.w_off;
        if (downward) {
          switch (k) {
            case 0: return {T2 + p2 + static_cast<size_t>(p2) * P2, s, s, P2};
            case 1: return {W, s, s, s};
            case 2: return {T1 + static_cast<size_t>(p1) * P1, P1, s, P1};
            default: return {T2 + static_cast<size_t>(p2) * P2, p2, p2 ? s : 0, P2};
          }
        }
        switch (k) {
          case 0: return {T1 + p1, s, p1, P1};
          case 1: return {T2 + p2, s, P2, P2};
          case 2: return {W, s, s, s};
          default: return {T1 + p1 + static_cast<size_t>(p1) * P1, s, s, P1};
        }
      };
      for (int gi = 0; gi < ng; ++gi) {
        const MergeRec& mr = L.merges[gi];
        WideMerge& w = wm[gi];
        w.in1s = ix + mr.in1_sep, w.in2s = ix + mr.in2_sep, w.in1p = ix + mr.in1_per;
        w.in2p = ix + mr.in2_per, w.out1p = ix + mr.out1_per, w.out2p = ix + mr.out2_per;
        w.s = mr.s, w.p1 = mr.p1, w.p2 = mr.p2;
      }
      size_t poff = 0;
      std::vector<int> cta_tiles(4 * static_cast<size_t>(G + 1), 0);
      for (int k = 0; k < 4; ++k) {
        // stage k's rows over all merges, times ncb column blocks so that a
        // CTA's range has >= 128 rows (2 KB column segments per bulk copy:
        // 32-row segments streamed at half the rate); equal contiguous
        // ranges per CTA
        long long NR = 0;
        for (int gi = 0; gi < ng; ++gi) {
          const OpD o = op_of(gi, k);
          wm[gi].R[k] = o.R;
          prefix[k * (ng + 1) + gi + 1] = prefix[k * (ng + 1) + gi] + o.R;
          if (o.C > 0) NR += o.R;
          D.bytes += 16.0 * o.R * o.C;
        }
        int cmax = 0;
        for (int gi = 0; gi < ng; ++gi) cmax = std::max(cmax, op_of(gi, k).C);
        const int ncb = NR > 0 ? static_cast<int>(std::max<long long>(
                                     (cmax + kTcCap - 1) / kTcCap, std::max<long long>(1, (128LL * G + NR - 1) / NR)))
                               : 0;
        for (int gi = 0; gi < ng; ++gi) {
          const OpD o = op_of(gi, k);
          WideMerge& w = wm[gi];
          w.ncb[k] = (o.R > 0 && o.C > 0) ? std::min(ncb, o.C) : 0;
          w.part[k] = static_cast<long long>(poff);
          poff += static_cast<size_t>(w.ncb[k]) * o.R;
        }
        // flattened (column block, merge, row) space of the merges with work
        std::vector<int> mlist;
        std::vector<long long> mpre(1, 0);
        for (int gi = 0; gi < ng; ++gi)
          if (wm[gi].ncb[k] > 0) mlist.push_back(gi), mpre.push_back(mpre.back() + wm[gi].R[k]);
        const long long N = NR * ncb;
        for (int bb = 0; bb < G; ++bb) {
          cta_tiles[k * (G + 1) + bb] = static_cast<int>(tiles.size());
          long long f = N * bb / G;
          const long long f1 = N * (bb + 1) / G;
          while (f < f1) {
            const int cb = static_cast<int>(f / NR);
            const long long rem = f % NR;
            const int mi = static_cast<int>(std::upper_bound(mpre.begin(), mpre.end(), rem) - mpre.begin()) - 1;
            const int gi = mlist[mi];
            const int row = static_cast<int>(rem - mpre[mi]);
            const OpD o = op_of(gi, k);
            const int nb = wm[gi].ncb[k];
            // (at most 32 rows per consumer warp in one tile)
            const long long take = std::min<long long>({f1 - f, o.R - row, 32LL * wl->shape.warps});
            if (cb < nb) {  // (a narrow operator may have fewer column blocks)
              const int TC = (o.C + nb - 1) / nb;
              WideTile t{};
              t.c0 = cb * TC, t.cols = std::min(TC, o.C - t.c0);
              t.r0 = row, t.rows = static_cast<int>(take);
              t.ld = o.ld, t.m = gi, t.cb = cb;
              t.A = o.src + row + static_cast<size_t>(t.c0) * o.ld;
              if (t.cols > 0) tiles.push_back(t);
            }
            f += take;
          }
        }
        cta_tiles[k * (G + 1) + G] = static_cast<int>(tiles.size());
      }
      part_max = std::max(part_max, poff);
      D.ntiles = static_cast<int>(tiles.size());
      D.tiles.upload(tiles, ctx->stream);
      D.merges.upload(wm, ctx->stream);
      D.prefix.upload(prefix, ctx->stream);
      D.cta_tiles.upload(cta_tiles, ctx->stream);
      D.args.cta_tiles = D.cta_tiles.p;
      D.args.tiles = D.tiles.p;
      D.args.merges = D.merges.p;
      D.args.nm = ng;
      D.args.row_prefix = D.prefix.p;
      D.args.down = downward ? 1 : 0;
      D.args.slot_entries = wl->shape.slot_entries;
      D.args.tc_max = wl->shape.tc_max;
    }
    wl->part.alloc(std::max<size_t>(part_max, 1));
    wl->bar.alloc(2);
    HPSB_CUDA(cudaMemsetAsync(wl->bar.p, 0, 2 * sizeof(unsigned), ctx->stream));
    for (auto& D : wl->dir) D.args.part = wl->part.p, D.args.bar = wl->bar.p;
    wl->level = l;
    if (std::getenv("HPSB_PROFILE_LEVELS")) wl->label = "vcycle_wide_L" + std::to_string(l);
    p->wides.push_back(std::move(wl));
    return static_cast<int>(p->wides.size()) - 1;
  };
  std::vector<int> small_of(cfg.depth, -1), cluster_of(cfg.depth, -1), fused_of(cfg.depth, -1),
      stream_of(cfg.depth, -1), wide_of(cfg.depth, -1);
  for (int l = 1; l < cfg.depth; ++l) {
    fused_of[l] = fused_level(l);
    if (fused_of[l] >= 0) continue;
    small_of[l] = small_level(l);
    stream_of[l] = stream_level(l);
    if (stream_of[l] >= 0 || small_of[l] >= 0) continue;
    wide_of[l] = wide_level(l);
    if (wide_of[l] < 0) cluster_of[l] = cluster_level(l);
  }
  p->small_level_of = small_of;
  mark("levels");
  auto add_step = [&](int l, bool downward) {
    Precond::Step st;
    st.level = l;
    st.small = small_of[l];
    st.cluster = cluster_of[l];
    st.stream = stream_of[l];
    st.wide = wide_of[l];
    if (st.stream >= 0) {
      p->bytes_small += downward ? p->streams[st.stream]->bytes_down : p->streams[st.stream]->bytes_up;
    } else if (st.wide >= 0) {
      p->bytes_small += p->wides[st.wide]->dir[downward ? 0 : 1].bytes;
    } else if (fused_of[l] >= 0) {
      const bool global_level = l > h->sk->el->part.last_local;
      VPlan& plan =
          downward ? (global_level ? p->down_g : p->down) : (global_level ? p->up_g : p->up);
      st.plan = &plan;
      st.p0 = static_cast<int>(plan.phases.size());
      const std::vector<VItem>& its = downward ? p->fused[fused_of[l]]->down : p->fused[fused_of[l]]->up;
      if (!its.empty()) {
        plan.phases[plan.begin_phase()].label =
            std::string(downward ? "vcycle_down" : "vcycle_up") +
            (std::getenv("HPSB_PROFILE_LEVELS") ? "_fused_L" + std::to_string(l) : "");
        int rows = 0;
        for (const VItem& it : its) rows += it.rows;
        for (const VItem& it : its) plan.add_split(it, split_rows(rows, sms));
      }
      st.p1 = static_cast<int>(plan.phases.size());
    } else if (st.cluster >= 0) {
      p->bytes_small += downward ? p->clusters[st.cluster]->bytes_down : p->clusters[st.cluster]->bytes_up;
    } else if (st.small < 0) {
      const bool global_level = l > h->sk->el->part.last_local;
      VPlan& plan =
          downward ? (global_level ? p->down_g : p->down) : (global_level ? p->up_g : p->up);
      st.plan = &plan;
      st.p0 = static_cast<int>(plan.phases.size());
      build_level(l, downward);
      st.p1 = static_cast<int>(plan.phases.size());
    } else {
      p->bytes_small += downward ? p->smalls[st.small]->bytes_down : p->smalls[st.small]->bytes_up;
    }
    (downward ? p->down_steps : p->up_steps).push_back(st);
  };
  for (int l = 1; l < cfg.depth; ++l) add_step(l, true);
  for (int l = cfg.depth - 1; l >= 1; --l) add_step(l, false);
  mark("steps");
  p->down.name = "vcycle_down";
  p->up.name = "vcycle_up";
  p->down_g.name = "vcycle_down";
  p->up_g.name = "vcycle_up";
  p->down.finalize(ctx->stream);
  p->up.finalize(ctx->stream);
  p->down_g.finalize(ctx->stream);
  p->up_g.finalize(ctx->stream);
  if (ctx->world() > 1) {
    const Partition& part = h->sk->el->part;
    std::vector<int> keep(part.face_owner.size());
    for (size_t f = 0; f < keep.size(); ++f)
      keep[f] = part.face_owner[f] == ctx->rank() || (part.face_owner[f] < 0 && ctx->rank() == 0);
    p->keep_face.upload(keep, ctx->stream);
    p->tail_off = static_cast<int64_t>(h->sk->graph.level_range[part.last_local].first) * h->sk->bs;
  }

  // stage lists for the multi-RHS phases (single GPU)
  p->tmp_total = std::max<size_t>(tmp_total, 1);
  for (int dir = 0; dir < 2; ++dir) {
    p->stage_items[dir].assign(cfg.depth, {});
    for (int l = 1; l < cfg.depth; ++l) {
      auto pm = level_stages(l, dir == 0);
      auto& lv = p->stage_items[dir][l];
      lv.assign(4, {});
      for (auto& st : pm)
        for (int k = 0; k < 4; ++k)
          for (auto& it : st[k]) lv[k].push_back(it);
    }
  }

  mark("plans");
  // ---- coarse level: M_depth = I + sum_boxes scatter(T_box) on the tail
  const LevelOps& C = *h->levels[cfg.depth - 1];
  p->off_d = static_cast<int64_t>(C.first_face) * sk->bs;
  p->dim_d = p->dim - p->off_d;
  if (cfg.exact_coarse && p->dim_d > kExactCoarseMax)
    throw InvalidArgument("MgPreconditioner: exact coarse system too large for a dense inverse");
  const int ci = cfg.exact_coarse ? 0 : cfg.coarse_iters;
  p->V.alloc(static_cast<size_t>(p->dim_d) * (ci + 1));
  p->cv.alloc(p->dim_d);
  p->cw.alloc(p->dim_d);
  p->Hm.alloc(static_cast<size_t>(ci + 1) * ci);
  p->gv.alloc(ci + 1);
  p->rs.alloc(ci);
  p->rc.alloc(ci);
  p->state.alloc(4);
  std::vector<int> lidx;
  std::vector<size_t> in_at, out_at;
  for (const ChildBox& c : C.children) {
    in_at.push_back(lidx.size());
    for (const auto& q : c.pos) lidx.push_back(q.in - static_cast<int>(p->off_d));
    out_at.push_back(lidx.size());
    for (const auto& q : c.pos) lidx.push_back(q.out - static_cast<int>(p->off_d));
  }
  p->coarse_idx.upload(lidx, ctx->stream);
  int crows = 0;
  for (const ChildBox& c : C.children) crows += c.P;
  const int crb = split_rows(crows, sms);
  p->coarse_mv.begin_phase();
  for (size_t k = 0; k < C.children.size(); ++k) {
    const ChildBox& c = C.children[k];
    const int* ci_in = p->coarse_idx.p + in_at[k];
    const int* ci_out = p->coarse_idx.p + out_at[k];
    p->coarse_mv.add_split(item(C.tperm.p + c.t_off, c.P, c.P, c.P, p->cv.p, ci_in, p->cv.p,
                                ci_out, p->cw.p, ci_out, 1.0, 0.0, 1.0),
                           crb);
  }
  p->coarse_mv.name = "coarse_matvec";
  p->coarse_mv.finalize(ctx->stream);
  // Fused single-launch coarse solve when the coarse maps are small enough
  // for one 16-CTA cluster to stream them quickly.
  {
    std::vector<VItem> whole;
    for (size_t k = 0; k < C.children.size(); ++k) {
      const ChildBox& c = C.children[k];
      const int* ci_in = p->coarse_idx.p + in_at[k];
      const int* ci_out = p->coarse_idx.p + out_at[k];
      whole.push_back(item(C.tperm.p + c.t_off, c.P, c.P, c.P, nullptr, ci_in, nullptr, ci_out,
                           nullptr, ci_out, 1.0, 0.0, 1.0));
      p->coarse_max_cols = std::max(p->coarse_max_cols, c.P);
    }
    // One cluster streams ~0.3 MB per CTA per matvec within a few us; larger
    // coarse systems need the whole GPU for their matvecs (split launches).
    p->coarse_fused = p->coarse_mv.bytes_per_run <= (4ll << 20) && ci <= kMaxCoarseIters;
    p->coarse_csize = 1;
    while (p->coarse_csize < 16 &&
           p->coarse_mv.bytes_per_run > p->coarse_csize * static_cast<int64_t>(64 << 10))
      p->coarse_csize *= 2;
    p->coarse_items.upload(whole, ctx->stream);
    p->coarse_nitems = static_cast<int>(whole.size());
    // On-chip variant: a cluster of 16 CTAs (else 8, 4, 2) whose CTAs hold
    // their rows of the coarse maps in shared memory.  The largest cluster
    // wins: each CTA's staging burst is on the critical path when the
    // previous kernel's CTAs still occupy the SMs (cfg1: 16 CTAs 116 us per
    // apply, 4 CTAs 149 us). 
    {
      for (int Cc = kCoarseMaxCluster; Cc >= 2 && !p->coarse_cluster; Cc /= 2) {
        size_t stage = 0;
        for (const VItem& it : whole)
          stage += static_cast<size_t>(std::min(it.rows, cluster_chunk(it.rows, Cc))) * it.cols;
        const int slice = static_cast<int>((p->dim_d + Cc - 1) / Cc);
        size_t nidx = 0, xs_total = 0;
        for (const VItem& it : whole) {
          nidx += it.cols + std::min(it.rows, cluster_chunk(it.rows, Cc));
          xs_total += it.cols;
        }
        const size_t smem = sizeof(double2) * (static_cast<size_t>(p->dim_d) +
                                               static_cast<size_t>(ci + 2) * slice +
                                               xs_total + stage) +
                            sizeof(int) * nidx;
        if (p->coarse_fused && smem <= (200u << 10) && slice <= kCoarseCThreads &&
            whole.size() <= static_cast<size_t>(kCoarseClusterItems) &&
            coarse_cluster_fits(smem, Cc)) {
          p->coarse_cluster = true;
          p->coarse_xs = static_cast<int>(xs_total);
          p->coarse_stage = stage;
          p->coarse_slice = slice;
          p->coarse_smem = smem;
          p->coarse_csize = Cc;
        }
      }
    }
  }
  if (!cfg.exact_coarse && cfg.gamma > 1) {
    // next.M.apply(z) of apply_level's gamma loop (multigrid.cpp:71-80):
    // M_l = I + sum_boxes scatter_out(T gather_in(.)) over the boxes entering level l
    p->level_mv.resize(cfg.depth + 1);
    p->gam_rc.alloc(static_cast<size_t>(cfg.depth) * p->dim);
    p->gam_z.alloc(static_cast<size_t>(cfg.depth) * p->dim);
    p->gam_t.alloc(p->dim);
    for (int l = 2; l <= cfg.depth; ++l) {
      const LevelOps& Lv = *h->levels[l - 1];
      std::vector<int> gidx;
      std::vector<size_t> in_at2, out_at2;
      for (const ChildBox& c : Lv.children) {
        in_at2.push_back(gidx.size());
        for (const auto& q : c.pos) gidx.push_back(q.in);
        out_at2.push_back(gidx.size());
        for (const auto& q : c.pos) gidx.push_back(q.out);
      }
      VPlan& mv = p->level_mv[l];
      mv.idx_store.upload(gidx, ctx->stream);
      int rows = 0;
      for (const ChildBox& c : Lv.children) rows += c.P;
      const int rb2 = split_rows(std::max(rows, 1), sms);
      mv.begin_phase();
      for (size_t k = 0; k < Lv.children.size(); ++k) {
        const ChildBox& c = Lv.children[k];
        const int* gi = mv.idx_store.p + in_at2[k];
        const int* go = mv.idx_store.p + out_at2[k];
        mv.add_split(item(Lv.tperm.p + c.t_off, c.P, c.P, c.P, p->gam_t.p, gi, p->gam_t.p, go, p->r.p,
                          go, 1.0, 0.0, 1.0),
                     rb2);
      }
      mv.name = "level_matvec";
      mv.finalize(ctx->stream);
    }
  }
  if (cfg.exact_coarse) {
    // exact_lu = LU(M_depth.to_dense()) (multigrid.cpp:22-27); here the dense
    // inverse (blocked Gauss-Jordan on the DMMA GEMMs) and one GEMV per apply.
    const int64_t nd = p->dim_d;
    p->cinv.alloc(static_cast<size_t>(nd) * nd);
    CopyBatch cb;
    cb.identity(p->cinv.p, static_cast<int>(nd), static_cast<int>(nd));
    cb.run(ctx);
    std::vector<int64_t> toff, at;
    std::vector<int> Ps;
    for (size_t k = 0; k < C.children.size(); ++k) {
      toff.push_back(static_cast<int64_t>(C.children[k].t_off));
      Ps.push_back(C.children[k].P);
      at.push_back(static_cast<int64_t>(in_at[k]));
      at.push_back(static_cast<int64_t>(out_at[k]));
    }
    DevBuf<int64_t> d_toff, d_at;
    DevBuf<int> d_P, d_status(1);
    d_toff.upload(toff, ctx->stream);
    d_at.upload(at, ctx->stream);
    d_P.upload(Ps, ctx->stream);
    HPSB_CUDA(cudaMemsetAsync(d_status.p, 0, sizeof(int), ctx->stream));
    if (!C.children.empty()) {
      KernelScope ks(ctx, "coarse_densify", 0.0, 0.0);
      coarse_densify_kernel<<<dim3(32, static_cast<unsigned>(C.children.size())), 256, 0, ctx->stream>>>(
          C.tperm.p, d_toff.p, d_P.p, p->coarse_idx.p, d_at.p, p->cinv.p, nd);
      HPSB_LAUNCHED(ctx);
    }
    InverseBatch inv;
    inv.ops.push_back(InvOp{p->cinv.p, static_cast<int>(nd), static_cast<int>(nd), 0, 0});
    inv.run(ctx, d_status.p);
    int st = 0;
    HPSB_CUDA(cudaMemcpyAsync(&st, d_status.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (st) throw std::runtime_error("MgPreconditioner: singular coarse system");
    std::vector<int> yi(nd);
    for (int64_t k = 0; k < nd; ++k) yi[k] = static_cast<int>(p->off_d + k);
    p->exact_yi.upload(yi, ctx->stream);
    // z_tail = M_depth^{-1} r_tail, column chunks accumulate (beta = 1)
    constexpr int kChunk = 4096;
    const int rows_blk = split_rows(static_cast<int>(nd), sms);
    for (int64_t c0 = 0; c0 < nd; c0 += kChunk) {
      const int cc = static_cast<int>(std::min<int64_t>(kChunk, nd - c0));
      p->exact_mv.begin_phase();
      p->exact_mv.add_split(item(p->cinv.p + c0 * nd, static_cast<int>(nd), static_cast<int>(nd), cc,
                                 p->r.p + p->off_d + c0, nullptr, nullptr, nullptr, p->out.p,
                                 p->exact_yi.p, 1.0, c0 > 0 ? 1.0 : 0.0, 0.0),
                            rows_blk);
    }
    p->exact_mv.name = "coarse_exact";
    p->exact_mv.finalize(ctx->stream);
    p->coarse_fused = false;
  }
  // Large coarse systems (>= 100 MB of box maps per matvec; the split-launch
  // path otherwise): the whole gmres_fixed_steps as one persistent
  // cooperative grid (vcycle_wide.cu).  (cfg3, 189 MB: solve -1%; cfg2,
  // 30 MB: +5% -- the grid barriers dominate small coarse systems.)
  if (!cfg.exact_coarse && !p->coarse_fused && !p->coarse_cluster && p->coarse_mv.bytes_per_run >= (100ll << 20) && ci >= 1 && ci <= kCoarseWideMax &&
      !C.children.empty()) {
    auto cw = std::make_unique<CoarseWide>();
    cw->shape = wide_level_shape(1024, sms);
    const int occ = cw->shape.ok ? coarse_wide_max_ctas_per_sm(cw->shape.smem) : 0;
    if (occ >= 1) {
      if (occ < cw->shape.ctas_per_sm) cw->shape.ctas_per_sm = occ, cw->shape.grid = sms * occ;
      const int G = cw->shape.grid, nb = static_cast<int>(C.children.size());
      long long NR = 0;
      int cmax = 0;
      for (const ChildBox& c : C.children) NR += c.P, cmax = std::max(cmax, c.P);
      const int ncb = static_cast<int>(std::max<long long>((cmax + 1023) / 1024, std::max<long long>(1, (128LL * G + NR - 1) / NR)));
      std::vector<WideMerge> boxes(nb);
      std::vector<long long> mpre(1, 0);
      size_t poff = 0;
      std::vector<int> inv_box(p->dim_d, -1), inv_row(p->dim_d, -1);
      for (int k = 0; k < nb; ++k) {
        const ChildBox& c = C.children[k];
        WideMerge& w = boxes[k];
        w.in1s = p->coarse_idx.p + in_at[k];
        w.R[0] = c.P, w.ncb[0] = std::min(ncb, c.P), w.part[0] = static_cast<long long>(poff);
        poff += static_cast<size_t>(w.ncb[0]) * c.P;
        mpre.push_back(mpre.back() + c.P);
        for (int r0 = 0; r0 < c.P; ++r0) {
          const int o = lidx[out_at[k] + r0];
          if (o < 0 || o >= p->dim_d || inv_box[o] >= 0) throw std::runtime_error("coarse map: bad output slot");
          inv_box[o] = k, inv_row[o] = r0;
        }
      }
      for (int64_t i = 0; i < p->dim_d; ++i)
        if (inv_box[i] < 0) throw std::runtime_error("coarse map: slot without a box row");
      std::vector<WideTile> tiles;
      std::vector<int> cta(G + 1, 0);
      const long long N = NR * ncb;
      for (int bb = 0; bb < G; ++bb) {
        cta[bb] = static_cast<int>(tiles.size());
        long long f = N * bb / G;
        const long long f1 = N * (bb + 1) / G;
        while (f < f1) {
          const int cb = static_cast<int>(f / NR);
          const long long rem = f % NR;
          const int k = static_cast<int>(std::upper_bound(mpre.begin(), mpre.end(), rem) - mpre.begin()) - 1;
          const ChildBox& c = C.children[k];
          const int row = static_cast<int>(rem - mpre[k]);
          const long long take = std::min<long long>({f1 - f, c.P - row, 32LL * cw->shape.warps});
          const int nbk = boxes[k].ncb[0];
          if (cb < nbk) {
            const int TC = (c.P + nbk - 1) / nbk;
            WideTile t{};
            t.c0 = cb * TC, t.cols = std::min(TC, c.P - t.c0);
            t.r0 = row, t.rows = static_cast<int>(take);
            t.ld = c.P, t.m = k, t.cb = cb;
            t.A = C.tperm.p + c.t_off + row + static_cast<size_t>(t.c0) * c.P;
            if (t.cols > 0) tiles.push_back(t);
          }
          f += take;
        }
      }
      cta[G] = static_cast<int>(tiles.size());
      cw->tiles.upload(tiles, ctx->stream);
      cw->boxes.upload(boxes, ctx->stream);
      cw->cta_tiles.upload(cta, ctx->stream);
      cw->inv_box.upload(inv_box, ctx->stream);
      cw->inv_row.upload(inv_row, ctx->stream);
      cw->part.alloc(std::max<size_t>(poff, 1));
      cw->pd.alloc(static_cast<size_t>(G) * (kCoarseWideMax + 1));
      cw->pn.alloc(G);
      cw->bar.alloc(2);
      HPSB_CUDA(cudaMemsetAsync(cw->bar.p, 0, 2 * sizeof(unsigned), ctx->stream));
      CoarseArgs& A = cw->args;
      A.tiles = cw->tiles.p, A.cta_tiles = cw->cta_tiles.p, A.boxes = cw->boxes.p;
      A.inv_box = cw->inv_box.p, A.inv_row = cw->inv_row.p, A.part = cw->part.p;
      A.V = p->V.p, A.W = p->cw.p, A.pd = cw->pd.p, A.pn = cw->pn.p, A.bar = cw->bar.p;
      A.n = p->dim_d, A.ci = ci, A.slot_entries = cw->shape.slot_entries, A.tc_max = cw->shape.tc_max;
      cw->bytes = static_cast<double>(ci) * p->coarse_mv.bytes_per_run;
      p->coarse_wide = std::move(cw);
    }
  }
  p->bytes_per_apply = static_cast<int64_t>(p->bytes_small) + p->down.bytes_per_run +
                       p->up.bytes_per_run + p->down_g.bytes_per_run +
                       p->up_g.bytes_per_run +
                       static_cast<int64_t>(ci) * p->coarse_mv.bytes_per_run +
                       p->exact_mv.bytes_per_run;
  HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
  mark("coarse");
  if (trace) {
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    mark("device_drain");
    std::fprintf(stderr, "[hpsb trace precond]%s\n", trace_line.c_str());
  }
  return p.release();
}

void destroy_precond(Precond* p) { delete p; }

namespace {
// The deepest level's solve: gmres_fixed_steps on M_depth (or the exact
// dense inverse), r[off_d:] -> z[off_d:].
void run_coarse(Precond* p, double2* z_dev) {
  Context* ctx = p->ctx;
  const int ci = p->cfg.coarse_iters;
  if (p->cfg.exact_coarse) {
    p->exact_mv.run(ctx, p->out.p, z_dev);
  } else if (p->coarse_wide) {
    p->coarse_wide->run(ctx, p->r.p + p->off_d, z_dev + p->off_d);
  } else if (p->coarse_cluster) {
    KernelScope ks(ctx, "coarse_fused", static_cast<double>(p->coarse_mv.bytes_per_run), 0.0);
    launch_k(ctx, coarse_cluster_kernel, dim3(p->coarse_csize), dim3(kCoarseCThreads),
             p->coarse_smem, p->coarse_csize, static_cast<const VItem*>(p->coarse_items.p),
             p->coarse_nitems, static_cast<int>(p->dim_d), p->coarse_slice, ci,
             std::max(p->coarse_xs, 1), p->coarse_stage,
             static_cast<const double2*>(p->r.p + p->off_d), z_dev + p->off_d);
  } else if (p->coarse_fused) {
    static const bool attr = [] {  // thread-safe one-time init
      HPSB_CUDA(cudaFuncSetAttribute(coarse_fused_kernel,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      return true;
    }();
    (void)attr;
    const size_t smem = sizeof(double2) * std::max(p->coarse_max_cols, 1);
    allow_smem<coarse_fused_kernel>(smem);
    KernelScope ks(ctx, "coarse_fused", static_cast<double>(ci) * p->coarse_mv.bytes_per_run, 0.0);
    launch_k(ctx, coarse_fused_kernel, dim3(p->coarse_csize), dim3(kGemvThreads), smem,
             p->coarse_csize, static_cast<const VItem*>(p->coarse_items.p), p->coarse_nitems,
             p->dim_d, ci, p->V.p, p->cw.p, static_cast<const double2*>(p->r.p + p->off_d),
             z_dev + p->off_d, p->coarse_max_cols);
  } else {
  {
  KernelScope ks(ctx, "coarse_gmres", 32.0 * p->dim_d, 0.0);
  launch_k(ctx, coarse_init_kernel, dim3(1), dim3(kCoarseThreads), 0, 1,
           static_cast<const double2*>(p->r.p + p->off_d), p->dim_d, p->V.p, p->cv.p, p->gv.p, ci,
           p->state.p, int64_t(0));
  }
  for (int j = 0; j < ci; ++j) {
    p->coarse_mv.run(ctx);
    KernelScope ks(ctx, "coarse_gmres", 16.0 * p->dim_d * (2 * j + 4), 0.0);
    launch_k(ctx, coarse_step_kernel, dim3(1), dim3(kCoarseThreads), 0, 1, j, p->dim_d, ci, p->V.p,
             p->cv.p, p->cw.p, p->Hm.p, p->gv.p, p->rc.p, p->rs.p, p->state.p, int64_t(0));
  }
  {
  KernelScope ks(ctx, "coarse_gmres", 16.0 * p->dim_d * (ci + 1), 0.0);
  launch_k(ctx, coarse_finish_kernel, dim3(1), dim3(kCoarseThreads), 0, 1, p->dim_d, ci,
           static_cast<const double2*>(p->V.p), static_cast<const double2*>(p->Hm.p),
           static_cast<const double2*>(p->gv.p), static_cast<const double*>(p->state.p),
           z_dev + p->off_d, int64_t(0));
  }
  }
}

void run_level(Precond* p, int l, bool down, double2* z) {
  for (const Precond::Step& st : down ? p->down_steps : p->up_steps) {
    if (st.level == l) p->run_step(st, down, z);
  }
}

// One level step of the gamma-cycle.  Sharded: a local level runs the rank's
// own merges and, going down, sums the residual changes on the global rows
// (each changed by at most one rank); a global level runs owner-computes with
// the exchanges of run_global_sharded (its separator rows of z zeroed first:
// the exchange sums them over the ranks and only the owner assigns them).
void level_step(Precond* p, int l, bool down, double2* z) {
  Context* ctx = p->ctx;
  if (ctx->world() == 1) {
    run_level(p, l, down, z);
    return;
  }
  const int last_local = p->h->sk->el->part.last_local;
  if (l > last_local) {
    for (const Precond::Step& st : down ? p->down_steps : p->up_steps) {
      if (st.level != l) continue;
      if (down) {
        const auto& g = p->h->sk->graph;
        const int64_t s0 = static_cast<int64_t>(g.level_range[l - 1].first) * p->h->sk->bs;
        const int64_t s1 = static_cast<int64_t>(g.level_range[l].first) * p->h->sk->bs;
        HPSB_CUDA(cudaMemsetAsync(z + s0, 0, sizeof(double2) * (s1 - s0), ctx->stream));
      }
      p->run_global_level(st, down, z);
    }
    return;
  }
  if (!down) {
    run_level(p, l, false, z);
    return;
  }
  const int64_t t0 = p->tail_off, n = p->dim - t0;
  if (p->xsave.n < static_cast<size_t>(n)) p->xsave.alloc(n);
  zcopy(ctx, p->xsave.p, p->r.p + t0, n);
  run_level(p, l, true, z);
  exchange_deltas(ctx, p->xbuf, {{p->r.p + t0, p->xsave.p, n}});
}

// apply_level (multigrid.cpp:30-100) with gamma > 1: F and restriction at
// level l (down step), gamma recursive coarse corrections with the level
// system residual rc - M_{l+1} z in between, prolongation (up step).
// Sharded: vectors valid on the rank's own rows and the (replicated) global
// rows; M_{l+1} z below the coarse level sums the ranks' box rows on the
// global rows (each produced by one box, i.e. one rank).
void apply_level_gamma(Precond* p, int l, double2* z) {
  Context* ctx = p->ctx;
  if (l == p->cfg.depth) {
    run_coarse(p, z);
    return;
  }
  level_step(p, l, true, z);
  const Hierarchy* h = p->h;
  const bool sharded = ctx->world() > 1;
  const int64_t off = static_cast<int64_t>(h->levels[l]->first_face) * h->sk->bs;  // level l+1 tail
  const int64_t len = p->dim - off;
  double2* rc = p->gam_rc.p + static_cast<size_t>(l) * p->dim;
  double2* zacc = p->gam_z.p + static_cast<size_t>(l) * p->dim;
  const int blocks = static_cast<int>(std::min<int64_t>((len + 255) / 256, 8 * ctx->num_sms));
  launch_k(ctx, copy_vec_kernel, dim3(blocks), dim3(256), 0, 1, rc + off, p->r.p + off, len);
  HPSB_CUDA(cudaMemsetAsync(zacc + off, 0, sizeof(double2) * len, ctx->stream));
  for (int step = 0; step < p->cfg.gamma; ++step) {
    if (step > 0) {
      // r = rc - M_{l+1} z on the tail
      const bool split = sharded && l + 1 < p->cfg.depth;  // (the coarse boxes are on every rank)
      const int64_t t0 = p->tail_off;
      if (split) HPSB_CUDA(cudaMemsetAsync(p->gam_t.p + t0, 0, sizeof(double2) * (p->dim - t0), ctx->stream));
      p->level_mv[l + 1].run(ctx, p->gam_t.p, zacc, p->r.p, p->gam_t.p);
      if (split) ctx->comm->allreduce_sum(p->gam_t.p + t0, p->dim - t0, ctx);
      launch_k(ctx, copy_vec_kernel, dim3(blocks), dim3(256), 0, 1, p->r.p + off,
               static_cast<const double2*>(rc + off), len);
      launch_k(ctx, axpy_vec_kernel, dim3(blocks), dim3(256), 0, 1, p->r.p + off,
               static_cast<const double2*>(p->gam_t.p + off), -1.0, len);
    }
    apply_level_gamma(p, l + 1, z);
    launch_k(ctx, axpy_vec_kernel, dim3(blocks), dim3(256), 0, 1, zacc + off,
             static_cast<const double2*>(z + off), 1.0, len);
  }
  launch_k(ctx, copy_vec_kernel, dim3(blocks), dim3(256), 0, 1, z + off,
           static_cast<const double2*>(zacc + off), len);
  level_step(p, l, false, z);
}
}  // namespace

bool precond_graph_safe(const Precond* p) {
  return p->ctx->world() == 1 && (p->cfg.exact_coarse || p->cfg.gamma <= 1);
}

// Sharded global levels (owner-computes: each merge of a level above the
// subtrees runs on one rank).  Every rank holds the same global rows of r
// and out before a level; a level's merges change out at their separator
// rows (assignments, down) or by increments (up) and r at their perimeter
// rows, each row on exactly one rank, so one allreduce of the changes per
// level makes every rank consistent again for the next level.
void Precond::run_global_level(const Step& st, bool down, double2* z) {
  const auto& g = h->sk->graph;
  const int bs = h->sk->bs;
  auto ff = [&](int l) { return static_cast<int64_t>(g.level_range[l - 1].first) * bs; };
  const int l = st.level;
  const int64_t s0 = ff(l), s1 = ff(l + 1);  // level-l separator rows; rows above: [s1, dim)
  if (down) {
    // baseline of r above the level; out at the level's separators is 0
    // on every rank (zeroed before the global sweep)
    if (xsave.n < static_cast<size_t>(dim - s1)) xsave.alloc(dim - s1);
    zcopy(ctx, xsave.p, r.p + s1, dim - s1);
    run_step(st, true, z);
    exchange_deltas(ctx, xbuf, {{z + s0, nullptr, s1 - s0}, {r.p + s1, xsave.p, dim - s1}});
  } else {
    if (xsave.n < static_cast<size_t>(s1 - s0)) xsave.alloc(s1 - s0);
    zcopy(ctx, xsave.p, z + s0, s1 - s0);
    run_step(st, false, z);
    exchange_deltas(ctx, xbuf, {{z + s0, xsave.p, s1 - s0}});
  }
}

void Precond::run_global_sharded(bool down, double2* z) {
  const int last_local = h->sk->el->part.last_local;
  for (const Step& st : down ? down_steps : up_steps)
    if (st.level > last_local) run_global_level(st, down, z);
}

void precond_apply(Precond* p, const double2* v_dev, double2* z_dev, bool distributed) {
  Context* ctx = p->ctx;
  const int vblocks = static_cast<int>(std::min<int64_t>((p->dim + 255) / 256, 8 * ctx->num_sms));
  launch_k(ctx, copy_vec_kernel, dim3(vblocks), dim3(256), 0, 1, p->r.p, v_dev, p->dim);
  if (!p->cfg.exact_coarse && p->cfg.gamma > 1) {
    apply_level_gamma(p, 1, z_dev);
    if (ctx->world() > 1 && !distributed) gather_distributed(p->h->sk, z_dev);
    return;
  }
  // `out` of the plans is bound to the caller's z: no copy-out.
  p->run_steps(true, false, z_dev);  // local levels, down
  const bool sharded = ctx->world() > 1;
  if (sharded) {
    // Only global rows (the tail) were changed by more than one rank's
    // subtree, each by at most one: r_tail = v_tail + sum_ranks (r_rank - v)_tail.
    const int64_t t0 = p->tail_off;
    exchange_deltas(ctx, p->xbuf, {{p->r.p + t0, v_dev + t0, p->dim - t0}});
    HPSB_CUDA(cudaMemsetAsync(z_dev + t0, 0, sizeof(double2) * (p->dim - t0), ctx->stream));
    p->run_global_sharded(true, z_dev);  // top (global) levels, down: owner-computes
  } else {
    p->run_steps(true, true, z_dev);
  }
  run_coarse(p, z_dev);  // replicated on every rank (identical inputs)
  if (sharded) p->run_global_sharded(false, z_dev);
  else p->run_steps(false, true, z_dev);
  p->run_steps(false, false, z_dev);
  // distributed: each rank's own (local-face) rows and the global rows are
  // valid -- what the sharded FGMRES consumes; else the full vector
  if (sharded && !distributed) gather_distributed(p->h->sk, z_dev);
}

namespace {
// Multi-RHS phases from the single-RHS item lists: every vector operand is
// mapped to its R-column block (r -> rB, tmp -> tmpB, coarse cv / cw -> their
// blocks); `out` stays as the rebinding marker of the caller's output block.
void build_batch(Precond* p) {
  Context* ctx = p->ctx;
  const int Rm = kBatchMaxRhs;
  const int64_t dim = p->dim, nd = p->dim_d;
  const int ci = p->cfg.exact_coarse ? 0 : p->cfg.coarse_iters;
  p->rB.alloc(static_cast<size_t>(Rm) * dim);
  p->tmpB.alloc(static_cast<size_t>(Rm) * p->tmp_total);
  p->VB.alloc(static_cast<size_t>(Rm) * (ci + 1) * nd);
  p->cvB.alloc(static_cast<size_t>(Rm) * nd);
  p->cwB.alloc(static_cast<size_t>(Rm) * nd);
  p->HmB.alloc(static_cast<size_t>(Rm) * (ci + 1) * std::max(ci, 1));
  p->gvB.alloc(static_cast<size_t>(Rm) * (ci + 1));
  p->rsB.alloc(static_cast<size_t>(Rm) * std::max(ci, 1));
  p->rcB.alloc(static_cast<size_t>(Rm) * std::max(ci, 1));
  p->stateB.alloc(static_cast<size_t>(Rm) * 4);
  auto map = [&](const double2* ptr, int& ld) -> const double2* {
    if (!ptr) return nullptr;
    if (ptr >= p->r.p && ptr < p->r.p + dim) return ld = static_cast<int>(dim), p->rB.p + (ptr - p->r.p);
    if (ptr >= p->out.p && ptr < p->out.p + dim) return ld = static_cast<int>(dim), ptr;
    if (ptr >= p->tmp.p && ptr < p->tmp.p + p->tmp_total)
      return ld = static_cast<int>(p->tmp_total), p->tmpB.p + (ptr - p->tmp.p);
    if (ptr >= p->cv.p && ptr < p->cv.p + nd) return ld = static_cast<int>(nd), p->cvB.p + (ptr - p->cv.p);
    if (ptr >= p->cw.p && ptr < p->cw.p + nd) return ld = static_cast<int>(nd), p->cwB.p + (ptr - p->cw.p);
    throw std::logic_error("batch: unmapped vector operand");
  };
  auto conv = [&](const VItem& it) {
    BDesc d{};
    d.A = it.A, d.lda = it.lda, d.M = it.rows, d.K = it.A ? it.cols : 0;
    d.B = d.K ? map(it.x, d.ldb) : nullptr, d.bidx = d.K ? it.xi : nullptr;
    d.C = const_cast<double2*>(map(it.y, d.ldc)), d.cidx = it.yi;
    d.Z = it.gamma != 0.0 ? map(it.z, d.ldz) : nullptr, d.zidx = it.gamma != 0.0 ? it.zi : nullptr;
    d.alpha = it.alpha, d.beta = it.beta, d.gamma = it.gamma;
    return d;
  };
  auto phase_of = [&](const std::vector<VItem>& items) {
    BPhase ph;
    for (const VItem& it : items) ph.add(conv(it));
    ph.finalize(ctx->stream);
    return ph;
  };
  const bool lv = std::getenv("HPSB_PROFILE_LEVELS") != nullptr;
  for (int l = 1; l < p->cfg.depth; ++l)
    for (int k = 0; k < 4; ++k) {
      p->bdown.push_back(phase_of(p->stage_items[0][l][k]));
      if (lv) p->bdown.back().label = "vcycle_down_batch_L" + std::to_string(l);
    }
  for (int l = p->cfg.depth - 1; l >= 1; --l)
    for (int k = 0; k < 4; ++k) {
      p->bup.push_back(phase_of(p->stage_items[1][l][k]));
      if (lv) p->bup.back().label = "vcycle_up_batch_L" + std::to_string(l);
    }
  if (p->cfg.exact_coarse) {
    for (const VPhase& vp : p->exact_mv.phases) {
      std::vector<VItem> items;
      for (int u = vp.unit_begin; u < vp.unit_begin + vp.unit_count; ++u)
        for (int it = p->exact_mv.units[u].first;
             it < p->exact_mv.units[u].first + p->exact_mv.units[u].count; ++it)
          items.push_back(p->exact_mv.items[it]);
      p->bexact.push_back(phase_of(items));
    }
  } else {
    p->bcoarse = phase_of(p->coarse_mv.items);
  }
  HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
  p->batch_ready = true;
}
}  // namespace

void precond_apply_batch(Precond* p, const double2* v, double2* z, int R, bool distributed) {
  Context* ctx = p->ctx;
  if (R < 1 || R > kBatchMaxRhs) throw InvalidArgument("precond_apply: 1 <= nrhs <= 32");
  if (!p->cfg.exact_coarse && p->cfg.gamma > 1)
    throw InvalidArgument("precond_apply: multi-RHS runs gamma = 1");
  if (!p->batch_ready) build_batch(p);
  const int64_t dim = p->dim, nd = p->dim_d;
  HPSB_CUDA(cudaMemcpyAsync(p->rB.p, v, sizeof(double2) * R * dim, cudaMemcpyDeviceToDevice,
                            ctx->stream));
  BBind bind;
  bind.from[0] = p->out.p, bind.to[0] = z;
  // levels of small merges: the fused per-merge chain when its R-wide
  // vectors fit in shared memory, else the level's four GEMM phases
  auto small_fits = [&](int l) {
    const int si = p->small_level_of[l];
    return si >= 0 && p->smalls[si]->batch_smem(R) <= (200u << 10);
  };
  const int depth = p->cfg.depth;
  auto level = [&](int l, bool down) {
    if (small_fits(l)) {
      p->smalls[p->small_level_of[l]]->run_batch(ctx, down, p->rB.p, z, R, dim);
      return;
    }
    for (int k = 0; k < 4; ++k) {
      if (down) p->bdown[(l - 1) * 4 + k].run(ctx, R, "vcycle_down_batch", bind);
      else p->bup[(depth - 1 - l) * 4 + k].run(ctx, R, "vcycle_up_batch", bind);
    }
  };
  // Sharded: the single-RHS exchanges (precond_apply) on R columns at once.
  const bool sharded = ctx->world() > 1;
  const int last_local = sharded ? p->h->sk->el->part.last_local : depth;
  const int bs = p->h->sk->bs;
  const auto& g = p->h->sk->graph;
  auto ff = [&](int l) { return static_cast<int64_t>(g.level_range[l - 1].first) * bs; };
  auto save = [&](const double2* src, int64_t rows) {
    if (p->xsave.n < static_cast<size_t>(rows) * R) p->xsave.alloc(static_cast<size_t>(rows) * R);
    HPSB_CUDA(cudaMemcpy2DAsync(p->xsave.p, rows * sizeof(double2), src, dim * sizeof(double2),
                                rows * sizeof(double2), R, cudaMemcpyDeviceToDevice, ctx->stream));
  };
  for (int l = 1; l < depth && l <= last_local; ++l) level(l, true);
  if (sharded) {
    const int64_t t0 = p->tail_off;
    exchange_deltas(ctx, p->xbuf, {{p->rB.p + t0, v + t0, dim - t0, R, dim, dim}});
    HPSB_CUDA(cudaMemset2DAsync(z + t0, dim * sizeof(double2), 0, (dim - t0) * sizeof(double2), R,
                                ctx->stream));
    for (int l = last_local + 1; l < depth; ++l) {
      const int64_t s0 = ff(l), s1 = ff(l + 1);
      save(p->rB.p + s1, dim - s1);
      level(l, true);
      exchange_deltas(ctx, p->xbuf, {{z + s0, nullptr, s1 - s0, R, dim, 0},
                                     {p->rB.p + s1, p->xsave.p, dim - s1, R, dim, dim - s1}});
    }
  }
  if (p->cfg.exact_coarse) {
    for (const BPhase& ph : p->bexact) ph.run(ctx, R, "coarse_exact_batch", bind);
  } else {
    const int ci = p->cfg.coarse_iters;
    launch_k(ctx, coarse_init_kernel, dim3(R), dim3(kCoarseThreads), 0, 1,
             static_cast<const double2*>(p->rB.p + p->off_d), nd, p->VB.p, p->cvB.p, p->gvB.p, ci,
             p->stateB.p, dim);
    for (int j = 0; j < ci; ++j) {
      p->bcoarse.run(ctx, R, "coarse_matvec_batch");
      launch_k(ctx, coarse_step_kernel, dim3(R), dim3(kCoarseThreads), 0, 1, j, nd, ci, p->VB.p,
               p->cvB.p, p->cwB.p, p->HmB.p, p->gvB.p, p->rcB.p, p->rsB.p, p->stateB.p, dim);
    }
    launch_k(ctx, coarse_finish_kernel, dim3(R), dim3(kCoarseThreads), 0, 1, nd, ci,
             static_cast<const double2*>(p->VB.p), static_cast<const double2*>(p->HmB.p),
             static_cast<const double2*>(p->gvB.p), static_cast<const double*>(p->stateB.p),
             z + p->off_d, dim);
  }
  if (sharded)
    for (int l = depth - 1; l > last_local; --l) {
      const int64_t s0 = ff(l), s1 = ff(l + 1);
      save(z + s0, s1 - s0);
      level(l, false);
      exchange_deltas(ctx, p->xbuf, {{z + s0, p->xsave.p, s1 - s0, R, dim, s1 - s0}});
    }
  for (int l = std::min(depth - 1, last_local); l >= 1; --l) level(l, false);
  if (sharded && !distributed) gather_distributed(p->h->sk, z, R);
}

int64_t precond_bytes(const Precond* p) { return p->bytes_per_apply; }

double precond_pinned_bytes(const Precond* p) {
  // 16 [nnz(M_1) + sum_l (2 LU_l + B_l + C_l) + ci nnz(M_depth)]
  const Skeleton* sk = p->h->sk;
  const int nb = sk->el->nb, ne = sk->el->n * sk->el->n;
  double m1 = 0;
  for (int e = 0; e < ne; ++e) {
    double k = 0;
    for (int b = 0; b < nb; ++b) k += sk->h_in[static_cast<size_t>(e) * nb + b] >= 0;
    m1 += k * k;
  }
  double levels = 0;
  hierarchy_pinned(p->h, nullptr, nullptr, &levels);
  double coarse = 0;
  for (const ChildBox& c : p->h->levels[p->cfg.depth - 1]->children)
    coarse += static_cast<double>(c.P) * c.P;
  if (p->cfg.exact_coarse) return 16.0 * (m1 + levels + double(p->dim_d) * p->dim_d);
  return 16.0 * (m1 + levels + p->cfg.coarse_iters * coarse);
}

void precond_apply_host(Precond* p, const double2* v, double2* z) {
  Context* ctx = p->ctx;
  DevBuf<double2> vd(p->dim), zd(p->dim);
  HPSB_CUDA(cudaMemcpyAsync(vd.p, v, vd.bytes(), cudaMemcpyHostToDevice, ctx->stream));
  precond_apply(p, vd.p, zd.p);
  HPSB_CUDA(cudaMemcpyAsync(z, zd.p, zd.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
  HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace hpsb
