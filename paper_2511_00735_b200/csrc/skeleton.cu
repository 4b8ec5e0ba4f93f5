// Skeleton system: the global ItI interface operator and its right-hand side.
//
// assemble_skeleton (proj/src/skeleton.cpp:88-137) stores M as a std::map of
// bs x bs blocks: identity slot diagonals plus +T couplings.  On the B200 the
// operator is never assembled: M = I + sum_e P_e T_e Q_e^T, where Q_e gathers
// element e's incoming unknowns (its own slot of each interior face) and P_e
// scatters the rows of its outgoing data to the neighbour's incoming slot of
// the same face.  Every skeleton entry is the scatter target of exactly one
// (element, side) pair, so the matvec is conflict-free with no atomics, and
// the operator bytes streamed are exactly the element ItI maps.
#include <algorithm>

#include "device.cuh"
#include "internal.hpp"
#include "vcycle_small.hpp"
#include "zgemv_batch.hpp"

namespace hpsb {

namespace {
// rhs[out_e(alpha)] = -H_e(alpha) - sum_{gamma physical} T_e(alpha, gamma) t_e(gamma)
// (skeleton.cpp:121-132), one CTA per element, one thread per boundary row.
__global__ void skeleton_rhs_kernel(const double2* __restrict__ T, const double2* __restrict__ H,
                                    const int* __restrict__ in_idx, const int* __restrict__ out_idx,
                                    const double2* __restrict__ tside, double2* rhs, int nb,
                                    int64_t dim, int ne, int nrhs, const int* __restrict__ elist) {
  const int e = elist ? elist[blockIdx.x] : blockIdx.x;
  const double2* Te = T + static_cast<size_t>(e) * nb * nb;
  const int* in_e = in_idx + static_cast<size_t>(e) * nb;
  const int* out_e = out_idx + static_cast<size_t>(e) * nb;
  for (int r = 0; r < nrhs; ++r) {
    const double2* t = tside + (static_cast<size_t>(r) * ne + e) * nb;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      const int o = out_e[b];
      if (o < 0) continue;
      double2 v = H[static_cast<size_t>(e) * nb + b];
      v = make_double2(-v.x, -v.y);
      for (int c = 0; c < nb; ++c)
        if (in_e[c] < 0) v = csub(v, cmul(Te[b + static_cast<size_t>(c) * nb], t[c]));
      rhs[static_cast<size_t>(r) * dim + o] = v;
    }
  }
}

// Expand the physical-boundary data tb[r][side][j][m] (boundary_side_data,
// proj/src/mesh.cpp:111-139: per physical side, its n elements in ascending
// order, N-1 nodes each) into the zeroed element layout t[r][e][nb]: side 0
// (x=0) is element side 0 of e = j*n, side 1 (x=1) side 1 of e = j*n+n-1,
// side 2 (y=0) side 2 of e = j, side 3 (y=1) side 3 of e = (n-1)*n+j.
__global__ void tside_expand_kernel(const double2* __restrict__ tb, double2* __restrict__ t, int n,
                                    int m, int nrhs) {
  const int64_t total = static_cast<int64_t>(nrhs) * 4 * n * m;
  const int nb = 4 * m;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % m);
    const int j = static_cast<int>((i / m) % n);
    const int side = static_cast<int>((i / (static_cast<int64_t>(m) * n)) % 4);
    const int64_t r = i / (4LL * n * m);
    const int e = side == 0 ? j * n : side == 1 ? j * n + n - 1 : side == 2 ? j : (n - 1) * n + j;
    t[(r * n * n + e) * nb + side * m + k] = tb[i];
  }
}
}  // namespace

std::unique_ptr<Skeleton> build_skeleton(Elements* el, const double2* tside_host, int nrhs,
                                         bool boundary_only) {
  Context* ctx = el->ctx;
  auto sk = std::make_unique<Skeleton>();
  sk->ctx = ctx;
  sk->el = el;
  sk->graph = build_face_graph(el->n);
  sk->m = el->m;
  sk->bs = 2 * el->m;
  sk->dim = static_cast<int64_t>(sk->graph.num_faces()) * sk->bs;
  sk->nrhs = nrhs;
  const int ne = el->n * el->n, nb = el->nb, m = el->m;
  // Element incoming / outgoing skeleton indices (slot_offset, skeleton.cpp:80-86).
  sk->h_in.assign(static_cast<size_t>(ne) * nb, -1);
  sk->h_out.assign(static_cast<size_t>(ne) * nb, -1);
  for (int e = 0; e < ne; ++e)
    for (int side = 0; side < 4; ++side) {
      const int f = sk->graph.face_of_element[e][side];
      if (f < 0) continue;
      const int own = sk->graph.faces[f].e1 == e ? 1 : 0;
      for (int k = 0; k < m; ++k) {
        sk->h_in[static_cast<size_t>(e) * nb + side * m + k] = f * sk->bs + own * m + k;
        sk->h_out[static_cast<size_t>(e) * nb + side * m + k] = f * sk->bs + (1 - own) * m + k;
      }
    }
  sk->d_in.upload(sk->h_in, ctx->stream);
  sk->d_out.upload(sk->h_out, ctx->stream);

  // Right-hand sides (sharded: each rank adds its elements' rows, then sum).
  const bool sharded = ctx->world() > 1;
  const std::vector<int>& own = el->part.own_elems;
  sk->rhs.alloc(static_cast<size_t>(nrhs) * sk->dim);
  HPSB_CUDA(cudaMemsetAsync(sk->rhs.p, 0, sk->rhs.bytes(), ctx->stream));
  DevBuf<double2>& d_t = sk->tside;  // kept for the solution recovery
  d_t.alloc(static_cast<size_t>(nrhs) * ne * nb);
  if (boundary_only) {
    // Only the 4n physical sides carry data: copy those (cfg4: 5.8 MB instead
    // of the 1.5 GB element layout) and expand on the device.
    DevBuf<double2> d_tb;
    d_tb.alloc(static_cast<size_t>(nrhs) * 4 * el->n * m);
    // through the pinned staging ring: a pageable cudaMemcpyAsync on a busy
    // stream (the element stage may still run) can return before it has
    // consumed the caller's buffer
    staged_upload(d_tb.p, tside_host, d_tb.bytes(), ctx->stream);
    HPSB_CUDA(cudaMemsetAsync(d_t.p, 0, d_t.bytes(), ctx->stream));
    KernelScope ks(ctx, "skeleton_tside", 32.0 * d_tb.n, 0.0);
    tside_expand_kernel<<<std::min<int64_t>((d_tb.n + 255) / 256, 148 * 8), 256, 0,
                          ctx->stream>>>(d_tb.p, d_t.p, el->n, m, nrhs);
    HPSB_LAUNCHED(ctx);
  } else {
    HPSB_CUDA(cudaMemcpyAsync(d_t.p, tside_host, d_t.bytes(), cudaMemcpyHostToDevice,
                              ctx->stream));
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));  // see above; this layout is large
  }
  DevBuf<int> d_own;
  if (sharded) d_own.upload(own, ctx->stream);
  const int nwork = sharded ? static_cast<int>(own.size()) : ne;
  {
    KernelScope ks(ctx, "skeleton_rhs", 16.0 * nwork * nb * nb, 0.0);
    skeleton_rhs_kernel<<<nwork, 64, 0, ctx->stream>>>(el->T.p, el->H.p, sk->d_in.p, sk->d_out.p,
                                                       d_t.p, sk->rhs.p, nb, sk->dim, ne, nrhs,
                                                       sharded ? d_own.p : nullptr);
    HPSB_LAUNCHED(ctx);
  }
  if (sharded) ctx->comm->allreduce_sum(sk->rhs.p, sk->rhs.n, ctx);

  // Matvec plan: one unit per (own) element, y[out] = x[out] + T_e x[in].
  sk->x_buf.alloc(sk->dim);
  sk->y_buf.alloc(sk->dim);
  sk->apply_plan.begin_phase();
  for (int e = 0; e < ne; ++e) {
    if (sharded && !el->part.owns_elem(e)) continue;
    VItem it{};
    it.A = el->T.p + static_cast<size_t>(e) * nb * nb;
    it.lda = nb, it.rows = nb, it.cols = nb;
    it.x = sk->x_buf.p, it.xi = sk->d_in.p + static_cast<size_t>(e) * nb;
    it.z = sk->x_buf.p, it.zi = sk->d_out.p + static_cast<size_t>(e) * nb;
    it.y = sk->y_buf.p, it.yi = sk->d_out.p + static_cast<size_t>(e) * nb;
    it.alpha = 1.0, it.beta = 0.0, it.gamma = 1.0;
    sk->apply_plan.add_unit({it});
  }
  sk->apply_plan.name = "skeleton_matvec";
  sk->apply_plan.finalize(ctx->stream);
  {
    // the same element GEMVs through the TMA-streamed kernel (the plan above
    // stays for the multi-RHS path)
    const GemvStream::Shape shp = gemv_stream_shape(nb, nb);
    if (shp.ok) {
      auto gs = std::make_shared<GemvStream>();
      std::vector<GemvItem> items;
      for (int e = 0; e < ne; ++e) {
        if (sharded && !el->part.owns_elem(e)) continue;
        items.push_back({el->T.p + static_cast<size_t>(e) * nb * nb, sk->d_in.p + static_cast<size_t>(e) * nb,
                         sk->d_out.p + static_cast<size_t>(e) * nb, nb, nb});
      }
      gs->shape = shp;
      gs->count = static_cast<int>(items.size());
      gs->bytes = 16.0 * nb * nb * items.size();
      gs->d.upload(items, ctx->stream);
      sk->apply_stream = gs;
    }
  }
  if (sharded) {
    const Partition& part = el->part;
    sk->tail_off = static_cast<int64_t>(sk->graph.level_range[part.last_local].first) * sk->bs;
    std::vector<int> rows, keep(sk->graph.num_faces());
    for (int f = 0; f < sk->graph.num_faces(); ++f) {
      keep[f] = part.face_owner[f] == ctx->rank() || (part.face_owner[f] < 0 && ctx->rank() == 0);
      if (part.face_owner[f] == ctx->rank())
        for (int k = 0; k < sk->bs; ++k) rows.push_back(f * sk->bs + k);
    }
    for (int64_t i = sk->tail_off; i < sk->dim; ++i)
      rows.push_back(ctx->rank() == 0 ? static_cast<int>(i) : -static_cast<int>(i) - 1);
    sk->n_dist_rows = static_cast<int64_t>(rows.size());
    sk->dist_rows.upload(rows, ctx->stream);
    sk->keep_face.upload(keep, ctx->stream);
  }
  // no synchronisation: buffers are freed stream-ordered, host uploads are
  // staged, and the element stage may still be running (Elements::pending)
  return sk;
}

void skeleton_apply(const Skeleton* sk, const double2* x_dev, double2* y_dev, bool distributed) {
  // The plan was built on x_buf / y_buf; bind the caller's vectors instead.
  Context* ctx = sk->ctx;
  const bool sharded = ctx->world() > 1;
  // Every skeleton row is produced by exactly one rank's element: zero, then
  // sum -- the whole vector, or (distributed) the global rows only: an
  // element reads and writes only its own subtree's rows and the global rows
  // (the subtree boundaries are global-level faces).
  const int64_t z0 = distributed ? sk->tail_off : 0;
  if (sharded)
    HPSB_CUDA(cudaMemsetAsync(y_dev + z0, 0, (sk->dim - z0) * sizeof(double2), ctx->stream));
  if (sk->apply_stream) sk->apply_stream->run(ctx, x_dev, y_dev);
  else sk->apply_plan.run(ctx, sk->x_buf.p, const_cast<double2*>(x_dev), sk->y_buf.p, y_dev);
  if (sharded) ctx->comm->allreduce_sum(y_dev + z0, sk->dim - z0, ctx);
}

namespace {
__global__ void keep_faces_kernel(double2* v, const int* __restrict__ keep, int bs) {
  if (keep[blockIdx.x]) return;
  for (int k = threadIdx.x; k < bs; k += blockDim.x)
    v[static_cast<int64_t>(blockIdx.x) * bs + k] = make_double2(0.0, 0.0);
}
}  // namespace

void gather_distributed(const Skeleton* sk, double2* v, int R) {
  Context* ctx = sk->ctx;
  if (ctx->world() == 1) return;
  for (int b = 0; b < R; ++b) {
    keep_faces_kernel<<<sk->graph.num_faces(), 64, 0, ctx->stream>>>(v + b * sk->dim,
                                                                      sk->keep_face.p, sk->bs);
    HPSB_LAUNCHED(ctx);
  }
  ctx->comm->allreduce_sum(v, static_cast<size_t>(R) * sk->dim, ctx);
}

void skeleton_apply_batch(const Skeleton* sk, const double2* x, double2* y, int R,
                          bool distributed) {
  Context* ctx = sk->ctx;
  const bool sharded = ctx->world() > 1;
  auto* self = const_cast<Skeleton*>(sk);
  if (!self->batch) {
    // Y = X + sum_e scatter(T_e gather(X)): the matvec plan's items as a
    // multi-RHS GEMM phase on the x_buf / y_buf markers.
    auto ph = std::make_shared<BPhase>();
    for (const VItem& it : sk->apply_plan.items) {
      BDesc d{};
      d.A = it.A, d.lda = it.lda, d.M = it.rows, d.K = it.cols;
      d.B = it.x, d.bidx = it.xi, d.ldb = static_cast<int>(sk->dim);
      d.C = it.y, d.cidx = it.yi, d.ldc = static_cast<int>(sk->dim);
      d.Z = it.z, d.zidx = it.zi, d.ldz = static_cast<int>(sk->dim);
      d.alpha = it.alpha, d.beta = it.beta, d.gamma = it.gamma;
      ph->add(d);
    }
    ph->finalize(ctx->stream);
    self->batch = ph;
  }
  // sharded: as skeleton_apply, on R columns (own elements' rows; the rows
  // several ranks produce are zeroed and summed)
  const int64_t z0 = distributed ? sk->tail_off : 0;
  if (sharded)
    HPSB_CUDA(cudaMemset2DAsync(y + z0, sk->dim * sizeof(double2), 0,
                                (sk->dim - z0) * sizeof(double2), R, ctx->stream));
  BBind bind;
  bind.from[0] = sk->x_buf.p, bind.to[0] = const_cast<double2*>(x);
  bind.from[1] = sk->y_buf.p, bind.to[1] = y;
  static_cast<const BPhase*>(sk->batch.get())->run(ctx, R, "skeleton_matvec_batch", bind);
  if (sharded)
    exchange_deltas(ctx, self->gather_buf, {{y + z0, nullptr, sk->dim - z0, R, sk->dim, 0}});
}

}  // namespace hpsb
