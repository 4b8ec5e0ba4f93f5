// Solution recovery: the per-element field from the skeleton solution.
//
// Replaces recover_solution (proj/src/problems.cpp:60-92), which gathers each
// element's incoming impedance data g (skeleton slots on interior faces, the
// physical data t on the domain boundary) and solves the full corner-free
// local system L u = [g; b~] again (Element::solve, element.cpp:176-188).
// Here nothing is refactored.  With S^{-1} = (I - T) / (2 i eta) and
// H = 2 i eta S^{-1} L_Gi L_ii^{-1} b~:
//     u_G = ((I - T) g - H) / (2 i eta),
//     u_i = L_ii^{-1} (b~ - L_iG u_G) = Y_b - Y_G u_G,
// where Y = L_ii^{-1} [L_iG | b~] is what K1 already computed and kept per
// element (Elements::Y).  Two GEMVs per element: HBM bound,
// 16 nb^2 + 8 ni (nb + 2) + 16 t bytes per element.
//
// Output: field[e][t] complex in the corner-free compressed node order
// (comp_of_full, element.cpp:47-53), t = (N+1)^2 - 4, as recover_solution
// returns it.
#include "device.cuh"
#include "internal.hpp"

namespace hpsb {

namespace {
constexpr int kRecThreads = 128;

__global__ void __launch_bounds__(kRecThreads)
    recover_kernel(const double2* __restrict__ T, const double2* __restrict__ H,
                   const double* __restrict__ Y, const int* __restrict__ in_idx,
                   const double2* __restrict__ tside, const double2* __restrict__ x,
                   const int* __restrict__ bpos, const int* __restrict__ ipos, double2* field,
                   int nb, int ni, int t, double eta, const int* __restrict__ elist) {
  extern __shared__ double2 sg[];  // g[nb], uG[nb]
  double2* su = sg + nb;
  const int e = elist ? elist[blockIdx.x] : blockIdx.x;
  const int tid = threadIdx.x;
  const int* in_e = in_idx + static_cast<size_t>(e) * nb;
  for (int b = tid; b < nb; b += blockDim.x) {
    const int k = in_e[b];
    sg[b] = k >= 0 ? x[k] : tside[static_cast<size_t>(e) * nb + b];
  }
  __syncthreads();
  const double2* Te = T + static_cast<size_t>(e) * nb * nb;
  double2* fe = field + static_cast<size_t>(e) * t;
  const double s = 0.5 / eta;  // 1 / (2 i eta) = -i s
  for (int b = tid; b < nb; b += blockDim.x) {
    double2 acc = csub(sg[b], H[static_cast<size_t>(e) * nb + b]);
    for (int c = 0; c < nb; ++c) acc = csub(acc, cmul(__ldg(Te + b + static_cast<size_t>(c) * nb), sg[c]));
    const double2 u = make_double2(s * acc.y, -s * acc.x);
    su[b] = u;
    fe[bpos[b]] = u;
  }
  __syncthreads();
  const double* Ye = Y + static_cast<size_t>(e) * ni * (nb + 2);
  for (int q = tid; q < ni; q += blockDim.x) {
    double re = __ldg(Ye + q + static_cast<size_t>(nb) * ni);
    double im = __ldg(Ye + q + static_cast<size_t>(nb + 1) * ni);
    for (int c = 0; c < nb; ++c) {
      const double y = __ldg(Ye + q + static_cast<size_t>(c) * ni);
      re -= y * su[c].x;
      im -= y * su[c].y;
    }
    fe[ipos[q]] = make_double2(re, im);
  }
}
}  // namespace

void recover_field(const Skeleton* sk, const double2* x_dev, int rhs_index, double2* field_dev) {
  Context* ctx = sk->ctx;
  const Elements* el = sk->el;
  if (rhs_index < 0 || rhs_index >= sk->nrhs)
    throw InvalidArgument("recover: rhs index out of range");
  const int ne = el->n * el->n, nb = el->nb, ni = el->m * el->m, np = el->order + 1;
  const int t = np * np - 4;
  const IndexSets sets = build_index_sets(el->order);
  std::vector<int> bpos(nb), ipos(ni);
  for (int b = 0; b < nb; ++b) bpos[b] = sets.comp_of_full[sets.boundary[b]];
  for (int q = 0; q < ni; ++q) ipos[q] = sets.comp_of_full[sets.interior[q]];
  DevBuf<int> d_b, d_i, d_own;
  d_b.upload(bpos, ctx->stream);
  d_i.upload(ipos, ctx->stream);
  // Sharded: each rank recovers its own elements into a zeroed field; one sum.
  const bool sharded = ctx->world() > 1;
  if (sharded) {
    HPSB_CUDA(cudaMemsetAsync(field_dev, 0, sizeof(double2) * ne * t, ctx->stream));
    d_own.upload(el->part.own_elems, ctx->stream);
  }
  const int nwork = sharded ? static_cast<int>(el->part.own_elems.size()) : ne;
  if (nwork > 0) {
    KernelScope ks(ctx, "recover_field",
                   double(nwork) * (16.0 * nb * nb + 8.0 * ni * (nb + 2) + 16.0 * (t + 2 * nb)),
                   double(nwork) * (8.0 * nb * nb + 4.0 * ni * nb));
    recover_kernel<<<nwork, kRecThreads, 2 * nb * sizeof(double2), ctx->stream>>>(
        el->T.p, el->H.p, el->Y.p, sk->d_in.p,
        sk->tside.p + static_cast<size_t>(rhs_index) * ne * nb, x_dev, d_b.p, d_i.p, field_dev, nb, ni,
        t, el->eta, sharded ? d_own.p : nullptr);
    HPSB_LAUNCHED(ctx);
  }
  if (sharded) ctx->comm->allreduce_sum(field_dev, static_cast<size_t>(ne) * t, ctx);
}

}  // namespace hpsb
