#include <mutex>
// K1 element_iti: batched local impedance-to-impedance build.
//
// Replaces ElementOperators (proj/src/element.cpp:127-160) + source_to_outgoing
// (:167-174), batched over the mesh as build_elements (proj/src/mesh.cpp:36-109).
// Instead of the reference's complex LU of the full corner-free operator L
// (t x t), the kernel uses the identity
//     T = I - 2 i eta (L^{-1})_GG,   (L^{-1})_GG = S^{-1},
//     S = L_GG - L_Gi L_ii^{-1} L_iG,
//     H = -2 i eta (L^{-1}[0; b~])_G = 2 i eta S^{-1} L_Gi L_ii^{-1} b~,
// where L_ii = Kx(x)My + Mx(x)Ky - diag(c) Mx(x)My on the interior nodes is
// real symmetric positive definite for the configs (Appendix B.2).  Per
// element: real Cholesky of L_ii (ni = (N-1)^2), two triangular solves with
// nb + 2 right-hand sides (nb = 4(N-1)), the sparse boundary rows, and a
// complex nb x nb Gauss-Jordan inverse.
//
// Data layout: coeff[e][(N+1)^2] real c = kappa^2 (1 - b); source[e][ni]
// complex samples of s; T[e] nb x nb complex column-major in the boundary
// order left|right|bottom|top; H[e] nb complex.
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"
#include "linalg.cuh"
#include "internal.hpp"
#include "element_common.cuh"

namespace hpsb {

namespace {

// v1 / fallback: unblocked right-looking Cholesky (pivoted LU when L_ii is
// indefinite) on the element's workspace.  Processes a.elist when given.
__global__ void __launch_bounds__(kThreads) element_kernel(ElemArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int m = a.m, ni = a.ni, nb = a.nb, np = a.order + 1, N = a.order;
  const int ncol = nb + 2;
  double2* S = reinterpret_cast<double2*>(smem_raw);       // nb*nb
  double2* f = S + nb * nb;                                // nb
  double* colk = reinterpret_cast<double*>(f + nb);        // ni
  double* mass = colk + ni;                                // np
  int* perm = reinterpret_cast<int*>(mass + np);           // nb
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_fail;

  double* Lii = a.ws + blockIdx.x * a.ws_stride;  // ni*ni
  double* Y = Lii + static_cast<size_t>(ni) * ni;   // ni*ncol

  for (int i = tid; i < np; i += blockDim.x) mass[i] = a.mass[i];
  auto K = [&](int r, int c) { return __ldg(a.stiff + r + c * np); };
  const int count = a.elist ? (a.nlist_dev ? *a.nlist_dev : a.nlist) : a.ne;

  for (int ii = blockIdx.x; ii < count; ii += gridDim.x) {
    const int e = a.elist ? a.elist[ii] : ii;
    __syncthreads();
    if (tid == 0) s_fail = 0;
    const double* ce = a.coeff + static_cast<size_t>(e) * np * np;
    // 1. interior block L_ii (element.cpp:57-90 restricted to interior nodes)
    auto assemble_lii = [&]() {
      for (int idx = tid; idx < ni * ni; idx += blockDim.x) {
        const int r = idx % ni, c = idx / ni;
        const int i = r / m + 1, j = r % m + 1, k = c / m + 1, l = c % m + 1;
        double v = 0.0;
        if (j == l) v += K(i, k) * mass[j];
        if (i == k) v += mass[i] * K(j, l);
        if (r == c) v -= __ldg(ce + i * np + j) * mass[i] * mass[j];
        Lii[idx] = v;
      }
    };
    assemble_lii();
    // 2. right-hand sides [L_iG | re b~ | im b~]
    for (int idx = tid; idx < ni * ncol; idx += blockDim.x) {
      const int q = idx % ni, b = idx / ni;
      const int i = q / m + 1, j = q % m + 1;
      double v = 0.0;
      if (b < nb) {
        const int side = b / m, t = b % m + 1;
        switch (side) {
          case 0: v = (j == t) ? K(i, 0) * mass[j] : 0.0; break;
          case 1: v = (j == t) ? K(i, N) * mass[j] : 0.0; break;
          case 2: v = (i == t) ? mass[i] * K(j, 0) : 0.0; break;
          default: v = (i == t) ? mass[i] * K(j, N) : 0.0; break;
        }
      } else if (a.source) {
        const double2 s = a.source[static_cast<size_t>(e) * ni + q];
        const double w = mass[i] * mass[j];
        v = (b == nb) ? s.x * w : s.y * w;
      }
      Y[idx] = v;
    }
    __syncthreads();
    // 3. Cholesky L_ii = R R^T (lower, in place), right-looking
    for (int k = 0; k < ni; ++k) {
      if (tid == 0) {
        const double d = Lii[k + k * ni];
        if (!(d > 0.0)) s_fail = 1;
        Lii[k + k * ni] = sqrt(fmax(d, 1e-300));
      }
      __syncthreads();
      const double inv = 1.0 / Lii[k + k * ni];
      for (int i = k + 1 + tid; i < ni; i += blockDim.x) {
        const double v = Lii[i + k * ni] * inv;
        Lii[i + k * ni] = v;
        colk[i] = v;
      }
      __syncthreads();
      const int rem = ni - k - 1;
      for (int idx = tid; idx < rem * rem; idx += blockDim.x) {
        const int i = k + 1 + idx % rem, j = k + 1 + idx / rem;
        if (j <= i) Lii[i + j * ni] -= colk[i] * colk[j];
      }
      __syncthreads();
      if (s_fail) break;  // indefinite: fall back to pivoted LU below
    }
    __syncthreads();
    if (s_fail) {
      // Pivoted-LU fallback for an indefinite L_ii (c h^2 above the first
      // Dirichlet eigenvalue): P L_ii = L U with
      // partial pivoting, the row swaps applied to the right-hand sides.
      assemble_lii();
      __syncthreads();
      if (tid == 0) s_fail = 0;
      for (int k = 0; k < ni; ++k) {
        double best = -1.0;
        int bi = k;
        for (int i = k + tid; i < ni; i += blockDim.x) {
          const double v = fabs(Lii[i + k * ni]);
          if (v > best) best = v, bi = i;
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > best || (ov == best && oi < bi)) best = ov, bi = oi;
        }
        if ((tid & 31) == 0) red_v[tid >> 5] = best, red_i[tid >> 5] = bi;
        __syncthreads();
        if (tid == 0) {
          double b = -1.0;
          int p = k;
          for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            if (red_v[w] > b || (red_v[w] == b && red_i[w] < p)) b = red_v[w], p = red_i[w];
          perm[0] = p;
          if (!(b > 0.0)) s_fail = 2;
        }
        __syncthreads();
        const int p = perm[0];
        if (p != k) {
          for (int j = tid; j < ni; j += blockDim.x) {
            const double t = Lii[k + j * ni];
            Lii[k + j * ni] = Lii[p + j * ni];
            Lii[p + j * ni] = t;
          }
          for (int c = tid; c < ncol; c += blockDim.x) {
            const double t = Y[k + c * ni];
            Y[k + c * ni] = Y[p + c * ni];
            Y[p + c * ni] = t;
          }
        }
        __syncthreads();
        const double piv = Lii[k + k * ni];
        const double inv = piv != 0.0 ? 1.0 / piv : 0.0;
        for (int i = k + 1 + tid; i < ni; i += blockDim.x) {
          const double v = Lii[i + k * ni] * inv;
          Lii[i + k * ni] = v;
          colk[i] = v;
        }
        __syncthreads();
        const int rem = ni - k - 1;
        for (int idx = tid; idx < rem * rem; idx += blockDim.x) {
          const int i = k + 1 + idx % rem, j = k + 1 + idx / rem;
          Lii[i + j * ni] -= colk[i] * Lii[k + j * ni];
        }
        __syncthreads();
      }
      for (int k = 0; k < ni; ++k) {  // unit-lower forward substitution
        const int rem = ni - k - 1;
        for (int idx = tid; idx < rem * ncol; idx += blockDim.x) {
          const int i = k + 1 + idx % rem, c = idx / rem;
          Y[i + c * ni] -= Lii[i + k * ni] * Y[k + c * ni];
        }
        __syncthreads();
      }
      for (int k = ni - 1; k >= 0; --k) {  // upper back substitution
        const double d = Lii[k + k * ni];
        const double inv = d != 0.0 ? 1.0 / d : 0.0;
        for (int c = tid; c < ncol; c += blockDim.x) Y[k + c * ni] *= inv;
        __syncthreads();
        for (int idx = tid; idx < k * ncol; idx += blockDim.x) {
          const int i = idx % k, c = idx / k;
          Y[i + c * ni] -= Lii[i + k * ni] * Y[k + c * ni];
        }
        __syncthreads();
      }
    } else {
    // 4. solve R R^T Y = B
    for (int k = 0; k < ni; ++k) {
      const double inv = 1.0 / Lii[k + k * ni];
      for (int c = tid; c < ncol; c += blockDim.x) Y[k + c * ni] *= inv;
      __syncthreads();
      const int rem = ni - k - 1;
      for (int idx = tid; idx < rem * ncol; idx += blockDim.x) {
        const int i = k + 1 + idx % rem, c = idx / rem;
        Y[i + c * ni] -= Lii[i + k * ni] * Y[k + c * ni];
      }
      __syncthreads();
    }
    for (int k = ni - 1; k >= 0; --k) {
      const double inv = 1.0 / Lii[k + k * ni];
      for (int c = tid; c < ncol; c += blockDim.x) Y[k + c * ni] *= inv;
      __syncthreads();
      for (int idx = tid; idx < k * ncol; idx += blockDim.x) {
        const int i = idx % k, c = idx / k;
        Y[i + c * ni] -= Lii[k + i * ni] * Y[k + c * ni];
      }
      __syncthreads();
    }
    }
    __syncthreads();
    keep_interior(a, e, Y, ni);
    const bool ok = iti_epilogue(a, e, Y, ni, S, f, perm, red_v, red_i);
    if (tid == 0) a.status[e] = (s_fail ? 1 : 0) | (ok ? 0 : 2);  // 1: singular L_ii
  }
}

}  // namespace

namespace {
// status bit 4 (indefinite interior block: redo with the pivoted LU) -> list
// every element of the stage (or of a.elist) -> the pivoted-LU kernel
__global__ void mark_all_kernel(int* status, const int* elist, int count) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
    status[elist ? elist[i] : i] |= 4;
}
__global__ void collect_redo_kernel(const int* __restrict__ status, int ne, int* list, int* count) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x)
    if (status[e] & 4) list[atomicAdd(count, 1)] = e;
}
}  // namespace

std::unique_ptr<Elements> build_elements(Context* ctx, int n, int order, double eta,
                                         const double* coeff_dev, const double2* source_dev) {
  if (n < 2 || (n & (n - 1)) != 0)
    throw InvalidArgument("Mesh: elements per side must be a power of two >= 2");
  if (order < 2) throw InvalidArgument("Mesh: degree must be >= 2");
  if (!(eta > 0.0)) throw InvalidArgument("Mesh: kappa and eta must be positive");
  auto el = std::make_unique<Elements>();
  el->ctx = ctx;
  el->n = n, el->order = order, el->m = order - 1, el->nb = 4 * (order - 1);
  el->eta = eta, el->h = 1.0 / n;
  const int ne = n * n, np = order + 1, m = order - 1, ni = m * m, nb = 4 * m;

  // 1-D operators on the element edge (proj/src/spectral.cpp:89-98).
  const Gll g = gll_rule(order);
  const double h = el->h;
  std::vector<double> mass(np), diff(np * np), stiff(np * np, 0.0);
  for (int i = 0; i < np; ++i) mass[i] = (0.5 * h) * g.weights[i];
  for (int k = 0; k < np * np; ++k) diff[k] = (2.0 / h) * g.diff[k];
  for (int j = 0; j < np; ++j)
    for (int i = 0; i < np; ++i) {
      double s = 0.0;
      for (int q = 0; q < np; ++q) s += (diff[q + i * np] * mass[q]) * diff[q + j * np];
      stiff[i + j * np] = s;
    }
  DevBuf<double> d_mass, d_diff, d_stiff;
  d_mass.upload(mass, ctx->stream);
  d_diff.upload(diff, ctx->stream);
  d_stiff.upload(stiff, ctx->stream);

  el->T.alloc(static_cast<size_t>(ne) * nb * nb);
  el->H.alloc(static_cast<size_t>(ne) * nb);
  el->status.alloc(ne);
  el->Y.alloc(static_cast<size_t>(ne) * ni * (nb + 2));
  HPSB_CUDA(cudaMemsetAsync(el->status.p, 0, ne * sizeof(int), ctx->stream));
  // Sharded (one rank per GPU): build only this rank's quadtree subtree.
  el->part = make_partition(build_face_graph(n), ctx->world(), ctx->rank());
  DevBuf<int> d_own;
  const bool sharded = ctx->world() > 1;
  if (sharded) {
    HPSB_CUDA(cudaMemsetAsync(el->T.p, 0, el->T.bytes(), ctx->stream));
    HPSB_CUDA(cudaMemsetAsync(el->H.p, 0, el->H.bytes(), ctx->stream));
    d_own.upload(el->part.own_elems, ctx->stream);
  }
  const int nwork = sharded ? static_cast<int>(el->part.own_elems.size()) : ne;

  ElemArgs a{};
  a.ne = ne, a.order = order, a.m = m, a.ni = ni, a.nb = nb, a.eta = eta;
  a.mass = d_mass.p, a.diff = d_diff.p, a.stiff = d_stiff.p;
  a.coeff = coeff_dev, a.source = source_dev;
  a.T = el->T.p, a.H = el->H.p, a.status = el->status.p, a.Y = el->Y.p;
  a.npad = (ni + 15) / 16 * 16;
  a.nbc = (nb + 2 + 7) / 8 * 8;
  if (sharded) a.elist = d_own.p, a.nlist = nwork;

  // v5: batched blocked Cholesky over element chunks (element_v5.cu).  Orders
  // it does not cover (N + 1 > 64 or 4 (N - 1) > 96) run every element through
  // the pivoted-LU kernel below.
  DevBuf<double> ws;
  HPSB_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  if (!element_v5_build(ctx, a, nwork)) {
    mark_all_kernel<<<std::max(1, std::min((nwork + 255) / 256, 4 * ctx->num_sms)), 256, 0,
                      ctx->stream>>>(el->status.p, a.elist, nwork);
    HPSB_LAUNCHED(ctx);
  }
  // Pivoted-LU fallback (v1) for elements whose interior block is
  // indefinite (status bit 4), without a host round trip: the flagged
  // elements are listed on the device and the v1 launch reads the count.
  {
    DevBuf<int> d_redo(ne + 1);
    HPSB_CUDA(cudaMemsetAsync(d_redo.p + ne, 0, sizeof(int), ctx->stream));
    collect_redo_kernel<<<std::max(1, std::min((ne + 255) / 256, 4 * ctx->num_sms)), 256, 0,
                          ctx->stream>>>(el->status.p, ne, d_redo.p, d_redo.p + ne);
    HPSB_LAUNCHED(ctx);
    const int slots = std::min(ne, ctx->num_sms);
    const size_t stride = static_cast<size_t>(ni) * ni + static_cast<size_t>(ni) * (nb + 2);
    ws.alloc(stride * slots);
    a.ws = ws.p, a.ws_stride = stride;
    a.elist = d_redo.p, a.nlist = ne, a.nlist_dev = d_redo.p + ne;
    const size_t smem = sizeof(double2) * (nb * nb + nb) + sizeof(double) * (ni + np) +
                        sizeof(int) * nb + 16;
    int smem_max = 0;
    HPSB_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    if (smem + 1024 > static_cast<size_t>(smem_max))
      throw InvalidArgument("build_elements: order " + std::to_string(order) +
                            " exceeds the element kernels' shared-memory limit (N <= 25)");
    allow_smem<element_kernel>(smem);
    KernelScope ks(ctx, "element_iti_lu", 0.0, 0.0);
    element_kernel<<<slots, kThreads, smem, ctx->stream>>>(a);
    HPSB_LAUNCHED(ctx);
    // h_status[ne] = number of elements the fallback redid
    el->h_status = pinned_ints_acquire(ne + 1, &el->h_status_cap);
    HPSB_CUDA(cudaMemcpyAsync(el->h_status, el->status.p, ne * sizeof(int),
                              cudaMemcpyDeviceToHost, ctx->stream));
    HPSB_CUDA(cudaMemcpyAsync(el->h_status + ne, d_redo.p + ne, sizeof(int),
                              cudaMemcpyDeviceToHost, ctx->stream));
  }
  HPSB_CUDA(cudaEventCreateWithFlags(&el->done, cudaEventDisableTiming));
  HPSB_CUDA(cudaEventRecord(el->done, ctx->stream));
  el->pending = true;
  return el;
}

// Pinned status buffers are recycled, never freed: cudaFreeHost (and often
// cudaMallocHost) synchronises the whole device, which would stall the next
// setup's overlapped pipeline when the previous Elements is released.
namespace {
std::mutex g_pinned_mu;
std::vector<std::pair<int*, size_t>> g_pinned_free;
}  // namespace

int* pinned_ints_acquire(size_t n, size_t* cap) {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    for (size_t i = 0; i < g_pinned_free.size(); ++i)
      if (g_pinned_free[i].second >= n) {
        auto pr = g_pinned_free[i];
        g_pinned_free.erase(g_pinned_free.begin() + i);
        *cap = pr.second;
        return pr.first;
      }
  }
  int* p = nullptr;
  HPSB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p), n * sizeof(int)));
  *cap = n;
  return p;
}

Elements::~Elements() {
  // the status copy behind `done` may still be landing in h_status: wait
  // before the buffer goes back to the pool (another stage could take it)
  if (done && pending) cudaEventSynchronize(done);
  if (done) cudaEventDestroy(done);
  if (h_status) {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    g_pinned_free.emplace_back(h_status, h_status_cap);
  }
}

void elements_wait(Elements* el) {
  if (!el || !el->pending) return;
  HPSB_CUDA(cudaEventSynchronize(el->done));
  el->pending = false;
  const int ne = el->n * el->n;
  el->fallbacks = el->h_status[ne];
  for (int e = 0; e < ne; ++e)
    if (el->h_status[e]) {
      // mesh.cpp:82-84 annotates element failures with the element id.
      throw std::runtime_error("element " + std::to_string(e) + ": " +
                               ((el->h_status[e] & 1) ? "singular interior block"
                                                      : "singular local operator"));
    }
}

}  // namespace hpsb
