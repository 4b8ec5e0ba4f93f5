// K6: restarted flexible GMRES on the skeleton system.
//
// Follows gmres_driver (proj/src/krylov.cpp:45-178) in flexible mode: the
// same cycle / restart / breakdown / true-residual logic, complex Givens
// rotations and convergence test on |g_{j+1}| / ||b||.  The Arnoldi
// orthogonalisation is classical Gram-Schmidt applied twice (CGS2) instead of
// the reference's modified Gram-Schmidt + reorthogonalisation pass: the same
// two passes over the basis, but each pass is one batched dot kernel (V^H w)
// and one batched axpy, so it streams the basis twice per pass instead of
// 2(j+1) dependent dot/axpy launches.  The (restart+1) x restart Hessenberg
// matrix and the Givens rotations live on the host (a few KB); the vectors
// stay in HBM.
#include <algorithm>
#include <cmath>
#include <complex>

#include "device.cuh"
#include "internal.hpp"

namespace hpsb {

namespace {
constexpr int kRowsPerThread = 4;
constexpr int kThreads = 256;
constexpr int kRowsPerBlock = kThreads * kRowsPerThread;

// partial[b * ncols + i] = sum_{rows of block b} conj(V[k, i]) w[k]
__global__ void __launch_bounds__(kThreads) dots_kernel(const double2* __restrict__ V, int64_t ld,
                                                       int ncols, const double2* __restrict__ w,
                                                       int64_t n, double2* partial) {
  __shared__ double2 sh[kThreads / 32][104];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock;
  double2 wv[kRowsPerThread];
#pragma unroll
  for (int r = 0; r < kRowsPerThread; ++r) {
    const int64_t k = base + threadIdx.x + r * kThreads;
    wv[r] = k < n ? w[k] : make_double2(0.0, 0.0);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = 0; i < ncols; ++i) {
    const double2* Vi = V + i * ld;
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < kRowsPerThread; ++r) {
      const int64_t k = base + threadIdx.x + r * kThreads;
      if (k < n) acc = cfma_conj(ldg2(Vi + k), wv[r], acc);
    }
    acc.x = warp_sum(acc.x);
    acc.y = warp_sum(acc.y);
    if (lane == 0) sh[warp][i] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ncols; i += kThreads) {
    double2 s = make_double2(0.0, 0.0);
    for (int q = 0; q < kThreads / 32; ++q) s = cadd(s, sh[q][i]);
    partial[static_cast<int64_t>(blockIdx.x) * ncols + i] = s;
  }
}

// out[0..ncols) = V^H w in one launch: block b reduces rows
// [b*chunk, (b+1)*chunk) into partial[b*ncols + i]; the last block to finish
// (atomic ticket) sums the partials in fixed block order (deterministic).
__global__ void __launch_bounds__(kThreads) dots_fused_kernel(
    const double2* __restrict__ V, int64_t ld, int ncols, const double2* __restrict__ w,
    int64_t n, int64_t chunk, double2* partial, double2* out, unsigned* ticket) {
  __shared__ double2 sh[kThreads / 32][104];
  __shared__ bool last;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = 0; i < ncols; ++i) {
    const double2* Vi = V + i * ld;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t k = r0 + threadIdx.x; k < r1; k += kThreads)
      acc = cfma_conj(ldg2(Vi + k), __ldcg(w + k), acc);
    acc.x = warp_sum(acc.x);
    acc.y = warp_sum(acc.y);
    if (lane == 0) sh[warp][i] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ncols; i += kThreads) {
    double2 s = make_double2(0.0, 0.0);
    for (int q = 0; q < kThreads / 32; ++q) s = cadd(s, sh[q][i]);
    __stcg(partial + static_cast<int64_t>(blockIdx.x) * ncols + i, s);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = threadIdx.x; i < ncols; i += kThreads) {
    double2 s = make_double2(0.0, 0.0);
    for (unsigned b = 0; b < gridDim.x; ++b) s = cadd(s, __ldcg(partial + b * ncols + i));
    out[i] = s;
  }
  if (threadIdx.x == 0) *ticket = 0;  // ready for the next launch (stream-ordered)
}

// out[i] = sum_b partial[b * ncols + i]  (fixed order: deterministic)
__global__ void reduce_kernel(const double2* __restrict__ partial, int nblocks, int ncols,
                              double2* out) {
  __shared__ double2 sh[256];
  const int i = blockIdx.x;
  double2 s = make_double2(0.0, 0.0);
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x)
    s = cadd(s, partial[static_cast<int64_t>(b) * ncols + i]);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = cadd(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[i] = sh[0];
}

// w[k] += sign * sum_i h[i] V[k, i]
__global__ void __launch_bounds__(kThreads) axpy_kernel(const double2* __restrict__ V, int64_t ld,
                                                       int ncols, const double2* __restrict__ h,
                                                       double sign, double2* w, int64_t n) {
  __shared__ double2 hs[104];
  for (int i = threadIdx.x; i < ncols; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < ncols; ++i) acc = cfma(hs[i], ldg2(V + i * ld + k), acc);
    w[k] = make_double2(w[k].x + sign * acc.x, w[k].y + sign * acc.y);
  }
}

__global__ void scale_kernel(const double2* __restrict__ src, double s, double2* dst, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[k] = make_double2(src[k].x * s, src[k].y * s);
}

// r = b - y
__global__ void sub_kernel(const double2* __restrict__ b, const double2* __restrict__ y, double2* r,
                           int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    r[k] = csub(b[k], y[k]);
}

using cd = std::complex<double>;

struct Givens {
  double c = 1.0;
  cd s{0.0, 0.0};
};
Givens make_givens(cd a, cd b) {  // krylov.cpp:17-31
  Givens g;
  const double na = std::abs(a), nb = std::abs(b);
  if (nb == 0.0) return g;
  const double r = std::hypot(na, nb);
  if (na == 0.0) {
    g.c = 0.0;
    g.s = std::conj(b) / nb;
  } else {
    g.c = na / r;
    g.s = (a / na) * std::conj(b) / r;
  }
  return g;
}
void apply_givens(const Givens& g, cd& a, cd& b) {  // krylov.cpp:33-37
  const cd t = g.c * a + g.s * b;
  b = -std::conj(g.s) * a + g.c * b;
  a = t;
}

struct Work {
  Context* ctx;
  int64_t n;
  int blocks;
  int64_t chunk;
  DevBuf<double2> partial, hdev;
  DevBuf<unsigned> ticket;
  explicit Work(Context* c, int64_t dim, int maxcols) : ctx(c), n(dim) {
    blocks = static_cast<int>((dim + kRowsPerBlock - 1) / kRowsPerBlock);
    chunk = kRowsPerBlock;
    partial.alloc(static_cast<size_t>(blocks) * maxcols);
    hdev.alloc(3 * static_cast<size_t>(maxcols) + 4);
    ticket.alloc(1);
    HPSB_CUDA(cudaMemsetAsync(ticket.p, 0, sizeof(unsigned), c->stream));
  }
  int grid() const { return static_cast<int>(std::min<int64_t>((n + 255) / 256, 8 * ctx->num_sms)); }
  // out[0..ncols) = V^H w.  Short vectors: one launch (last-block reduction);
  // long vectors: many row blocks + a column-parallel reduce launch.
  void dots(const double2* V, int ncols, const double2* w, double2* out) {
    KernelScope ks(ctx, "gmres_dots", 16.0 * n * (ncols + 1), 8.0 * n * ncols);
    if (blocks <= 64) {
      dots_fused_kernel<<<blocks, kThreads, 0, ctx->stream>>>(V, n, ncols, w, n, chunk, partial.p,
                                                              out, ticket.p);
      HPSB_LAUNCHED(ctx);
    } else {
      dots_kernel<<<blocks, kThreads, 0, ctx->stream>>>(V, n, ncols, w, n, partial.p);
      HPSB_LAUNCHED(ctx);
      reduce_kernel<<<ncols, 256, 0, ctx->stream>>>(partial.p, blocks, ncols, out);
      HPSB_LAUNCHED(ctx);
    }
  }
  void axpy(const double2* V, int ncols, const double2* h, double sign, double2* w) {
    KernelScope ks(ctx, "gmres_axpy", 16.0 * n * (ncols + 2), 8.0 * n * ncols);
    axpy_kernel<<<grid(), kThreads, 0, ctx->stream>>>(V, n, ncols, h, sign, w, n);
    HPSB_LAUNCHED(ctx);
  }
  double norm(const double2* w) {
    dots(w, 1, w, hdev.p);
    double2 v;
    HPSB_CUDA(cudaMemcpyAsync(&v, hdev.p, sizeof(v), cudaMemcpyDeviceToHost, ctx->stream));
    HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    return std::sqrt(std::max(v.x, 0.0));
  }
  void scale(const double2* src, double s, double2* dst) {
    KernelScope ks(ctx, "gmres_scale", 32.0 * n, 0.0);
    scale_kernel<<<grid(), 256, 0, ctx->stream>>>(src, s, dst, n);
    HPSB_LAUNCHED(ctx);
  }
  void sub(const double2* b, const double2* y, double2* r) {
    KernelScope ks(ctx, "gmres_sub", 48.0 * n, 0.0);
    sub_kernel<<<grid(), 256, 0, ctx->stream>>>(b, y, r, n);
    HPSB_LAUNCHED(ctx);
  }
};
}  // namespace

hpsb_status fgmres(Skeleton* sk, Precond* pc, const double2* rhs, double2* x,
                   const hpsb_krylov_config& cfg, hpsb_solve_report* rep) {
  if (cfg.restart < 1) throw InvalidArgument("gmres: restart must be >= 1");
  if (cfg.restart > 100) throw InvalidArgument("gmres: restart must be <= 100 on the B200 path");
  if (!(cfg.tol > 0.0 && cfg.tol < 1.0)) throw InvalidArgument("gmres: tol must lie in (0, 1)");
  if (cfg.max_iters < 1) throw InvalidArgument("gmres: max_iters must be >= 1");
  Context* ctx = sk->ctx;
  const int64_t n = sk->dim;
  const int restart = cfg.restart;
  *rep = hpsb_solve_report{};
  Work wk(ctx, n, restart + 2);
  DevBuf<double2> V(static_cast<size_t>(n) * (restart + 1));
  DevBuf<double2> Z(pc ? static_cast<size_t>(n) * restart : 0);
  DevBuf<double2> w(n), tmp(n);
  HPSB_CUDA(cudaEventRecord(ctx->ev[2], ctx->stream));
  HPSB_CUDA(cudaMemsetAsync(x, 0, sizeof(double2) * n, ctx->stream));
  const double bnorm = wk.norm(rhs);
  auto finish_time = [&] {
    HPSB_CUDA(cudaEventRecord(ctx->ev[3], ctx->stream));
    HPSB_CUDA(cudaEventSynchronize(ctx->ev[3]));
    float ms = 0;
    HPSB_CUDA(cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]));
    rep->seconds = ms * 1e-3;
  };
  if (bnorm == 0.0) {
    rep->converged = 1;
    finish_time();
    return HPSB_OK;
  }
  auto true_residual = [&]() {
    skeleton_apply(sk, x, tmp.p);
    wk.sub(rhs, tmp.p, tmp.p);
    return wk.norm(tmp.p) / bnorm;
  };
  std::vector<cd> H(static_cast<size_t>(restart + 1) * restart), gv(restart + 1);
  std::vector<Givens> rot(restart);
  std::vector<double2> hh(2 * (restart + 1) + 1);
  auto Hm = [&](int i, int j) -> cd& { return H[i + static_cast<size_t>(j) * (restart + 1)]; };
  int total = 0;
  bool converged = false;
  while (total < cfg.max_iters && !converged) {
    double beta;
    if (total == 0) {
      zcopy(ctx, tmp.p, rhs, n);
      beta = bnorm;
    } else {
      beta = true_residual() * bnorm;  // r0 = rhs - M x (krylov.cpp:72-73)
    }
    if (beta / bnorm <= cfg.tol) {
      converged = true;
      break;
    }
    wk.scale(tmp.p, 1.0 / beta, V.p);
    std::fill(gv.begin(), gv.end(), cd(0.0, 0.0));
    gv[0] = beta;
    int j = 0;
    bool breakdown = false;
    for (; j < restart && total < cfg.max_iters; ++j, ++total) {
      double2* Vj = V.p + static_cast<size_t>(j) * n;
      if (pc) {
        double2* Zj = Z.p + static_cast<size_t>(j) * n;
        precond_apply(pc, Vj, Zj);
        skeleton_apply(sk, Zj, w.p);
      } else {
        skeleton_apply(sk, Vj, w.p);
      }
      // CGS2: two passes of h = V^H w, w -= V h
      double2* h1 = wk.hdev.p;
      double2* h2 = wk.hdev.p + (j + 1);
      double2* nn = wk.hdev.p + 2 * (j + 1);
      wk.dots(V.p, j + 1, w.p, h1);
      wk.axpy(V.p, j + 1, h1, -1.0, w.p);
      wk.dots(V.p, j + 1, w.p, h2);
      wk.axpy(V.p, j + 1, h2, -1.0, w.p);
      wk.dots(w.p, 1, w.p, nn);
      HPSB_CUDA(cudaMemcpyAsync(hh.data(), wk.hdev.p, sizeof(double2) * (2 * (j + 1) + 1),
                                cudaMemcpyDeviceToHost, ctx->stream));
      HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
      for (int i = 0; i <= j; ++i)
        Hm(i, j) = cd(hh[i].x + hh[j + 1 + i].x, hh[i].y + hh[j + 1 + i].y);
      const double hnext = std::sqrt(std::max(hh[2 * (j + 1)].x, 0.0));
      Hm(j + 1, j) = hnext;
      for (int i = 0; i < j; ++i) apply_givens(rot[i], Hm(i, j), Hm(i + 1, j));
      rot[j] = make_givens(Hm(j, j), Hm(j + 1, j));
      apply_givens(rot[j], Hm(j, j), Hm(j + 1, j));
      apply_givens(rot[j], gv[j], gv[j + 1]);
      const double rel = std::abs(gv[j + 1]) / bnorm;
      if (hnext <= 1e-14 * bnorm) {
        breakdown = true;
        ++j;
        ++total;
        break;
      }
      wk.scale(w.p, 1.0 / hnext, V.p + static_cast<size_t>(j + 1) * n);
      if (rel <= cfg.tol) {
        ++j;
        ++total;
        break;
      }
    }
    if (j > 0) {
      std::vector<cd> y(j);
      for (int i = j - 1; i >= 0; --i) {
        cd s = gv[i];
        for (int k = i + 1; k < j; ++k) s -= Hm(i, k) * y[k];
        y[i] = s / Hm(i, i);
      }
      std::vector<double2> yd(j);
      for (int i = 0; i < j; ++i) yd[i] = make_double2(y[i].real(), y[i].imag());
      HPSB_CUDA(cudaMemcpyAsync(wk.hdev.p, yd.data(), sizeof(double2) * j, cudaMemcpyHostToDevice,
                                ctx->stream));
      wk.axpy(pc ? Z.p : V.p, j, wk.hdev.p, 1.0, x);
      HPSB_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    const double true_rel = true_residual();
    rep->final_residual = true_rel;
    if (true_rel <= cfg.tol) converged = true;
    if (breakdown && !converged) {
      finish_time();
      rep->iterations = total;
      throw std::runtime_error("gmres: numerical breakdown before convergence");
    }
  }
  rep->iterations = total;
  rep->final_residual = true_residual();
  rep->converged = rep->final_residual <= cfg.tol;
  finish_time();
  return rep->converged ? HPSB_OK : HPSB_NO_CONVERGENCE;
}

}  // namespace hpsb
