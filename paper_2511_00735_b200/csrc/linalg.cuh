// CTA-level dense linear algebra device routines shared by the kernels.
#pragma once

#include "device.cuh"

namespace hpsb {

// Complex Gauss-Jordan inverse with partial pivoting, in place (n x n,
// column-major, leading dimension n), executed by the whole CTA.  Row swaps
// are undone as column swaps at the end.  Returns false if a pivot is 0.
static __device__ __noinline__ bool gj_inverse_cta(double2* A, int n, int* perm, double* red_v, int* red_i) {
  const int tid = threadIdx.x;
  __shared__ int s_piv;
  __shared__ double2 s_inv;
  __shared__ bool s_ok;
  if (tid == 0) s_ok = true;
  for (int k = 0; k < n; ++k) {
    // pivot search in column k, rows k..n-1
    double best = -1.0;
    int bi = k;
    for (int i = k + tid; i < n; i += blockDim.x) {
      const double v = cabs2(A[i + k * n]);
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
      s_piv = p;
      perm[k] = p;
      if (!(b > 0.0)) s_ok = false;
    }
    __syncthreads();
    const int p = s_piv;
    if (p != k)
      for (int j = tid; j < n; j += blockDim.x) {
        const double2 t = A[k + j * n];
        A[k + j * n] = A[p + j * n];
        A[p + j * n] = t;
      }
    __syncthreads();
    if (tid == 0) s_inv = cinv(A[k + k * n]);
    __syncthreads();
    const double2 inv = s_inv;
    for (int j = tid; j < n; j += blockDim.x)
      if (j != k) A[k + j * n] = cmul(A[k + j * n], inv);
    __syncthreads();
    // eliminate column k from all other rows (columns j != k)
    for (int idx = tid; idx < n * n; idx += blockDim.x) {
      const int i = idx % n, j = idx / n;
      if (i == k || j == k) continue;
      A[idx] = csub(A[idx], cmul(A[i + k * n], A[k + j * n]));
    }
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) {
      if (i == k) A[k + k * n] = inv;
      else A[i + k * n] = cmul(make_double2(-A[i + k * n].x, -A[i + k * n].y), inv);
    }
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {
    const int p = perm[k];
    if (p != k)
      for (int i = tid; i < n; i += blockDim.x) {
        const double2 t = A[i + k * n];
        A[i + k * n] = A[i + p * n];
        A[i + p * n] = t;
      }
    __syncthreads();
  }
  return s_ok;
}

}  // namespace hpsb
