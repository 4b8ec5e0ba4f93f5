// CTA-level dense linear algebra device routines shared by the kernels.
#pragma once

#include "device.cuh"

namespace hpsb {

// Complex Gauss-Jordan inverse with partial pivoting, in place (n x n,
// column-major, leading dimension n), executed by the whole CTA.  Row swaps
// are undone as column swaps at the end.  Returns false if a pivot is 0.
// Per column k: warp 0 finds the pivot (max |a_ik|, lowest index on ties);
// the pivot row is swapped in and scaled; the rank-1 elimination runs with
// columns over warps and rows over lanes (no index division); column k is
// finalised.  Four barriers per column; the closing column swaps are applied
// row-wise by independent threads (one barrier in total).
static __device__ __noinline__ bool gj_inverse_cta(double2* A, int n, int* perm, double* red_v, int* red_i) {
  (void)red_v, (void)red_i;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  __shared__ int s_piv;
  __shared__ double2 s_inv;
  __shared__ bool s_ok;
  if (tid == 0) s_ok = true;
  for (int k = 0; k < n; ++k) {
    if (warp == 0) {
      double best = -1.0;
      int bi = k;
      for (int i = k + lane; i < n; i += 32) {
        const double v = cabs2(A[i + k * n]);
        if (v > best) best = v, bi = i;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) best = ov, bi = oi;
      }
      if (lane == 0) {
        s_piv = bi;
        perm[k] = bi;
        if (!(best > 0.0)) s_ok = false;
        s_inv = cinv(A[bi + k * n]);
      }
    }
    __syncthreads();
    const int p = s_piv;
    const double2 inv = s_inv;
    // swap rows k <-> p and scale row k (its column-k entry stays the pivot)
    for (int j = tid; j < n; j += blockDim.x) {
      const double2 t = A[p + j * n];
      if (p != k) A[p + j * n] = A[k + j * n];
      A[k + j * n] = (j == k) ? t : cmul(t, inv);
    }
    __syncthreads();
    // eliminate column k from every other row (columns j != k)
    for (int j = warp; j < n; j += nwarps) {
      if (j == k) continue;
      const double2 akj = A[k + j * n];
      for (int i = lane; i < n; i += 32)
        if (i != k) A[i + j * n] = csub(A[i + j * n], cmul(A[i + k * n], akj));
    }
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) {
      if (i == k) A[k + k * n] = inv;
      else A[i + k * n] = cmul(make_double2(-A[i + k * n].x, -A[i + k * n].y), inv);
    }
    __syncthreads();
  }
  // undo the row swaps as column swaps, each thread on its own rows
  for (int i = tid; i < n; i += blockDim.x)
    for (int k = n - 1; k >= 0; --k) {
      const int p = perm[k];
      if (p != k) {
        const double2 t = A[i + k * n];
        A[i + k * n] = A[i + p * n];
        A[i + p * n] = t;
      }
    }
  __syncthreads();
  return s_ok;
}

}  // namespace hpsb
