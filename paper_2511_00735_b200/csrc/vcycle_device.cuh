// Device helpers shared by the fused V-cycle merge kernels
// (vcycle_small.cu: one CTA per merge; vcycle_cluster.cu: one cluster).
#pragma once

#include "device.cuh"

namespace hpsb {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// y = A x (A in smem, col-major ld lda, rows <= blockDim.x); returns row
// tid's value (zero for tid >= rows).  Column groups split the K loop, the
// partial sums reduce through `red` (blockDim.x double2).  Block-wide: every
// thread must call it.
template <int kThreads>
__device__ double2 smem_gemv(const double2* A, int lda, int rows, int cols, const double2* x,
                             double2* red) {
  const int tid = threadIdx.x;
  const int rpad = rows <= 8 ? 8 : rows <= 16 ? 16 : (rows + 31) & ~31;
  const int groups = kThreads / rpad;
  const int r = tid % rpad, g = tid / rpad;
  double2 acc = make_double2(0.0, 0.0);
  if (g < groups && r < rows)
    for (int j = g; j < cols; j += groups) acc = cfma(A[r + j * lda], x[j], acc);
  double2 s = make_double2(0.0, 0.0);
  if (rpad <= 32) {
    // a warp holds 32 / rpad groups of the same rows: fold them with
    // shuffles, then one partial per warp and row goes through `red`
    const int lane = tid & 31, warp = tid >> 5;
    for (int o = rpad; o < 32; o <<= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane < rpad) red[warp * rpad + lane] = acc;
    __syncthreads();
    if (tid < rows) {
      s = red[tid];
      for (int w = 1; w < kThreads / 32; ++w) s = cadd(s, red[w * rpad + tid]);
    }
  } else {
    red[tid] = acc;
    __syncthreads();
    if (tid < rows) {
      s = red[tid];
      for (int q = 1; q < groups; ++q) s = cadd(s, red[tid + q * rpad]);
    }
  }
  __syncthreads();
  return s;
}

}  // namespace hpsb
