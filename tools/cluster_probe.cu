// Microbenchmark: thread-block cluster barrier and DSMEM reduction latency.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void bar_only(int iters, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    acc = acc * 1.0000001 + 1.0;
    cl.sync();
  }
  if (acc == -1.0) sink[0] = acc;
}

__global__ void bar_split(int iters, double* sink) {
  // barrier.cluster.arrive.release + wait.acquire written out
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    acc = acc * 1.0000001 + 1.0;
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  if (acc == -1.0) sink[0] = acc;
}

__global__ void reduce_dsmem(int iters, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double part[2];
  const int C = cl.num_blocks();
  double acc = 0;
  int slot = 0;
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) part[slot] = acc + 1.0;
    cl.sync();
    double t = 0;
    for (int q = 0; q < C; ++q) t += *cl.map_shared_rank(&part[slot], q);
    acc = t * 1e-9;
    slot ^= 1;
  }
  cl.sync();
  if (acc == -1.0) sink[0] = acc;
}

__global__ void remote_store(int iters, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double2 buf[512];
  const int C = cl.num_blocks(), me = cl.block_rank();
  double2 v = make_double2(threadIdx.x, 1.0);
  for (int i = 0; i < iters; ++i) {
    if ((threadIdx.x & 31) == 0 && threadIdx.x < 256) {
      for (int q = 0; q < 4; ++q) {
        const int k = (me * 32 + (threadIdx.x >> 5) * 4 + q + i) & 511;
        cl.map_shared_rank(buf, k % C)[k] = v;
      }
    }
    cl.sync();
  }
  if (buf[threadIdx.x].x == -1.0) sink[0] = 1.0;
}

__global__ void local_smem_gemv(int iters, double* sink) {
  // 32 rows x 240 cols, warp per row, smem operands (the coarse matvec shape)
  extern __shared__ double2 A[];
  double2* x = A + 32 * 240;
  for (int k = threadIdx.x; k < 33 * 240; k += blockDim.x) A[k] = make_double2(k * 1e-3, 1.0);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double tot = 0;
  for (int i = 0; i < iters; ++i) {
    for (int r = warp; r < 32; r += 8) {
      double2 acc = make_double2(0.0, 0.0);
      for (int c = lane; c < 240; c += 32) {
        const double2 a = A[r * 240 + c], b = x[c];
        acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
        acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
      }
      for (int o = 16; o > 0; o >>= 1) acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      tot += acc.x;
    }
    __syncthreads();
  }
  if (tot == -1.0) sink[0] = tot;
}

template <class K>
float run(K kernel, int C, int threads, int iters, double* sink) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(threads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, iters, sink);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, kernel, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return 1e3f * ms / iters;
}

int main() {
  double* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(bar_only, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(bar_split, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(reduce_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(remote_store, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int C : {8, 16}) printf("C=%2d  32 remote stores + cl.sync %.3f us\n", C, run(remote_store, C, 256, 5000, sink));
  {
    cudaFuncSetAttribute(local_smem_gemv, cudaFuncAttributeMaxDynamicSharedMemorySize, 33 * 240 * 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    local_smem_gemv<<<1, 256, 33 * 240 * 16>>>(10, sink);
    cudaEventRecord(a);
    local_smem_gemv<<<1, 256, 33 * 240 * 16>>>(2000, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("smem gemv 32x240 warp-per-row: %.3f us (%s)\n", 1e3 * ms / 2000, cudaGetErrorString(cudaGetLastError()));
  }
  for (int C : {2, 4, 8, 16}) {
    printf("C=%2d  cl.sync %.3f us  arrive/wait %.3f us  dsmem-reduce %.3f us  (%s)\n", C,
           run(bar_only, C, 256, 5000, sink), run(bar_split, C, 256, 5000, sink),
           run(reduce_dsmem, C, 256, 5000, sink), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
