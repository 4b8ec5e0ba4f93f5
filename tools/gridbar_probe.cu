// Microbenchmark: cost of a software grid barrier (atomic arrive + generation
// spin) in a cooperative persistent kernel on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (ld_acquire(bar + 1) == gen) {
      }
    }
  }
  __syncthreads();
}

__global__ void probe(unsigned* bar, int iters, double* sink) {
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    acc = acc * 1.0000001 + 1.0;
    grid_barrier(bar, gridDim.x);
  }
  if (acc == -1.0) sink[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* bar;
  double* sink;
  cudaMalloc(&bar, 8);
  cudaMalloc(&sink, 8);
  cudaMemset(bar, 0, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int per : {1, 2, 4}) {
    for (int threads : {256, 512}) {
      int grid = sms * per;
      int iters = 2000;
      void* args[] = {&bar, &iters, &sink};
      cudaLaunchCooperativeKernel((void*)probe, grid, threads, args, 0, 0);
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)probe, grid, threads, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %4d x %3d threads: %.3f us per barrier (%s)\n", grid, threads, 1e3 * ms / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  // launch overhead reference: empty cooperative kernel
  {
    int iters = 0;
    int grid = sms;
    void* args[] = {&bar, &iters, &sink};
    cudaEventRecord(a);
    for (int k = 0; k < 100; ++k) cudaLaunchCooperativeKernel((void*)probe, grid, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("empty cooperative launch: %.3f us each\n", 1e3 * ms / 100);
    cudaEventRecord(a);
    for (int k = 0; k < 100; ++k) probe<<<grid, 256>>>(bar, 0, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("empty regular launch: %.3f us each\n", 1e3 * ms / 100);
  }
  return 0;
}
