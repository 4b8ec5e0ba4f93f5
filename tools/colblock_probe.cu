// Microbenchmark: HBM read bandwidth of the V-cycle's split-phase access
// pattern (CTA = a block of `rb` consecutive rows of a column-major matrix,
// threads over rows x column groups, 16-byte loads) against a contiguous
// stream of the same bytes.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rows_kernel(const double2* __restrict__ A, int lda, int cols, int rb, double* out) {
  const int rpad = rb <= 8 ? 8 : rb <= 16 ? 16 : (rb + 31) & ~31;
  const int groups = 256 / rpad;
  const int r = threadIdx.x % rpad, g = threadIdx.x / rpad;
  const double2* Ar = A + (size_t)blockIdx.x * rb + r;
  double acc = 0;
  if (r < rb)
    for (int j = g; j < cols; j += 8 * groups) {
      double2 a[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = (j + q * groups < cols) ? __ldg(Ar + (size_t)(j + q * groups) * lda) : make_double2(0, 0);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc += a[q].x + a[q].y;
    }
  if (acc == -1.0) out[0] = acc;
}

// the same with the V-cycle's prologue: gather x (cols entries, through an
// index map) into shared memory before streaming, and multiply by it
__global__ void rows_gather_kernel(const double2* __restrict__ A, int lda, int cols, int rb,
                                   const double2* __restrict__ x, const int* __restrict__ xi,
                                   double* out) {
  extern __shared__ double2 xs[];
  for (int j = threadIdx.x; j < (cols ? cols : lda); j += blockDim.x) xs[j] = __ldcg(x + __ldg(xi + j));
  __syncthreads();
  const int rpad = rb <= 8 ? 8 : rb <= 16 ? 16 : (rb + 31) & ~31;
  const int groups = 256 / rpad;
  const int r = threadIdx.x % rpad, g = threadIdx.x / rpad;
  const double2* Ar = A + (size_t)blockIdx.x * rb + r;
  double acc = 0;
  if (r < rb)
    for (int j = g; j < cols; j += 8 * groups) {
      double2 a[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = (j + q * groups < cols) ? __ldg(Ar + (size_t)(j + q * groups) * lda) : make_double2(0, 0);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (j + q * groups < cols) acc += a[q].x * xs[j + q * groups].x + a[q].y * xs[j + q * groups].y;
    }
  if (acc == -1.0) out[0] = acc;
}

__global__ void contig_kernel(const double2* __restrict__ A, size_t n, double* out) {
  double acc = 0;
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
    const double2 v = __ldg(A + k);
    acc += v.x + v.y;
  }
  if (acc == -1.0) out[0] = acc;
}

int main() {
  const int n = 4864;  // rows = cols (a cfg3 top-level block)
  double2* A;
  double* out;
  cudaMalloc(&A, (size_t)n * n * sizeof(double2));
  cudaMalloc(&out, 8);
  cudaMemset(A, 0, (size_t)n * n * sizeof(double2));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = (double)n * n * 16;
  for (int rb : {8, 16, 32, 64, 128, 256}) {
    const int grid = n / rb;
    rows_kernel<<<grid, 256>>>(A, n, n, rb, out);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) rows_kernel<<<grid, 256>>>(A, n, n, rb, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("row blocks of %3d (%4d CTAs): %7.1f GB/s\n", rb, grid, bytes * 10 / (ms * 1e-3) / 1e9);
  }
  {
    double2* x;
    int* xi;
    cudaMalloc(&x, n * sizeof(double2));
    cudaMalloc(&xi, n * sizeof(int));
    int* hx = new int[n];
    for (int j = 0; j < n; ++j) hx[j] = (j * 7919) % n;
    cudaMemcpy(xi, hx, n * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemset(x, 0, n * sizeof(double2));
    cudaFuncSetAttribute(rows_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, n * 16);
    for (int cols : {n, n / 2, n / 4})
      for (int rb : {8, 16}) {
        const int grid = n / rb;
        const double by = (double)n * cols * 16;
        rows_gather_kernel<<<grid, 256, cols * 16>>>(A, n, cols, rb, x, xi, out);
        cudaEventRecord(a);
        for (int it = 0; it < 10; ++it) rows_gather_kernel<<<grid, 256, cols * 16>>>(A, n, cols, rb, x, xi, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("gather(%4d cols, %5.1f KB smem) + row blocks of %3d (%4d CTAs): %7.1f GB/s\n", cols,
               cols * 16 / 1024.0, rb, grid, by * 10 / (ms * 1e-3) / 1e9);
      }
    // the x gather alone (no matrix)
    {
      const int grid = n / 8;
      rows_gather_kernel<<<grid, 256, n * 16>>>(A, n, 0, 8, x, xi, out);
      cudaEventRecord(a);
      for (int it = 0; it < 10; ++it) rows_gather_kernel<<<grid, 256, n * 16>>>(A, n, 0, 8, x, xi, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("empty-matrix launch with %d-entry gather: %.1f us\n", n, ms * 100);
    }
  }
  contig_kernel<<<148 * 8, 256>>>(A, (size_t)n * n, out);
  cudaEventRecord(a);
  for (int it = 0; it < 10; ++it) contig_kernel<<<148 * 8, 256>>>(A, (size_t)n * n, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("contiguous stream           : %7.1f GB/s (%s)\n", bytes * 10 / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
