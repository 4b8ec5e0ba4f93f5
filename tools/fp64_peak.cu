// FP64 peak probe for B200: DFMA vs DMMA (mma.sync f64) throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dmma_m8n8k4_loop(double* out, int iters) {
  double acc[4][2];
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dmma_m16n8k16_loop(double* out, int iters) {
  double acc[4][4];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-6 * i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-6 * i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += acc[i][j];
  if (s == 12345.0) out[threadIdx.x] = s;
}

// Mixed: even warps run DMMA chains, odd warps DFMA chains (do the DMMA and
// DFMA pipes overlap?).  Reports the combined rate; fl counts both.
__global__ void mixed_loop(double* out, int iters, int dfma_per_dmma) {
  const bool mm = ((threadIdx.x >> 5) & 1) == 0;
  double s = 0;
  if (mm) {
    double acc[4][2];
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
    for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
  } else {
    double a[8], b = 1.0000001, c = 0.9999999;
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters * dfma_per_dmma; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    for (int i = 0; i < 8; ++i) s += a[i];
  }
  if (s == 12345.0) out[threadIdx.x] = s;
}

// Sustained DMMA rate: m8n8k4 chains launched back to back for `seconds`
// (4 s as MEASURED_PEAKS' sustained bf16 figure), one CUDA-event pair around
// the whole run; the burst figure is the best single launch.
static void sustained(double seconds, int sms) {
  double* d; cudaMalloc(&d, 4096 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = sms * 4, threads = 256, iters = 20000;
  const double fl = 2.0 * 256 * 4 * iters * (double)grid * (threads / 32);
  float best = 1e30f, ms = 0;
  for (int i = 0; i < 5; ++i) {
    cudaEventRecord(e0); dmma_m8n8k4_loop<<<grid, threads>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const int launches = (int)(seconds * 1e3 / best) + 1;
  cudaEventRecord(e0);
  for (int i = 0; i < launches; ++i) dmma_m8n8k4_loop<<<grid, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"dmma_burst_tflops\": %.2f, \"dmma_sustained_tflops\": %.2f, \"sustained_seconds\": %.2f, "
         "\"launches\": %d, \"err\": \"%s\"}\n",
         fl / best / 1e9, fl * launches / ms / 1e9, ms * 1e-3, launches,
         cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (argc > 1) {  // fp64_peak <seconds>: sustained mode (JSON line)
    sustained(atof(argv[1]), sms);
    return 0;
  }
  double* d; cudaMalloc(&d, 4096 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 3; ++rep) {
    for (int blocks_per_sm : {2, 4, 8}) {
      int grid = sms * blocks_per_sm, threads = 256;
      float ms;
      dfma_loop<<<grid, threads>>>(d, iters);
      cudaEventRecord(e0); dfma_loop<<<grid, threads>>>(d, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * iters * (double)grid * threads;
      printf("dfma          bps=%d  %.2f TFLOP/s\n", blocks_per_sm, fl / ms / 1e9);
      dmma_m8n8k4_loop<<<grid, threads>>>(d, iters);
      cudaEventRecord(e0); dmma_m8n8k4_loop<<<grid, threads>>>(d, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 256 * 4 * iters * (double)grid * (threads / 32);
      printf("dmma m8n8k4   bps=%d  %.2f TFLOP/s\n", blocks_per_sm, fl / ms / 1e9);
      dmma_m16n8k16_loop<<<grid, threads>>>(d, iters / 4);
      cudaEventRecord(e0); dmma_m16n8k16_loop<<<grid, threads>>>(d, iters / 4); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 16 * 8 * 16 * 4 * (iters / 4) * (double)grid * (threads / 32);
      printf("dmma m16n8k16 bps=%d  %.2f TFLOP/s\n", blocks_per_sm, fl / ms / 1e9);
    }
  }
  for (int ratio : {1, 2, 4}) {
    int grid = sms * 4, threads = 256;
    float ms;
    mixed_loop<<<grid, threads>>>(d, iters, ratio);
    cudaEventRecord(e0); mixed_loop<<<grid, threads>>>(d, iters, ratio); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    const double half_warps = (double)grid * (threads / 32) / 2;
    const double fl = 2.0 * 256 * 4 * iters * half_warps + 2.0 * 8 * iters * ratio * half_warps * 32;
    printf("mixed dmma+dfma ratio=%d  %.2f TFLOP/s combined\n", ratio, fl / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
