// TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on shared-memory
// mbarriers with transaction counts, for the streamed GEMV kernels.
#pragma once

#include <cuda_runtime.h>

namespace hpsb {

__device__ __forceinline__ unsigned tma_smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tma_mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tma_smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void tma_mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tma_smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tma_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(tma_smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          tma_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tma_smem_u32(bar))
      : "memory");
}
// A consumer warp hands a ring slot back to the producer: its generic-proxy
// reads of the slot are ordered before the next TMA (async-proxy) write into
// it by a proxy fence, then one lane arrives on the slot's empty barrier.
// (Without the fence the CGS2 kernel's results varied run to run.)
__device__ __forceinline__ void tma_release(unsigned long long* empty, int lane) {
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (lane == 0) tma_arrive(empty);
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace hpsb
