// tma.cuh — bulk (TMA) global->shared copies completed on an mbarrier (sm_90+/sm_100a PTX).
//
// The residue loop stages each input line into shared memory with cp.async.bulk while the
// previous transform computes, so the SMs never wait on HBM latency at the start of a
// forward FFT (kernels.cuh, STAGE path).  One elected thread per line group issues the copy;
// every thread of the group waits on the mbarrier phase.
#pragma once
#include <cstdint>

namespace hc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// order this thread's (and, after a barrier, the CTA's) generic-proxy accesses before
// subsequent async-proxy (TMA) accesses
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Copy `bytes` (multiple of 16, both addresses 16-B aligned) in chunks onto one barrier.
// Called by a single thread.
__device__ __forceinline__ void tma_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  constexpr uint32_t kChunk = 32768;
  fence_proxy_async();
  mbar_expect_tx(bar, bytes);
  for (uint32_t off = 0; off < bytes; off += kChunk) {
    const uint32_t n = bytes - off < kChunk ? bytes - off : kChunk;
    tma_load_1d(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, n, bar);
  }
}

// Warm L2 with a line that will be staged later (no shared-memory destination, no barrier).
__device__ __forceinline__ void l2_prefetch(const void* src, uint32_t bytes) {
  constexpr uint32_t kChunk = 32768;
  for (uint32_t off = 0; off < bytes; off += kChunk) {
    const uint32_t n = bytes - off < kChunk ? bytes - off : kChunk;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(static_cast<const char*>(src) + off), "r"(n)
                 : "memory");
  }
}

}  // namespace hc
