// tma.cuh — bulk (TMA) global->shared copies completed on an mbarrier (sm_90+/sm_100a PTX).
//
// The residue loop stages each input line into shared memory with cp.async.bulk while the
// previous transform computes, so the SMs never wait on HBM latency at the start of a
// forward FFT (kernels.cuh, STAGE path).  One elected thread per line group issues the copy;
// every thread of the group waits on the mbarrier phase.
#pragma once
#include <cuda.h>  // CUtensorMap (the maps are encoded on the host, hconv_lib.cu)
#include <cstdint>

// HC_TMA_FENCE=1: a generic->async proxy fence before every bulk load (off by default: every
// load is issued after a group barrier that follows the buffer's last generic accesses -- its
// loads have returned and its stores have been performed in shared memory; measured 2% of c2)
#ifndef HC_TMA_FENCE
#define HC_TMA_FENCE 0
#endif
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

// this thread's generic-proxy global stores before subsequent async-proxy (TMA) reads of them
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

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
  if (HC_TMA_FENCE) fence_proxy_async();
  mbar_expect_tx(bar, bytes);
  for (uint32_t off = 0; off < bytes; off += kChunk) {
    const uint32_t n = bytes - off < kChunk ? bytes - off : kChunk;
    tma_load_1d(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, n, bar);
  }
}

// ---- shared -> global bulk stores (bulk-group completion) ----
// Each thread that wrote the source through ordinary stores runs fence_proxy_async_smem(), then
// the group synchronises, then one thread issues the copy and commits the group.  Before the
// source is overwritten, the same thread waits with bulk_wait_read().
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// bytes: multiple of 16, both addresses 16-B aligned; evict_first: streaming output
__device__ __forceinline__ void tma_store(void* dst, const void* src, uint32_t bytes, bool evict_first) {
  constexpr uint32_t kChunk = 32768;
  const uint64_t pol = l2_policy_evict_first();
  for (uint32_t off = 0; off < bytes; off += kChunk) {
    const uint32_t n = bytes - off < kChunk ? bytes - off : kChunk;
    if (evict_first)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                       static_cast<char*>(dst) + off),
                   "r"(smem_u32(static_cast<const char*>(src) + off)), "r"(n), "l"(pol)
                   : "memory");
    else
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(static_cast<char*>(dst) + off),
                   "r"(smem_u32(static_cast<const char*>(src) + off)), "r"(n)
                   : "memory");
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// all committed bulk stores of this thread have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// all committed bulk stores of this thread are complete (their global writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Warm L2 with a line that will be staged later (no shared-memory destination, no barrier).
__device__ __forceinline__ void l2_prefetch(const void* src, uint32_t bytes) {
  constexpr uint32_t kChunk = 32768;
  for (uint32_t off = 0; off < bytes; off += kChunk) {
    const uint32_t n = bytes - off < kChunk ? bytes - off : kChunk;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(static_cast<const char*>(src) + off), "r"(n)
                 : "memory");
  }
}

// ---- per-thread asynchronous 16-byte global->shared copies (cp.async, LDGSTS) ----
// Used where a tile is gathered from strided rows (column tiles of the N-D outer axes): each
// thread copies its elements into the tile's shared-memory layout without staging them in
// registers; completion per thread through commit/wait groups, then a CTA barrier.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- tensor-map (cp.async.bulk.tensor) tiles: 3D maps {inner, rows, outer} of float64 ----
// Load one box at element coordinates (c0, c1, c2) into shared memory, completing on `bar`.
__device__ __forceinline__ void tma_tensor_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                   uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// Store one box from shared memory (bulk-group completion; commit with bulk_commit()).
__device__ __forceinline__ void tma_tensor_store_3d(const CUtensorMap* map, int c0, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

}  // namespace hc
