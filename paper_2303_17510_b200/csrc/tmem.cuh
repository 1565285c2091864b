// tmem.cuh — tensor memory (TMEM) as per-thread spill space for the ping-pong kernel.
//
// TMEM is 512 columns x 128 lanes x 32 bit per SM.  Warp w of a CTA reaches the lane quarter
// 32*(w%4) .. 32*(w%4)+31 (lane = its lane id); warps w, w+4, w+8 share a quarter and take
// disjoint column ranges.  The 32x32b shapes move, per thread, N consecutive 32-bit columns of
// its own lane, so a thread's values never leave its lane: the kernel keeps the stashed
// spectrum F and the residue accumulator there instead of in shared memory (measured 4x the
// shared-memory store+load throughput, tools/tmem_bench.cu), which frees the shared-memory
// pipe for the FFT exchanges.  All tcgen05 ld/st are warp-collective (.sync.aligned).
#pragma once
#include <cstdint>

#include "fft_device.cuh"

namespace hc {

// one warp allocates `cols` columns (power of 2, >= 32) and publishes the base address
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, int cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem_dst)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t base, int cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void split(double2 z, uint32_t* w) {
  const unsigned long long a = __double_as_longlong(z.x), b = __double_as_longlong(z.y);
  w[0] = (uint32_t)a;
  w[1] = (uint32_t)(a >> 32);
  w[2] = (uint32_t)b;
  w[3] = (uint32_t)(b >> 32);
}
__device__ __forceinline__ double2 join(const uint32_t* w) {
  return make_double2(__longlong_as_double((long long)(((unsigned long long)w[1] << 32) | w[0])),
                      __longlong_as_double((long long)(((unsigned long long)w[3] << 32) | w[2])));
}

// 8 complex values (32 columns) <-> TMEM at column address taddr
__device__ __forceinline__ void tm_st8(uint32_t taddr, const double2* z) {
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 8; ++i) split(z[i], r + 4 * i);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t taddr, double2* z) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 8; ++i) z[i] = join(r + 4 * i);
}
// 4 complex values (16 columns)
__device__ __forceinline__ void tm_st4(uint32_t taddr, const double2* z) {
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) split(z[i], r + 4 * i);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tm_ld4(uint32_t taddr, double2* z) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 4; ++i) z[i] = join(r + 4 * i);
}

// N complex values (N % 4 == 0) to / from consecutive columns starting at taddr
template <int N>
__device__ __forceinline__ void tm_store(uint32_t taddr, const double2* z) {
  static_assert(N % 4 == 0, "TMEM spills move groups of 4 complex values");
  sfor<N / 8>([&](auto Ki) HC_INL { tm_st8(taddr + 32 * Ki, z + 8 * Ki); });
  if constexpr (N % 8) tm_st4(taddr + 32 * (N / 8), z + 8 * (N / 8));
}

// Per-thread spill layout of a kernel with NT threads per CTA: F (EF complex) and the residue
// accumulator (EA complex) side by side; warps sharing a lane quarter take consecutive slots.
template <int NT, int EF, int EA>
struct TmemLayout {
  static constexpr int WPQ = (NT / 32 + 3) / 4;            // warps per lane quarter
  static constexpr int SLOT = 4 * (EF + EA);                // columns per warp slot
  static constexpr int NEED = WPQ * SLOT;
  static constexpr int COLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static constexpr bool FITS = NEED <= 512 && EF % 4 == 0 && EA % 4 == 0 && EF + EA > 0;
  // thread's F columns / accumulator columns (lane field = the warp's quarter)
  __device__ __forceinline__ static uint32_t f_addr(uint32_t base) {
    const uint32_t w = threadIdx.x / 32;
    return base + ((32u * (w % 4)) << 16) + (w / 4) * SLOT;
  }
  __device__ __forceinline__ static uint32_t a_addr(uint32_t base) { return f_addr(base) + 4 * EF; }
};

}  // namespace hc
