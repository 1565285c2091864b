// tmem_bench.cu — throughput of thread-private spills to tensor memory (tcgen05.st / tcgen05.ld,
// 32x32b shapes) against shared memory (STS.128 / LDS.128) for 384 threads per SM, 96 32-bit
// words per thread (the ping-pong kernel's stash of 24 complex values).  Diagnostics only.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void tm_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tm_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

template <bool TMEM>
__global__ void __launch_bounds__(384, 1) k(unsigned long long* cyc, uint32_t* out, int iters) {
  __shared__ uint32_t tbase;
  extern __shared__ __align__(16) uint32_t sm[];
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (TMEM) {
    if (w == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * 7 + i;
  const uint32_t taddr = TMEM ? tbase + ((uint32_t)(32 * (w % 4)) << 16) + (uint32_t)(160 * (w / 4)) : 0;
  uint4* s4 = reinterpret_cast<uint4*>(sm);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (TMEM) {
#pragma unroll
      for (int c = 0; c < 3; ++c) tm_st32(taddr + 32 * c, r);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      __syncthreads();
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        uint32_t q[32];
        tm_ld32(taddr + 32 * c, q);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] += q[i];
      }
      __syncthreads();
    } else {
#pragma unroll
      for (int c = 0; c < 24; ++c)
        s4[c * 384 + threadIdx.x] = make_uint4(r[(4 * c) % 32], r[(4 * c + 1) % 32], r[(4 * c + 2) % 32], r[(4 * c + 3) % 32]);
      __syncthreads();
#pragma unroll
      for (int c = 0; c < 24; ++c) {
        uint4 q = s4[c * 384 + threadIdx.x];
        r[(4 * c) % 32] += q.x; r[(4 * c + 1) % 32] += q.y; r[(4 * c + 2) % 32] += q.z; r[(4 * c + 3) % 32] += q.w;
      }
      __syncthreads();
    }
  }
  unsigned long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 32; ++i) s += r[i];
  out[blockIdx.x * 384 + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  if (TMEM) {
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
}

int main() {
  unsigned long long* cyc;
  uint32_t* out;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&out, 148 * 384 * 4);
  const int iters = 200;
  for (int t = 0; t < 2; ++t) {
    unsigned long long c = 0;
    if (t == 0) {
      cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      k<true><<<148, 384, 160 * 1024>>>(cyc, out, iters);
    } else {
      cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      k<false><<<148, 384, 160 * 1024>>>(cyc, out, iters);
    }
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    // bytes moved per iteration per SM: 384 threads x 384 B written + read
    printf("%s: %.0f cycles/iter (store+load of 147456 B each), %s\n", t == 0 ? "TMEM" : "SMEM", (double)c / iters,
           cudaGetErrorString(e));
  }
  return 0;
}
