// Step-0 box measurement: FP64 DFMA / DADD throughput, device attributes.
// Not product code: measures the FP64 roofline denominator (absent from MEASURED_PEAKS.json).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void fp64_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (OP == 0) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
      } else {
        x0 = x0 + b; x1 = x1 + b; x2 = x2 + b; x3 = x3 + b; x4 = x4 + b; x5 = x5 + b; x6 = x6 + b; x7 = x7 + b;
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int l2 = 0, smemOptin = 0, clk = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  cudaDeviceGetAttribute(&smemOptin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"name\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %d, \"smem_per_sm\": %zu, \"regs_per_sm\": %d, \"clock_khz\": %d, \"cc\": \"%d.%d\"}\n",
         p.name, p.multiProcessorCount, l2, smemOptin, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor, clk, p.major, p.minor);
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int op = 0; op < 2; ++op) {
    for (int rep = 0; rep < 3; ++rep) {
      int blocks = p.multiProcessorCount * 4, threads = 512, iters = 4000;
      if (op == 0) fp64_loop<0><<<blocks, threads>>>(out, 10, 0.999, 1e-3); else fp64_loop<1><<<blocks, threads>>>(out, 10, 0.999, 1e-3);
      cudaEventRecord(e0);
      if (op == 0) fp64_loop<0><<<blocks, threads>>>(out, iters, 0.999, 1e-3); else fp64_loop<1><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double instr = (double)blocks * threads * iters * 16 * 8;
      double flops = instr * (op == 0 ? 2 : 1);
      printf("{\"op\": \"%s\", \"ms\": %.3f, \"dp_instr_per_s\": %.4e, \"tflops\": %.3f}\n", op == 0 ? "dfma" : "dadd", ms, instr / (ms * 1e-3), flops / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
