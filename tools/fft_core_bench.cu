// fft_core_bench.cu — microbenchmark of the block-FFT core (fft_forward + fft_inverse on data
// resident in registers / shared memory, no global traffic), one CTA per SM.  Diagnostics
// only: reports cycles per 6144-point (etc.) FFT to separate FFT-core efficiency from the
// convolution pipeline around it.
#include <cstdio>
#include <vector>
#include "../paper_2303_17510_b200/csrc/kernels.cuh"

using namespace hc;

struct Unit {
  __device__ void operator()(int, double2& t, double2& w) const {
    t = make_double2(1.0, 0.0);
    w = make_double2(0.9999, 0.01);
  }
};

template <class Cfg, int G = 1>
__global__ void __launch_bounds__(Cfg::T * G, 1) k_core(double2* out, const double2* mt_g, int iters, unsigned long long* cyc) {
  extern __shared__ __align__(16) double2 smem[];
  double2* mt = smem;
  const int g = threadIdx.x / Cfg::T;
  double2* X = smem + (Cfg::MT > 0 ? Cfg::MT : 1) + g * Cfg::XS;
  for (int i = threadIdx.x; i < Cfg::MT; i += blockDim.x) mt[i] = mt_g[i];
  __syncthreads();
  const int tid = threadIdx.x % Cfg::T;
  double2 v[Cfg::E];
  for (int i = 0; i < Cfg::E; ++i) v[i] = make_double2(tid * 1e-3 + i, i * 0.5);
  const GroupSync sync{g + 1, Cfg::T};
  const Unit p0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    fft_forward<Cfg>(v, X, mt, tid, sync, p0);
    fft_inverse<Cfg>(v, X, mt, tid, sync, p0);
#pragma unroll
    for (int i = 0; i < Cfg::E; ++i) v[i] = cscale(v[i], 1.0 / Cfg::N);
  }
  unsigned long long t1 = clock64();
  if (tid == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  double2 s = make_double2(0, 0);
  for (int i = 0; i < Cfg::E; ++i) s = cadd(s, v[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class Cfg, int G = 1>
void run(const char* name) {
  const int iters = 50;
  double2 *out, *mt;
  unsigned long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(double2));
  cudaMalloc(&mt, (Cfg::MT + 1) * sizeof(double2));
  cudaMemset(mt, 0, (Cfg::MT + 1) * sizeof(double2));
  cudaMalloc(&cyc, 8);
  size_t sm = (Cfg::MT + 1 + G * Cfg::XS) * sizeof(double2);
  cudaFuncSetAttribute(k_core<Cfg, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_core<Cfg, G>, Cfg::T * G, sm);
  k_core<Cfg, G><<<148 * nb, Cfg::T * G, sm>>>(out, mt, 2, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_core<Cfg, G><<<148 * nb, Cfg::T * G, sm>>>(out, mt, iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double ffts = 2.0 * iters * 148 * nb * G;
  const double per_fft_ns = ms * 1e6 / (ffts / 148);  // per SM
  // FP64 flops: 5 N log2 N per FFT (nominal)
  const double flops = 5.0 * Cfg::N * std::log2((double)Cfg::N) * ffts;
  printf("%-14s G=%d N=%5d T=%4d ctas/sm=%d  cycles/FFT(cta0)=%8.0f  ns/FFT/SM=%8.1f  nominal TFLOP/s=%6.2f  err=%s\n", name,
         G, Cfg::N, Cfg::T, nb, (double)c / (2.0 * iters), per_fft_ns, flops / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<FFTCfg<Radices<16, 16, 24>, 384>>("16x16x24");
  run<FFTCfg<Radices<16, 24, 16>, 384>>("16x24x16");
  run<FFTCfg<Radices<24, 16, 16>, 384>>("24x16x16");
  run<FFTCfg<Radices<16, 16, 16>, 256>>("16x16x16");
  return 0;
}
