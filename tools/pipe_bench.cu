// pipe_bench.cu — how the FP64 pipe and the shared-memory pipe overlap for radix-16 butterfly jobs
// (16 LDS.128 -> DFT16 + 15 complex twiddles -> 16 STS.128 per thread), one CTA per SM.
// Diagnostics only.  modes: 0 compute only, 1 load+store only, 2 load->compute->store,
// 3 the same with a CTA barrier per job, 4 double-buffered (loads of job k+1 before the butterflies
// of job k), 5 double-buffered with a barrier every job.
#include <cstdio>
#include "../paper_2303_17510_b200/csrc/conv_ip.cuh"
using namespace hc;

template <int MODE>
__global__ void __launch_bounds__(384, 1) k(double2* out, int iters, int n_elems) {
  extern __shared__ __align__(128) double2 sm[];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < n_elems; i += nt) sm[i] = make_double2(1e-3 * i, 0.5);
  __syncthreads();
  double2 v[16], u[16];
  const int pos = tid ^ ((tid / 24) & 7);
  const int stride = n_elems / 16;  // element a at a * stride + pos
  const double2 w = make_double2(0.9999, 0.01);
  for (int a = 0; a < 16; ++a) v[a] = make_double2(tid + a, a), u[a] = v[a];
  auto LD = [&](double2(&x)[16]) HC_INL { sfor<16>([&](auto A) HC_INL { x[A] = sm[A * stride + pos]; }); };
  auto ST = [&](const double2(&x)[16]) HC_INL { sfor<16>([&](auto A) HC_INL { sm[A * stride + pos] = x[A]; }); };
  auto C = [&](double2(&x)[16]) HC_INL {
    DFT<16, +1>::run(x);
    double2 t = w;
    sfor<15>([&](auto K) HC_INL {
      x[K + 1] = cmul(x[K + 1], t);
      t = cmul(t, w);
    });
    sfor<16>([&](auto A) HC_INL { x[A] = cscale(x[A], 0.0625); });
  };
  __shared__ __align__(8) uint64_t bars[2];
  if (tid == 0) {
    mbar_init(&bars[0], nt / 32);
    mbar_init(&bars[1], nt / 32);
    fence_mbar_init();
  }
  __syncthreads();
  WarpBar bX{smem_u32(&bars[0])}, bY{smem_u32(&bars[1])};
  double2* sy = sm + n_elems;
  auto LDY = [&](double2(&x)[16]) HC_INL { sfor<16>([&](auto A) HC_INL { x[A] = sy[A * stride + pos]; }); };
  auto STY = [&](const double2(&x)[16]) HC_INL { sfor<16>([&](auto A) HC_INL { sy[A * stride + pos] = x[A]; }); };
  if (MODE == 6 || MODE == 7) {
    bX.arrive();
    bY.arrive();
  }
  if (MODE == 4 || MODE == 5) LD(v);
  for (int it = 0; it < iters; ++it) {
    if (MODE == 6) {  // two buffers alternating, split mbarrier per buffer (k_conv1d_ip's paired passes)
      bX.wait();
      LD(v);
      C(v);
      ST(v);
      bX.arrive();
      bY.wait();
      LDY(u);
      C(u);
      STY(u);
      bY.arrive();
      continue;
    }
    if (MODE == 7) {  // one buffer, split mbarrier right around (k_conv1d_ip's solo passes)
      bX.wait();
      LD(v);
      C(v);
      ST(v);
      bX.arrive();
      continue;
    }
    if (MODE == 0) {
      C(v);
    } else if (MODE == 1) {
      LD(v);
      ST(v);
    } else if (MODE == 2 || MODE == 3) {
      LD(v);
      C(v);
      ST(v);
      if (MODE == 3) __syncthreads();
    } else {
      LD(u);
      C(v);
      ST(v);
      if (MODE == 5) __syncthreads();
      LD(v);
      C(u);
      ST(u);
      if (MODE == 5) __syncthreads();
    }
  }
  double2 s = make_double2(0, 0);
  for (int a = 0; a < 16; ++a) s = cadd(s, cadd(v[a], u[a]));
  out[blockIdx.x * nt + tid] = s;
}

template <int MODE>
void run(int nt, const char* name) {
  const int iters = 2000;
  double2* out;
  cudaMalloc(&out, 148 * 1024 * sizeof(double2));
  const int n_elems = 16 * nt;
  const size_t smb = (size_t)n_elems * 16 * 2;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
  k<MODE><<<148, nt, smb>>>(out, 10, n_elems);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<148, nt, smb>>>(out, iters, n_elems);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double jobs = ((MODE >= 4 && MODE <= 6) ? 2.0 : 1.0) * iters;  // jobs per thread
  const double cyc_per_job = ms * 1e-3 * 1.965e9 / jobs;  // SM cycles per (all warps do one job)
  printf("%-26s threads=%3d  cycles per job-round=%8.1f  per warp-job/SMSP=%7.1f  %s\n", name, nt, cyc_per_job,
         cyc_per_job / (nt / 128.0), cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int nt : {128, 256, 384}) {
    run<0>(nt, "compute only");
    run<1>(nt, "load+store only");
    run<2>(nt, "load->compute->store");
    run<3>(nt, "  + barrier per job");
    run<4>(nt, "double-buffered");
    run<5>(nt, "  + barrier per job");
    run<6>(nt, "two buffers, mbarriers");
    run<7>(nt, "one buffer, mbarrier");
  }
  return 0;
}
