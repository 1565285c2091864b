// inst_ip.cu — instantiations of the in-place interleaved convolution kernel (conv_ip.cuh) and
// the host's access to them by complex FFT length.
#include "conv_ip.cuh"

namespace hc {

#ifndef HC_IP6144_PLAN
#define HC_IP6144_PLAN 2
#endif
// 16 x 24 x 16: the product pass (forward g, product, inverse: the heaviest) runs on all 12 warps with 16
// values per thread; the radix-24 pass in the middle on 8 (16 x 16 x 24 spills there at 168 registers)
#if HC_IP6144_PLAN == 1
using CfgIp6144 = FFTCfg<Radices<16, 16, 24>, 384>;
#else
using CfgIp6144 = FFTCfg<Radices<16, 24, 16>, 384>;
#endif

// HC_IP_KERNEL=1: k_conv1d_ip (12 warps, a barrier per pass); 2: k_conv1d_ip2 (8 warps, software-pipelined
// jobs); 3: k_conv1d_ip3 (12 warps, group-local hand-offs between passes 1 and 2)
#ifndef HC_IP_KERNEL
#define HC_IP_KERNEL 4
#endif
#if HC_IP_KERNEL == 2
using CfgIp = FFTCfg<Radices<16, 16, 24>, 384>;  // (thread count unused: the kernel runs 256 threads)
#define HC_IP_K k_conv1d_ip2<SYM_COMPLEX, CfgIp>
constexpr int kIpThreads = 256;
#elif HC_IP_KERNEL == 3
using CfgIp = FFTCfg<Radices<16, 24, 16>, 384>;
#define HC_IP_K k_conv1d_ip3<SYM_COMPLEX, CfgIp>
constexpr int kIpThreads = CfgIp::T;
#elif HC_IP_KERNEL == 4
using CfgIp = FFTCfg<Radices<16, 24, 16>, 384>;
#define HC_IP_K k_conv1d_ip4<SYM_COMPLEX, CfgIp>
constexpr int kIpThreads = CfgIp::T;
#else
using CfgIp = CfgIp6144;
#define HC_IP_K k_conv1d_ip<SYM_COMPLEX, CfgIp>
constexpr int kIpThreads = CfgIp::T;
#endif

const void* conv_ip_fn(int sym, int Bc) {
  if (sym == SYM_COMPLEX && Bc == 6144) return (const void*)HC_IP_K;
  return nullptr;
}
int conv_ip_threads(int) { return kIpThreads; }
// residue blocks the kernel requires (0: any)
int conv_ip_residues(int) { return HC_IP_KERNEL == 4 ? 2 : 0; }

size_t conv_ip_smem_bytes(int Bc, int tabn) {
  return Bc == 6144 ? conv_ip_smem<CfgIp>(tabn) : 0;
}

// radix plan of the in-place kernel (the host builds its middle-pass tables from it)
void conv_ip_radices(int Bc, int* P, int* R, int* mt) {
  if (Bc == 6144) {
    *P = CfgIp::P;
    for (int i = 0; i < CfgIp::P; ++i) R[i] = CfgIp::R(i);
    *mt = CfgIp::MT;
  }
}

#if defined(HC_IP_DIAG) && HC_IP_KERNEL == 3
// timing builds: the kernel with parts compiled out, selected by HCONV_DBG (results are wrong)
template <int D>
bool diag_launch(const ConvArgs& a, int grid, size_t smem, cudaStream_t s) {
  if (a.dbg != D) return false;
  auto k = k_conv1d_ip3<SYM_COMPLEX, CfgIp, D>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<grid, kIpThreads, smem, s>>>(a);
  return true;
}
#endif

void conv_ip_launch(int Bc, const ConvArgs& a, int grid, size_t smem, cudaStream_t s) {
#if defined(HC_IP_DIAG) && HC_IP_KERNEL == 3
  if (diag_launch<13>(a, grid, smem, s) || diag_launch<13 + 16>(a, grid, smem, s) || diag_launch<13 + 32>(a, grid, smem, s) ||
      diag_launch<13 + 64>(a, grid, smem, s) || diag_launch<13 + 128>(a, grid, smem, s) ||
      diag_launch<13 + 256>(a, grid, smem, s) || diag_launch<13 + 496 - 16>(a, grid, smem, s) ||
      diag_launch<13 + 496 - 32>(a, grid, smem, s) || diag_launch<13 + 496 - 64>(a, grid, smem, s) ||
      diag_launch<13 + 496 - 128>(a, grid, smem, s) || diag_launch<13 + 496 - 256>(a, grid, smem, s) ||
      diag_launch<13 + 496>(a, grid, smem, s) || diag_launch<13 + 496 - 16 + 512>(a, grid, smem, s) ||
      diag_launch<13 + 496 + 512>(a, grid, smem, s) || diag_launch<13 + 1024>(a, grid, smem, s) || diag_launch<13 + 496 - 32 + 512>(a, grid, smem, s) || diag_launch<13 + 496 - 48>(a, grid, smem, s))
    return;
#endif
  if (Bc == 6144) HC_IP_K<<<grid, kIpThreads, smem, s>>>(a);
}

}  // namespace hc
