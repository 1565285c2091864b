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

const void* conv_ip_fn(int sym, int Bc) {
  if (sym == SYM_COMPLEX && Bc == 6144) return (const void*)k_conv1d_ip<SYM_COMPLEX, CfgIp6144>;
  return nullptr;
}

size_t conv_ip_smem_bytes(int Bc, int tabn) {
  return Bc == 6144 ? conv_ip_smem<CfgIp6144>(tabn) : 0;
}

// radix plan of the in-place kernel (the host builds its middle-pass tables from it)
void conv_ip_radices(int Bc, int* P, int* R, int* mt) {
  if (Bc == 6144) {
    *P = CfgIp6144::P;
    for (int i = 0; i < CfgIp6144::P; ++i) R[i] = CfgIp6144::R(i);
    *mt = CfgIp6144::MT;
  }
}

void conv_ip_launch(int Bc, const ConvArgs& a, int grid, size_t smem, cudaStream_t s) {
  if (Bc == 6144) k_conv1d_ip<SYM_COMPLEX, CfgIp6144><<<grid, CfgIp6144::T, smem, s>>>(a);
}

}  // namespace hc
