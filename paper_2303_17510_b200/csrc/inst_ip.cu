// inst_ip.cu — instantiation of the in-place two-residue convolution kernel (conv_ip.cuh) and the
// host's access to it by complex FFT length.
#include "conv_ip.cuh"

namespace hc {

// 16 x 24 x 16 at 12 warps: passes 0 and 2 (radix 16) on every warp, pass 1 (radix 24) on 8
// (HC_IP_PLAN=2: 16 x 16 x 24, the radix-24 pass last and free of twiddles, on 8 warps with 24 values each:
// spills at 168 registers, c2 0.70 -> 0.91 ms)
#ifndef HC_IP_PLAN
#define HC_IP_PLAN 1
#endif
#if HC_IP_PLAN == 2
using CfgIp6144 = FFTCfg<Radices<16, 16, 24>, 384>;
#else
using CfgIp6144 = FFTCfg<Radices<16, 24, 16>, 384>;
#endif

const void* conv_ip_fn(int sym, int Bc) {
  if (sym == SYM_COMPLEX && Bc == 6144) return (const void*)k_conv1d_ip4<SYM_COMPLEX, CfgIp6144>;
  return nullptr;
}
int conv_ip_threads(int) { return CfgIp6144::T; }
// residue blocks the kernel requires
int conv_ip_residues(int) { return 2; }

size_t conv_ip_smem_bytes(int Bc, int tabn) { return Bc == 6144 ? conv_ip_smem<CfgIp6144>(tabn) : 0; }

// radix plan of the in-place kernel (the host builds its middle-pass tables from it)
void conv_ip_radices(int Bc, int* P, int* R, int* mt) {
  if (Bc == 6144) {
    *P = CfgIp6144::P;
    for (int i = 0; i < CfgIp6144::P; ++i) R[i] = CfgIp6144::R(i);
    *mt = CfgIp6144::MT;
  }
}

void conv_ip_launch(int Bc, const ConvArgs& a, int grid, size_t smem, cudaStream_t s) {
  if (Bc == 6144) k_conv1d_ip4<SYM_COMPLEX, CfgIp6144><<<grid, CfgIp6144::T, smem, s>>>(a);
}

}  // namespace hc
