// registry.cuh — kernel instantiations available to the host (one table per symmetry).
#pragma once
#include <cuda_runtime.h>

#include "naive.cuh"

namespace hc {

struct KernelEntry {
  int Bc = 0;      // complex FFT length (0 for the naive entry: any length <= kNaiveMax)
  int T = 0, G = 0;
  bool naive = false;
  size_t smem_conv = 0, smem_fwd = 0, smem_bwd = 0;  // per CTA (naive: per complex point)
  const void* conv_fn = nullptr;
  const void* fwd_fn = nullptr;
  const void* bwd_fn = nullptr;
  void (*conv)(const ConvArgs&, int grid, size_t smem, cudaStream_t) = nullptr;
  void (*fwd)(const FwdArgs&, int grid, size_t smem, cudaStream_t) = nullptr;
  void (*bwd)(const BwdArgs&, int grid, size_t smem, cudaStream_t) = nullptr;
  const char* radix = "";
  int P = 0, R[4] = {0, 0, 0, 0};  // radix plan (host builds the pass-0 / middle-pass tables from it)
  int mt = 0;                      // middle-pass table entries (FFTCfg::MT)
  int xs = 0, stash = 0;           // exchange buffer / shared-memory stash per group (complex)
  const void* convpp2_fn = nullptr;  // paired ping-pong variant (k_conv1d_pp2: complex, L <= B)
  void (*convpp2)(const ConvArgs&, int grid, size_t smem, cudaStream_t) = nullptr;
  const void* convpp_fn = nullptr;  // ping-pong variant (k_conv1d_pp)
  void (*convpp)(const ConvArgs&, int grid, size_t smem, cudaStream_t) = nullptr;
  // column-tile outer-axis passes (complex / centered only): GC interleaved column groups
  int gc = 0, gcp = 0;  // column groups per CTA: unpipelined / pipelined kernels
  const void* fwdc_fn = nullptr;
  const void* bwdc_fn = nullptr;
  void (*fwdc)(const FwdArgs&, int grid, size_t smem, cudaStream_t) = nullptr;
  void (*bwdc)(const BwdArgs&, int grid, size_t smem, cudaStream_t) = nullptr;
  // pipelined column tiles (two tile buffers of GC x max(XS, rows) values)
  const void* fwdcp_fn = nullptr;
  const void* bwdcp_fn = nullptr;
  void (*fwdcp)(const FwdArgs&, int grid, size_t smem, cudaStream_t) = nullptr;
  void (*bwdcp)(const BwdArgs&, int grid, size_t smem, cudaStream_t) = nullptr;
  // the same tiles moved by tensor-map TMA (k_pfft_*_cols_tma; gcp columns per tile)
  const void* fwdct_fn = nullptr;
  const void* bwdct_fn = nullptr;
  void (*fwdct)(const FwdArgs&, const TileMaps&, const CUtensorMap&, const CUtensorMap&, int grid, size_t smem,
                cudaStream_t) = nullptr;
  void (*bwdct)(const BwdArgs&, const TileMaps&, const CUtensorMap&, int grid, size_t smem, cudaStream_t) = nullptr;
  // one-buffer TMA tiles at the full width gc (k_pfft_*_cols_tma1), for blocks whose two-buffer
  // tiles would be narrower (gcp < gc)
  const void* fwdc1_fn = nullptr;
  const void* bwdc1_fn = nullptr;
  void (*fwdc1)(const FwdArgs&, const TileMaps&, const CUtensorMap&, const CUtensorMap&, int grid, size_t smem,
                cudaStream_t) = nullptr;
  void (*bwdc1)(const BwdArgs&, const TileMaps&, const CUtensorMap&, int grid, size_t smem, cudaStream_t) = nullptr;
};

// column groups per CTA: up to 8 adjacent columns (128 B rows), <= 1024 threads, and the
// interleaved exchange buffers within ~200 KB of shared memory
template <class Cfg>
constexpr int column_groups() {
  int g = 8;
  while (g > 1 && (g * Cfg::T > 1024 || (long long)g * Cfg::XS * 16 > 200 * 1024)) g /= 2;
  return g;
}

// pipelined column tiles: two tile buffers per CTA, so up to half the groups of column_groups
// (4 columns per tile -- 64-byte rows, two CTAs per SM -- measured slower: c5 9.91 -> 12.42 ms)
template <class Cfg>
constexpr int column_groups_pp() {
  int g = 8;
  while (g > 1 && (g * Cfg::T > 1024 || 2LL * g * Cfg::XS * 16 > 200 * 1024)) g /= 2;
  return g;
}

// SMEM_STASH: keep the first spectrum in shared memory even when it would fit in registers
// (lets G > 1 line groups share an SM within the register budget).
// MINB: minimum resident CTAs per SM requested from ptxas (caps registers per thread)
template <int SYM, class Cfg, int G, bool SMEM_STASH = false, int MINB = 1>
KernelEntry make_entry(const char* radix) {
  constexpr bool SR = Cfg::E <= 16 && !SMEM_STASH;
  KernelEntry e;
  e.Bc = Cfg::N;
  e.T = Cfg::T;
  e.G = G;
  e.radix = radix;
  e.smem_conv = (Cfg::MT + (size_t)G * (Cfg::XS + (SR ? 0 : Cfg::N))) * sizeof(double2);
  e.smem_fwd = e.smem_bwd = (Cfg::MT + (size_t)G * Cfg::XS) * sizeof(double2);
  e.P = Cfg::P;
  for (int i = 0; i < Cfg::P; ++i) e.R[i] = Cfg::R(i);
  e.mt = Cfg::MT;
  e.xs = Cfg::XS;
  e.stash = SR ? 0 : Cfg::N;
  e.conv_fn = (const void*)k_conv1d<SYM, Cfg, G, SR, MINB>;
  e.fwd_fn = (const void*)k_pfft_fwd<SYM, Cfg, G>;
  e.bwd_fn = (const void*)k_pfft_bwd<SYM, Cfg, G>;
  e.conv = [](const ConvArgs& a, int grid, size_t sm, cudaStream_t s) {
    k_conv1d<SYM, Cfg, G, SR, MINB><<<grid, Cfg::T * G, sm, s>>>(a);
  };
  // paired ping-pong (complex): kernels that own the SM with at most 16 last-pass values per
  // thread (B200: 4096-point blocks 0.560 -> 0.484 ms for L = 4000 x 4096 lines; the split
  // last-pass variant for 16x16x24 spills at 384 threads, 0.79 -> 0.91 ms; the smaller plans,
  // several CTAs per SM at capped registers, spill too: 2048 0.29 -> 0.35, 512 0.24 -> 0.30 ms)
  if constexpr (SYM == SYM_COMPLEX && Cfg::ES <= 16 && Cfg::T <= 256 && (2 * Cfg::XS * G * 16 > 116 * 1024)) {
    e.convpp2_fn = (const void*)k_conv1d_pp2<Cfg, G, MINB>;
    e.convpp2 = [](const ConvArgs& a, int grid, size_t sm, cudaStream_t s) {
      k_conv1d_pp2<Cfg, G, MINB><<<grid, Cfg::T * G, sm, s>>>(a);
    };
  }
  e.convpp_fn = (const void*)k_conv1d_pp<SYM, Cfg, G, SR, MINB>;
  e.convpp = [](const ConvArgs& a, int grid, size_t sm, cudaStream_t s) {
    k_conv1d_pp<SYM, Cfg, G, SR, MINB><<<grid, Cfg::T * G, sm, s>>>(a);
  };
  e.fwd = [](const FwdArgs& a, int grid, size_t sm, cudaStream_t s) {
    k_pfft_fwd<SYM, Cfg, G><<<grid, Cfg::T * G, sm, s>>>(a);
  };
  e.bwd = [](const BwdArgs& a, int grid, size_t sm, cudaStream_t s) {
    k_pfft_bwd<SYM, Cfg, G><<<grid, Cfg::T * G, sm, s>>>(a);
  };
  if constexpr (SYM != SYM_HERMITIAN) {
    constexpr int GC = column_groups<Cfg>();
    e.gc = GC;
    e.fwdc_fn = (const void*)k_pfft_fwd_cols<SYM, Cfg, GC>;
    e.bwdc_fn = (const void*)k_pfft_bwd_cols<SYM, Cfg, GC>;
    e.fwdc = [](const FwdArgs& a, int grid, size_t sm, cudaStream_t s) {
      k_pfft_fwd_cols<SYM, Cfg, GC><<<grid, Cfg::T * GC, sm, s>>>(a);
    };
    e.bwdc = [](const BwdArgs& a, int grid, size_t sm, cudaStream_t s) {
      k_pfft_bwd_cols<SYM, Cfg, GC><<<grid, Cfg::T * GC, sm, s>>>(a);
    };
    constexpr int GP = column_groups_pp<Cfg>();
    e.gcp = GP;
    e.fwdcp_fn = (const void*)k_pfft_fwd_cols_pp<SYM, Cfg, GP>;
    e.bwdcp_fn = (const void*)k_pfft_bwd_cols_pp<SYM, Cfg, GP>;
    e.fwdcp = [](const FwdArgs& a, int grid, size_t sm, cudaStream_t s) {
      k_pfft_fwd_cols_pp<SYM, Cfg, GP><<<grid, Cfg::T * GP, sm, s>>>(a);
    };
    e.bwdcp = [](const BwdArgs& a, int grid, size_t sm, cudaStream_t s) {
      k_pfft_bwd_cols_pp<SYM, Cfg, GP><<<grid, Cfg::T * GP, sm, s>>>(a);
    };
    e.fwdct_fn = (const void*)k_pfft_fwd_cols_tma<SYM, Cfg, GP>;
    e.bwdct_fn = (const void*)k_pfft_bwd_cols_tma<SYM, Cfg, GP>;
    e.fwdct = [](const FwdArgs& a, const TileMaps& tm, const CUtensorMap& mi, const CUtensorMap& mo, int grid, size_t sm,
                 cudaStream_t s) { k_pfft_fwd_cols_tma<SYM, Cfg, GP><<<grid, Cfg::T * GP, sm, s>>>(a, tm, mi, mo); };
    e.bwdct = [](const BwdArgs& a, const TileMaps& tm, const CUtensorMap& mi, int grid, size_t sm, cudaStream_t s) {
      k_pfft_bwd_cols_tma<SYM, Cfg, GP><<<grid, Cfg::T * GP, sm, s>>>(a, tm, mi);
    };
    // (plans of more than 16 values per thread run GC x T > 512 threads at capped registers: their
    // tiles stay with the plain-load kernels)
    if constexpr (GP < GC && Cfg::E <= 16) {
      e.fwdc1_fn = (const void*)k_pfft_fwd_cols_tma1<SYM, Cfg, GC>;
      e.bwdc1_fn = (const void*)k_pfft_bwd_cols_tma1<SYM, Cfg, GC>;
      e.fwdc1 = [](const FwdArgs& a, const TileMaps& tm, const CUtensorMap& mi, const CUtensorMap& mo, int grid,
                   size_t sm, cudaStream_t s) {
        k_pfft_fwd_cols_tma1<SYM, Cfg, GC><<<grid, Cfg::T * GC, sm, s>>>(a, tm, mi, mo);
      };
      e.bwdc1 = [](const BwdArgs& a, const TileMaps& tm, const CUtensorMap& mi, int grid, size_t sm, cudaStream_t s) {
        k_pfft_bwd_cols_tma1<SYM, Cfg, GC><<<grid, Cfg::T * GC, sm, s>>>(a, tm, mi);
      };
    }
  }
  return e;
}

template <int SYM>
KernelEntry make_naive_entry() {
  KernelEntry e;
  e.Bc = 0;
  e.T = kNaiveT;
  e.G = 1;
  e.naive = true;
  e.radix = "direct";
  e.smem_conv = 3 * sizeof(double2);
  e.smem_fwd = 1 * sizeof(double2);
  e.smem_bwd = 2 * sizeof(double2);
  e.conv_fn = (const void*)k_conv1d_naive<SYM>;
  e.fwd_fn = (const void*)k_pfft_fwd_naive<SYM>;
  e.bwd_fn = (const void*)k_pfft_bwd_naive<SYM>;
  e.conv = [](const ConvArgs& a, int grid, size_t sm, cudaStream_t s) { k_conv1d_naive<SYM><<<grid, kNaiveT, sm, s>>>(a); };
  e.fwd = [](const FwdArgs& a, int grid, size_t sm, cudaStream_t s) { k_pfft_fwd_naive<SYM><<<grid, kNaiveT, sm, s>>>(a); };
  e.bwd = [](const BwdArgs& a, int grid, size_t sm, cudaStream_t s) { k_pfft_bwd_naive<SYM><<<grid, kNaiveT, sm, s>>>(a); };
  return e;
}

// 512-point plan occupancy knobs (A/B builds; c5's z-lines: one line group per CTA and 8 CTAs per
// SM measured 3 % faster than 2 groups x 4 CTAs, 0.586 -> 0.568 ms for 65536 Hermitian lines)
#ifndef HC_R512_G
#define HC_R512_G 1
#endif
#ifndef HC_R512_MINB
#define HC_R512_MINB 8
#endif
#ifndef HC_R6144_PLAN
#define HC_R6144_PLAN 1
#endif
#ifndef HC_R4096_MINB
#define HC_R4096_MINB 1
#endif
#ifndef HC_R4096_SMEM_STASH
#define HC_R4096_SMEM_STASH false
#endif
// (1024-point plan: G = 1 with 5 CTAs per SM measured no faster for c1, 0.0466 vs 0.0457 ms)
#ifndef HC_R1024_G
#define HC_R1024_G 2
#endif
#ifndef HC_R1024_MINB
#define HC_R1024_MINB 1
#endif
// Radix plans (complex FFT length -> passes, threads per line group, groups per CTA).  The table of a
// symmetry is built by two translation units (PART 0: blocks up to 3072 points, PART 1: the long
// blocks and the direct-sum entry) so that the build's critical path is half a symmetry.
template <int SYM, int PART>
inline void build_registry(KernelEntry* out, int* count) {
  int k = *count;
#ifdef HC_REGISTRY_MIN
  // development builds (make VARIANT=dev EXTRA=-DHC_REGISTRY_MIN): the plans of c3 / c4 / c5 only
  if constexpr (PART == 0) {
    out[k++] = make_entry<SYM, FFTCfg<Radices<8, 8, 8>, 64>, HC_R512_G, false, HC_R512_MINB>("8x8x8");
    out[k++] = make_entry<SYM, FFTCfg<Radices<16, 16, 3>, 64>, 2>("16x16x3");
  } else {
    out[k++] = make_entry<SYM, FFTCfg<Radices<16, 16, 16>, 256>, 1, HC_R4096_SMEM_STASH, HC_R4096_MINB>("16x16x16");
#ifdef HC_REGISTRY_C2  // + c2's 6144-point plan (the in-place kernel's host plumbing hangs off it)
    out[k++] = make_entry<SYM, FFTCfg<Radices<16, 16, 24>, 384>, 1>("16x16x24");
#endif
    out[k++] = make_naive_entry<SYM>();
  }
#else
  if constexpr (PART == 0) {
    out[k++] = make_entry<SYM, FFTCfg<Radices<8, 8>, 32>, 4, false, 4>("8x8");
    out[k++] = make_entry<SYM, FFTCfg<Radices<16, 8>, 32>, 4, false, 4>("16x8");
    out[k++] = make_entry<SYM, FFTCfg<Radices<4, 8, 8>, 32>, 4, false, 4>("4x8x8");
    // 384 = 8x8x6: the explicit 768-point Hermitian block of c5's z axis (M = 766)
    out[k++] = make_entry<SYM, FFTCfg<Radices<8, 8, 6>, 64>, 1, false, 8>("8x8x6");
    out[k++] = make_entry<SYM, FFTCfg<Radices<8, 8, 8>, 64>, HC_R512_G, false, HC_R512_MINB>("8x8x8");
    out[k++] = make_entry<SYM, FFTCfg<Radices<16, 16, 3>, 64>, 2>("16x16x3");
    out[k++] = make_entry<SYM, FFTCfg<Radices<16, 16, 4>, 64>, HC_R1024_G, false, HC_R1024_MINB>("16x16x4");
    out[k++] = make_entry<SYM, FFTCfg<Radices<16, 16, 6>, 96>, 1>("16x16x6");
    out[k++] = make_entry<SYM, FFTCfg<Radices<16, 16, 8>, 128>, 1, true, 3>("16x16x8");
    out[k++] = make_entry<SYM, FFTCfg<Radices<16, 16, 12>, 192>, 1>("16x16x12");
  } else {
    out[k++] = make_entry<SYM, FFTCfg<Radices<16, 16, 16>, 256>, 1, HC_R4096_SMEM_STASH, HC_R4096_MINB>("16x16x16");
    // measured on B200 (r01): 16x16x24/T384 1.146 ms for c2, 8x8x8x12/T768 1.231 ms
#if HC_R6144_PLAN == 2
    out[k++] = make_entry<SYM, FFTCfg<Radices<24, 16, 16>, 256>, 1>("24x16x16");
#else
    out[k++] = make_entry<SYM, FFTCfg<Radices<16, 16, 24>, 384>, 1>("16x16x24");
#endif
    // radix-7 plan: 3584 = 16 x 14 x 16 (the 7-smooth sizes of SPEC.md:523; DFT14 = 2 x 7 with the
    // pair-form DFT7): blocks of 3584 complex / 7168 Hermitian points
    out[k++] = make_entry<SYM, FFTCfg<Radices<16, 14, 16>, 256>, 1>("16x14x16");
    // radix-5 plan: 6000 = 10 x 24 x 25 (the 5-smooth sizes of SPEC.md:523's search space, e.g.
    // c2's m = 6000 = L, p = 1, q = 2)
    out[k++] = make_entry<SYM, FFTCfg<Radices<10, 24, 25>, 320>, 1>("10x24x25");
    out[k++] = make_naive_entry<SYM>();
  }
#endif
  *count = k;
}

}  // namespace hc
