// conv_ip.cuh — k_conv1d_ip: Alg. convolve for complex lines with L <= B,
// fused like k_conv1d_pp (kernels.cuh) but with IN-PLACE block FFT passes and the two forward
// transforms interleaved.
//
// The block FFT of N = R0 R1 R2 points runs as three decimation-in-frequency passes that read and
// write the SAME shared-memory positions (pass 0: butterfly b over elements N1 a + b; pass 1:
// sub-sequence k0, elements N1 k0 + N2 a + b1; pass 2: R2 contiguous elements), so the spectrum
// is left in digit-reversed positions.  A convolution does not care: F and G share the order, the
// product is pointwise, and the inverse runs the mirrored decimation-in-time passes from the same
// positions.  In place means
//   * no write-after-read hazard between the threads of a pass: ONE barrier per pass instead of
//     two, and it is split (arrive after the pass, wait before the next pass on that buffer);
//   * the f line (buffer X) and the g line (buffer Y) are transformed pass by pass, alternating,
//     each with its own barrier: a warp arrives on X's barrier, runs g's pass on Y, and by the
//     time it waits on X's barrier the other warps have arrived too.  Warps drift apart, so the
//     shared-memory phases of some overlap the FP64 phases of others (in k_conv1d_pp the whole
//     line group moves in lockstep and the two pipes take turns);
//   * the raw line staged by TMA is consumed in place by pass 0, the residue accumulator and the
//     first spectrum live in tensor memory, the last residue writes its outputs straight from
//     registers: Y is free as soon as the inverse's last pass has loaded it, and the next g line
//     is on its way while the outputs are computed.
// Bank conflicts: pass 2 reads R2 contiguous values per thread (a stride of R2 x 16 B between
// threads).  Positions are swizzled within aligned groups of 8 values, j -> j ^ ((j / R2) & 7):
// every quarter-warp access of every pass then covers the 8 distinct 16-byte slots of the 32
// banks (R1, R2 multiples of 8).  The swizzle permutes within 8 consecutive lanes of one warp, so
// pass 0 (linear reads of the TMA-staged line, swizzled writes) stays hazard-free across warps.
#pragma once
#include "kernels.cuh"

namespace hc {

// Split-phase barrier over the warps of a CTA: mbarrier with one arrival per warp.
struct WarpBar {
  uint32_t addr;
  uint32_t ph = 0;
  __device__ __forceinline__ void arrive() const {
    __syncwarp();
    if ((threadIdx.x & 31) == 0)
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
  }
  __device__ __forceinline__ void wait() {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITB_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITB_%=;\n"
        "}\n" ::"r"(addr),
        "r"(ph)
        : "memory");
    ph ^= 1;
  }
  // the phase completes without this thread waiting for it
  __device__ __forceinline__ void skip() { ph ^= 1; }
};

#ifndef HC_IP_DIRECT_OUT
#define HC_IP_DIRECT_OUT 1
#endif

template <int SYM, class Cfg>
__global__ void __launch_bounds__(Cfg::T, 1) k_conv1d_ip(ConvArgs p) {
  static_assert(SYM == SYM_COMPLEX, "in-place kernel: complex lines");
  static_assert(Cfg::P == 3, "three-pass plans");
  constexpr int T = Cfg::T, R0 = Cfg::R(0), R1 = Cfg::R(1), R2 = Cfg::R(2);
  constexpr int N = Cfg::N, N1 = R1 * R2, N2 = R2;
  constexpr int NB0 = N1, NB1 = R0 * R2, NB2 = R0 * R1;
  static_assert(NB0 <= T && NB1 <= T && NB2 <= T, "one butterfly per thread and pass");
  static_assert(NB0 % 32 == 0 && NB1 % 32 == 0 && NB2 % 32 == 0, "warp-uniform passes");
  static_assert(R1 % 8 == 0 && R2 % 8 == 0, "swizzle keys");
  using TL = TmemLayout<T, R2, R0>;
  static_assert(TL::FITS, "F and the accumulator live in tensor memory");
  extern __shared__ __align__(16) double2 smem[];
  __shared__ __align__(8) uint64_t bars[4];  // TMA f, TMA g, passes on X, passes on Y
  __shared__ uint32_t tm_base;
  const int tid = threadIdx.x;
  const AxisDev& a = p.ax;
  double2* tb = smem;
  const double2* mt = tb;
  // line buffers on a 128-byte boundary (the swizzle's bank argument)
  double2* X;
  {
    const uint32_t s0 = smem_u32(smem + a.tabn);
    X = smem + a.tabn + (((128u - (s0 & 127u)) & 127u) >> 4);
  }
  double2* Y = X + N;
  stage_tables(tb, a, a.tabn);
  uint64_t* bar_f = &bars[0];
  uint64_t* bar_g = &bars[1];
  if (tid == 0) {
    mbar_init(bar_f, 1);
    mbar_init(bar_g, 1);
    mbar_init(&bars[2], T / 32);
    mbar_init(&bars[3], T / 32);
    fence_mbar_init();
  }
  if (tid < 32) tmem_alloc(&tm_base, TL::COLS);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tf = TL::f_addr(tm_base), ta = TL::a_addr(tm_base);
  WarpBar bX{smem_u32(&bars[2])}, bY{smem_u32(&bars[3])};
  uint32_t ph_f = 0, ph_g = 0;
  const int L = a.L;
  const uint32_t row_bytes = (uint32_t)a.S * 16u;
  const long long step = gridDim.x;
  long long item = blockIdx.x;
  if (tid == 0 && item < p.lin.count) {
    tma_copy(X, p.f + p.lin.base(item), row_bytes, bar_f);
    tma_copy(Y, p.g + p.lin.base(item), row_bytes, bar_g);
  }
  // per-thread positions
  const int pos0 = tid ^ ((tid / R2) & 7);     // pass 0: element N1 k + tid sits at N1 k + pos0
  const int k0_1 = tid / N2, b1 = tid % N2;    // pass 1: sub-sequence and butterfly
  const int base1 = N1 * k0_1;
  const int base2 = N2 * tid, key2 = tid & 7;  // pass 2: butterfly tid, element a at base2 + (a ^ key2)
  const double scale = 1.0 / (double)a.qm;

  for (; item < p.lin.count; item += step) {
    const long long base = p.lin.base(item);
    const long long nitem = item + step;
    const long long nline = nitem < p.lin.count ? p.lin.base(nitem) : -1;
    if (tid == 0 && nline >= 0) {
      l2_prefetch(p.f + nline, row_bytes);
      l2_prefetch(p.g + nline, row_bytes);
    }
    for (int res = 0; res < a.n; ++res) {
      const bool last = res == a.n - 1;
      const long long nbase = !last ? base : nline;
      const P0Res<SYM> p0{&a, tb, res};
      const double2* U = tb + (a.oU + res * a.nu);
      // ---- pass 0 of f (X) and g (Y): raw line -> pre-twiddle -> DFT -> twiddle, in place
      auto fwd0 = [&](double2* Z) HC_INL {
        if (NB0 == T || tid < NB0) {
          double2 v[R0];
          sfor<R0>([&](auto Ai) HC_INL {
            const int s = N1 * Ai + tid;
            v[Ai] = s < L ? Z[s] : make_double2(0.0, 0.0);
          });
          if (res) sfor<R0>([&](auto Ai) HC_INL { v[Ai] = cmul(v[Ai], U[Ai]); });
          DFT<R0, +1>::run(v);
          pass0_twiddle<+1, R0>(v, tid, p0);
          __syncwarp();  // the swizzle moves values between lanes of the warp: all have loaded
          sfor<R0>([&](auto Ki) HC_INL { Z[N1 * Ki + pos0] = v[Ki]; });
        }
      };
      auto fwd1 = [&](double2* Z) HC_INL {
        if (NB1 == T || tid < NB1) {
          double2 v[R1];
          sfor<R1>([&](auto Ai) HC_INL { v[Ai] = Z[base1 + N2 * Ai + (b1 ^ (Ai & 7))]; });
          DFT<R1, +1>::run(v);
          sfor<R1 - 1>([&](auto Ki) HC_INL {
            constexpr int k = Ki + 1;
            v[k] = cmul(v[k], mt[(k - 1) * N2 + b1]);
          });
          sfor<R1>([&](auto Ki) HC_INL { Z[base1 + N2 * Ki + (b1 ^ (Ki & 7))] = v[Ki]; });
        }
      };
      mbar_wait(bar_f, ph_f);
      ph_f ^= 1;
      fwd0(X);
      bX.arrive();
      mbar_wait(bar_g, ph_g);
      ph_g ^= 1;
      fwd0(Y);
      bY.arrive();
      // ---- pass 1
      bX.wait();
      fwd1(X);
      bX.arrive();
      bY.wait();
      fwd1(Y);
      bY.arrive();
      // ---- pass 2 of f: spectrum to tensor memory; X is free once every warp has loaded
      bX.wait();
      {
        double2 v[R2];
        if (NB2 == T || tid < NB2) sfor<R2>([&](auto Ai) HC_INL { v[Ai] = X[base2 + (Ai ^ key2)]; });
        bX.arrive();
        if (NB2 == T || tid < NB2) {
          DFT<R2, +1>::run(v);
          tm_store<R2>(tf, v);
        }
      }
      if (tid == 0) {
        bX.wait();
        if (nbase >= 0) {
          fence_proxy_async_smem();
          tma_copy(X, p.f + nbase, row_bytes, bar_f);
        }
      } else {
        bX.skip();
      }
      // ---- pass 2 of g, product, inverse pass 2 (in registers), back to Y
      bY.wait();
      if (NB2 == T || tid < NB2) {
        double2 v[R2];
        sfor<R2>([&](auto Ai) HC_INL { v[Ai] = Y[base2 + (Ai ^ key2)]; });
        DFT<R2, +1>::run(v);
        tmem_wait_st();
        sfor<R2 / 4>([&](auto Ki) HC_INL {
          double2 F4[4];
          tm_ld4(tf + 16 * Ki, F4);
          sfor<4>([&](auto i) HC_INL { v[4 * Ki + i] = cmul(v[4 * Ki + i], F4[i]); });
        });
        DFT<R2, -1>::run(v);
        sfor<R2>([&](auto Ai) HC_INL { Y[base2 + (Ai ^ key2)] = v[Ai]; });
      }
      bY.arrive();
      // ---- inverse pass 1
      bY.wait();
      if (NB1 == T || tid < NB1) {
        double2 v[R1];
        sfor<R1>([&](auto Ki) HC_INL { v[Ki] = Y[base1 + N2 * Ki + (b1 ^ (Ki & 7))]; });
        sfor<R1 - 1>([&](auto Ki) HC_INL {
          constexpr int k = Ki + 1;
          v[k] = cmulc(v[k], mt[(k - 1) * N2 + b1]);
        });
        DFT<R1, -1>::run(v);
        sfor<R1>([&](auto Ai) HC_INL { Y[base1 + N2 * Ai + (b1 ^ (Ai & 7))] = v[Ai]; });
      }
      bY.arrive();
      // ---- inverse pass 0: Y is free once every warp has loaded; outputs from registers
      bY.wait();
      {
        double2 v[R0];
        const bool act = NB0 == T || tid < NB0;
        if (act) sfor<R0>([&](auto Ki) HC_INL { v[Ki] = Y[N1 * Ki + pos0]; });
        bY.arrive();
        if (tid == 0) {
          bY.wait();
          if (nbase >= 0) {
            fence_proxy_async_smem();
            tma_copy(Y, p.g + nbase, row_bytes, bar_g);
          }
        } else {
          bY.skip();
        }
        if (act) {
          pass0_twiddle<-1, R0>(v, tid, p0);
          DFT<R0, -1>::run(v);
          if (res) sfor<R0>([&](auto Ai) HC_INL { v[Ai] = cmulc(v[Ai], U[Ai]); });
        }
        // residue accumulator in the thread's own tensor-memory columns (warp-collective)
        if (NB0 == T || tid < NB0) {
          if (res > 0) {
            tmem_wait_st();
            sfor<R0 / 4>([&](auto Ki) HC_INL {
              double2 t4[4];
              tm_ld4(ta + 16 * Ki, t4);
              sfor<4>([&](auto i) HC_INL { v[4 * Ki + i] = cadd(v[4 * Ki + i], t4[i]); });
            });
          }
          if (!last) {
            tm_store<R0>(ta, v);
          } else {
            double2* o = p.out + base;
            sfor<R0>([&](auto Ai) HC_INL {
              const int s = N1 * Ai + tid;
              if (s < L) __stcs(o + s, cscale(v[Ai], scale));
            });
          }
        }
      }
    }
  }
  tmem_wait_st();
  tmem_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc(tm_base, TL::COLS);
}

// shared memory of k_conv1d_ip for `tabn` staged table entries (128 bytes of alignment slack)
template <class Cfg>
constexpr size_t conv_ip_smem(int tabn) {
  return ((size_t)tabn + 2 * (size_t)Cfg::N) * sizeof(double2) + 128;
}

}  // namespace hc
