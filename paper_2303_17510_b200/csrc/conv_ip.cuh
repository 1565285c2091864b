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
  bool off = false;  // diagnostics (HCONV_DBG bit 2): never wait (timing runs only, results are wrong)
  __device__ __forceinline__ void arrive() const {
    if (off) return;
    __syncwarp();
    if ((threadIdx.x & 31) == 0)
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
  }
  __device__ __forceinline__ void wait() {
    if (off) {
      ph ^= 1;
      return;
    }
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

// Load-order ring of k_conv1d_ip (HC_IP_RING): the three warps of every SM sub-partition (roles
// w / 4 = 0, 1, 2) would otherwise issue the loads of a pass in round-robin, receive their values
// at the same time, compete for the FP64 pipe at the same time and store at the same time -- the
// shared-memory pipe and the FP64 pipe taking turns.  The ring hands a token from role to role
// (named barriers, producer arrive / consumer sync): role 0's loads are queued first, it computes
// while roles 1 and 2 still load, stores while they compute, and the stagger persists through the
// alternating f / g passes (nothing re-aligns the roles until the next real barrier stall).
#ifndef HC_IP_RING
#define HC_IP_RING 1
#endif
__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
template <int PAR>
__device__ __forceinline__ void ring_acquire(int role) {
  if (HC_IP_RING) {
    if (role == 1) nbar_sync(1 + 2 * PAR, 256);
    if (role == 2) nbar_sync(2 + 2 * PAR, 256);
  }
}
template <int PAR>
__device__ __forceinline__ void ring_pass(int role) {
  if (HC_IP_RING) {
    if (role == 0) nbar_arrive(1 + 2 * PAR, 256);
    if (role == 1) nbar_arrive(2 + 2 * PAR, 256);
  }
}

#ifndef HC_IP2_F_TMEM
#define HC_IP2_F_TMEM 1
#endif
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
  const int role = tid >> 7;  // warp / 4: the SM sub-partition's first, second, third warp
  static_assert(!HC_IP_RING || T == 384, "load-order ring: three roles of four warps");
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
  bX.off = bY.off = (p.dbg & 2) != 0;
  const bool no_tm = (p.dbg & 4) != 0, no_out = (p.dbg & 1) != 0;  // diagnostics (timing runs only)
  // HCONV_TRACE: clock64 at the phase boundaries of warps 0, 5 and 11 of CTA 0 (128 stamps each)
  const int tw = tid == 0 ? 0 : tid == 5 * 32 ? 1 : tid == 11 * 32 ? 2 : -1;
  const bool tr = p.trace && blockIdx.x == 0 && tw >= 0;
  int tn = 0;
#define HC_TR()                                                              \
  do {                                                                       \
    if (tr && tn < 128) p.trace[tw * 128 + tn++] = (unsigned long long)clock64(); \
  } while (0)
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
      auto fwd0 = [&](double2* Z, auto Par) HC_INL {
        if (NB0 == T || tid < NB0) {
          double2 v[R0];
          ring_acquire<decltype(Par)::value>(role);
          sfor<R0>([&](auto Ai) HC_INL {
            const int s = N1 * Ai + tid;
            v[Ai] = s < L ? Z[s] : make_double2(0.0, 0.0);
          });
          ring_pass<decltype(Par)::value>(role);
          if (res) sfor<R0>([&](auto Ai) HC_INL { v[Ai] = cmul(v[Ai], U[Ai]); });
          DFT<R0, +1>::run(v);
          pass0_twiddle<+1, R0>(v, tid, p0);
          __syncwarp();  // the swizzle moves values between lanes of the warp: all have loaded
          sfor<R0>([&](auto Ki) HC_INL { Z[N1 * Ki + pos0] = v[Ki]; });
        }
      };
      auto fwd1 = [&](double2* Z, auto Par) HC_INL {
        ring_acquire<decltype(Par)::value>(role);
        if (NB1 == T || tid < NB1) {
          double2 v[R1];
          sfor<R1>([&](auto Ai) HC_INL { v[Ai] = Z[base1 + N2 * Ai + (b1 ^ (Ai & 7))]; });
          ring_pass<decltype(Par)::value>(role);
          DFT<R1, +1>::run(v);
          sfor<R1 - 1>([&](auto Ki) HC_INL {
            constexpr int k = Ki + 1;
            v[k] = cmul(v[k], mt[(k - 1) * N2 + b1]);
          });
          sfor<R1>([&](auto Ki) HC_INL { Z[base1 + N2 * Ki + (b1 ^ (Ki & 7))] = v[Ki]; });
        } else {
          ring_pass<decltype(Par)::value>(role);
        }
      };
      using P0_ = std::integral_constant<int, 0>;
      using P1_ = std::integral_constant<int, 1>;
      HC_TR();  // 0
      mbar_wait(bar_f, ph_f);
      ph_f ^= 1;
      HC_TR();  // 1: waited f
      fwd0(X, P0_{});
      bX.arrive();
      HC_TR();  // 2: pass 0 f
      mbar_wait(bar_g, ph_g);
      ph_g ^= 1;
      HC_TR();  // 3: waited g
      fwd0(Y, P1_{});
      bY.arrive();
      HC_TR();  // 4: pass 0 g
      // ---- pass 1
      bX.wait();
      HC_TR();  // 5
      fwd1(X, P0_{});
      bX.arrive();
      HC_TR();  // 6: pass 1 f
      bY.wait();
      HC_TR();  // 7
      fwd1(Y, P1_{});
      bY.arrive();
      HC_TR();  // 8: pass 1 g
      // ---- pass 2 of f: spectrum to tensor memory; X is free once every warp has loaded
      bX.wait();
      HC_TR();  // 9
      {
        double2 v[R2];
        ring_acquire<0>(role);
        if (NB2 == T || tid < NB2) sfor<R2>([&](auto Ai) HC_INL { v[Ai] = X[base2 + (Ai ^ key2)]; });
        ring_pass<0>(role);
        bX.arrive();
        if (NB2 == T || tid < NB2) {
          DFT<R2, +1>::run(v);
          if (!no_tm) tm_store<R2>(tf, v);
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
      HC_TR();  // 10: pass 2 f (+ thread 0's TMA issue)
      bY.wait();
      HC_TR();  // 11
      ring_acquire<1>(role);
      if (NB2 == T || tid < NB2) {
        double2 v[R2];
        sfor<R2>([&](auto Ai) HC_INL { v[Ai] = Y[base2 + (Ai ^ key2)]; });
        ring_pass<1>(role);
        DFT<R2, +1>::run(v);
        if (!no_tm) {
          tmem_wait_st();
          sfor<R2 / 4>([&](auto Ki) HC_INL {
            double2 F4[4];
            tm_ld4(tf + 16 * Ki, F4);
            sfor<4>([&](auto i) HC_INL { v[4 * Ki + i] = cmul(v[4 * Ki + i], F4[i]); });
          });
        } else {
          sfor<R2>([&](auto Ki) HC_INL { v[Ki] = cmul(v[Ki], v[(Ki + 1) % R2]); });
        }
        DFT<R2, -1>::run(v);
        sfor<R2>([&](auto Ai) HC_INL { Y[base2 + (Ai ^ key2)] = v[Ai]; });
      } else {
        ring_pass<1>(role);
      }
      bY.arrive();
      // ---- inverse pass 1
      HC_TR();  // 12: pass 2 g, product, inverse pass 2
      bY.wait();
      HC_TR();  // 13
      ring_acquire<0>(role);
      if (NB1 == T || tid < NB1) {
        double2 v[R1];
        sfor<R1>([&](auto Ki) HC_INL { v[Ki] = Y[base1 + N2 * Ki + (b1 ^ (Ki & 7))]; });
        ring_pass<0>(role);
        sfor<R1 - 1>([&](auto Ki) HC_INL {
          constexpr int k = Ki + 1;
          v[k] = cmulc(v[k], mt[(k - 1) * N2 + b1]);
        });
        DFT<R1, -1>::run(v);
        sfor<R1>([&](auto Ai) HC_INL { Y[base1 + N2 * Ai + (b1 ^ (Ai & 7))] = v[Ai]; });
      } else {
        ring_pass<0>(role);
      }
      bY.arrive();
      // ---- inverse pass 0: Y is free once every warp has loaded; outputs from registers
      HC_TR();  // 14: inverse pass 1
      bY.wait();
      HC_TR();  // 15
      {
        double2 v[R0];
        const bool act = NB0 == T || tid < NB0;
        ring_acquire<1>(role);
        if (act) sfor<R0>([&](auto Ki) HC_INL { v[Ki] = Y[N1 * Ki + pos0]; });
        ring_pass<1>(role);
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
          if (res > 0 && !no_tm) {
            tmem_wait_st();
            sfor<R0 / 4>([&](auto Ki) HC_INL {
              double2 t4[4];
              tm_ld4(ta + 16 * Ki, t4);
              sfor<4>([&](auto i) HC_INL { v[4 * Ki + i] = cadd(v[4 * Ki + i], t4[i]); });
            });
          }
          if (!last) {
            if (!no_tm) tm_store<R0>(ta, v);
            else if (v[0].x == 12345.678) p.out[0] = v[1];
          } else if (!no_out || v[0].x == 12345.678) {
            double2* o = p.out + base;
            sfor<R0>([&](auto Ai) HC_INL {
              const int s = N1 * Ai + tid;
              if (s < L) __stcs(o + s, cscale(v[Ai], scale));
            });
          }
        }
      }
      HC_TR();  // 16: inverse pass 0, outputs
    }
  }
#undef HC_TR
  tmem_wait_st();
  tmem_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc(tm_base, TL::COLS);
}

// ------------------------------------------------------------------------------------------
// k_conv1d_ip3: k_conv1d_ip with group-local hand-offs between passes 1 and 2.
//
// Only the pass 0 <-> pass 1 boundary is all-to-all.  After pass 0 the N-point line is R0
// independent sub-sequences; with R0 = 16 they form 4 groups of 4 sub-sequences (N / 4 points),
// each transformed in pass 1 by 2 warps (radix R1 = 24: 16 butterflies per sub-sequence) and in
// pass 2 by 3 warps (radix R2 = 16: 24 butterflies per sub-sequence).  The hand-off pass 1 ->
// pass 2 -> inverse pass 1 stays inside a group (one mbarrier per group, line and direction), so
// the groups -- and with them the shared-memory and FP64 phases of the warps -- drift apart
// instead of meeting at a CTA-wide barrier after every pass (tools/pipe_bench.cu: a barrier per
// pass costs 40 % on top of load -> butterflies -> store; without it the two pipes overlap to
// within 15 % of the FP64 time).  Pass 2 of f and g, the product and the inverse pass 2 are one
// step with F and G in registers (no stash: tensor-memory reads run at 64 B/clk, half the
// shared-memory rate).  CTA-wide barriers left per residue: pass 0 -> pass 1 of f and of g
// (hidden: the other line's pass runs in between) and inverse pass 1 -> inverse pass 0.
// DBG: compile-time diagnostics mask (timing builds only, HC_IP_DIAG in inst_ip.cu)
template <int SYM, class Cfg, int DBG = 0>
__global__ void __launch_bounds__(Cfg::T, 1) k_conv1d_ip3(ConvArgs p) {
  static_assert(SYM == SYM_COMPLEX, "in-place kernel: complex lines");
  static_assert(Cfg::P == 3, "three-pass plans");
  constexpr int T = Cfg::T, R0 = Cfg::R(0), R1 = Cfg::R(1), R2 = Cfg::R(2);
  constexpr int N = Cfg::N, N1 = R1 * R2, N2 = R2;
  constexpr int NB0 = N1, NB1 = R0 * R2, NB2 = R0 * R1;
  static_assert(T == 384 && NB0 == T && NB2 == T && NB1 == 256, "12 warps: pass 1 on 8, passes 0 and 2 on all");
  static_assert(R0 == 16 && R1 == 24 && R2 == 16, "4 groups of 4 sub-sequences: 2 pass-1 warps, 3 pass-2 warps each");
  // diagnostics (HCONV_DBG, timing runs only -- results are wrong): 1 no output stores, 4 no
  // accumulator, 8 no line copies (the buffers keep stale data)
  constexpr bool no_out = DBG & 1, no_acc = DBG & 4, no_tma = DBG & 8;
  // 16 / 32 / 64 / 128 / 256: skip pass 0 / pass 1 / pass 2 + product / inverse pass 1 / inverse pass 0
  constexpr bool sk0 = DBG & 16, sk1 = DBG & 32, sk2 = DBG & 64, sk3 = DBG & 128, sk4 = DBG & 256;
  extern __shared__ __align__(16) double2 smem[];
  __shared__ __align__(8) uint64_t bars[16];  // TMA f, TMA g, X, Y, then per group: pass 1 of f, of g, inverse pass 2
  __shared__ uint32_t tm_base;
  const int tid = threadIdx.x, w = tid >> 5;
  const AxisDev& a = p.ax;
  double2* tb = smem;
  const double2* mt = tb;
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
    for (int m = 0; m < 4; ++m) {
      mbar_init(&bars[4 + m], 2);   // pass 1 of f done in group m (2 warps)
      mbar_init(&bars[8 + m], 2);   // pass 1 of g
      mbar_init(&bars[12 + m], 3);  // inverse pass 2 (3 warps)
    }
    fence_mbar_init();
  }
  // residue accumulator in tensor memory: R0 values per thread
  using TL = TmemLayout<T, 0, R0>;
  static_assert(TL::FITS, "accumulator in tensor memory");
  if (tid < 32) tmem_alloc(&tm_base, TL::COLS);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t ta = TL::a_addr(tm_base);
  const int m1 = (w >> 1) & 3, m2 = w / 3;  // group as a pass-1 warp (w < 8) / as a pass-2 warp
  WarpBar bX{smem_u32(&bars[2])}, bY{smem_u32(&bars[3])};
  WarpBar gF1{smem_u32(&bars[4 + m1])}, gG1{smem_u32(&bars[8 + m1])};    // arrive (pass-1 warp)
  WarpBar gF2{smem_u32(&bars[4 + m2])}, gG2{smem_u32(&bars[8 + m2])};    // wait (pass-2 warp)
  WarpBar gI2{smem_u32(&bars[12 + m2])}, gI1{smem_u32(&bars[12 + m1])};  // arrive (pass 2) / wait (pass 1)
  if constexpr ((DBG & 512) != 0)  // free-running: no barrier at all (pass-0-only timing runs)
    bX.off = bY.off = gF1.off = gG1.off = gF2.off = gG2.off = gI2.off = gI1.off = true;
  uint32_t ph_f = 0, ph_g = 0;
  const int L = a.L;
  const uint32_t row_bytes = (uint32_t)a.S * 16u;
  const long long step = gridDim.x;
  long long item = blockIdx.x;
  if (tid == 0 && item < p.lin.count && !no_tma) {
    tma_copy(X, p.f + p.lin.base(item), row_bytes, bar_f);
    tma_copy(Y, p.g + p.lin.base(item), row_bytes, bar_g);
  }
  const int pos0 = tid ^ ((tid / R2) & 7);
  const int k0_1 = tid / N2, b1 = tid % N2;
  const int base1 = N1 * k0_1;
  const int base2 = N2 * tid, key2 = tid & 7;
  const double scale = 1.0 / (double)a.qm;
  const bool w1 = w < 8;  // pass-1 warp
  // HCONV_TRACE: clock64 at the phase boundaries of warps 0, 5 and 11 of CTA 0 (128 stamps each)
  const int tw = tid == 0 ? 0 : tid == 5 * 32 ? 1 : tid == 11 * 32 ? 2 : -1;
  const bool tr = p.trace && blockIdx.x == 0 && tw >= 0;
  int tn = 0;
#define HC_TR()                                                                   \
  do {                                                                            \
    if (tr && tn < 128) p.trace[tw * 128 + tn++] = (unsigned long long)clock64(); \
  } while (0)

  for (; item < p.lin.count; item += step) {
    const long long base = p.lin.base(item);
    const long long nitem = item + step;
    const long long nline = nitem < p.lin.count ? p.lin.base(nitem) : -1;
    if (tid == 0 && nline >= 0 && !no_tma) {
      l2_prefetch(p.f + nline, row_bytes);
      l2_prefetch(p.g + nline, row_bytes);
    }
    for (int res = 0; res < a.n; ++res) {
      const bool last = res == a.n - 1;
      const long long nbase = !last ? base : nline;
      const P0Res<SYM> p0{&a, tb, res};
      const double2* U = tb + (a.oU + res * a.nu);
      auto fwd0 = [&](double2* Z) HC_INL {
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
      };
      auto fwd1 = [&](double2* Z) HC_INL {
        double2 v[R1];
        sfor<R1>([&](auto Ai) HC_INL { v[Ai] = Z[base1 + N2 * Ai + (b1 ^ (Ai & 7))]; });
        DFT<R1, +1>::run(v);
        sfor<R1 - 1>([&](auto Ki) HC_INL {
          constexpr int k = Ki + 1;
          v[k] = cmul(v[k], mt[(k - 1) * N2 + b1]);
        });
        sfor<R1>([&](auto Ki) HC_INL { Z[base1 + N2 * Ki + (b1 ^ (Ki & 7))] = v[Ki]; });
      };
      if constexpr ((DBG & 1024) != 0) {
        // timing experiment: passes 0 and 1 of both lines only, every barrier hidden behind the other
        // line's pass (the steady state of a schedule without solo phases)
        if (item != blockIdx.x || res) bX.wait();
        fwd0(X);
        bX.arrive();
        if (item != blockIdx.x || res) bY.wait();
        fwd0(Y);
        bY.arrive();
        bX.wait();
        if (w1) fwd1(X);
        bX.arrive();
        bY.wait();
        if (w1) fwd1(Y);
        bY.arrive();
        continue;
      }
      // ---- pass 0 of f (X) and g (Y)
      HC_TR();  // 0
      if (!no_tma) mbar_wait(bar_f, ph_f);
      ph_f ^= 1;
      HC_TR();  // 1
      if constexpr (!sk0) fwd0(X);
      bX.arrive();
      HC_TR();  // 2
      if (!no_tma) mbar_wait(bar_g, ph_g);
      ph_g ^= 1;
      HC_TR();  // 3
      if constexpr (!sk0) fwd0(Y);
      bY.arrive();
      HC_TR();  // 4
      // ---- pass 1 (warps 0..7), handed to the group's pass-2 warps
      bX.wait();
      HC_TR();  // 5
      if (w1) {
        if constexpr (!sk1) fwd1(X);
        gF1.arrive();
      }
      HC_TR();  // 6
      bY.wait();
      HC_TR();  // 7
      if (w1) {
        if constexpr (!sk1) fwd1(Y);
        gG1.arrive();
      }
      HC_TR();  // 8
      // ---- pass 2 of f and g, product, inverse pass 2: F and G in registers
      {
        double2 vf[R2], vg[R2];
        gF2.wait();
        HC_TR();  // 9
        if constexpr (!sk2) sfor<R2>([&](auto Ai) HC_INL { vf[Ai] = X[base2 + (Ai ^ key2)]; });
        gG2.wait();
        HC_TR();  // 10
        if constexpr (!sk2) {
          sfor<R2>([&](auto Ai) HC_INL { vg[Ai] = Y[base2 + (Ai ^ key2)]; });
          DFT<R2, +1>::run(vf);
        }
        bX.arrive();  // (release: this warp's loads of X are performed) X is free once every warp is here
        if constexpr (!sk2) {
          DFT<R2, +1>::run(vg);
          sfor<R2>([&](auto Ki) HC_INL { vg[Ki] = cmul(vg[Ki], vf[Ki]); });
          DFT<R2, -1>::run(vg);
          sfor<R2>([&](auto Ai) HC_INL { Y[base2 + (Ai ^ key2)] = vg[Ai]; });
        }
        gI2.arrive();
      }
      HC_TR();  // 11
      if (tid == 0) {
        bX.wait();
        if (nbase >= 0 && !no_tma) {
          fence_proxy_async_smem();
          tma_copy(X, p.f + nbase, row_bytes, bar_f);
        }
      } else {
        bX.skip();
      }
      __syncwarp();
      // ---- inverse pass 1 (warps 0..7)
      HC_TR();  // 12
      if (w1) {
        double2 v[R1];
        gI1.wait();
        HC_TR();  // 13 (pass-1 warps only)
        if constexpr (!sk3) {
          sfor<R1>([&](auto Ki) HC_INL { v[Ki] = Y[base1 + N2 * Ki + (b1 ^ (Ki & 7))]; });
          sfor<R1 - 1>([&](auto Ki) HC_INL {
            constexpr int k = Ki + 1;
            v[k] = cmulc(v[k], mt[(k - 1) * N2 + b1]);
          });
          DFT<R1, -1>::run(v);
          sfor<R1>([&](auto Ai) HC_INL { Y[base1 + N2 * Ai + (b1 ^ (Ai & 7))] = v[Ai]; });
        }
      }
      bY.arrive();
      // ---- inverse pass 0: Y is free once every warp has loaded; outputs from registers
      HC_TR();  // 14 (13 for warps 8..11)
      bY.wait();
      HC_TR();  // 15
      {
        double2 v[R0];
        if constexpr (!sk4) sfor<R0>([&](auto Ki) HC_INL { v[Ki] = Y[N1 * Ki + pos0]; });
        bY.arrive();
        if (tid == 0) {
          bY.wait();
          if (nbase >= 0 && !no_tma) {
            fence_proxy_async_smem();
            tma_copy(Y, p.g + nbase, row_bytes, bar_g);
          }
        } else {
          bY.skip();
        }
        __syncwarp();
        if constexpr (!sk4) {
          pass0_twiddle<-1, R0>(v, tid, p0);
          DFT<R0, -1>::run(v);
          if (res) sfor<R0>([&](auto Ai) HC_INL { v[Ai] = cmulc(v[Ai], U[Ai]); });
        }
        if (res > 0 && !no_acc) {
          tmem_wait_st();
          sfor<R0 / 4>([&](auto Ki) HC_INL {
            double2 t4[4];
            tm_ld4(ta + 16 * Ki, t4);
            sfor<4>([&](auto i) HC_INL { v[4 * Ki + i] = cadd(v[4 * Ki + i], t4[i]); });
          });
        }
        if (!last) {
          if (!no_acc) tm_store<R0>(ta, v);
          else if (v[0].x == 12345.678) p.out[0] = v[1];
        } else if (!no_out || v[0].x == 12345.678) {
          double2* o = p.out + base;
          sfor<R0>([&](auto Ai) HC_INL {
            const int s = N1 * Ai + tid;
            if (s < L) __stcs(o + s, cscale(v[Ai], scale));
          });
        }
      }
      HC_TR();  // 16
    }
  }
#undef HC_TR
  tmem_wait_st();
  tmem_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc(tm_base, TL::COLS);
}

// ------------------------------------------------------------------------------------------
// k_conv1d_ip4: both residues of a line at once (plans with n = 2 residue blocks).
//
// Measured on k_conv1d_ip3 (compile-time diagnostics, inst_ip.cu): its phases cost the sum of
// what each costs alone, and a chain of phases whose barriers are all hidden behind another
// line's phase runs 35 % faster than the same phases followed by solo phases -- every real
// barrier stall re-aligns the warps, and aligned warps load together, compute together and store
// together.  Here no phase is solo: residue 0 of the line lives in buffer X, residue 1 in buffer Y,
// each buffer runs the whole chain f: pass 0, 1, 2 (F to tensor memory) -> g: pass 0, 1, 2 + product
// + inverse pass 2 -> inverse pass 1 -> inverse pass 0 in place, and every warp alternates
// between the two buffers phase by phase, so each barrier has the other residue's phase to
// complete behind.  The two inverse outputs meet in registers (same thread, same elements): no
// residue accumulator.  A buffer is refilled (g after pass 2 of f, the next line's f after inverse
// pass 0) by whichever warp is last to finish loading it (shared-memory counter): nobody waits.
struct IpChain {
  double2* Z;         // line buffer
  int res;            // residue block
  WarpBar b;          // CTA-wide barrier of the buffer
  WarpBar g1a, g1w;   // pass 1 done in a group: arrive (pass-1 warp's group) / wait (pass-2 warp's group)
  WarpBar gIa, gIw;   // inverse pass 2 done in a group: arrive (pass-2 warp) / wait (pass-1 warp)
  uint64_t* bar_tma;  // line copies into the buffer
  uint32_t ph_tma;
  uint32_t tf;        // the thread's F columns in tensor memory
  int* readers;       // warps that have finished loading the buffer in the current phase
};

template <int SYM, class Cfg>
__global__ void __launch_bounds__(Cfg::T, 1) k_conv1d_ip4(ConvArgs p) {
  static_assert(SYM == SYM_COMPLEX, "in-place kernel: complex lines");
  static_assert(Cfg::P == 3, "three-pass plans");
  constexpr int T = Cfg::T, R0 = Cfg::R(0), R1 = Cfg::R(1), R2 = Cfg::R(2);
  constexpr int N = Cfg::N, N1 = R1 * R2, N2 = R2;
  static_assert(T == 384 && R0 == 16 && R1 == 24 && R2 == 16, "12 warps; 4 groups: 2 pass-1 warps, 3 pass-2 warps");
  extern __shared__ __align__(16) double2 smem[];
  // TMA X, TMA Y, barrier X, barrier Y, then per buffer and group: pass 1 done, inverse pass 2 done
  __shared__ __align__(8) uint64_t bars[20];
  __shared__ int readers[2];
  __shared__ uint32_t tm_base;
  const int tid = threadIdx.x, w = tid >> 5;
  const AxisDev& a = p.ax;
  double2* tb = smem;
  const double2* mt = tb;
  double2* X;
  {
    const uint32_t s0 = smem_u32(smem + a.tabn);
    X = smem + a.tabn + (((128u - (s0 & 127u)) & 127u) >> 4);
  }
  stage_tables(tb, a, a.tabn);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], T / 32);
    mbar_init(&bars[3], T / 32);
    for (int i = 0; i < 8; ++i) {
      mbar_init(&bars[4 + i], 2);   // pass 1 done (2 warps): buffer i / 4, group i % 4
      mbar_init(&bars[12 + i], 3);  // inverse pass 2 done (3 warps)
    }
    readers[0] = readers[1] = 0;
    fence_mbar_init();
  }
  using TL = TmemLayout<T, 2 * R2, 0>;  // F of both residues
  static_assert(TL::FITS, "both spectra in tensor memory");
  if (tid < 32) tmem_alloc(&tm_base, TL::COLS);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const int m1 = (w >> 1) & 3, m2 = w / 3;  // group as a pass-1 warp (w < 8) / as a pass-2 warp
  IpChain cA{X, 0, {smem_u32(&bars[2])}, {smem_u32(&bars[4 + m1])}, {smem_u32(&bars[4 + m2])},
             {smem_u32(&bars[12 + m2])}, {smem_u32(&bars[12 + m1])}, &bars[0], 0u, TL::f_addr(tm_base), &readers[0]};
  IpChain cB{X + N, 1, {smem_u32(&bars[3])}, {smem_u32(&bars[8 + m1])}, {smem_u32(&bars[8 + m2])},
             {smem_u32(&bars[16 + m2])}, {smem_u32(&bars[16 + m1])}, &bars[1], 0u, TL::f_addr(tm_base) + 4 * R2, &readers[1]};
  const int L = a.L;
  const uint32_t row_bytes = (uint32_t)a.S * 16u;
  const long long step = gridDim.x;
  long long item = blockIdx.x;
  if (tid == 0 && item < p.lin.count) {
    tma_copy(cA.Z, p.f + p.lin.base(item), row_bytes, cA.bar_tma);
    tma_copy(cB.Z, p.f + p.lin.base(item), row_bytes, cB.bar_tma);
  }
  const int pos0 = tid ^ ((tid / R2) & 7);
  const int k0_1 = tid / N2, b1 = tid % N2;
  const int base1 = N1 * k0_1;
  const int base2 = N2 * tid, key2 = tid & 7;
  const double scale = 1.0 / (double)a.qm;
  const bool w1 = w < 8;  // pass-1 warp
  const double2* U1 = tb + (a.oU + a.nu);  // residue 1

  // the warp has finished loading the chain's buffer; the last one refills it from `src`
  auto release = [&](IpChain& c, const double2* src) HC_INL {
    __syncwarp();
    if ((tid & 31) == 0) {
      const int old = atomicAdd(c.readers, 1);
      if (old == T / 32 - 1) {
        *c.readers = 0;
        if (src) {
          fence_proxy_async_smem();
          tma_copy(c.Z, src, row_bytes, c.bar_tma);
        }
      }
    }
  };
  auto wait_line = [&](IpChain& c) HC_INL {
    mbar_wait(c.bar_tma, c.ph_tma);
    c.ph_tma ^= 1;
  };
  auto fwd0 = [&](IpChain& c) HC_INL {
    const P0Res<SYM> p0{&a, tb, c.res};
    double2* Z = c.Z;
    double2 v[R0];
    sfor<R0>([&](auto Ai) HC_INL {
      const int s = N1 * Ai + tid;
      v[Ai] = s < L ? Z[s] : make_double2(0.0, 0.0);
    });
    if (c.res) sfor<R0>([&](auto Ai) HC_INL { v[Ai] = cmul(v[Ai], U1[Ai]); });
    DFT<R0, +1>::run(v);
    pass0_twiddle<+1, R0>(v, tid, p0);
    __syncwarp();  // the swizzle moves values between lanes of the warp: all have loaded
    sfor<R0>([&](auto Ki) HC_INL { Z[N1 * Ki + pos0] = v[Ki]; });
    c.b.arrive();
  };
  auto fwd1 = [&](IpChain& c) HC_INL {
    c.b.wait();
    if (w1) {
      double2* Z = c.Z;
      double2 v[R1];
      sfor<R1>([&](auto Ai) HC_INL { v[Ai] = Z[base1 + N2 * Ai + (b1 ^ (Ai & 7))]; });
      DFT<R1, +1>::run(v);
      sfor<R1 - 1>([&](auto Ki) HC_INL {
        constexpr int k = Ki + 1;
        v[k] = cmul(v[k], mt[(k - 1) * N2 + b1]);
      });
      sfor<R1>([&](auto Ki) HC_INL { Z[base1 + N2 * Ki + (b1 ^ (Ki & 7))] = v[Ki]; });
      c.g1a.arrive();
    }
  };

  for (; item < p.lin.count; item += step) {
    const long long base = p.lin.base(item);
    const long long nitem = item + step;
    const long long nline = nitem < p.lin.count ? p.lin.base(nitem) : -1;
    if (tid == 0 && nline >= 0) {
      l2_prefetch(p.f + nline, row_bytes);
      l2_prefetch(p.g + nline, row_bytes);
    }
    const double2* gsrc = p.g + base;
    const double2* fnext = nline >= 0 ? p.f + nline : nullptr;
    // ---- f: passes 0, 1, 2; the spectrum goes to tensor memory, the buffer is refilled with g
    wait_line(cA);
    fwd0(cA);
    wait_line(cB);
    fwd0(cB);
    fwd1(cA);
    fwd1(cB);
    auto fwd2f = [&](IpChain& c) HC_INL {
      double2 v[R2];
      c.g1w.wait();
      sfor<R2>([&](auto Ai) HC_INL { v[Ai] = c.Z[base2 + (Ai ^ key2)]; });
      DFT<R2, +1>::run(v);
      release(c, gsrc);
      tm_store<R2>(c.tf, v);
    };
    fwd2f(cA);
    fwd2f(cB);
    // ---- g: passes 0, 1, 2 + product + inverse pass 2
    wait_line(cA);
    fwd0(cA);
    wait_line(cB);
    fwd0(cB);
    fwd1(cA);
    fwd1(cB);
    auto fwd2g = [&](IpChain& c) HC_INL {
      double2 v[R2];
      c.g1w.wait();
      sfor<R2>([&](auto Ai) HC_INL { v[Ai] = c.Z[base2 + (Ai ^ key2)]; });
      DFT<R2, +1>::run(v);
      tmem_wait_st();
      sfor<R2 / 4>([&](auto Ki) HC_INL {
        double2 F4[4];
        tm_ld4(c.tf + 16 * Ki, F4);
        sfor<4>([&](auto i) HC_INL { v[4 * Ki + i] = cmul(v[4 * Ki + i], F4[i]); });
      });
      DFT<R2, -1>::run(v);
      sfor<R2>([&](auto Ai) HC_INL { c.Z[base2 + (Ai ^ key2)] = v[Ai]; });
      c.gIa.arrive();
    };
    fwd2g(cA);
    fwd2g(cB);
    // ---- inverse pass 1 (warps 0..7)
    auto inv1 = [&](IpChain& c) HC_INL {
      if (w1) {
        double2* Z = c.Z;
        double2 v[R1];
        c.gIw.wait();
        sfor<R1>([&](auto Ki) HC_INL { v[Ki] = Z[base1 + N2 * Ki + (b1 ^ (Ki & 7))]; });
        sfor<R1 - 1>([&](auto Ki) HC_INL {
          constexpr int k = Ki + 1;
          v[k] = cmulc(v[k], mt[(k - 1) * N2 + b1]);
        });
        DFT<R1, -1>::run(v);
        sfor<R1>([&](auto Ai) HC_INL { Z[base1 + N2 * Ai + (b1 ^ (Ai & 7))] = v[Ai]; });
      }
      c.b.arrive();
    };
    inv1(cA);
    inv1(cB);
    // ---- inverse pass 0 of both residues; their sum is the output (both in this thread's registers)
    double2 h[R0];
    {
      const P0Res<SYM> p0{&a, tb, 0};
      cA.b.wait();
      sfor<R0>([&](auto Ki) HC_INL { h[Ki] = cA.Z[N1 * Ki + pos0]; });
      pass0_twiddle<-1, R0>(h, tid, p0);
      release(cA, fnext);
      DFT<R0, -1>::run(h);
    }
    {
      const P0Res<SYM> p0{&a, tb, 1};
      double2 v[R0];
      cB.b.wait();
      sfor<R0>([&](auto Ki) HC_INL { v[Ki] = cB.Z[N1 * Ki + pos0]; });
      pass0_twiddle<-1, R0>(v, tid, p0);
      release(cB, fnext);
      DFT<R0, -1>::run(v);
      double2* o = p.out + base;
      sfor<R0>([&](auto Ai) HC_INL {
        const int s = N1 * Ai + tid;
        const double2 x = cadd(h[Ai], cmulc(v[Ai], U1[Ai]));
        if (s < L) __stcs(o + s, cscale(x, scale));
      });
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc(tm_base, TL::COLS);
}

// ------------------------------------------------------------------------------------------
// k_conv1d_ip2: the same in-place passes, software-pipelined inside each thread.
//
// k_conv1d_ip's warps move in phase (fair scheduling keeps them together), so within a pass
// every warp loads, then every warp computes, then every warp stores: the shared-memory pipe and
// the FP64 pipe still take turns.  Here a CTA of 8 warps (255 registers per thread) treats a
// radix-R0/R1 pass over a line as 12 jobs of 32 butterflies and each warp runs 3 jobs per pass
// pair (f line in X, g line in Y) -- warps 0..3: X, X, Y; warps 4..7: X, Y, Y -- with two
// register sets: the loads of job k+1 are issued before the butterflies of job k, the stores of
// job k drain behind the butterflies of job k+1.  Each SM sub-partition hosts one warp of each
// flavour, i.e. 3 jobs per line and pass.  Every warp does its X jobs first, so X's barrier
// completes two thirds into the pass and the first loads of the next pass are issued before the
// pass's last butterflies; Y's barrier is only needed a job later.  Pass 2 (256 radix-24
// butterflies, one per thread) keeps F in registers next to G: no stash at all.  The inverse
// (one line) runs 2 jobs on warps 0..3 and 1 on warps 4..7 per pass.
template <int SYM, class Cfg>
__global__ void __launch_bounds__(256, 1) k_conv1d_ip2(ConvArgs p) {
  static_assert(SYM == SYM_COMPLEX, "in-place kernel: complex lines");
  static_assert(Cfg::P == 3, "three-pass plans");
  constexpr int T = 256, R0 = Cfg::R(0), R1 = Cfg::R(1), R2 = Cfg::R(2);
  constexpr int N = Cfg::N, N1 = R1 * R2, N2 = R2;
  static_assert(R0 == 16 && R1 == 16, "two register sets of 16 values");
  static_assert(N1 == 12 * 32 && R0 * R2 == 12 * 32, "12 jobs of 32 butterflies in passes 0 and 1");
  static_assert(R0 * R1 == T, "one pass-2 butterfly per thread");
  static_assert(R1 % 8 == 0 && R2 % 8 == 0, "swizzle keys");
  extern __shared__ __align__(16) double2 smem[];
  __shared__ __align__(8) uint64_t bars[4];  // TMA f, TMA g, passes on X, passes on Y
  __shared__ uint32_t tm_base;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const bool fa = w < 4;  // flavour A: jobs X, X, Y; flavour B: X, Y, Y
  const int u = w & 3;
  const AxisDev& a = p.ax;
  double2* tb = smem;
  const double2* mt = tb;
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
  // residue accumulator in tensor memory: per lane quarter, flavour A's two jobs then B's one
  // (HC_IP2_F_TMEM: F too, behind the accumulators, instead of registers)
  constexpr int TM_COLS = HC_IP2_F_TMEM ? 512 : 256;
  if (tid < 32) tmem_alloc(&tm_base, TM_COLS);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t ta = tm_base + ((32u * (uint32_t)u) << 16) + (fa ? 0u : 128u);
  const uint32_t tal = fa ? ta + 64 : ta;
  const uint32_t tf = tm_base + ((32u * (uint32_t)u) << 16) + 192u + (fa ? 0u : 96u);
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
  // jobs of the pair passes: butterflies 32 job + lane of the line in Z1 / Z2 / Z3
  double2* const Z1 = X;
  double2* const Z2 = fa ? X : Y;
  double2* const Z3 = Y;
  const int be1_ = 32 * (fa ? u : 8 + u) + lane;
  const double scale = 1.0 / (double)a.qm;

  // ---- building blocks (be: butterfly index of the job)
  auto ld0 = [&](double2(&v)[16], const double2* Z, int be) HC_INL {
    sfor<R0>([&](auto Ai) HC_INL {
      const int s = N1 * Ai + be;
      v[Ai] = s < L ? Z[s] : make_double2(0.0, 0.0);
    });
  };
  auto pos0 = [&](int be) HC_INL { return be ^ ((be / R2) & 7); };
  auto st0 = [&](const double2(&v)[16], double2* Z, int be) HC_INL {
    const int q = pos0(be);
    __syncwarp();  // the swizzle moves values between lanes of the warp: all have loaded
    sfor<R0>([&](auto Ki) HC_INL { Z[N1 * Ki + q] = v[Ki]; });
  };
  auto ld1 = [&](double2(&v)[16], const double2* Z, int be) HC_INL {
    const int k0 = be / N2, b1 = be - k0 * N2;
    const double2* zz = Z + N1 * k0;
    sfor<R1>([&](auto Ai) HC_INL { v[Ai] = zz[N2 * Ai + (b1 ^ (Ai & 7))]; });
  };
  auto st1 = [&](const double2(&v)[16], double2* Z, int be) HC_INL {
    const int k0 = be / N2, b1 = be - k0 * N2;
    double2* zz = Z + N1 * k0;
    sfor<R1>([&](auto Ai) HC_INL { zz[N2 * Ai + (b1 ^ (Ai & 7))] = v[Ai]; });
  };
  auto ldk0 = [&](double2(&v)[16], const double2* Z, int be) HC_INL {  // pass-0 outputs (inverse pass 0 input)
    const int q = pos0(be);
    sfor<R0>([&](auto Ki) HC_INL { v[Ki] = Z[N1 * Ki + q]; });
  };

  double2 va[16], vb[16];
  // first job of pass 0 (line f in X) for the first line
  if (item < p.lin.count) {
    mbar_wait(bar_f, ph_f);
    ph_f ^= 1;
    ld0(va, Z1, be1_);
  }
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
      // butterfly indices recomputed per residue behind an opaque zero: hoisted out of the loops the
      // dozens of shared-memory offsets derived from them would be spilled to local memory
      int lz;
      asm volatile("mov.b32 %0, %1;" : "=r"(lz) : "r"(lane));
      const int be1 = 32 * (fa ? u : 8 + u) + lz;
      const int be2 = 32 * (fa ? u + 4 : u) + lz;
      const int be3 = 32 * (fa ? 8 + u : u + 4) + lz;
      // jobs of the inverse (line in Y): A: u, u + 4; B: 8 + u
      const int bi1 = be1;
      const int bi2 = 32 * (u + 4) + lz;  // flavour A only
      const int bil = fa ? bi2 : bi1;     // the warp's last inverse job (register set vb)
      const int tidz = 32 * w + lz;
      const int base2 = N2 * tidz, key2 = tidz & 7;  // pass 2
      auto c0 = [&](double2(&v)[16], int be) HC_INL {
        if (res) sfor<R0>([&](auto Ai) HC_INL { v[Ai] = cmul(v[Ai], U[Ai]); });
        DFT<R0, +1>::run(v);
        pass0_twiddle<+1, R0>(v, be, p0);
      };
      auto c1 = [&](double2(&v)[16], int be) HC_INL {
        const int b1 = be % N2;
        DFT<R1, +1>::run(v);
        sfor<R1 - 1>([&](auto Ki) HC_INL {
          constexpr int k = Ki + 1;
          v[k] = cmul(v[k], mt[(k - 1) * N2 + b1]);
        });
      };
      // ---- pass 0 (va holds job 1, loaded ahead)
      if (!fa) {
        mbar_wait(bar_g, ph_g);
      }
      ld0(vb, Z2, be2);
      c0(va, be1);
      st0(va, Z1, be1);
      if (!fa) bX.arrive();
      if (fa) {
        mbar_wait(bar_g, ph_g);
      }
      ph_g ^= 1;
      ld0(va, Z3, be3);
      c0(vb, be2);
      st0(vb, Z2, be2);
      if (fa) bX.arrive();
      bX.wait();
      ld1(vb, Z1, be1);  // pass 1, job 1
      c0(va, be3);
      st0(va, Z3, be3);
      bY.arrive();
      // ---- pass 1 (vb holds job 1)
      if (!fa) bY.wait();
      ld1(va, Z2, be2);
      c1(vb, be1);
      st1(vb, Z1, be1);
      if (!fa) bX.arrive();
      if (fa) bY.wait();
      ld1(vb, Z3, be3);
      c1(va, be2);
      st1(va, Z2, be2);
      if (fa) bX.arrive();
      bX.wait();
      double2 vf[R2], vg[R2];
      sfor<R2>([&](auto Ai) HC_INL { vf[Ai] = X[base2 + (Ai ^ key2)]; });  // pass 2 of f
      c1(vb, be3);
      st1(vb, Z3, be3);
      bY.arrive();
      // ---- pass 2: F and G in registers, product, inverse pass 2, back to Y
      bY.wait();
      sfor<R2>([&](auto Ai) HC_INL { vg[Ai] = Y[base2 + (Ai ^ key2)]; });
      DFT<R2, +1>::run(vf);
      bX.arrive();  // X has been read by this warp
      if (tid == 0) {
        bX.wait();
        if (nbase >= 0) {
          fence_proxy_async_smem();
          tma_copy(X, p.f + nbase, row_bytes, bar_f);
        }
      } else {
        bX.skip();
      }
      __syncwarp();
      if constexpr (HC_IP2_F_TMEM) tm_store<R2>(tf, vf);
      DFT<R2, +1>::run(vg);
      if constexpr (HC_IP2_F_TMEM) {
        tmem_wait_st();
        sfor<R2 / 4>([&](auto Ki) HC_INL {
          double2 F4[4];
          tm_ld4(tf + 16 * Ki, F4);
          sfor<4>([&](auto i) HC_INL { vg[4 * Ki + i] = cmul(vg[4 * Ki + i], F4[i]); });
        });
      } else {
        sfor<R2>([&](auto Ki) HC_INL { vg[Ki] = cmul(vg[Ki], vf[Ki]); });
      }
      DFT<R2, -1>::run(vg);
      sfor<R2>([&](auto Ai) HC_INL { Y[base2 + (Ai ^ key2)] = vg[Ai]; });
      bY.arrive();
      // ---- inverse pass 1 (Y): A two jobs, B one
      auto ci1 = [&](double2(&v)[16], int be) HC_INL {
        const int b1 = be % N2;
        sfor<R1 - 1>([&](auto Ki) HC_INL {
          constexpr int k = Ki + 1;
          v[k] = cmulc(v[k], mt[(k - 1) * N2 + b1]);
        });
        DFT<R1, -1>::run(v);
      };
      bY.wait();
      if (fa) ld1(va, Y, bi1);
      ld1(vb, Y, bil);
      if (fa) {
        ci1(va, bi1);
        st1(va, Y, bi1);
      }
      ci1(vb, bil);
      st1(vb, Y, bil);
      bY.arrive();
      // ---- inverse pass 0: outputs from registers, accumulator in tensor memory
      auto ci0 = [&](double2(&v)[16], int be, uint32_t tacc) HC_INL {
        pass0_twiddle<-1, R0>(v, be, p0);
        DFT<R0, -1>::run(v);
        if (res) sfor<R0>([&](auto Ai) HC_INL { v[Ai] = cmulc(v[Ai], U[Ai]); });
        if (res > 0) {
          tmem_wait_st();
          sfor<R0 / 4>([&](auto Ki) HC_INL {
            double2 t4[4];
            tm_ld4(tacc + 16 * Ki, t4);
            sfor<4>([&](auto i) HC_INL { v[4 * Ki + i] = cadd(v[4 * Ki + i], t4[i]); });
          });
        }
        if (!last) {
          tm_store<R0>(tacc, v);
        } else {
          double2* o = p.out + base;
          sfor<R0>([&](auto Ai) HC_INL {
            const int s = N1 * Ai + be;
            if (s < L) __stcs(o + s, cscale(v[Ai], scale));
          });
        }
      };
      bY.wait();
      if (fa) ldk0(va, Y, bi1);
      ldk0(vb, Y, bil);
      bY.arrive();  // (release: the loads above are performed) Y is free once every warp is here
      if (tid == 0) {
        bY.wait();
        if (nbase >= 0) {
          fence_proxy_async_smem();
          tma_copy(Y, p.g + nbase, row_bytes, bar_g);
        }
      } else {
        bY.skip();
      }
      __syncwarp();
      if (fa) ci0(va, bi1, ta);
      // first job of the next pass 0 (f line in X, on its way since pass 2), behind the last butterflies
      if (nbase >= 0) {
        mbar_wait(bar_f, ph_f);
        ph_f ^= 1;
        ld0(va, Z1, be1);
      }
      ci0(vb, bil, tal);
    }
  }
  tmem_wait_st();
  tmem_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc(tm_base, TM_COLS);
}

// shared memory of k_conv1d_ip for `tabn` staged table entries (128 bytes of alignment slack)
template <class Cfg>
constexpr size_t conv_ip_smem(int tabn) {
  return ((size_t)tabn + 2 * (size_t)Cfg::N) * sizeof(double2) + 128;
}

}  // namespace hc
