// conv_ip.cuh — k_conv1d_ip4: Alg. convolve for complex lines with L <= B and
// n = 2 residue blocks (c2: L = 6000, m = 6144, q = 2), fused like k_conv1d_pp (kernels.cuh) but with
// IN-PLACE block-FFT passes, group-local hand-offs and both residues in flight.
//
// In-place passes.  The block FFT of N = R0 R1 R2 points runs as three decimation-in-frequency
// passes that read and write the SAME shared-memory positions (pass 0: butterfly b over elements
// N1 a + b; pass 1: sub-sequence k0, elements N1 k0 + N2 a + b1; pass 2: R2 contiguous elements), so
// the spectrum is left in digit-reversed positions.  A convolution does not care: F and G share the
// order, the product is pointwise, and the inverse runs the mirrored decimation-in-time passes from
// the same positions.  No write-after-read hazard between the threads of a pass: ONE barrier per
// pass instead of two, and it is split (arrive after the pass, wait before the next pass on that
// buffer).  The raw line staged by TMA is consumed in place by pass 0; the last pass writes its
// outputs straight from registers.
//
// Bank conflicts.  Pass 2 reads R2 contiguous values per thread (a stride of R2 x 16 B between
// threads).  Positions are swizzled within aligned groups of 8 values, j -> j ^ ((j / R2) & 7):
// every quarter-warp access of every pass then covers the 8 distinct 16-byte slots of the 32
// banks (R1, R2 multiples of 8).  The swizzle permutes within 8 consecutive lanes of one warp, so
// pass 0 (linear reads of the TMA-staged line, swizzled writes) stays hazard-free across warps.
//
// Group-local hand-offs.  Only the pass 0 <-> pass 1 boundary is all-to-all.  After pass 0 the line
// is R0 = 16 independent sub-sequences; they form 4 groups of 4, each transformed in pass 1 (radix
// 24) by 2 warps and in pass 2 (radix 16) by 3 warps.  Pass 1 -> pass 2 -> inverse pass 1 hand over
// inside a group (one mbarrier per group and direction).
//
// What the measurements said (tools/pipe_bench.cu, and compile-time variants of this kernel with
// phases removed): load -> butterflies -> store loops overlap the shared-memory pipe and the FP64
// pipe to within 15 % of the FP64 time as long as the warps drift freely; every real barrier stall
// re-aligns them, and aligned warps load together, compute together and store together (a phase
// then costs shared-memory time PLUS FP64 time).  A chain of phases whose barriers all complete
// behind another line's phase runs at the free-running speed.  Variants that kept solo phases (one
// line per CTA with f in X and g in Y: the f / g passes paired but pass 2, the inverse passes solo;
// 8 warps with software-pipelined jobs; a token ring ordering the loads of the three warps of a
// sub-partition) all landed on the ping-pong kernel's 0.76 ms for c2.
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

// Both residues of a line at once.  Residue 0 of the line lives in buffer X, residue 1 in buffer Y;
// each buffer runs the whole chain  f: pass 0, 1, 2 (F to tensor memory)  ->  g: pass 0, 1, 2 + product
// + inverse pass 2  ->  inverse pass 1  ->  inverse pass 0  in place, and every warp alternates between
// the two buffers phase by phase, so each barrier has the other residue's phase to complete behind:
// no phase is solo.  The two inverse outputs meet in registers (same thread, same elements): no
// residue accumulator.  A buffer is refilled (g after pass 2 of f, the next line's f after inverse
// pass 0) by whichever warp is last to finish loading it (shared-memory counter): nobody waits.
// Measured and dropped: buffer Y one phase behind buffer X (0.705 vs 0.694 ms for c2), pass 1 of
// buffer Y on warps 4..11 instead of 0..7 (0.719 ms).
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
  // pass 1: R0 R2 butterflies on W1 warps, pass 2: R0 R1 butterflies on W2 warps; 4 groups of R0 / 4
  // sub-sequences, each with W1 / 4 pass-1 warps and W2 / 4 pass-2 warps
  constexpr int W1 = R0 * R2 / 32, W2 = R0 * R1 / 32, G1 = W1 / 4, G2 = W2 / 4;
  static_assert(T == 384 && R0 == 16 && N1 == T && W1 % 4 == 0 && W2 % 4 == 0 && W1 <= 12 && W2 <= 12,
                "12 warps; pass 0 on all of them; 4 groups");
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
      mbar_init(&bars[4 + i], G1);   // pass 1 done (G1 warps): buffer i / 4, group i % 4
      mbar_init(&bars[12 + i], G2);  // inverse pass 2 done (G2 warps)
    }
    readers[0] = readers[1] = 0;
    fence_mbar_init();
  }
  using TL = TmemLayout<32 * W2, 2 * R2, 0>;  // F of both residues, in the pass-2 warps' columns
  static_assert(TL::FITS, "both spectra in tensor memory");
  if (tid < 32) tmem_alloc(&tm_base, TL::COLS);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  // groups: as a pass-1 warp (warps 0..W1-1) m1, as a pass-2 warp (warps 0..W2-1) m2
  const int m1 = (w / G1) & 3, m2 = (w / G2) & 3;
  const bool w1 = w < W1, w2 = w < W2;
  const int base1 = N1 * (tid / N2), b1 = tid % N2;  // pass 1: sub-sequence offset and butterfly
  IpChain cA{X, 0, {smem_u32(&bars[2])}, {smem_u32(&bars[4 + m1])}, {smem_u32(&bars[4 + m2])},
             {smem_u32(&bars[12 + m2])}, {smem_u32(&bars[12 + m1])}, &bars[0], 0u, TL::f_addr(tm_base), &readers[0]};
  IpChain cB{X + N, 1, {smem_u32(&bars[3])}, {smem_u32(&bars[8 + m1])}, {smem_u32(&bars[8 + m2])},
             {smem_u32(&bars[16 + m2])}, {smem_u32(&bars[16 + m1])}, &bars[1], 0u, TL::f_addr(tm_base) + 4 * R2,
             &readers[1]};
  const int L = a.L;
  const uint32_t row_bytes = (uint32_t)a.S * 16u;
  const long long step = gridDim.x;
  long long item = blockIdx.x;
  if (tid == 0 && item < p.lin.count) {
    tma_copy(cA.Z, p.f + p.lin.base(item), row_bytes, cA.bar_tma);
    tma_copy(cB.Z, p.f + p.lin.base(item), row_bytes, cB.bar_tma);
  }
  const int pos0 = tid ^ ((tid / R2) & 7);
  const int base2 = N2 * tid, key2 = tid & 7;
  const double scale = 1.0 / (double)a.qm;
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

  const double2* gsrc = nullptr;   // the line's g (refill after pass 2 of f)
  const double2* fnext = nullptr;  // the next line's f (refill after inverse pass 0)
  auto fwd2f = [&](IpChain& c) HC_INL {
    if (!w2) {
      release(c, gsrc);
      return;
    }
    double2 v[R2];
    c.g1w.wait();
    sfor<R2>([&](auto Ai) HC_INL { v[Ai] = c.Z[base2 + (Ai ^ key2)]; });
    DFT<R2, +1>::run(v);
    release(c, gsrc);
    tm_store<R2>(c.tf, v);
  };
  auto fwd2g = [&](IpChain& c) HC_INL {
    if (!w2) return;
    double2 v[R2];
    c.g1w.wait();
    sfor<R2>([&](auto Ai) HC_INL { v[Ai] = c.Z[base2 + (Ai ^ key2)]; });
    DFT<R2, +1>::run(v);
    tmem_wait_st();
    // (issuing these tensor-memory loads before the butterflies measured slower: 0.715 vs 0.701 ms)
    sfor<R2 / 4>([&](auto Ki) HC_INL {
      double2 F4[4];
      tm_ld4(c.tf + 16 * Ki, F4);
      sfor<4>([&](auto i) HC_INL { v[4 * Ki + i] = cmul(v[4 * Ki + i], F4[i]); });
    });
    DFT<R2, -1>::run(v);
    sfor<R2>([&](auto Ai) HC_INL { c.Z[base2 + (Ai ^ key2)] = v[Ai]; });
    c.gIa.arrive();
  };
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
  // inverse pass 0 of a buffer into h (pass-0 layout, before the residue's post-twiddle)
  auto inv0 = [&](IpChain& c, double2(&h)[R0], const double2* refill) HC_INL {
    const P0Res<SYM> p0{&a, tb, c.res};
    c.b.wait();
    sfor<R0>([&](auto Ki) HC_INL { h[Ki] = c.Z[N1 * Ki + pos0]; });
    pass0_twiddle<-1, R0>(h, tid, p0);
    release(c, refill);
    DFT<R0, -1>::run(h);
  };
  // h (residue 0) + v (residue 1, post-twiddled) -> output line
  auto emit = [&](const double2(&h)[R0], const double2(&v)[R0], long long base) HC_INL {
    double2* o = p.out + base;
    sfor<R0>([&](auto Ai) HC_INL {
      const int s = N1 * Ai + tid;
      const double2 x = cadd(h[Ai], cmulc(v[Ai], U1[Ai]));
      if (s < L) __stcs(o + s, cscale(x, scale));
    });
  };
  auto set_line = [&](long long it) HC_INL {
    const long long nitem = it + step;
    const long long nline = nitem < p.lin.count ? p.lin.base(nitem) : -1;
    if (tid == 0 && nline >= 0) {
      l2_prefetch(p.f + nline, row_bytes);
      l2_prefetch(p.g + nline, row_bytes);
    }
    gsrc = p.g + p.lin.base(it);
    fnext = nline >= 0 ? p.f + nline : nullptr;
  };
  for (; item < p.lin.count; item += step) {
    const long long base = p.lin.base(item);
    set_line(item);
    // ---- f: passes 0, 1, 2; the spectrum goes to tensor memory, the buffer is refilled with g
    wait_line(cA);
    fwd0(cA);
    wait_line(cB);
    fwd0(cB);
    fwd1(cA);
    fwd1(cB);
    fwd2f(cA);
    fwd2f(cB);
    // ---- g: passes 0, 1, 2 + product + inverse pass 2
    wait_line(cA);
    fwd0(cA);
    wait_line(cB);
    fwd0(cB);
    fwd1(cA);
    fwd1(cB);
    fwd2g(cA);
    fwd2g(cB);
    // ---- inverse passes 1 and 0; the two residues' outputs meet in registers
    inv1(cA);
    inv1(cB);
    double2 h[R0], v[R0];
    inv0(cA, h, fnext);
    inv0(cB, v, fnext);
    emit(h, v, base);
  }
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
