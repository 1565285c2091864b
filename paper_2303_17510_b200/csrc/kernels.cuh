// kernels.cuh — fused residue-loop kernels (templated on the block-FFT radix plan).
//
//  k_conv1d   : Alg. convolve / convolveX for a batch of lines, fully
//               fused: for every residue block v the A = 2 forward padded FFTs, the product
//               (SPEC.md:424 builtin_mult_product) and the backward padded FFT with
//               accumulation run on chip; HBM sees f, g once (second residue re-reads hit L2)
//               and h once.  One CTA hosts G independent line groups of T threads.
//  k_pfft_fwd : one residue of forward1/2/Inner[C|H] for a batch of lines (SPEC pfft-*),
//               output in reference order or natural block order.
//  k_pfft_bwd : one residue of backward1/2/Inner[C|H] with accumulation (SPEC pfft-*).
#pragma once
#include "block_io.cuh"
#include "tma.cuh"
#include "tmem.cuh"

namespace hc {

struct ConvArgs {
  AxisDev ax;
  Lines lin;             // input/output line addressing (inputs and output share the layout)
  const double2* f;
  const double2* g;
  double2* out;
  double2* scratch;      // per-group accumulator slots (S complex each)
  int stage;             // 0: pass-0 reads global; 1: lines staged by TMA into X; 2: into a separate buffer
  int gs;                // group stride in shared memory (complex)
  int in_off;            // stage 2: offset of the staging buffer inside the group region
                         // stage 3: ping-pong kernel (k_conv1d_pp), X and Y of XS each
  unsigned long long* trace;  // optional phase timestamps of CTA 0 / thread 0 (HCONV_TRACE)
  int dbg;                    // diagnostics (HCONV_DBG bits, ping-pong kernel): 1 skip stores,
                              // 2 skip pass-0 loads, 4 skip the product, 8 skip the inverse
  int tm_acc = 0;             // k_conv1d, Hermitian: the CTA owns the SM, so the residue
                              // accumulator may live in tensor memory (512 columns)
};

struct FwdArgs {
  AxisDev ax;
  Lines lin;             // input lines
  Lines lout;            // output lines (block values at element stride lout.es)
  const double2* f;
  void* F;               // complex128 (complex/centered) or float64 (Hermitian)
  int v;
  int ref_order;         // 1: SPEC order F[u m + l]; 0: natural k'
};

struct BwdArgs {
  AxisDev ax;
  Lines lin;             // block lines (input)
  Lines lout;            // output lines
  const void* F;
  double2* dst;
  const double2* acc;    // may alias dst; lines addressed like lout
  double scale;
  int v;
  int ref_order;
};

// butterfly c of pass I exists for this thread (compile-time pass index: the radix tables are
// host constexpr arrays and must only be indexed with constants in device code)
template <class Cfg, int I>
__device__ __forceinline__ bool bvalid(int c, int tid) {
  constexpr int NB = Cfg::NB(I);
  return NB % Cfg::T == 0 || tid + c * Cfg::T < NB;
}

// pass-0 load of one input line (radix kernels: table-driven, no runtime modulo)
template <int SYM, class Cfg>
__device__ __forceinline__ void load_pass0(double2 (&v)[Cfg::E], const AxisDev& a, const double2* tb, const double2* f,
                                           long long es, int res, int tid) {
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), Ns1 = Cfg::Ns(1);
  sfor<C0>([&](auto Ci) HC_INL {
    constexpr int c = Ci;
    const int b = tid + c * Cfg::T;
    if (bvalid<Cfg, 0>(c, tid)) {
      sfor<R0>([&](auto Ai) HC_INL {
        constexpr int ai = Ai;
        if constexpr (SYM == SYM_HERMITIAN) v[c * R0 + ai] = load_Zp_fast(a, tb, f, es, Ns1 * ai + b, res, ai, b);
        else v[c * R0 + ai] = load_fast<SYM>(a, tb, f, es, Ns1 * ai + b, res, ai);
      });
    }
  });
}

// pass-0 output twiddle source: omega_Bc^{b k} times (complex / centered) the folded residue
// factor zeta_qm^{v b}
template <int SYM>
struct P0Res {
  const AxisDev* a;
  const double2* tb;
  int v;
  __device__ __forceinline__ void operator()(int b, double2& t, double2& w) const {
    w = tA(*a, tb, b);
    t = (SYM != SYM_HERMITIAN && v) ? tZ(*a, tb, v, b) : make_double2(1.0, 0.0);
  }
};

// inverse post-processing from pass-0 layout (complex / centered)
template <int SYM, class Cfg>
__device__ __forceinline__ void store_pass0(const double2 (&v)[Cfg::E], const AxisDev& a, const double2* tb,
                                            const Emit& em, int res, int tid) {
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), Ns1 = Cfg::Ns(1);
  sfor<C0>([&](auto Ci) HC_INL {
    constexpr int c = Ci;
    const int b = tid + c * Cfg::T;
    if (bvalid<Cfg, 0>(c, tid)) {
      sfor<R0>([&](auto Ai) HC_INL { store_fast<SYM>(a, tb, em, Ns1 * Ai + b, res, Ai, v[c * R0 + Ai]); });
    }
  });
}

// Hermitian post-processing: pass-0 layout -> Z in shared memory -> outputs j < S
template <class Cfg, class Sync>
__device__ __forceinline__ void store_herm(const double2 (&v)[Cfg::E], const AxisDev& a, const double2* tb,
                                           const Emit& em, int res, int tid, double2* Z, const Sync& sync) {
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), Ns1 = Cfg::Ns(1);
  sfor<C0>([&](auto Ci) HC_INL {
    constexpr int c = Ci;
    const int b = tid + c * Cfg::T;
    if (bvalid<Cfg, 0>(c, tid)) sfor<R0>([&](auto Ai) HC_INL { Z[Ns1 * Ai + b] = v[c * R0 + Ai]; });
  });
  sync();
  herm_store_quads<Ns1>(a, tb, em, Z, res, tid, Cfg::T);
  sync();
}

// Hermitian pass-0 input from a line staged in shared memory: the packed values Z'_k
// (load_Zp_fast) are built IN PLACE, one quad {k, Bc-k, Bc+k, B-k} per thread -- the quad's four
// stored values are read before its two outputs Z'_k, Z'_{Bc-k} are written, and quads are
// disjoint -- so each W_s is formed once (load_Zp_fast forms it twice) with int offsets:
//   W_s = (f_s + conj f_{B-s} [zeta^{-vB}]) zeta^{vs},  e = W_k + conj W_{Bc-k},
//   o = (W_k - conj W_{Bc-k}) zeta_B^k,  Z'_k = e + i o,  Z'_{Bc-k} = conj e + i conj o.
// The caller synchronises before reading Z' in pass-0 layout (load_plain).
template <int NT, int NS1>
__device__ __forceinline__ void herm_pack(double2* X, const AxisDev& a, const double2* tb, int v, int tid) {
  const int Bc = a.Bc, B = a.B, S = a.S, half = Bc / 2;
  constexpr int ns1 = NS1;  // == a.ns1 (Bc / R0): compile-time, so k / ns1 is a shift or a multiply
  const double2 one = make_double2(1.0, 0.0);
  const double2 cH = v ? tb[a.oH + v] : one;            // zeta_qm^{v Bc}
  const double2 c1 = v ? tb[a.oC + v * a.nc + 1] : one;  // zeta_qm^{v B}
  const double2* Zr = tb + (a.oZ + v * ns1);
  const double2* Ur = tb + (a.oU + v * a.nu);
  const double2* Bl = tb + a.oBl;
  const double2* Bh = tb + a.oBh;
  if (S <= half) {
    // heavily padded lines (S <= Bc/2, e.g. c5's z-lines, 256 of 1024): only x1 = f_k is
    // nonzero in a quad (Bc - k, B - k and Bc + k all lie beyond the data), so W_{Bc-k} = 0,
    // e = W_k and o = W_k zeta_B^k; quads with k >= S write zeros
    for (int k = tid; k <= half; k += NT) {
      const int kh = k / ns1, kl = k - kh * ns1;
      double2 wk = k < S ? X[k] : make_double2(0.0, 0.0);
      if (v) wk = cmul(wk, cmul(Zr[kl], Ur[kh]));  // zeta_qm^{v k}
      const double2 o = cmul(wk, cmul(Bh[kh], Bl[kl]));
      X[k] = make_double2(wk.x - o.y, wk.y + o.x);
      if (k != 0 && k != half) X[Bc - k] = make_double2(wk.x + o.y, o.x - wk.y);
    }
    return;
  }
  for (int k = tid; k <= half; k += NT) {
    const int kh = k / ns1, kl = k - kh * ns1;
    const int s2 = Bc - k;
    double2 x1 = k < S ? X[k] : make_double2(0.0, 0.0);
    double2 x2 = s2 < S ? X[s2] : make_double2(0.0, 0.0);
    const int r1 = B - k, r2 = B - s2;  // r1 > 0 always (k <= Bc/2 < B)
    const double2 y1 = r1 < S ? cconj(X[r1]) : make_double2(0.0, 0.0);
    const double2 y2 = (r2 > 0 && r2 < S) ? cconj(X[r2]) : make_double2(0.0, 0.0);
    double2 wk, wm;
    if (v) {
      const double2 zk = cmul(Zr[kl], Ur[kh]);  // zeta_qm^{v k}
      const double2 zm = cmulc(cH, zk);         // zeta_qm^{v (Bc - k)}
      wk = cmul(cadd(x1, cmulc(y1, c1)), zk);
      wm = cconj(cmul(cadd(x2, cmulc(y2, c1)), zm));
    } else {
      wk = cadd(x1, y1);
      wm = cconj(cadd(x2, y2));
    }
    const double2 e = cadd(wk, wm);
    const double2 o = cmul(csub(wk, wm), cmul(Bh[kh], Bl[kl]));  // zeta_B^k
    X[k] = make_double2(e.x - o.y, e.y + o.x);
    if (k != 0 && k != half) X[s2] = make_double2(e.x + o.y, o.x - e.y);
  }
}

// Heavily padded Hermitian lines (S <= Bc/2, herm_pack's fast path) straight into pass-0 layout:
// element j = Ns1 a + b of Z' depends on one stored value only (k = j below Bc/2, k = Bc - j
// above: W_{Bc-k} = 0), so the packed line never takes the round trip through shared memory
// (herm_pack writes 2 values per quad, load_plain reads them back) and one barrier goes away; the
// low factor of zeta_B^k is the same for a thread's lower (kl = b) and upper (kl = -b mod Ns1)
// elements and is read once each.  Same values as herm_pack + load_plain (each Z'_j is formed by
// the same operations on the same operands).
template <class Cfg>
__device__ __forceinline__ void herm_load_padded(double2 (&v)[Cfg::E], const double2* X, const AxisDev& a,
                                                 const double2* tb, int res, int tid) {
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), Ns1 = Cfg::Ns(1), Bc = Cfg::N, half = Bc / 2;
  const int S = a.S;
  const double2* Zr = tb + (a.oZ + res * Ns1);
  const double2* Ur = tb + (a.oU + res * a.nu);
  const double2* Bl = tb + a.oBl;
  const double2* Bh = tb + a.oBh;
  sfor<C0>([&](auto Ci) HC_INL {
    constexpr int c = Ci;
    const int b = tid + c * Cfg::T;
    if (bvalid<Cfg, 0>(c, tid)) {
      const int bu = (Ns1 - b) % Ns1;  // kl of the upper elements
      const double2 blo = Bl[b], bup = Bl[bu];
      double2 zlo = make_double2(1.0, 0.0), zup = zlo;
      if (res) {
        zlo = Zr[b];
        zup = Zr[bu];
      }
      sfor<R0>([&](auto Ai) HC_INL {
        constexpr int ai = Ai;
        const int j = Ns1 * ai + b;
        const bool low = j <= half;
        const int k = low ? j : Bc - j;
        const int kh = k / Ns1;
        double2 wk = k < S ? X[k] : make_double2(0.0, 0.0);
        if (res) wk = cmul(wk, cmul(low ? zlo : zup, Ur[kh]));  // zeta_qm^{v k}
        const double2 o = cmul(wk, cmul(Bh[kh], low ? blo : bup));
        v[c * R0 + ai] = low ? make_double2(wk.x - o.y, wk.y + o.x) : make_double2(wk.x + o.y, o.x - wk.y);
      });
    }
  });
}

// pass-0 values straight from a shared-memory line in natural order (v[c R0 + a] = X[Ns1 a + b])
template <class Cfg>
__device__ __forceinline__ void load_plain(double2 (&v)[Cfg::E], const double2* X, int tid) {
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), Ns1 = Cfg::Ns(1);
  sfor<C0>([&](auto Ci) HC_INL {
    constexpr int c = Ci;
    const int b = tid + c * Cfg::T;
    if (bvalid<Cfg, 0>(c, tid)) sfor<R0>([&](auto Ai) HC_INL { v[c * R0 + Ai] = X[Ns1 * Ai + b]; });
  });
}

// stage the per-axis tables (block_io.cuh: A Z U C MT [H Bl Bh]) into shared memory (whole CTA)
__device__ __forceinline__ void stage_tables(double2* tb, const AxisDev& a, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) tb[i] = __ldg(a.tab + i);
  __syncthreads();
}

// ------------------------------------------------------------------ conv1d --
// STASH_REGS: keep the first forward spectrum in registers instead of shared memory.
// Staged mode (p.stage != 0, unit element stride): every input line (f, g) and the residue
// accumulator are brought on chip by TMA bulk copies issued one phase ahead -- the next line
// copy starts as soon as the previous transform has released the exchange buffer, so the
// HBM/L2 latency overlaps the butterflies of the current transform.
// Hermitian post-processing with the residue accumulator in tensor memory: the same quads as
// herm_store_quads (block_io.cuh), iterated a fixed NIT times per thread so that the
// warp-collective tcgen05 loads / stores stay convergent; each iteration's four outputs keep
// their four accumulator values in the thread's own TMEM columns (16 per iteration).  FIRST: no
// accumulator yet; FINAL: add, scale and write the outputs instead of storing back.
template <int NIT, int NS1>
__device__ __forceinline__ void herm_quads_tm(const AxisDev& a, const double2* tb, double2* out, long long es,
                                              double scale, const double2* Z, int v, int tid, int T, uint32_t ta,
                                              bool first, bool final_) {
  const int Bc = a.Bc, B = a.B, S = a.S, half = Bc / 2;
  const double2 one = make_double2(1.0, 0.0);
  const double2 zBc = v ? tH(a, tb, v) : one;
  const double2 zB = v ? tC(a, tb, v, 1) : one;
#pragma unroll 1
  for (int it = 0; it < NIT; ++it) {
    const int k0 = tid + it * T;
    const bool kv = k0 <= half;
    const int k = kv ? k0 : 0;
    const int j[4] = {k, B - k, Bc - k, Bc + k};
    const bool ok[4] = {kv && k < S, kv && k > 0 && B - k < S, kv && Bc - k != k && Bc - k < S,
                        kv && k > 0 && k != half && Bc + k < S};
    const double2 zk = Z[k];
    const double2 zm = cconj(Z[k == 0 ? 0 : Bc - k]);
    const double2 e = cscale(cadd(zk, zm), 0.5);
    const double2 d = cscale(csub(zk, zm), 0.5);
    const double2 o = make_double2(d.y, -d.x);
    const double2 tB = cmul(tBh(a, tb, k / NS1), tBl(a, tb, k % NS1));
    const double2 wk = cadd(e, cmulc(o, tB));
    const double2 wm = csub(cconj(e), cmul(tB, cconj(o)));
    double2 w[4] = {wk, cconj(wk), wm, cconj(wm)};
    if (v) {
      const double2 zvk = cmul(tZ(a, tb, v, k % NS1), tU(a, tb, v, k / NS1));
      w[0] = cmulc(w[0], zvk);
      w[1] = cmulc(cmul(w[1], zvk), zB);
      w[2] = cmulc(cmul(w[2], zvk), zBc);
      w[3] = cmulc(cmulc(w[3], zvk), zBc);
    }
    if (!first) {
      double2 acc[4];
      tm_ld4(ta + 16 * it, acc);
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = cadd(w[u], acc[u]);
    }
    if (!final_) {
      tm_st4(ta + 16 * it, w);
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (ok[u]) __stcs(out + (long long)j[u] * es, cscale(w[u], scale));
    }
  }
}

// HC_CONV_TMEM=1: the register stash of the first spectrum (STASH_REGS) lives in tensor memory
// instead (frees Cfg::ES complex registers per thread; 128 columns per CTA at most)
#ifndef HC_CONV_TMEM
#define HC_CONV_TMEM 1
#endif
template <int SYM, class Cfg, int G, bool STASH_REGS, int MINB = 1>
__global__ void __launch_bounds__(Cfg::T * G, MINB) k_conv1d(ConvArgs p) {
  extern __shared__ __align__(16) double2 smem[];
  __shared__ __align__(8) uint64_t bars[2 * G];
  __shared__ uint32_t tm_base;
  using TLc = TmemLayout<Cfg::T * G, Cfg::ES, 0>;
  constexpr bool TMST = HC_CONV_TMEM && STASH_REGS && TLc::FITS && TLc::COLS <= 128;
  // Hermitian accumulator in TMEM (host sets p.tm_acc when the CTA owns the SM)
  constexpr int NIT = (Cfg::N / 2) / Cfg::T + 1;
  using TLa = TmemLayout<Cfg::T * G, Cfg::ES, 4 * NIT>;
  constexpr bool TMACC = TMST && SYM == SYM_HERMITIAN && TLa::FITS && G == 1;
  const bool tm_acc = TMACC && p.tm_acc;
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), NBL = Cfg::NB(Cfg::P - 1);
  const int g = threadIdx.x / T, tid = threadIdx.x % T;
  double2* tb = smem;
  const double2* mt = tb;  // middle-pass tables sit at offset 0
  double2* X = smem + p.ax.tabn + g * p.gs;
  double2* stash = X + Cfg::XS;
  double2* IN = p.stage == 2 ? X + p.in_off : X;
  uint64_t* bar_in = &bars[2 * g];
  uint64_t* bar_acc = &bars[2 * g + 1];
  const GroupSync sync{g + 1, T};
  const AxisDev& a = p.ax;
  stage_tables(tb, a, a.tabn);
  const double2* tp = a.tabn >= a.tabfull ? tb : a.tab;
  const int stage = p.stage;
  const bool stage_acc = stage != 0 && !STASH_REGS && a.S <= Cfg::N;
  if (stage && tid == 0) {
    mbar_init(bar_in, 1);
    mbar_init(bar_acc, 1);
    fence_mbar_init();
  }
  if constexpr (TMST) {
    if (threadIdx.x < 32) tmem_alloc(&tm_base, tm_acc ? TLa::COLS : TLc::COLS);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
  }
  sync();
  const uint32_t tf = TMST ? (tm_acc ? TLa::f_addr(tm_base) : TLc::f_addr(tm_base)) : 0u;
  const uint32_t ta = tm_acc ? TLa::a_addr(tm_base) : 0u;
  uint32_t ph_in = 0, ph_acc = 0;
  const uint32_t row_bytes = (uint32_t)a.S * 16u;
  const long long es = p.lin.es, step = (long long)gridDim.x * G;
  double2* slot = p.scratch + (long long)(blockIdx.x * G + g) * a.S;
  long long item = (long long)blockIdx.x * G + g;
  if (stage && tid == 0 && item < p.lin.count) tma_copy(IN, p.f + p.lin.base(item), row_bytes, bar_in);
  const bool tr = p.trace && blockIdx.x == 0 && threadIdx.x == 0;
  int tn = 0;
  // trace points are preceded by a group barrier (when tracing) so they mark phase boundaries
#define HC_TRACE()                                   \
  do {                                               \
    if (p.trace) {                                   \
      sync();                                        \
      if (tr && tn < 256) p.trace[tn++] = clock64(); \
    }                                                \
  } while (0)
  for (; item < p.lin.count; item += step) {
    const long long base = p.lin.base(item);
    for (int res = 0; res < a.n; ++res) {
      HC_TRACE();
      const bool last = res == a.n - 1;
      // next f line: the same line for the next residue, else the next item's line
      const double2* fnext = !last ? p.f + base : (item + step < p.lin.count ? p.f + p.lin.base(item + step) : nullptr);
      double2 v[Cfg::E];
      double2 Fr[STASH_REGS && !TMST ? Cfg::E : 1];
      const P0Res<SYM> p0{&a, tp, res};
      // ---- forward padded FFTs of the A = 2 inputs (one code copy: keeps the kernel inside
      //      the instruction cache); input 0 is stashed, input 1 multiplied by it
#pragma unroll 1
      for (int inp = 0; inp < 2; ++inp) {
        const double2* src = inp == 0 ? p.f : p.g;
        // TMA issued when this input releases the staging buffer: g after f, then the next f
        const double2* nxt = inp == 0 ? p.g + base : fnext;
        if (stage) {
          mbar_wait(bar_in, ph_in);
          ph_in ^= 1;
          HC_TRACE();
          if constexpr (SYM == SYM_HERMITIAN) {
            herm_pack<T, Cfg::Ns(1)>(IN, a, tp, res, tid);
            sync();
            load_plain<Cfg>(v, IN, tid);
          } else {
            load_pass0<SYM, Cfg>(v, a, tp, IN, 1, res, tid);
          }
          sync();  // IN (X in mode 1) fully read before the exchange writes / the next copy
          if (stage == 2 && tid == 0 && nxt) tma_copy(IN, nxt, row_bytes, bar_in);
        } else {
          load_pass0<SYM, Cfg>(v, a, tp, src + base, es, res, tid);
        }
        HC_TRACE();
        fft_forward<Cfg>(v, X, mt, tid, sync, p0, [&]() HC_INL {
          if (stage == 1 && inp == 0 && tid == 0) tma_copy(IN, p.g + base, row_bytes, bar_in);
        });
        HC_TRACE();
        if (inp == 0) {
          if constexpr (TMST) {
            tm_store<Cfg::ES>(tf, v);
          } else {
            sfor<CL>([&](auto Ci) HC_INL {
              constexpr int c = Ci;
              if (bvalid<Cfg, Cfg::P - 1>(c, tid))
                sfor<RL>([&](auto Ki) HC_INL {
                  if constexpr (STASH_REGS) Fr[c * RL + Ki] = v[c * RL + Ki];
                  else stash[Ki * NBL + tid + c * T] = v[c * RL + Ki];
                });
            });
          }
        } else if constexpr (TMST) {
          tmem_wait_st();
          sfor<Cfg::ES / 4>([&](auto Ki) HC_INL {
            double2 F4[4];
            tm_ld4(tf + 16 * Ki, F4);
            sfor<4>([&](auto i) HC_INL {
              double2& G_ = v[4 * Ki + i];
              const double2 F = F4[i];
              if constexpr (SYM == SYM_HERMITIAN) G_ = make_double2(G_.x * F.x, G_.y * F.y);
              else G_ = cmul(G_, F);
            });
          });
        } else {
          sfor<CL>([&](auto Ci) HC_INL {
            constexpr int c = Ci;
            if (bvalid<Cfg, Cfg::P - 1>(c, tid))
              sfor<RL>([&](auto Ki) HC_INL {
                double2 F;
                if constexpr (STASH_REGS) F = Fr[c * RL + Ki];
                else F = stash[Ki * NBL + tid + c * T];
                double2& G_ = v[c * RL + Ki];
                if constexpr (SYM == SYM_HERMITIAN) G_ = make_double2(G_.x * F.x, G_.y * F.y);  // real residues
                else G_ = cmul(G_, F);
              });
          });
        }
      }
      HC_TRACE();
      // ---- residue accumulator -> stash (its last reader was the product above)
      if (stage_acc && res > 0) {
        // the slot was written by this group's generic stores (store_pass0 / store_herm of the
        // previous residue) and is now read by the async proxy: every writer fences first
        fence_proxy_async_global();
        sync();
        if (tid == 0) tma_copy(stash, slot, row_bytes, bar_acc);
      }
      // ---- inverse; the next f copy into X starts once X is released (not for the
      //      Hermitian store, which uses X as its Z buffer)
      HC_TRACE();
      fft_inverse<Cfg>(v, X, mt, tid, sync, p0, [&]() HC_INL {
        if (SYM != SYM_HERMITIAN && stage == 1 && tid == 0 && fnext) tma_copy(IN, fnext, row_bytes, bar_in);
      });
      HC_TRACE();
      const double2* acc = nullptr;
      if (res > 0 && !tm_acc) {
        if (stage_acc) {
          mbar_wait(bar_acc, ph_acc);
          ph_acc ^= 1;
          acc = stash;
        } else {
          acc = slot;
        }
      }
      const Emit em = last ? Emit{p.out + base, es, acc, 1, 1.0 / (double)a.qm, true} : Emit{slot, 1, acc, 1, 1.0, false};
      if constexpr (SYM == SYM_HERMITIAN) {
        if (tm_acc) {
          constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), Ns1 = Cfg::Ns(1);
          sfor<C0>([&](auto Ci) HC_INL {
            constexpr int c = Ci;
            const int b = tid + c * Cfg::T;
            if (bvalid<Cfg, 0>(c, tid)) sfor<R0>([&](auto Ai) HC_INL { X[Ns1 * Ai + b] = v[c * R0 + Ai]; });
          });
          sync();
          herm_quads_tm<NIT, Ns1>(a, tp, p.out + base, es, 1.0 / (double)a.qm, X, res, tid, Cfg::T, ta, res == 0, last);
          sync();
        } else {
          store_herm<Cfg>(v, a, tp, em, res, tid, X, sync);
        }
        if (stage == 1 && tid == 0 && fnext) tma_copy(IN, fnext, row_bytes, bar_in);
      } else {
        store_pass0<SYM, Cfg>(v, a, tp, em, res, tid);
      }
      HC_TRACE();
      if (stage_acc) sync();  // stash (acc) reads done before the next residue stashes F
    }
  }
  if constexpr (TMST) {
    tmem_wait_st();
    tmem_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tm_base, tm_acc ? TLa::COLS : TLc::COLS);
  }
#undef HC_TRACE
}

// ------------------------------------------- ping-pong fast paths (complex / centered) --
// The ping-pong kernel sees unit-stride lines staged in shared memory and (host:
// conv_layout) every table staged in shared memory, so its pass-0 loads and post-processing
// stores are written with int offsets into shared memory, table rows hoisted per residue, and
// the fold terms (L > B only) in one uniform branch after the main loop instead of a loop per
// element.  Same arithmetic as load_fast / store_fast (block_io.cuh).
template <int SYM, class Cfg>
__device__ __forceinline__ void load_pass0_pp(double2 (&v)[Cfg::E], const AxisDev& a, const double2* tb,
                                              const double2* X, int res, int tid) {
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), Ns1 = Cfg::Ns(1);
  const int L = a.L, B = a.B;
  const double2* Cv = tb + (a.oC + res * a.nc);  // row res (rows from 1, see build_tables)
  if constexpr (SYM == SYM_COMPLEX) {
    sfor<C0>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int b = tid + c * Cfg::T;
      if (bvalid<Cfg, 0>(c, tid))
        sfor<R0>([&](auto Ai) HC_INL {
          const int s = Ns1 * Ai + b;
          v[c * R0 + Ai] = s < L ? X[s] : make_double2(0.0, 0.0);
        });
    });
    if (L > B) {
      sfor<C0>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        const int b = tid + c * Cfg::T;
        if (bvalid<Cfg, 0>(c, tid))
          sfor<R0>([&](auto Ai) HC_INL {
            double2& x = v[c * R0 + Ai];
            int t = 1;
            for (int j = Ns1 * Ai + b + B; j < L; j += B, ++t) x = cadd(x, res ? cmul(X[j], Cv[t]) : X[j]);
          });
      });
    }
  } else {
    const int H = a.H, LH = L - H, BH = B - H;
    const double2 c1 = res ? Cv[1] : make_double2(1.0, 0.0);
    sfor<C0>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int b = tid + c * Cfg::T;
      if (bvalid<Cfg, 0>(c, tid))
        sfor<R0>([&](auto Ai) HC_INL {
          const int s = Ns1 * Ai + b;
          double2 x = s < LH ? X[s + H] : make_double2(0.0, 0.0);
          if (s >= BH) x = cadd(x, res ? cmulc(X[s - BH], c1) : X[s - BH]);
          v[c * R0 + Ai] = x;
        });
    });
  }
  if (res) {
    const double2* U = tb + (a.oU + res * a.nu);
    sfor<C0>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      if (bvalid<Cfg, 0>(c, tid)) sfor<R0>([&](auto Ai) HC_INL { v[c * R0 + Ai] = cmul(v[c * R0 + Ai], U[Ai]); });
    });
  }
}

// dst[j] = (ACC ? acc[j] : 0) + w_j, times `scale` with streaming stores when FINAL; acc is the
// residue accumulator staged in shared memory (unit stride), dst a unit-stride line.
// SMEM: dst is a shared-memory line (possibly == acc, updated in place) that a bulk copy
// writes out afterwards.
template <int SYM, class Cfg, bool ACC, bool FINAL, bool SMEM = false>
__device__ __forceinline__ void store_pass0_pp(double2 (&v)[Cfg::E], const AxisDev& a, const double2* tb, double2* dst,
                                               const double2* acc, double scale, int res, int tid) {
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), Ns1 = Cfg::Ns(1);
  const int L = a.L, B = a.B;
  const double2* Cv = tb + (a.oC + res * a.nc);  // row res (rows from 1, see build_tables)
  auto put = [&](int j, double2 w) HC_INL {
    if constexpr (ACC) w = cadd(w, acc[j]);
    if constexpr (FINAL) w = cscale(w, scale);
    if constexpr (FINAL && !SMEM) __stcs(dst + j, w);
    else dst[j] = w;
  };
  if (res) {
    const double2* U = tb + (a.oU + res * a.nu);
    sfor<C0>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      if (bvalid<Cfg, 0>(c, tid)) sfor<R0>([&](auto Ai) HC_INL { v[c * R0 + Ai] = cmulc(v[c * R0 + Ai], U[Ai]); });
    });
  }
  if constexpr (SYM == SYM_COMPLEX) {
    sfor<C0>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int b = tid + c * Cfg::T;
      if (bvalid<Cfg, 0>(c, tid))
        sfor<R0>([&](auto Ai) HC_INL {
          const int s = Ns1 * Ai + b;
          if (s < L) put(s, v[c * R0 + Ai]);
        });
    });
    if (L > B) {
      sfor<C0>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        const int b = tid + c * Cfg::T;
        if (bvalid<Cfg, 0>(c, tid))
          sfor<R0>([&](auto Ai) HC_INL {
            const double2 w = v[c * R0 + Ai];
            int t = 1;
            for (int j = Ns1 * Ai + b + B; j < L; j += B, ++t) put(j, res ? cmulc(w, Cv[t]) : w);
          });
      });
    }
  } else {
    const int H = a.H, LH = L - H, BH = B - H;
    const double2 c1 = res ? Cv[1] : make_double2(1.0, 0.0);
    sfor<C0>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int b = tid + c * Cfg::T;
      if (bvalid<Cfg, 0>(c, tid))
        sfor<R0>([&](auto Ai) HC_INL {
          const int s = Ns1 * Ai + b;
          const double2 w = v[c * R0 + Ai];
          if (s < LH) put(s + H, w);
          if (s >= BH) put(s - BH, res ? cmul(w, c1) : w);
        });
    });
  }
}

// Residue accumulator in tensor memory (complex / centered, no folding: L <= B, so every pass-0
// element s feeds at most one output).  v holds the inverse block in pass-0 layout; it is
// post-twiddled in place, added to the thread's accumulator columns (unless FIRST) and either
// stored back (not FINAL) or scaled and written to the output line staged in Y (FINAL).  Same
// arithmetic as store_pass0_pp.
template <int SYM, class Cfg, bool FIRST, bool FINAL>
__device__ __forceinline__ void acc_tmem_pp(double2 (&v)[Cfg::E], const AxisDev& a, const double2* tb, uint32_t ta,
                                            double2* Y, double scale, int res, int tid) {
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), Ns1 = Cfg::Ns(1), E0 = C0 * R0;
  const int L = a.L, H = a.H, LH = L - H, BH = a.B - H;
  if (res) {
    const double2* U = tb + (a.oU + res * a.nu);
    const double2 c1 = tb[a.oC + res * a.nc + 1];
    sfor<C0>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      sfor<R0>([&](auto Ai) HC_INL {
        double2 w = cmulc(v[c * R0 + Ai], U[Ai]);
        if constexpr (SYM == SYM_CENTERED) {
          if (Ns1 * Ai + tid + c * Cfg::T >= BH) w = cmul(w, c1);  // logical s - B
        }
        v[c * R0 + Ai] = w;
      });
    });
  }
  if constexpr (!FIRST) {
    sfor<E0 / 4>([&](auto Ki) HC_INL {
      double2 t4[4];
      tm_ld4(ta + 16 * Ki, t4);
      sfor<4>([&](auto i) HC_INL { v[4 * Ki + i] = cadd(v[4 * Ki + i], t4[i]); });
    });
  }
  if constexpr (!FINAL) {
    tm_store<E0>(ta, v);  // completion awaited before the next tcgen05.ld (the product's)
  } else {
    sfor<C0>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int b = tid + c * Cfg::T;
      if (bvalid<Cfg, 0>(c, tid))
        sfor<R0>([&](auto Ai) HC_INL {
          const int s = Ns1 * Ai + b;
          const double2 w = cscale(v[c * R0 + Ai], scale);
          if constexpr (SYM == SYM_COMPLEX) {
            if (s < L) Y[s] = w;
          } else {
            if (s < LH) Y[s + H] = w;
            else if (s >= BH) Y[s - BH] = w;
          }
        });
    });
  }
}

// --------------------------------------------------------- conv1d, ping-pong --
#ifndef HC_PP_BULK
#define HC_PP_BULK 1
#endif
#ifndef HC_PP_TMEM
#define HC_PP_TMEM 1
#endif
#ifndef HC_PP_TMEM_F
#define HC_PP_TMEM_F 1
#endif
// Two line buffers X and Y per group.  X stages f and then serves f's exchanges (and holds the
// stashed spectrum F), Y stages g and then serves g's and the inverse's exchanges.  The copy of
// the next f line into X starts as soon as F has been consumed by the product, the next g line
// into Y as soon as the inverse releases Y: each copy gets a full transform of lead time.
// Requires unit-stride lines of at most XS values (host: conv_layout).
template <int SYM, class Cfg, int G, bool STASH_REGS, int MINB = 1>
__global__ void __launch_bounds__(Cfg::T * G, MINB) k_conv1d_pp(ConvArgs p) {
  extern __shared__ __align__(16) double2 smem[];
  __shared__ __align__(8) uint64_t bars[2 * G];
  __shared__ uint32_t tm_base;
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), NBL = Cfg::NB(Cfg::P - 1);
  // tensor memory for the stashed spectrum F and the residue accumulator: kernels whose two
  // line buffers exclude a second CTA on the SM (so the whole TMEM is this CTA's)
  // (F in TMEM too frees X right after the f transform: c2 0.795 ms vs 0.815 with F in X;
  // sharing TMEM between several CTAs per SM measured slower for c1's 2048-point plan)
  using TLmax = TmemLayout<T * G, Cfg::ES, Cfg::C(0) * Cfg::R(0)>;
  constexpr bool TM_OK = !STASH_REGS && TLmax::FITS && 2 * Cfg::XS * G * 16 > 116 * 1024;
  constexpr bool TM_F = HC_PP_TMEM_F && TM_OK;
  using TL = TmemLayout<T * G, TM_F ? Cfg::ES : 0, Cfg::C(0) * Cfg::R(0)>;
  constexpr bool TMS = HC_PP_TMEM && TM_OK && TL::FITS;
  constexpr bool TMF = TMS && TM_F;
  constexpr bool F_OFF = STASH_REGS || TMF;  // F does not occupy X after the f transform
  const int g = threadIdx.x / T, tid = threadIdx.x % T;
  double2* tb = smem;
  const double2* mt = tb;
  double2* X = smem + p.ax.tabn + g * p.gs;
  double2* Y = X + Cfg::XS;
  uint64_t* bar_f = &bars[2 * g];
  uint64_t* bar_g = &bars[2 * g + 1];
  const GroupSync sync{g + 1, T};
  const AxisDev& a = p.ax;
  stage_tables(tb, a, a.tabn);
  const double2* tp = tb;  // host: the ping-pong kernel runs only with every table staged
  if (tid == 0) {
    mbar_init(bar_f, 1);
    mbar_init(bar_g, 1);
    fence_mbar_init();
  }
  if constexpr (TMS) {
    if (threadIdx.x < 32) tmem_alloc(&tm_base, TL::COLS);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
  }
  sync();
  const uint32_t tf = TMS ? TL::f_addr(tm_base) : 0u, ta = TMS ? TL::a_addr(tm_base) : 0u;
  // accumulator in TMEM: complex / centered without folding (L <= B)
  const bool acc_tm = TMS && SYM != SYM_HERMITIAN && a.L <= a.B;
  uint32_t ph_f = 0, ph_g = 0;
  const uint32_t row_bytes = (uint32_t)a.S * 16u;
  const long long es = p.lin.es, step = (long long)gridDim.x * G;
  double2* slot = p.scratch + (long long)(blockIdx.x * G + g) * a.S;
  long long item = (long long)blockIdx.x * G + g;
  if (tid == 0 && item < p.lin.count) {
    tma_copy(X, p.f + p.lin.base(item), row_bytes, bar_f);
    tma_copy(Y, p.g + p.lin.base(item), row_bytes, bar_g);
  }
  // complex / centered: each residue's output is assembled in Y and written out by a bulk
  // copy (the SM moves on while it drains); the next g copy into Y waits for its reads
  constexpr bool BULK = SYM != SYM_HERMITIAN && HC_PP_BULK;
  const double2* g_next = nullptr;  // pending next-g copy (issued once the bulk store read Y)
  const bool tr = p.trace && blockIdx.x == 0 && threadIdx.x == 0;
  int tn = 0;
#define HC_TRACE()                                   \
  do {                                               \
    if (p.trace) {                                   \
      sync();                                        \
      if (tr && tn < 256) p.trace[tn++] = clock64(); \
    }                                                \
  } while (0)
  for (; item < p.lin.count; item += step) {
    const long long base = p.lin.base(item);
    for (int res = 0; res < a.n; ++res) {
      HC_TRACE();
      const bool last = res == a.n - 1;
      const long long nbase = !last ? base : (item + step < p.lin.count ? p.lin.base(item + step) : -1);
      double2 v[Cfg::E];
      double2 Fr[STASH_REGS ? Cfg::E : 1];
      const P0Res<SYM> p0{&a, tp, res};
      // ---- forward f (staged in X, exchanges in X)
      mbar_wait(bar_f, ph_f);
      ph_f ^= 1;
      HC_TRACE();
      if (!(p.dbg & 2)) {
        if constexpr (SYM == SYM_HERMITIAN) {
          if (a.S <= Cfg::N / 2) {
            herm_load_padded<Cfg>(v, X, a, tb, res, tid);
          } else {
            herm_pack<T, Cfg::Ns(1)>(X, a, tb, res, tid);
            sync();
            load_plain<Cfg>(v, X, tid);
          }
        } else {
          load_pass0_pp<SYM, Cfg>(v, a, tb, X, res, tid);
        }
      }
      sync();
      HC_TRACE();
      auto hk = [&]() HC_INL {
        // F kept in registers / TMEM: X is free right away for the next f line
        if (F_OFF && tid == 0 && nbase >= 0) tma_copy(X, p.f + nbase, row_bytes, bar_f);
      };
      auto hk0 = [&]() HC_INL {
        // the previous residue's bulk store has had a load and a pass to read Y
        if (BULK && g_next && tid == 0) {
          bulk_wait_read();
          tma_copy(Y, g_next, row_bytes, bar_g);
        }
      };
      fft_forward<Cfg, GroupSync, P0Res<SYM>, decltype(hk), 1, decltype(hk0)>(v, X, mt, tid, sync, p0, hk, hk0);
      if constexpr (BULK) g_next = nullptr;
      sfor<CL>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        if (bvalid<Cfg, Cfg::P - 1>(c, tid))
          sfor<RL>([&](auto Ki) HC_INL {
            if constexpr (STASH_REGS) Fr[c * RL + Ki] = v[c * RL + Ki];
            else if constexpr (!TMF) X[Ki * NBL + tid + c * T] = v[c * RL + Ki];
          });
      });
      if constexpr (TMF) tm_store<Cfg::ES>(tf, v);  // completion awaited just before the product
      HC_TRACE();
      // ---- forward g (staged in Y, exchanges in Y)
      mbar_wait(bar_g, ph_g);
      ph_g ^= 1;
      HC_TRACE();
      if (!(p.dbg & 2)) {
        if constexpr (SYM == SYM_HERMITIAN) {
          if (a.S <= Cfg::N / 2) {
            herm_load_padded<Cfg>(v, Y, a, tb, res, tid);
          } else {
            herm_pack<T, Cfg::Ns(1)>(Y, a, tb, res, tid);
            sync();
            load_plain<Cfg>(v, Y, tid);
          }
        } else {
          load_pass0_pp<SYM, Cfg>(v, a, tb, Y, res, tid);
        }
      }
      sync();
      HC_TRACE();
      fft_forward<Cfg>(v, Y, mt, tid, sync, p0);
      HC_TRACE();
      if constexpr (TMS) tmem_wait_st();  // the previous residue's accumulator stores
      if constexpr (TMF) {
        // F back from TMEM four values at a time (the whole F does not fit beside G in registers);
        if (!(p.dbg & 4)) sfor<Cfg::ES / 4>([&](auto Ki) HC_INL {
          double2 F4[4];
          tm_ld4(tf + 16 * Ki, F4);
          sfor<4>([&](auto i) HC_INL {
            double2& G_ = v[4 * Ki + i];
            const double2 F = F4[i];
            if constexpr (SYM == SYM_HERMITIAN) G_ = make_double2(G_.x * F.x, G_.y * F.y);
            else G_ = cmul(G_, F);
          });
        });
      } else if (!(p.dbg & 4)) sfor<CL>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        if (bvalid<Cfg, Cfg::P - 1>(c, tid))
          sfor<RL>([&](auto Ki) HC_INL {
            double2 F;
            if constexpr (STASH_REGS) F = Fr[c * RL + Ki];
            else F = X[Ki * NBL + tid + c * T];
            double2& G_ = v[c * RL + Ki];
            if constexpr (SYM == SYM_HERMITIAN) G_ = make_double2(G_.x * F.x, G_.y * F.y);
            else G_ = cmul(G_, F);
          });
      });
      if constexpr (!F_OFF) {
        sync();  // every thread has read its stashed F: X is free for the next f line
        if (tid == 0 && nbase >= 0) tma_copy(X, p.f + nbase, row_bytes, bar_f);
      }
      // ---- inverse (exchanges in Y).  Once Y is released it receives the accumulator slot
      //      (after residue 0, so the stores' read-modify-write never waits on L2) and then,
      //      after the stores, the next g line; at residue 0 the next g line directly.
      const bool acc_y = SYM != SYM_HERMITIAN && res > 0 && !acc_tm;
      auto release_y = [&]() HC_INL {
        if (SYM != SYM_HERMITIAN && tid == 0) {
          if (acc_tm) {
            // outputs of a non-final residue go to TMEM: Y is free for the next g line now
            // (writing the final residue straight from registers instead of a bulk store from Y
            // measured slower: c2 0.795 -> 0.825 ms)
            if (!last && nbase >= 0) tma_copy(Y, p.g + nbase, row_bytes, bar_g);
          } else if (acc_y) {
            if constexpr (BULK) bulk_wait_all();  // the slot's bulk store has landed
            tma_copy(Y, slot, row_bytes, bar_g);
          } else if (!BULK && nbase >= 0) {
            tma_copy(Y, p.g + nbase, row_bytes, bar_g);
          }
        }
      };
      HC_TRACE();
      if (!(p.dbg & 8)) {
        fft_inverse<Cfg>(v, Y, mt, tid, sync, p0, release_y);
      } else {
        sync();
        release_y();
      }
      HC_TRACE();
      const double2* acc = res > 0 ? slot : nullptr;
      if (acc_y) {
        mbar_wait(bar_g, ph_g);
        ph_g ^= 1;
        acc = Y;
      }
      HC_TRACE();
      const Emit em = last ? Emit{p.out + base, es, acc, 1, 1.0 / (double)a.qm, true} : Emit{slot, 1, acc, 1, 1.0, false};
      if constexpr (SYM == SYM_HERMITIAN) {
        store_herm<Cfg>(v, a, tp, em, res, tid, Y, sync);
        if (tid == 0 && nbase >= 0) tma_copy(Y, p.g + nbase, row_bytes, bar_g);
      } else if (BULK && acc_tm) {
        if (last) {
          if (!(p.dbg & 1)) {
            if (res) acc_tmem_pp<SYM, Cfg, false, true>(v, a, tb, ta, Y, em.scale, res, tid);
            else acc_tmem_pp<SYM, Cfg, true, true>(v, a, tb, ta, Y, em.scale, res, tid);
          }
          fence_proxy_async_smem();
          sync();
          if (tid == 0) tma_store(p.out + base, Y, row_bytes, true);
          g_next = nbase >= 0 ? p.g + nbase : nullptr;
        } else {
          if (res) acc_tmem_pp<SYM, Cfg, false, false>(v, a, tb, ta, Y, 1.0, res, tid);
          else acc_tmem_pp<SYM, Cfg, true, false>(v, a, tb, ta, Y, 1.0, res, tid);
        }
      } else if constexpr (BULK) {
        // acc_y <=> res > 0: the accumulator is staged in Y, updated in place
        if (!(p.dbg & 1)) {
          if (last) {
            if (acc_y) store_pass0_pp<SYM, Cfg, true, true, true>(v, a, tb, Y, Y, em.scale, res, tid);
            else store_pass0_pp<SYM, Cfg, false, true, true>(v, a, tb, Y, Y, em.scale, res, tid);
          } else {
            if (acc_y) store_pass0_pp<SYM, Cfg, true, false, true>(v, a, tb, Y, Y, 1.0, res, tid);
            else store_pass0_pp<SYM, Cfg, false, false, true>(v, a, tb, Y, Y, 1.0, res, tid);
          }
        }
        fence_proxy_async_smem();
        sync();
        if (tid == 0) tma_store(last ? p.out + base : slot, Y, row_bytes, last);
        g_next = nbase >= 0 ? p.g + nbase : nullptr;
      } else {
        if (!(p.dbg & 1)) {
          // acc_y <=> res > 0: the accumulator is staged in Y
          if (last) {
            if (acc_y) store_pass0_pp<SYM, Cfg, true, true>(v, a, tb, p.out + base, Y, em.scale, res, tid);
            else store_pass0_pp<SYM, Cfg, false, true>(v, a, tb, p.out + base, Y, em.scale, res, tid);
          } else {
            if (acc_y) store_pass0_pp<SYM, Cfg, true, false>(v, a, tb, slot, Y, 1.0, res, tid);
            else store_pass0_pp<SYM, Cfg, false, false>(v, a, tb, slot, Y, 1.0, res, tid);
          }
        }
        if (acc_y) {
          sync();  // every thread has read its accumulator values from Y
          if (tid == 0 && nbase >= 0) tma_copy(Y, p.g + nbase, row_bytes, bar_g);
        }
      }
    }
  }
  if (BULK && tid == 0) bulk_wait_all();  // shared memory stays valid until the last store read it
  if constexpr (TMS) {
    tmem_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tm_base, TL::COLS);
  }
#undef HC_TRACE
}

// ------------------------------------------------- conv1d, ping-pong, paired --
// Complex lines with L <= B (no folding) in kernels that own the SM (X, Y and TMEM): the f and g
// forward FFTs run as ONE interleaved pair (fft_forward_pair: f's exchanges in X, g's in Y, half
// the barrier phases of two transforms, and one stream's butterflies overlap the other's
// shared-memory traffic); the product needs no stash.  TMEM keeps the residue accumulator and,
// for residues after the first, g's raw pass-0 values (the next residue re-reads only f).
//   copies: next f into X right after the pair's last exchange (a whole inverse of lead time);
//   next line's g into Y right after the inverse's last exchange, from L2 (prefetched at the
//   start of the line's last inverse); the last residue writes its outputs straight from
//   registers (streaming stores), so Y is free as soon as the inverse is done.
template <class Cfg>
__device__ __forceinline__ void load_raw_pp2(double2 (&v)[Cfg::E], int L, const double2* X, int tid) {
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), Ns1 = Cfg::Ns(1);
  sfor<C0>([&](auto Ci) HC_INL {
    constexpr int c = Ci;
    const int b = tid + c * Cfg::T;
    if (bvalid<Cfg, 0>(c, tid))
      sfor<R0>([&](auto Ai) HC_INL {
        const int s = Ns1 * Ai + b;
        v[c * R0 + Ai] = s < L ? X[s] : make_double2(0.0, 0.0);
      });
  });
}
template <class Cfg, int DIR>
__device__ __forceinline__ void twiddle_u_pp2(double2 (&v)[Cfg::E], const double2* U, int tid) {
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0);
  sfor<C0>([&](auto Ci) HC_INL {
    constexpr int c = Ci;
    if (bvalid<Cfg, 0>(c, tid)) sfor<R0>([&](auto Ai) HC_INL { v[c * R0 + Ai] = mul_tw<DIR>(v[c * R0 + Ai], U[Ai]); });
  });
}

// fft_forward_pair with the LAST pass split: passes 0 .. P-2 run paired (f through X, g through
// Y), then f's last-pass DFT runs alone and its spectrum is stashed (stash_f, e.g. to TMEM),
// then g's: at most one stream's last-pass values are live at a time (radix plans whose last
// pass holds more values per thread than two streams fit in registers, 16x16x24 at 384
// threads).  hook() runs once X is free (f's last-pass inputs loaded by every thread); Y is
// read by the time the function returns (the caller synchronises before reusing it).
template <class Cfg, class Sync, class P0, class Hook, class StashF>
__device__ __forceinline__ void fft_forward_pair_split(double2 (&v)[Cfg::E], double2 (&w)[Cfg::E], double2* X, double2* Y,
                                                       const double2* mt, int tid, const Sync& sync, const P0& p0,
                                                       const Hook& hook, const StashF& stash_f) {
  constexpr int P = Cfg::P, T = Cfg::T;
  static_assert(P >= 2, "radix plans have at least two passes");
  sfor<P - 1>([&](auto I) HC_INL {
    constexpr int i = I;
    constexpr int R = Cfg::R(i), C = Cfg::C(i), NB = Cfg::NB(i), Ns1 = Cfg::Ns(i + 1), Rp = Cfg::Rprod(i);
    sfor<C>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (NB % T == 0 || beta < NB) {
        DFT<R, +1>::run(v + c * R);
        DFT<R, +1>::run(w + c * R);
        if constexpr (i == 0) {
          double2 t, tw;
          p0(beta, t, tw);
          sfor<R>([&](auto Ki) HC_INL {
            constexpr int k = Ki;
            v[c * R + k] = cmul(v[c * R + k], t);
            w[c * R + k] = cmul(w[c * R + k], t);
            if constexpr (k + 1 < R) t = cmul(t, tw);
          });
        } else {
          const int b = beta % Ns1;
          sfor<R - 1>([&](auto Ki) HC_INL {
            constexpr int k = Ki + 1;
            const double2 tw = mt[Cfg::MTo(i) + (k - 1) * Ns1 + b];
            v[c * R + k] = cmul(v[c * R + k], tw);
            w[c * R + k] = cmul(w[c * R + k], tw);
          });
        }
        const int K = beta / Ns1, b = beta % Ns1;
        constexpr int St = Cfg::St(i + 1);
        sfor<R>([&](auto Ki) HC_INL {
          X[(K + Rp * Ki) * St + b] = v[c * R + Ki];
          Y[(K + Rp * Ki) * St + b] = w[c * R + Ki];
        });
      }
    });
    sync();
    constexpr int R2 = Cfg::R(i + 1), C2 = Cfg::C(i + 1), NB2 = Cfg::NB(i + 1), Ns2 = Cfg::Ns(i + 2);
    constexpr int St = Cfg::St(i + 1);
    if constexpr (i + 1 < P - 1) {
      sfor<C2>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        const int beta = tid + c * T;
        if (NB2 % T == 0 || beta < NB2) {
          const int K = beta / Ns2, b = beta % Ns2;
          sfor<R2>([&](auto Ai) HC_INL {
            v[c * R2 + Ai] = X[K * St + Ns2 * Ai + b];
            w[c * R2 + Ai] = Y[K * St + Ns2 * Ai + b];
          });
        }
      });
      sync();
    } else {
      // last pass: f alone (X), stash, then g (Y)
      sfor<C2>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        const int beta = tid + c * T;
        if (NB2 % T == 0 || beta < NB2) {
          const int K = beta / Ns2, b = beta % Ns2;
          sfor<R2>([&](auto Ai) HC_INL { v[c * R2 + Ai] = X[K * St + Ns2 * Ai + b]; });
        }
      });
      sync();
      hook();
      sfor<C2>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        if (NB2 % T == 0 || tid + c * T < NB2) DFT<R2, +1>::run(v + c * R2);
      });
      stash_f(v);
      sfor<C2>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        const int beta = tid + c * T;
        if (NB2 % T == 0 || beta < NB2) {
          const int K = beta / Ns2, b = beta % Ns2;
          sfor<R2>([&](auto Ai) HC_INL { w[c * R2 + Ai] = Y[K * St + Ns2 * Ai + b]; });
          DFT<R2, +1>::run(w + c * R2);
        }
      });
    }
  });
}

template <class Cfg, int G, int MINB = 1>
__global__ void __launch_bounds__(Cfg::T * G, MINB) k_conv1d_pp2(ConvArgs p) {
  extern __shared__ __align__(16) double2 smem[];
  __shared__ __align__(8) uint64_t bars[2 * G];
  __shared__ uint32_t tm_base;
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1);
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), E0 = C0 * R0, Ns1 = Cfg::Ns(1);
  // split last pass (more than 16 last-pass values per thread): f's spectrum parks in TMEM in
  // place of g's raw values (TMEM holds 512 columns), and g is re-copied for every residue
  constexpr bool SPLIT = Cfg::ES > 16;
  using TL = TmemLayout<T * G, SPLIT ? Cfg::ES : E0, E0>;  // g raw (or f spectrum), accumulator
  static_assert(TL::FITS, "TMEM layout");
  const int g = threadIdx.x / T, tid = threadIdx.x % T;
  double2* tb = smem;
  const double2* mt = tb;
  double2* X = smem + p.ax.tabn + g * p.gs;
  double2* Y = X + Cfg::XS;
  uint64_t* bar_f = &bars[2 * g];
  uint64_t* bar_g = &bars[2 * g + 1];
  const GroupSync sync{g + 1, T};
  const AxisDev& a = p.ax;
  stage_tables(tb, a, a.tabn);
  if (tid == 0) {
    mbar_init(bar_f, 1);
    mbar_init(bar_g, 1);
    fence_mbar_init();
  }
  // TMEM only with several residues (g stash, accumulator); every CTA resident on the SM fits
  // its columns (registry: pp2 instantiated only when they do)
  const bool use_tm = a.n > 1;
  if (use_tm && threadIdx.x < 32) tmem_alloc(&tm_base, TL::COLS);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tg = use_tm ? TL::f_addr(tm_base) : 0u, ta = use_tm ? TL::a_addr(tm_base) : 0u, tf = tg;
  uint32_t ph_f = 0, ph_g = 0;
  const uint32_t row_bytes = (uint32_t)a.S * 16u;
  const long long es = p.lin.es, step = (long long)gridDim.x * G;
  const int L = a.L, n = a.n;
  const double scale = 1.0 / (double)a.qm;
  long long item = (long long)blockIdx.x * G + g;
  if (tid == 0 && item < p.lin.count) {
    tma_copy(X, p.f + p.lin.base(item), row_bytes, bar_f);
    tma_copy(Y, p.g + p.lin.base(item), row_bytes, bar_g);
  }
  for (; item < p.lin.count; item += step) {
    const long long base = p.lin.base(item);
    const long long next = item + step < p.lin.count ? p.lin.base(item + step) : -1;
    for (int res = 0; res < n; ++res) {
      const bool last = res == n - 1;
      const P0Res<SYM_COMPLEX> p0{&a, tb, res};
      const double2* U = tb + (a.oU + res * a.nu);
      double2 v[Cfg::E], w[Cfg::E];
      if (use_tm) tmem_wait_st();  // the previous residue's TMEM stores (accumulator, g stash)
      mbar_wait(bar_f, ph_f);
      ph_f ^= 1;
      load_raw_pp2<Cfg>(v, L, X, tid);
      if (res == 0 || SPLIT) {
        mbar_wait(bar_g, ph_g);
        ph_g ^= 1;
        load_raw_pp2<Cfg>(w, L, Y, tid);
        if constexpr (!SPLIT) {
          if (n > 1) tm_store<E0>(tg, w);
        }
        if (res) {
          twiddle_u_pp2<Cfg, +1>(v, U, tid);
          twiddle_u_pp2<Cfg, +1>(w, U, tid);
        }
      } else {
        sfor<E0 / 4>([&](auto Ki) HC_INL { tm_ld4(tg + 16 * Ki, w + 4 * Ki); });
        twiddle_u_pp2<Cfg, +1>(v, U, tid);
        twiddle_u_pp2<Cfg, +1>(w, U, tid);
      }
      sync();  // X and Y consumed before the pair's first exchange overwrites them
      auto hk = [&]() HC_INL {  // X and Y free: next f (this line's next residue, or the next line)
        if (tid == 0) {
          const long long nb = last ? next : base;
          if (nb >= 0) tma_copy(X, p.f + nb, row_bytes, bar_f);
          if (last && next >= 0) l2_prefetch(p.g + next, row_bytes);
        }
      };
      if constexpr (SPLIT) {
        // f's spectrum parks in TMEM while g's last pass runs; the product lands in v
        auto stash = [&](const double2(&x)[Cfg::E]) HC_INL { tm_store<Cfg::ES>(tf, x); };
        fft_forward_pair_split<Cfg, GroupSync, P0Res<SYM_COMPLEX>, decltype(hk), decltype(stash)>(v, w, X, Y, mt, tid,
                                                                                                  sync, p0, hk, stash);
        tmem_wait_st();
        sfor<Cfg::ES / 4>([&](auto Ki) HC_INL {
          double2 F4[4];
          tm_ld4(tf + 16 * Ki, F4);
          sfor<4>([&](auto i) HC_INL { v[4 * Ki + i] = cmul(w[4 * Ki + i], F4[i]); });
        });
        sync();  // Y read by every thread before the inverse's first exchange
      } else {
        fft_forward_pair<Cfg, GroupSync, P0Res<SYM_COMPLEX>, decltype(hk)>(v, w, X, Y, mt, tid, sync, p0, hk);
        sfor<CL>([&](auto Ci) HC_INL {
          constexpr int c = Ci;
          if (bvalid<Cfg, Cfg::P - 1>(c, tid)) sfor<RL>([&](auto Ki) HC_INL { v[c * RL + Ki] = cmul(v[c * RL + Ki], w[c * RL + Ki]); });
        });
      }
      auto hki = [&]() HC_INL {  // Y free: the next line's g (L2-prefetched); SPLIT: this line's again
        if (tid == 0) {
          if (last && next >= 0) tma_copy(Y, p.g + next, row_bytes, bar_g);
          else if (SPLIT && !last) tma_copy(Y, p.g + base, row_bytes, bar_g);
        }
      };
      fft_inverse<Cfg, GroupSync, P0Res<SYM_COMPLEX>, decltype(hki)>(v, Y, mt, tid, sync, p0, hki);
      if (res) twiddle_u_pp2<Cfg, -1>(v, U, tid);
      if (res) {
        sfor<E0 / 4>([&](auto Ki) HC_INL {
          double2 t4[4];
          tm_ld4(ta + 16 * Ki, t4);
          sfor<4>([&](auto i) HC_INL { v[4 * Ki + i] = cadd(v[4 * Ki + i], t4[i]); });
        });
      }
      if (!last) {
        tm_store<E0>(ta, v);
      } else {
        double2* out = p.out + base;
        sfor<C0>([&](auto Ci) HC_INL {
          constexpr int c = Ci;
          const int b = tid + c * T;
          if (bvalid<Cfg, 0>(c, tid))
            sfor<R0>([&](auto Ai) HC_INL {
              const int s = Ns1 * Ai + b;
              if (s < L) __stcs(out + (long long)s * es, cscale(v[c * R0 + Ai], scale));
            });
        });
      }
    }
  }
  if (use_tm) tmem_wait_st();
  tmem_fence_before();
  __syncthreads();
  if (use_tm && threadIdx.x < 32) tmem_dealloc(tm_base, TL::COLS);
}

// --------------------------------------------------------- column-tile pfft --
// Outer-axis passes of the N-D driver read columns at a large element stride.  Here the GC
// line groups of a CTA take GC ADJACENT columns and interleave thread by thread (thread t ->
// group t % GC), so every load/store instruction of a warp touches GC consecutive columns
// (coalesced), and the groups' exchange buffers interleave element by element (conflict-free).
// Complex / centered data only (Hermitian is always the innermost, contiguous axis).
template <int SYM, class Cfg, int GC>
__global__ void __launch_bounds__(Cfg::T * GC, 1) k_pfft_fwd_cols(FwdArgs p) {
  static_assert(SYM != SYM_HERMITIAN, "column tiles serve outer (non-Hermitian) axes");
  extern __shared__ __align__(16) double2 smem[];
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), RpL = Cfg::Rprod(Cfg::P - 1);
  const int g = threadIdx.x % GC, tid = threadIdx.x / GC;
  double2* tb = smem;
  const double2* mt = tb;
  double2* X = smem + p.ax.tabn + g;
  const CtaSync sync;
  const AxisDev& a = p.ax;
  stage_tables(tb, a, a.tabn);
  const double2* tp = a.tabn >= a.tabfull ? tb : a.tab;
  const P0Res<SYM> p0{&a, tp, p.v};
  const long long rounds = (p.lin.count + (long long)gridDim.x * GC - 1) / ((long long)gridDim.x * GC);
  for (long long rd = 0; rd < rounds; ++rd) {
    const long long item = (rd * gridDim.x + blockIdx.x) * GC + g;
    const bool live = item < p.lin.count;
    double2 v[Cfg::E];
    if (live) load_pass0<SYM, Cfg>(v, a, tp, p.f + p.lin.base(item), p.lin.es, p.v, tid);
    fft_forward<Cfg, CtaSync, P0Res<SYM>, NoHook, GC>(v, X, mt, tid, sync, p0);
    if (!live) continue;
    const long long ob = p.lout.base(item), oes = p.lout.es;
    double2* F = (double2*)p.F;
    sfor<CL>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (bvalid<Cfg, Cfg::P - 1>(c, tid))
        sfor<RL>([&](auto Ki) HC_INL {
          const long long kp = beta + (long long)RpL * Ki;
          F[ob + (p.ref_order ? ref_index(a, kp) : kp) * oes] = v[c * RL + Ki];
        });
    });
  }
}

template <int SYM, class Cfg, int GC>
__global__ void __launch_bounds__(Cfg::T * GC, 1) k_pfft_bwd_cols(BwdArgs p) {
  static_assert(SYM != SYM_HERMITIAN, "column tiles serve outer (non-Hermitian) axes");
  extern __shared__ __align__(16) double2 smem[];
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), RpL = Cfg::Rprod(Cfg::P - 1);
  const int g = threadIdx.x % GC, tid = threadIdx.x / GC;
  double2* tb = smem;
  const double2* mt = tb;
  double2* X = smem + p.ax.tabn + g;
  const CtaSync sync;
  const AxisDev& a = p.ax;
  stage_tables(tb, a, a.tabn);
  const double2* tp = a.tabn >= a.tabfull ? tb : a.tab;
  const P0Res<SYM> p0{&a, tp, p.v};
  const long long rounds = (p.lin.count + (long long)gridDim.x * GC - 1) / ((long long)gridDim.x * GC);
  for (long long rd = 0; rd < rounds; ++rd) {
    const long long item = (rd * gridDim.x + blockIdx.x) * GC + g;
    const bool live = item < p.lin.count;
    double2 v[Cfg::E];
    if (live) {
      const long long ib = p.lin.base(item), ies = p.lin.es;
      const double2* F = (const double2*)p.F;
      sfor<CL>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        const int beta = tid + c * T;
        if (bvalid<Cfg, Cfg::P - 1>(c, tid))
          sfor<RL>([&](auto Ki) HC_INL {
            const long long kp = beta + (long long)RpL * Ki;
            v[c * RL + Ki] = F[ib + (p.ref_order ? ref_index(a, kp) : kp) * ies];
          });
      });
    }
    fft_inverse<Cfg, CtaSync, P0Res<SYM>, NoHook, GC>(v, X, mt, tid, sync, p0);
    if (!live) continue;
    const long long ob = p.lout.base(item);
    const Emit em{p.dst + ob, p.lout.es, p.acc ? p.acc + ob : nullptr, p.lout.es, p.scale};
    store_pass0<SYM, Cfg>(v, a, tp, em, p.v, tid);
  }
}

// ------------------------------------------------- column-tile pfft, pipelined --
// The same column tiles as k_pfft_fwd_cols / k_pfft_bwd_cols, software-pipelined: the CTA owns
// two tile buffers of GC x max(XS, rows) values (element j of column g at [j GC + g]).  While
// the FFT of tile k runs in one buffer (its staged input, then its exchanges), every thread's
// cp.async copies gather tile k + gridDim.x into the other, so the strided row reads overlap
// the butterflies instead of stalling them (the unpipelined kernels are ~40 % long-scoreboard
// stalls at one CTA per SM).  Natural block order only (the N-D driver's work arrays).
template <int SYM, class Cfg, int GC>
__global__ void __launch_bounds__(Cfg::T * GC, 1) k_pfft_fwd_cols_pp(FwdArgs p) {
  static_assert(SYM != SYM_HERMITIAN, "column tiles serve outer (non-Hermitian) axes");
  extern __shared__ __align__(16) double2 smem[];
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), RpL = Cfg::Rprod(Cfg::P - 1);
  const int g = threadIdx.x % GC, tid = threadIdx.x / GC;
  const AxisDev& a = p.ax;
  double2* tb = smem;
  const double2* mt = tb;
  stage_tables(tb, a, a.tabn);
  const double2* tp = a.tabn >= a.tabfull ? tb : a.tab;
  const P0Res<SYM> p0{&a, tp, p.v};
  const int rows = a.S;
  const int bufn = GC * (rows > Cfg::XS ? rows : Cfg::XS);
  // (buffer k & 1 is addressed by arithmetic on the shared-memory base: selecting from an array of
  // pointers hides the address space from the compiler and every access turns generic, LD.E / ST.E)
  double2* const buf0 = smem + a.tabn;
  const long long ntiles = (p.lin.count + GC - 1) / GC;
  const long long es = p.lin.es;
  auto gather = [&](long long t, double2* B) HC_INL {
    const long long item = t * GC + g;
    if (t < ntiles && item < p.lin.count) {
      const double2* src = p.f + p.lin.base(item);
      for (int j = tid; j < rows; j += T) cp_async16(B + j * GC + g, src + j * es);
    }
    cp_async_commit();
  };
  gather(blockIdx.x, buf0);
  int k = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    double2* X = buf0 + (k & 1) * bufn;
    __syncthreads();  // the previous tile's exchanges in the other buffer are finished
    gather(t + gridDim.x, buf0 + ((k + 1) & 1) * bufn);
    cp_async_wait<1>();
    __syncthreads();  // tile t has landed (every thread's copies)
    const long long item = t * GC + g;
    const bool live = item < p.lin.count;
    double2 v[Cfg::E];
    if (live) load_pass0<SYM, Cfg>(v, a, tp, X + g, GC, p.v, tid);
    __syncthreads();  // the staged tile is consumed before the first exchange overwrites it
    fft_forward<Cfg, CtaSync, P0Res<SYM>, NoHook, GC>(v, X + g, mt, tid, CtaSync(), p0);
    if (!live) continue;
    const long long ob = p.lout.base(item), oes = p.lout.es;
    double2* F = (double2*)p.F;
    sfor<CL>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (bvalid<Cfg, Cfg::P - 1>(c, tid))
        sfor<RL>([&](auto Ki) HC_INL { F[ob + (beta + (long long)RpL * Ki) * oes] = v[c * RL + Ki]; });
    });
  }
  cp_async_wait<0>();
}

template <int SYM, class Cfg, int GC>
__global__ void __launch_bounds__(Cfg::T * GC, 1) k_pfft_bwd_cols_pp(BwdArgs p) {
  static_assert(SYM != SYM_HERMITIAN, "column tiles serve outer (non-Hermitian) axes");
  extern __shared__ __align__(16) double2 smem[];
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), RpL = Cfg::Rprod(Cfg::P - 1);
  const int g = threadIdx.x % GC, tid = threadIdx.x / GC;
  const AxisDev& a = p.ax;
  double2* tb = smem;
  const double2* mt = tb;
  stage_tables(tb, a, a.tabn);
  const double2* tp = a.tabn >= a.tabfull ? tb : a.tab;
  const P0Res<SYM> p0{&a, tp, p.v};
  constexpr int rows = Cfg::N;  // block values (complex)
  constexpr int bufn = GC * Cfg::XS;
  // (buffer k & 1 is addressed by arithmetic on the shared-memory base: selecting from an array of
  // pointers hides the address space from the compiler and every access turns generic, LD.E / ST.E)
  double2* const buf0 = smem + a.tabn;
  const long long ntiles = (p.lin.count + GC - 1) / GC;
  const long long ies = p.lin.es;
  const double2* F = (const double2*)p.F;
  auto gather = [&](long long t, double2* B) HC_INL {
    const long long item = t * GC + g;
    if (t < ntiles && item < p.lin.count) {
      const double2* src = F + p.lin.base(item);
      for (int j = tid; j < rows; j += T) cp_async16(B + j * GC + g, src + j * ies);
    }
    cp_async_commit();
  };
  gather(blockIdx.x, buf0);
  int k = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    double2* X = buf0 + (k & 1) * bufn;
    __syncthreads();
    gather(t + gridDim.x, buf0 + ((k + 1) & 1) * bufn);
    cp_async_wait<1>();
    __syncthreads();
    const long long item = t * GC + g;
    const bool live = item < p.lin.count;
    double2 v[Cfg::E];
    sfor<CL>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (bvalid<Cfg, Cfg::P - 1>(c, tid))
        sfor<RL>([&](auto Ki) HC_INL { v[c * RL + Ki] = X[(beta + RpL * Ki) * GC + g]; });
    });
    __syncthreads();
    fft_inverse<Cfg, CtaSync, P0Res<SYM>, NoHook, GC>(v, X + g, mt, tid, CtaSync(), p0);
    if (!live) continue;
    const long long ob = p.lout.base(item);
    const Emit em{p.dst + ob, p.lout.es, p.acc ? p.acc + ob : nullptr, p.lout.es, p.scale};
    store_pass0<SYM, Cfg>(v, a, tp, em, p.v, tid);
  }
  cp_async_wait<0>();
}

// Whole-CTA barriers whose first write-after-read wait (before the first exchange's stores) runs a
// gate instead: used when the exchange buffer is released by something other than this transform.
template <class Gate>
struct GatedCtaSync {
  const Gate& gate;
  mutable bool open = false;
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
  __device__ __forceinline__ void war_arrive() const { __syncthreads(); }
  __device__ __forceinline__ void war_wait() const {
    if (!open) gate();
    open = true;
  }
};
// ------------------------------------------ column-tile pfft, tensor-map TMA --
// The pipelined column tiles with every tile moved by the TMA engine instead of per-thread
// copies: a 3D tensor map {inner columns, rows, outer} (float64 pairs) describes the strided
// columns, one thread issues the box loads of the next tile (<= 256 rows per box) onto the
// buffer's mbarrier, and -- forward -- the finished block is staged in the tile buffer and
// written back by tensor stores (bulk groups), so neither direction occupies the LSU and the
// SM computes the next tile while the copies run.  Tiles never straddle an outer index (host:
// GC divides the inner extent).  Natural block order only.
__device__ __forceinline__ double2* align_smem128(double2* p) {
  const uint32_t a = smem_u32(p);
  return p + (((a + 127u) & ~127u) - a) / 16u;
}
struct TileMaps {
  int inner;           // columns per outer index (nin)
  int rows_in;         // rows of the input tile (data rows, or the block for the inverse)
  int box_in, box_out; // rows per tensor box (<= 256) of the input and output maps
  int bufn;            // complex values per tile buffer (host: >= every box row written or read)
  int nb_stage = 0;    // k_pfft_bwd_cols_tma1: leading input boxes prefetched into the staging area
};
template <int SYM, class Cfg, int GC>
__global__ void __launch_bounds__(Cfg::T * GC, 1)
    k_pfft_fwd_cols_tma(FwdArgs p, TileMaps tm, const __grid_constant__ CUtensorMap min,
                        const __grid_constant__ CUtensorMap mout) {
  static_assert(SYM != SYM_HERMITIAN, "column tiles serve outer (non-Hermitian) axes");
  extern __shared__ __align__(16) double2 smem[];
  __shared__ __align__(8) uint64_t bars[2];
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), RpL = Cfg::Rprod(Cfg::P - 1);
  constexpr int N = Cfg::N;
  const int g = threadIdx.x % GC, tid = threadIdx.x / GC;
  const AxisDev& a = p.ax;
  double2* tb = smem;
  const double2* mt = tb;
  stage_tables(tb, a, a.tabn);
  const double2* tp = a.tabn >= a.tabfull ? tb : a.tab;
  const P0Res<SYM> p0{&a, tp, p.v};
  const int rows = tm.rows_in;
  // tensor copies need 128-byte-aligned shared addresses (the dynamic segment follows the static
  // mbarriers, so align the absolute address; the host adds the slack)
  double2* buf0 = align_smem128(smem + a.tabn);
  // (buffer b is buf0 + b * bufn: arithmetic on the shared-memory base keeps the accesses LDS / STS)
  const long long ntiles = p.lin.count / GC;
  const bool leader = threadIdx.x == 0;
  const int kBox = tm.box_in;
  const int nbox_in = (rows + kBox - 1) / kBox;
  const uint32_t box_bytes = (uint32_t)GC * 16u * (uint32_t)kBox;
  auto issue = [&](long long t, int b) HC_INL {
    if (t >= ntiles) return;
    const long long item = t * GC;
    const int c0 = (int)(2 * (item % tm.inner)), c2 = (int)(item / tm.inner);
    mbar_expect_tx(&bars[b], box_bytes * (uint32_t)nbox_in);
    for (int r = 0; r < nbox_in; ++r) tma_tensor_load_3d(buf0 + (size_t)b * tm.bufn + (size_t)r * kBox * GC, &min, c0, r * kBox, c2, &bars[b]);
  };
  if (leader) {
    tma_prefetch_map(&min);
    tma_prefetch_map(&mout);
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (leader) issue(blockIdx.x, 0);
  uint32_t ph[2] = {0, 0};
  int k = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int b = k & 1;
    double2* X = buf0 + (size_t)b * tm.bufn;
    mbar_wait(&bars[b], ph[b]);
    ph[b] ^= 1;
    double2 v[Cfg::E];
    load_pass0<SYM, Cfg>(v, a, tp, X + g, GC, p.v, tid);
    // behind the pass-0 butterflies: the next tile's copy into the other buffer, once that buffer's
    // last tensor store has read its block (waiting for it at the top of the tile stalled the
    // leader, and with it the CTA, for the store's whole shared-memory read), and the barrier that
    // says the staged tile is consumed before the first exchange overwrites it
    auto gate = [&]() HC_INL {
      if (leader) {
        bulk_wait_read();
        issue(t + gridDim.x, b ^ 1);
      }
      __syncthreads();
    };
    const GatedCtaSync<decltype(gate)> gs{gate};
    fft_forward<Cfg, GatedCtaSync<decltype(gate)>, P0Res<SYM>, NoHook, GC>(v, X + g, mt, tid, gs, p0);
    // (fft_forward ends its last exchange with a CTA barrier: every read of X is done, X takes the block [k][GC])
    sfor<CL>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (bvalid<Cfg, Cfg::P - 1>(c, tid))
        sfor<RL>([&](auto Ki) HC_INL { X[(beta + RpL * Ki) * GC + g] = v[c * RL + Ki]; });
    });
    fence_proxy_async_smem();
    __syncthreads();
    if (leader) {
      const long long item = t * GC;
      const int c0 = (int)(2 * (item % tm.inner)), c2 = (int)(item / tm.inner);
      for (int r = 0; r * tm.box_out < N; ++r)
        tma_tensor_store_3d(&mout, c0, r * tm.box_out, c2, X + (size_t)r * tm.box_out * GC);
      bulk_commit();
    }
  }
  if (leader) bulk_wait_all();
}

template <int SYM, class Cfg, int GC>
__global__ void __launch_bounds__(Cfg::T * GC, 1)
    k_pfft_bwd_cols_tma(BwdArgs p, TileMaps tm, const __grid_constant__ CUtensorMap min) {
  static_assert(SYM != SYM_HERMITIAN, "column tiles serve outer (non-Hermitian) axes");
  extern __shared__ __align__(16) double2 smem[];
  __shared__ __align__(8) uint64_t bars[2];
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), RpL = Cfg::Rprod(Cfg::P - 1);
  constexpr int N = Cfg::N;
  const int g = threadIdx.x % GC, tid = threadIdx.x / GC;
  const AxisDev& a = p.ax;
  double2* tb = smem;
  const double2* mt = tb;
  stage_tables(tb, a, a.tabn);
  const double2* tp = a.tabn >= a.tabfull ? tb : a.tab;
  const P0Res<SYM> p0{&a, tp, p.v};
  double2* buf0 = align_smem128(smem + a.tabn);
  // (buffer b is buf0 + b * bufn: arithmetic on the shared-memory base keeps the accesses LDS / STS)
  const long long ntiles = p.lin.count / GC;
  const bool leader = threadIdx.x == 0;
  const int kBox = tm.box_in;
  const int nbox = (N + kBox - 1) / kBox;
  const uint32_t box_bytes = (uint32_t)GC * 16u * (uint32_t)kBox;
  auto issue = [&](long long t, int b) HC_INL {
    if (t >= ntiles) return;
    const long long item = t * GC;
    const int c0 = (int)(2 * (item % tm.inner)), c2 = (int)(item / tm.inner);
    mbar_expect_tx(&bars[b], box_bytes * (uint32_t)nbox);
    for (int r = 0; r < nbox; ++r) tma_tensor_load_3d(buf0 + (size_t)b * tm.bufn + (size_t)r * kBox * GC, &min, c0, r * kBox, c2, &bars[b]);
  };
  if (leader) {
    tma_prefetch_map(&min);
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (leader) issue(blockIdx.x, 0);
  uint32_t ph[2] = {0, 0};
  int k = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int b = k & 1;
    double2* X = buf0 + (size_t)b * tm.bufn;
    // the other buffer's exchanges (previous tile) ended at the barrier closing that tile
    if (leader) issue(t + gridDim.x, b ^ 1);
    mbar_wait(&bars[b], ph[b]);
    ph[b] ^= 1;
    double2 v[Cfg::E];
    sfor<CL>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (bvalid<Cfg, Cfg::P - 1>(c, tid))
        sfor<RL>([&](auto Ki) HC_INL { v[c * RL + Ki] = X[(beta + RpL * Ki) * GC + g]; });
    });
    __syncthreads();
    fft_inverse<Cfg, CtaSync, P0Res<SYM>, NoHook, GC>(v, X + g, mt, tid, CtaSync(), p0);
    const long long ob = p.lout.base(t * GC + g);
    const Emit em{p.dst + ob, p.lout.es, p.acc ? p.acc + ob : nullptr, p.lout.es, p.scale};
    store_pass0<SYM, Cfg>(v, a, tp, em, p.v, tid);
    // (X is free for the next issue into it: fft_inverse ends its last exchange with a CTA barrier)
  }
}

// ------------------------------- column-tile pfft, tensor-map TMA, one tile buffer --
// Blocks too long for two tile buffers at the full tile width (c4's 4096-point columns: one
// buffer of 2 columns is 139 KB) still overlap their copies with the butterflies:
//  * forward: the raw tile is only the data rows (half a block or less for explicit padding), so
//    it is prefetched by TMA into a separate staging area IN behind the exchange buffer X while
//    the previous tile transforms; the finished block leaves X by tensor stores, whose
//    shared-memory reads are waited for just before the next tile's first exchange;
//  * inverse: the leading boxes of the next block tile (as many as fit behind X) are prefetched
//    into a staging area while the current tile transforms; the rest is loaded into X itself as
//    soon as the last exchange of the current tile has been read (fft_inverse's hook), i.e. behind
//    the pass-0 butterflies, the post-twiddles and the strided output stores.
// Same tiles, maps and arithmetic as the two-buffer kernels above (bit-identical results).
template <int SYM, class Cfg, int GC>
__global__ void __launch_bounds__(Cfg::T * GC, 1)
    k_pfft_fwd_cols_tma1(FwdArgs p, TileMaps tm, const __grid_constant__ CUtensorMap min,
                         const __grid_constant__ CUtensorMap mout) {
  static_assert(SYM != SYM_HERMITIAN, "column tiles serve outer (non-Hermitian) axes");
  extern __shared__ __align__(16) double2 smem[];
  __shared__ __align__(8) uint64_t bar;
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), RpL = Cfg::Rprod(Cfg::P - 1);
  constexpr int N = Cfg::N;
  const int g = threadIdx.x % GC, tid = threadIdx.x / GC;
  const AxisDev& a = p.ax;
  double2* tb = smem;
  const double2* mt = tb;
  stage_tables(tb, a, a.tabn);
  const double2* tp = a.tabn >= a.tabfull ? tb : a.tab;
  const P0Res<SYM> p0{&a, tp, p.v};
  const int rows = tm.rows_in;
  double2* X = align_smem128(smem + a.tabn);
  double2* IN = X + tm.bufn;  // bufn is a multiple of 8 values: IN stays 128-byte aligned
  const long long ntiles = p.lin.count / GC;
  const bool leader = threadIdx.x == 0;
  const int kBox = tm.box_in;
  const int nbox_in = (rows + kBox - 1) / kBox;
  const uint32_t box_bytes = (uint32_t)GC * 16u * (uint32_t)kBox;
  auto issue = [&](long long t) HC_INL {
    if (t >= ntiles) return;
    const long long item = t * GC;
    const int c0 = (int)(2 * (item % tm.inner)), c2 = (int)(item / tm.inner);
    mbar_expect_tx(&bar, box_bytes * (uint32_t)nbox_in);
    for (int r = 0; r < nbox_in; ++r) tma_tensor_load_3d(IN + (size_t)r * kBox * GC, &min, c0, r * kBox, c2, &bar);
  };
  if (leader) {
    tma_prefetch_map(&min);
    tma_prefetch_map(&mout);
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (leader) issue(blockIdx.x);
  uint32_t ph = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(&bar, ph);
    ph ^= 1;
    double2 v[Cfg::E];
    load_pass0<SYM, Cfg>(v, a, tp, IN + g, GC, p.v, tid);
    // one barrier behind the pass-0 butterflies says both "IN is consumed" (the next tile's copy
    // may start) and "X is free" (the previous tile's tensor stores have read it)
    auto gate = [&]() HC_INL {
      if (leader) bulk_wait_read();
      __syncthreads();
      if (leader) issue(t + gridDim.x);
    };
    const GatedCtaSync<decltype(gate)> gs{gate};
    fft_forward<Cfg, GatedCtaSync<decltype(gate)>, P0Res<SYM>, NoHook, GC>(v, X + g, mt, tid, gs, p0);
    // (fft_forward ends its last exchange with a CTA barrier: every read of X is done, X takes the block [k][GC])
    sfor<CL>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (bvalid<Cfg, Cfg::P - 1>(c, tid))
        sfor<RL>([&](auto Ki) HC_INL { X[(beta + RpL * Ki) * GC + g] = v[c * RL + Ki]; });
    });
    fence_proxy_async_smem();
    __syncthreads();
    if (leader) {
      const long long item = t * GC;
      const int c0 = (int)(2 * (item % tm.inner)), c2 = (int)(item / tm.inner);
      for (int r = 0; r * tm.box_out < N; ++r)
        tma_tensor_store_3d(&mout, c0, r * tm.box_out, c2, X + (size_t)r * tm.box_out * GC);
      bulk_commit();
    }
  }
  if (leader) bulk_wait_all();
}

template <int SYM, class Cfg, int GC>
__global__ void __launch_bounds__(Cfg::T * GC, 1)
    k_pfft_bwd_cols_tma1(BwdArgs p, TileMaps tm, const __grid_constant__ CUtensorMap min) {
  static_assert(SYM != SYM_HERMITIAN, "column tiles serve outer (non-Hermitian) axes");
  extern __shared__ __align__(16) double2 smem[];
  __shared__ __align__(8) uint64_t bars[2];  // 0: the staged leading boxes (S), 1: the boxes loaded into X
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), RpL = Cfg::Rprod(Cfg::P - 1);
  constexpr int N = Cfg::N;
  const int g = threadIdx.x % GC, tid = threadIdx.x / GC;
  const AxisDev& a = p.ax;
  double2* tb = smem;
  const double2* mt = tb;
  stage_tables(tb, a, a.tabn);
  const double2* tp = a.tabn >= a.tabfull ? tb : a.tab;
  const P0Res<SYM> p0{&a, tp, p.v};
  double2* X = align_smem128(smem + a.tabn);
  double2* S = X + tm.bufn;  // the first nb_stage boxes of the next tile wait here
  const long long ntiles = p.lin.count / GC;
  const bool leader = threadIdx.x == 0;
  const int kBox = tm.box_in;
  const int nbox = (N + kBox - 1) / kBox, nbs = tm.nb_stage;
  const int rows_s = nbs * kBox;  // block rows below this are read from S
  const uint32_t box_bytes = (uint32_t)GC * 16u * (uint32_t)kBox;
  auto issue = [&](long long t, int r0, int r1, double2* dst, uint64_t* bar) HC_INL {
    if (t >= ntiles || r0 >= r1) return;
    const long long item = t * GC;
    const int c0 = (int)(2 * (item % tm.inner)), c2 = (int)(item / tm.inner);
    mbar_expect_tx(bar, box_bytes * (uint32_t)(r1 - r0));
    for (int r = r0; r < r1; ++r) tma_tensor_load_3d(dst + (size_t)r * kBox * GC, &min, c0, r * kBox, c2, bar);
  };
  if (leader) {
    tma_prefetch_map(&min);
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (leader) {
    issue(blockIdx.x, 0, nbs, S, &bars[0]);
    issue(blockIdx.x, nbs, nbox, X, &bars[1]);
  }
  uint32_t ph = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (nbs > 0) mbar_wait(&bars[0], ph);
    if (nbs < nbox) mbar_wait(&bars[1], ph);
    ph ^= 1;
    double2 v[Cfg::E];
    sfor<CL>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (bvalid<Cfg, Cfg::P - 1>(c, tid))
        sfor<RL>([&](auto Ki) HC_INL {
          const int row = beta + RpL * Ki;
          v[c * RL + Ki] = X[(row < rows_s ? tm.bufn : 0) + row * GC + g];  // S = X + bufn (one shared base)
        });
    });
    __syncthreads();  // the block is in registers: S may be refilled, the exchanges may use X
    if (leader) issue(t + gridDim.x, 0, nbs, S, &bars[0]);
    // the rest of the next block goes into X itself behind the barrier that ends the last exchange
    // (fft_inverse's hook), i.e. behind the pass-0 butterflies and the strided output stores
    auto next = [&]() HC_INL {
      if (leader) issue(t + gridDim.x, nbs, nbox, X, &bars[1]);
    };
    fft_inverse<Cfg, CtaSync, P0Res<SYM>, decltype(next), GC>(v, X + g, mt, tid, CtaSync(), p0, next);
    const long long ob = p.lout.base(t * GC + g);
    const Emit em{p.dst + ob, p.lout.es, p.acc ? p.acc + ob : nullptr, p.lout.es, p.scale};
    store_pass0<SYM, Cfg>(v, a, tp, em, p.v, tid);
  }
}

// ---------------------------------------------------------------- pfft fwd --
template <int SYM, class Cfg, int G>
__global__ void __launch_bounds__(Cfg::T * G, 1) k_pfft_fwd(FwdArgs p) {
  extern __shared__ double2 smem[];
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), RpL = Cfg::Rprod(Cfg::P - 1);
  const int g = threadIdx.x / T, tid = threadIdx.x % T;
  double2* tb = smem;
  const double2* mt = tb;  // middle-pass tables sit at offset 0
  double2* X = smem + p.ax.tabn + g * Cfg::XS;
  const GroupSync sync{g + 1, T};
  const AxisDev& a = p.ax;
  stage_tables(tb, a, a.tabn);
  const double2* tp = a.tabn >= a.tabfull ? tb : a.tab;
  const P0Res<SYM> p0{&a, tp, p.v};
  for (long long item = (long long)blockIdx.x * G + g; item < p.lin.count; item += (long long)gridDim.x * G) {
    double2 v[Cfg::E];
    load_pass0<SYM, Cfg>(v, a, tp, p.f + p.lin.base(item), p.lin.es, p.v, tid);
    fft_forward<Cfg>(v, X, mt, tid, sync, p0);
    const long long ob = p.lout.base(item), oes = p.lout.es;
    sfor<CL>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (bvalid<Cfg, Cfg::P - 1>(c, tid))
        sfor<RL>([&](auto Ki) HC_INL {
          const long long kp = beta + (long long)RpL * Ki;
          const double2 val = v[c * RL + Ki];
          if constexpr (SYM == SYM_HERMITIAN) {
            double* F = (double*)p.F;
            const long long i0 = p.ref_order ? ref_index(a, 2 * kp) : 2 * kp;
            const long long i1 = p.ref_order ? ref_index(a, 2 * kp + 1) : 2 * kp + 1;
            F[ob + i0 * oes] = val.x;
            F[ob + i1 * oes] = val.y;
          } else {
            double2* F = (double2*)p.F;
            F[ob + (p.ref_order ? ref_index(a, kp) : kp) * oes] = val;
          }
        });
    });
  }
}

// ---------------------------------------------------------------- pfft bwd --
template <int SYM, class Cfg, int G>
__global__ void __launch_bounds__(Cfg::T * G, 1) k_pfft_bwd(BwdArgs p) {
  extern __shared__ double2 smem[];
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), RpL = Cfg::Rprod(Cfg::P - 1);
  const int g = threadIdx.x / T, tid = threadIdx.x % T;
  double2* tb = smem;
  const double2* mt = tb;  // middle-pass tables sit at offset 0
  double2* X = smem + p.ax.tabn + g * Cfg::XS;
  const GroupSync sync{g + 1, T};
  const AxisDev& a = p.ax;
  stage_tables(tb, a, a.tabn);
  const double2* tp = a.tabn >= a.tabfull ? tb : a.tab;
  const P0Res<SYM> p0{&a, tp, p.v};
  for (long long item = (long long)blockIdx.x * G + g; item < p.lin.count; item += (long long)gridDim.x * G) {
    double2 v[Cfg::E];
    const long long ib = p.lin.base(item), ies = p.lin.es;
    sfor<CL>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (bvalid<Cfg, Cfg::P - 1>(c, tid))
        sfor<RL>([&](auto Ki) HC_INL {
          const long long kp = beta + (long long)RpL * Ki;
          if constexpr (SYM == SYM_HERMITIAN) {
            const double* F = (const double*)p.F;
            const long long i0 = p.ref_order ? ref_index(a, 2 * kp) : 2 * kp;
            const long long i1 = p.ref_order ? ref_index(a, 2 * kp + 1) : 2 * kp + 1;
            v[c * RL + Ki] = make_double2(F[ib + i0 * ies], F[ib + i1 * ies]);
          } else {
            const double2* F = (const double2*)p.F;
            v[c * RL + Ki] = F[ib + (p.ref_order ? ref_index(a, kp) : kp) * ies];
          }
        });
    });
    fft_inverse<Cfg>(v, X, mt, tid, sync, p0);
    const long long ob = p.lout.base(item);
    const Emit em{p.dst + ob, p.lout.es, p.acc ? p.acc + ob : nullptr, p.lout.es, p.scale};
    if constexpr (SYM == SYM_HERMITIAN) store_herm<Cfg>(v, a, tp, em, p.v, tid, X, sync);
    else store_pass0<SYM, Cfg>(v, a, tp, em, p.v, tid);
  }
}

}  // namespace hc
