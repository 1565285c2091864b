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

namespace hc {

struct ConvArgs {
  AxisDev ax;
  Lines lin;             // input/output line addressing (inputs and output share the layout)
  const double2* f;
  const double2* g;
  double2* out;
  double2* scratch;      // per-group accumulator slots (S complex each)
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
__device__ __forceinline__ void load_pass0(double2 (&v)[Cfg::E], const AxisDev& a, const double2* f, long long es,
                                           int res, int tid) {
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), Ns1 = Cfg::Ns(1);
  sfor<C0>([&](auto Ci) {
    constexpr int c = Ci;
    const int b = tid + c * Cfg::T;
    if (bvalid<Cfg, 0>(c, tid)) {
      sfor<R0>([&](auto Ai) {
        constexpr int ai = Ai;
        if constexpr (SYM == SYM_HERMITIAN) v[c * R0 + ai] = load_Zp_fast(a, f, es, Ns1 * ai + b, res, ai, b);
        else v[c * R0 + ai] = load_fast<SYM>(a, f, es, Ns1 * ai + b, res, ai);
      });
    }
  });
}

// pass-0 output twiddle source: omega_Bc^{b k} times (complex / centered) the folded residue
// factor zeta_qm^{v b}
template <int SYM>
struct P0Res {
  const AxisDev* a;
  int v;
  __device__ __forceinline__ void operator()(int b, double2& t, double2& w) const {
    w = tA(*a, b);
    t = (SYM != SYM_HERMITIAN && v) ? tZ(*a, v, b) : make_double2(1.0, 0.0);
  }
};

// inverse post-processing from pass-0 layout (complex / centered)
template <int SYM, class Cfg>
__device__ __forceinline__ void store_pass0(const double2 (&v)[Cfg::E], const AxisDev& a, const Emit& em, int res,
                                            int tid) {
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), Ns1 = Cfg::Ns(1);
  sfor<C0>([&](auto Ci) {
    constexpr int c = Ci;
    const int b = tid + c * Cfg::T;
    if (bvalid<Cfg, 0>(c, tid)) {
      sfor<R0>([&](auto Ai) { store_fast<SYM>(a, em, Ns1 * Ai + b, res, Ai, v[c * R0 + Ai]); });
    }
  });
}

// Hermitian post-processing: pass-0 layout -> Z in shared memory -> outputs j < S
template <class Cfg, class Sync>
__device__ __forceinline__ void store_herm(const double2 (&v)[Cfg::E], const AxisDev& a, const Emit& em, int res,
                                           int tid, double2* Z, const Sync& sync) {
  constexpr int R0 = Cfg::R(0), C0 = Cfg::C(0), Ns1 = Cfg::Ns(1);
  sfor<C0>([&](auto Ci) {
    constexpr int c = Ci;
    const int b = tid + c * Cfg::T;
    if (bvalid<Cfg, 0>(c, tid)) sfor<R0>([&](auto Ai) { Z[Ns1 * Ai + b] = v[c * R0 + Ai]; });
  });
  sync();
  for (int j = tid; j < a.S; j += Cfg::T) em(j, herm_w_fast<Ns1>(a, Z, j, res));
  sync();
}

// stage the middle-pass twiddle tables into shared memory (whole CTA)
template <class Cfg>
__device__ __forceinline__ void stage_mt(double2* mt, const AxisDev& a) {
  if constexpr (Cfg::MT > 0) {
    for (int i = threadIdx.x; i < Cfg::MT; i += blockDim.x) mt[i] = __ldg(a.tab + a.oMT + i);
    __syncthreads();
  }
}

// ------------------------------------------------------------------ conv1d --
// STASH_REGS: keep the first forward spectrum in registers instead of shared memory.
template <int SYM, class Cfg, int G, bool STASH_REGS>
__global__ void __launch_bounds__(Cfg::T * G, 1) k_conv1d(ConvArgs p) {
  extern __shared__ double2 smem[];
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), NBL = Cfg::NB(Cfg::P - 1);
  constexpr int GS = Cfg::XS + (STASH_REGS ? 0 : Cfg::N);
  const int g = threadIdx.x / T, tid = threadIdx.x % T;
  double2* mt = smem;
  double2* X = smem + Cfg::MT + g * GS;
  double2* stash = X + Cfg::XS;
  const GroupSync sync{g + 1, T};
  const AxisDev& a = p.ax;
  stage_mt<Cfg>(mt, a);
  const long long es = p.lin.es;
  double2* slot = p.scratch + (long long)(blockIdx.x * G + g) * a.S;
  for (long long item = (long long)blockIdx.x * G + g; item < p.lin.count; item += (long long)gridDim.x * G) {
    const long long base = p.lin.base(item);
    for (int res = 0; res < a.n; ++res) {
      double2 v[Cfg::E];
      double2 Fr[STASH_REGS ? Cfg::E : 1];
      const P0Res<SYM> p0{&a, res};
      load_pass0<SYM, Cfg>(v, a, p.f + base, es, res, tid);
      fft_forward<Cfg>(v, X, mt, tid, sync, p0);
      sfor<CL>([&](auto Ci) {
        constexpr int c = Ci;
        if (bvalid<Cfg, Cfg::P - 1>(c, tid))
          sfor<RL>([&](auto Ki) {
            if constexpr (STASH_REGS) Fr[c * RL + Ki] = v[c * RL + Ki];
            else stash[Ki * NBL + tid + c * T] = v[c * RL + Ki];
          });
      });
      load_pass0<SYM, Cfg>(v, a, p.g + base, es, res, tid);
      fft_forward<Cfg>(v, X, mt, tid, sync, p0);
      sfor<CL>([&](auto Ci) {
        constexpr int c = Ci;
        if (bvalid<Cfg, Cfg::P - 1>(c, tid))
          sfor<RL>([&](auto Ki) {
            double2 F;
            if constexpr (STASH_REGS) F = Fr[c * RL + Ki];
            else F = stash[Ki * NBL + tid + c * T];
            double2& G_ = v[c * RL + Ki];
            if constexpr (SYM == SYM_HERMITIAN) G_ = make_double2(G_.x * F.x, G_.y * F.y);  // real residues
            else G_ = cmul(G_, F);
          });
      });
      fft_inverse<Cfg>(v, X, mt, tid, sync, p0);
      Emit em;
      const bool last = res == a.n - 1;
      if (last) {
        em = Emit{p.out + base, es, res > 0 ? slot : nullptr, 1, 1.0 / (double)a.qm};
      } else {
        em = Emit{slot, 1, res > 0 ? slot : nullptr, 1, 1.0};
      }
      if constexpr (SYM == SYM_HERMITIAN) store_herm<Cfg>(v, a, em, res, tid, X, sync);
      else store_pass0<SYM, Cfg>(v, a, em, res, tid);
    }
  }
}

// ---------------------------------------------------------------- pfft fwd --
template <int SYM, class Cfg, int G>
__global__ void __launch_bounds__(Cfg::T * G, 1) k_pfft_fwd(FwdArgs p) {
  extern __shared__ double2 smem[];
  constexpr int T = Cfg::T, RL = Cfg::R(Cfg::P - 1), CL = Cfg::C(Cfg::P - 1), RpL = Cfg::Rprod(Cfg::P - 1);
  const int g = threadIdx.x / T, tid = threadIdx.x % T;
  double2* mt = smem;
  double2* X = smem + Cfg::MT + g * Cfg::XS;
  const GroupSync sync{g + 1, T};
  const AxisDev& a = p.ax;
  stage_mt<Cfg>(mt, a);
  const P0Res<SYM> p0{&a, p.v};
  for (long long item = (long long)blockIdx.x * G + g; item < p.lin.count; item += (long long)gridDim.x * G) {
    double2 v[Cfg::E];
    load_pass0<SYM, Cfg>(v, a, p.f + p.lin.base(item), p.lin.es, p.v, tid);
    fft_forward<Cfg>(v, X, mt, tid, sync, p0);
    const long long ob = p.lout.base(item), oes = p.lout.es;
    sfor<CL>([&](auto Ci) {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (bvalid<Cfg, Cfg::P - 1>(c, tid))
        sfor<RL>([&](auto Ki) {
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
  double2* mt = smem;
  double2* X = smem + Cfg::MT + g * Cfg::XS;
  const GroupSync sync{g + 1, T};
  const AxisDev& a = p.ax;
  stage_mt<Cfg>(mt, a);
  const P0Res<SYM> p0{&a, p.v};
  for (long long item = (long long)blockIdx.x * G + g; item < p.lin.count; item += (long long)gridDim.x * G) {
    double2 v[Cfg::E];
    const long long ib = p.lin.base(item), ies = p.lin.es;
    sfor<CL>([&](auto Ci) {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (bvalid<Cfg, Cfg::P - 1>(c, tid))
        sfor<RL>([&](auto Ki) {
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
    if constexpr (SYM == SYM_HERMITIAN) store_herm<Cfg>(v, a, em, p.v, tid, X, sync);
    else store_pass0<SYM, Cfg>(v, a, em, p.v, tid);
  }
}

}  // namespace hc
