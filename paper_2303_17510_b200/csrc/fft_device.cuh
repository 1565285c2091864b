// fft_device.cuh — in-register / shared-memory FP64 complex FFT building blocks (sm_100a).
//
// Sign convention of the paper: the forward transform uses
// zeta_N = exp(+2 pi i / N) (DIR = +1); the unnormalised inverse uses DIR = -1.
//
// A block FFT of compile-time length N = R_0 R_1 ... R_{P-1} runs as P passes.  Pass i
// takes the sub-sequences left by passes 0..i-1 (indexed by K = k_0 + R_0 k_1 + ..., each of
// length Ns_i = R_i ... R_{P-1}), does an R_i-point DFT in registers over the elements
// (K, Ns_{i+1} a + b), a < R_i, multiplies output k by omega_{Ns_i}^{b k} and hands
// element (K + Rprod_i k, b) to pass i+1 through one shared-memory exchange.  Input is in
// natural order, output index K = k_0 + R_0 k_1 + ... is the natural frequency.  Because a
// convolution only needs F and G in the SAME order, the forward leaves its last pass in
// registers, the pointwise product is taken there, and the inverse runs the passes in
// reverse from the same registers (no bit-reversal, no extra round trip).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "tw_consts.h"

// Every lambda on the hot path is force-inlined: the same lambda bodies are shared by several
// kernels, and an out-of-line call would push the register arrays it touches to local memory.
#define HC_INL __attribute__((always_inline))

namespace hc {

template <int N, int I = 0, class F>
__device__ __forceinline__ void sfor(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    sfor<N, I + 1>(static_cast<F&&>(f));
  }
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// a + s b, componentwise (radix-7 butterflies)
__device__ __forceinline__ double2 cfma7(double s, double2 b, double2 a) { return make_double2(fma(s, b.x, a.x), fma(s, b.y, a.y)); }
// a * i^DIR
template <int DIR>
__device__ __forceinline__ double2 mul_i(double2 a) {
  if constexpr (DIR > 0) return make_double2(-a.y, a.x);
  else return make_double2(a.y, -a.x);
}
// multiply by a table twiddle (DIR = +1) or its conjugate (DIR = -1)
template <int DIR>
__device__ __forceinline__ double2 mul_tw(double2 a, double2 w) {
  if constexpr (DIR > 0) return cmul(a, w);
  else return cmulc(a, w);
}

// x * zeta_R^{DIR*E}, trivial angles folded at compile time.
template <int R, int E, int DIR>
__device__ __forceinline__ double2 twc(double2 x) {
  constexpr int e = ((E % R) + R) % R;
  if constexpr (e == 0) {
    return x;
  } else if constexpr (2 * e == R) {
    return make_double2(-x.x, -x.y);
  } else if constexpr (4 * e == R) {
    return mul_i<DIR>(x);
  } else if constexpr (4 * e == 3 * R) {
    return mul_i<-DIR>(x);
  } else {
    constexpr double c = TwC<R>::c[e];
    constexpr double s = DIR * TwC<R>::s[e];
    return make_double2(fma(x.x, c, -x.y * s), fma(x.x, s, x.y * c));
  }
}

#ifndef HC_FF_MODE
#define HC_FF_MODE 1
#endif
constexpr int first_factor(int R) {
  if (HC_FF_MODE == 1 && R % 8 == 0 && R != 8 && R % 3 == 0) return 8;   // 24 = 8 x 3
  if (HC_FF_MODE == 2 && R % 3 == 0 && R != 3) return 3;                 // 24 = 3 x 8, 12 = 3 x 4
  if (R % 4 == 0 && R != 4) return 4;
  for (int f : {2, 3, 5, 7}) if (R % f == 0 && R != f) return f;
  return R;  // prime
}

// In-place R-point DFT of x[0..R) in registers, natural-order output.
template <int R, int DIR>
struct DFT {
  static __device__ __forceinline__ void run(double2* x) {
    constexpr int A = first_factor(R);
    if constexpr (A == R) {  // prime: direct sum with compile-time twiddles
      double2 y[R];
      sfor<R>([&](auto K) HC_INL {
        constexpr int k = K;
        double2 acc = x[0];
        sfor<R - 1>([&](auto J) HC_INL {
          constexpr int j = J + 1;
          acc = cadd(acc, twc<R, j * k, DIR>(x[j]));
        });
        y[k] = acc;
      });
      sfor<R>([&](auto K) HC_INL { x[K] = y[K]; });
    } else {  // four-step: n = Bf a + b, k = ka + A kb
      constexpr int Bf = R / A;
      double2 t[R];
      sfor<Bf>([&](auto Bi) HC_INL {
        constexpr int b = Bi;
        double2 y[A];
        sfor<A>([&](auto Ai) HC_INL { y[Ai] = x[Bf * Ai + b]; });
        DFT<A, DIR>::run(y);
        sfor<A>([&](auto Ki) HC_INL {
          constexpr int ka = Ki;
          t[ka * Bf + b] = twc<R, b * ka, DIR>(y[ka]);
        });
      });
      sfor<A>([&](auto Ki) HC_INL {
        constexpr int ka = Ki;
        double2 z[Bf];
        sfor<Bf>([&](auto Bi) HC_INL { z[Bi] = t[ka * Bf + Bi]; });
        DFT<Bf, DIR>::run(z);
        sfor<Bf>([&](auto Kb) HC_INL { x[ka + A * Kb] = z[Kb]; });
      });
    }
  }
};
template <int DIR>
struct DFT<1, DIR> {
  static __device__ __forceinline__ void run(double2*) {}
};
template <int DIR>
struct DFT<2, DIR> {
  static __device__ __forceinline__ void run(double2* x) {
    const double2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
  }
};
template <int DIR>
struct DFT<3, DIR> {
  static __device__ __forceinline__ void run(double2* x) {
    constexpr double s3 = DIR * 0.8660254037844386;  // sin(2 pi / 3)
    const double2 t1 = cadd(x[1], x[2]);
    const double2 t2 = make_double2(fma(-0.5, t1.x, x[0].x), fma(-0.5, t1.y, x[0].y));
    const double2 d = csub(x[1], x[2]);
    const double2 t3 = make_double2(-s3 * d.y, s3 * d.x);  // i * s3 * d
    x[0] = cadd(x[0], t1);
    x[1] = cadd(t2, t3);
    x[2] = csub(t2, t3);
  }
};
template <int DIR>
struct DFT<4, DIR> {
  static __device__ __forceinline__ void run(double2* x) {
    const double2 t0 = cadd(x[0], x[2]), t1 = csub(x[0], x[2]);
    const double2 t2 = cadd(x[1], x[3]), t3 = mul_i<DIR>(csub(x[1], x[3]));
    x[0] = cadd(t0, t2);
    x[2] = csub(t0, t2);
    x[1] = cadd(t1, t3);
    x[3] = csub(t1, t3);
  }
};

// 5-point DFT through the two real symmetric / antisymmetric pairs (x1 +- x4, x2 +- x3):
// 40 FP64 instructions instead of the direct sum's ~96 (radix-5 plans, SPEC.md:523's 7-smooth
// sizes).  y_k = sum_j x_j zeta_5^{DIR j k}.
template <int DIR>
struct DFT<5, DIR> {
  static __device__ __forceinline__ void run(double2* x) {
    constexpr double c1 = 0.30901699437494745, c2 = -0.8090169943749475;     // cos(2 pi/5), cos(4 pi/5)
    constexpr double s1 = DIR * 0.9510565162951535, s2 = DIR * 0.5877852522924731;  // sin(2 pi/5), sin(4 pi/5)
    const double2 t1 = cadd(x[1], x[4]), t2 = cadd(x[2], x[3]);
    const double2 t3 = csub(x[1], x[4]), t4 = csub(x[2], x[3]);
    const double2 a1 = make_double2(fma(c2, t2.x, fma(c1, t1.x, x[0].x)), fma(c2, t2.y, fma(c1, t1.y, x[0].y)));
    const double2 a2 = make_double2(fma(c1, t2.x, fma(c2, t1.x, x[0].x)), fma(c1, t2.y, fma(c2, t1.y, x[0].y)));
    // i b1, i b2 with b1 = s1 t3 + s2 t4, b2 = s2 t3 - s1 t4
    const double2 b1 = make_double2(fma(s2, t4.x, s1 * t3.x), fma(s2, t4.y, s1 * t3.y));
    const double2 b2 = make_double2(fma(-s1, t4.x, s2 * t3.x), fma(-s1, t4.y, s2 * t3.y));
    x[0] = cadd(x[0], cadd(t1, t2));
    x[1] = make_double2(a1.x - b1.y, a1.y + b1.x);
    x[4] = make_double2(a1.x + b1.y, a1.y - b1.x);
    x[2] = make_double2(a2.x - b2.y, a2.y + b2.x);
    x[3] = make_double2(a2.x + b2.y, a2.y - b2.x);
  }
};

// 7-point DFT through the three symmetric / antisymmetric pairs (x_j +- x_{7-j}): 66 FP64
// instructions instead of the direct sum's ~170 (radix-7 plans: the 7-smooth sizes of SPEC.md:523).
template <int DIR>
struct DFT<7, DIR> {
  static __device__ __forceinline__ void run(double2* x) {
    constexpr double c1 = TwC<7>::c[1], c2 = TwC<7>::c[2], c3 = TwC<7>::c[3];
    constexpr double s1 = DIR * TwC<7>::s[1], s2 = DIR * TwC<7>::s[2], s3 = DIR * TwC<7>::s[3];
    const double2 t1 = cadd(x[1], x[6]), t2 = cadd(x[2], x[5]), t3 = cadd(x[3], x[4]);
    const double2 d1 = csub(x[1], x[6]), d2 = csub(x[2], x[5]), d3 = csub(x[3], x[4]);
    // a_k = x0 + sum_j cos(2 pi j k / 7) t_j,  b_k = sum_j sin(2 pi j k / 7) d_j   (k = 1, 2, 3)
    const double2 a1 = cfma7(c3, t3, cfma7(c2, t2, cfma7(c1, t1, x[0])));
    const double2 a2 = cfma7(c1, t3, cfma7(c3, t2, cfma7(c2, t1, x[0])));
    const double2 a3 = cfma7(c2, t3, cfma7(c1, t2, cfma7(c3, t1, x[0])));
    const double2 b1 = cfma7(s3, d3, cfma7(s2, d2, make_double2(s1 * d1.x, s1 * d1.y)));
    const double2 b2 = cfma7(-s1, d3, cfma7(-s3, d2, make_double2(s2 * d1.x, s2 * d1.y)));
    const double2 b3 = cfma7(s2, d3, cfma7(-s1, d2, make_double2(s3 * d1.x, s3 * d1.y)));
    x[0] = cadd(x[0], cadd(t1, cadd(t2, t3)));
    x[1] = make_double2(a1.x - b1.y, a1.y + b1.x);
    x[6] = make_double2(a1.x + b1.y, a1.y - b1.x);
    x[2] = make_double2(a2.x - b2.y, a2.y + b2.x);
    x[5] = make_double2(a2.x + b2.y, a2.y - b2.x);
    x[3] = make_double2(a3.x - b3.y, a3.y + b3.x);
    x[4] = make_double2(a3.x + b3.y, a3.y - b3.x);
  }
};

#ifndef HC_DFT_FMA
#define HC_DFT_FMA 1
#endif
#if HC_DFT_FMA
// Hand-scheduled 8- and 16-point DFTs: the four-step form of the generic template, with every
// non-trivial internal twiddle written as c (1 + i DIR t) (t = tan of the angle) or
// sqrt(1/2) (+-1 + i DIR) and its scale c folded into the FMAs of the following radix-4 / radix-2
// butterflies (the ratio of two scales is again a tangent, c3/c1 = tan(pi/8)).  DFT16: 144 FP64
// instructions instead of 160; DFT8: 52 instead of 56.  Natural-order output, same as DFT<R>.
namespace dftc {
constexpr double h = 0.70710678118654752440084436210484903928;   // sqrt(1/2)
constexpr double c1 = 0.92387953251128675612818318939678828682;  // cos(pi/8)
constexpr double c3 = 0.38268343236508977172845998403039886676;  // cos(3pi/8)
constexpr double t1 = 0.41421356237309504880168872420969807857;  // tan(pi/8) = c3/c1
constexpr double t3 = 2.41421356237309504880168872420969807857;  // tan(3pi/8) = c1/c3
}  // namespace dftc
// y (1 + i DIR t)
template <int DIR>
__device__ __forceinline__ double2 tan_rot(double2 y, double t) {
  return make_double2(fma(-DIR * t, y.y, y.x), fma(DIR * t, y.x, y.y));
}
// a + s b, componentwise
__device__ __forceinline__ double2 cfma(double s, double2 b, double2 a) { return make_double2(fma(s, b.x, a.x), fma(s, b.y, a.y)); }

template <int DIR>
struct DFT<16, DIR> {
  static __device__ __forceinline__ void run(double2* x) {
    using namespace dftc;
    double2 y[4][4];  // y[b][ka]: DFT4 over a of x[4a + b]
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      double2 q[4] = {x[b], x[4 + b], x[8 + b], x[12 + b]};
      DFT<4, DIR>::run(q);
#pragma unroll
      for (int k = 0; k < 4; ++k) y[b][k] = q[k];
    }
    {  // ka = 0: no twiddles
      double2 z[4] = {y[0][0], y[1][0], y[2][0], y[3][0]};
      DFT<4, DIR>::run(z);
      x[0] = z[0], x[4] = z[1], x[8] = z[2], x[12] = z[3];
    }
    {  // ka = 1: zeta^1 = c1 (1 + i DIR t1), zeta^2 = h (1 + i DIR), zeta^3 = c3 (1 + i DIR t3)
      const double2 u1 = tan_rot<DIR>(y[1][1], t1), u2 = tan_rot<DIR>(y[2][1], 1.0), u3 = tan_rot<DIR>(y[3][1], t3);
      const double2 s02 = cfma(h, u2, y[0][1]), d02 = cfma(-h, u2, y[0][1]);
      const double2 p = cfma(t1, u3, u1), q = cfma(-t1, u3, u1);  // (z1 +- z3) / c1
      const double2 rq = mul_i<DIR>(q);
      x[1] = cfma(c1, p, s02), x[9] = cfma(-c1, p, s02);
      x[5] = cfma(c1, rq, d02), x[13] = cfma(-c1, rq, d02);
    }
    {  // ka = 2: zeta^2 = h (1 + i DIR), zeta^4 = i^DIR, zeta^6 = h (-1 + i DIR)
      const double2 v1 = tan_rot<DIR>(y[1][2], 1.0);
      const double2 w = y[3][2];
      const double2 v3 = make_double2(-w.x - DIR * w.y, -w.y + DIR * w.x);
      const double2 r2 = mul_i<DIR>(y[2][2]);
      const double2 s02 = cadd(y[0][2], r2), d02 = csub(y[0][2], r2);
      const double2 p = cadd(v1, v3), q = csub(v1, v3);
      const double2 rq = mul_i<DIR>(q);
      x[2] = cfma(h, p, s02), x[10] = cfma(-h, p, s02);
      x[6] = cfma(h, rq, d02), x[14] = cfma(-h, rq, d02);
    }
    {  // ka = 3: zeta^3 = c3 (1 + i DIR t3), zeta^6 = h (-1 + i DIR), zeta^9 = -c1 (1 + i DIR t1)
      const double2 w1 = tan_rot<DIR>(y[1][3], t3), w3 = tan_rot<DIR>(y[3][3], t1);
      const double2 g = y[2][3];
      const double2 w2 = make_double2(-g.x - DIR * g.y, -g.y + DIR * g.x);
      const double2 s02 = cfma(h, w2, y[0][3]), d02 = cfma(-h, w2, y[0][3]);
      const double2 p = cfma(-t3, w3, w1), q = cfma(t3, w3, w1);  // (z1 +- z3) / c3
      const double2 rq = mul_i<DIR>(q);
      x[3] = cfma(c3, p, s02), x[11] = cfma(-c3, p, s02);
      x[7] = cfma(c3, rq, d02), x[15] = cfma(-c3, rq, d02);
    }
  }
};

template <int DIR>
struct DFT<8, DIR> {
  static __device__ __forceinline__ void run(double2* x) {
    using namespace dftc;
    double2 y0[4] = {x[0], x[2], x[4], x[6]}, y1[4] = {x[1], x[3], x[5], x[7]};  // DFT4 over a of x[2a + b]
    DFT<4, DIR>::run(y0);
    DFT<4, DIR>::run(y1);
    x[0] = cadd(y0[0], y1[0]), x[4] = csub(y0[0], y1[0]);
    const double2 u1 = tan_rot<DIR>(y1[1], 1.0);  // zeta8^1 = h (1 + i DIR)
    x[1] = cfma(h, u1, y0[1]), x[5] = cfma(-h, u1, y0[1]);
    const double2 r2 = mul_i<DIR>(y1[2]);         // zeta8^2 = i^DIR
    x[2] = cadd(y0[2], r2), x[6] = csub(y0[2], r2);
    const double2 w = y1[3];                       // zeta8^3 = h (-1 + i DIR)
    const double2 u3 = make_double2(-w.x - DIR * w.y, -w.y + DIR * w.x);
    x[3] = cfma(h, u3, y0[3]), x[7] = cfma(-h, u3, y0[3]);
  }
};

// 24 = 8 x 3: the radix-3 butterflies of the second stage take both twiddled inputs in tangent
// form, z1 = c1 u1 and z2 = c2 u2 (u = y (1 + i tan)), with c1 factored out of the butterfly
// (r = c2 / c1 inside, c1 folded into the output FMAs): 16 FP64 instructions instead of 22 per
// group whose two twiddles are both non-trivial (ka = 1, 2, 4, 5, 7); the other groups as before.
template <int DIR, int KA>
__device__ __forceinline__ void dft3_tw24(double2 z0, double2 y1, double2 y2, double2* out) {
  constexpr int e1 = KA % 24, e2 = (2 * KA) % 24;
  constexpr bool triv1 = e1 % 6 == 0, triv2 = e2 % 6 == 0;
  if constexpr (!triv1 && !triv2) {
    constexpr double ca = TwC<24>::c[e1], sa = DIR * TwC<24>::s[e1];
    constexpr double cb = TwC<24>::c[e2], sb = DIR * TwC<24>::s[e2];
    constexpr double ta = sa / ca, tb = sb / cb, r = cb / ca;
    const double2 u1 = make_double2(fma(-ta, y1.y, y1.x), fma(ta, y1.x, y1.y));
    const double2 u2 = make_double2(fma(-tb, y2.y, y2.x), fma(tb, y2.x, y2.y));
    const double2 p = cfma(r, u2, u1), q = cfma(-r, u2, u1);  // (z1 + z2) / ca, (z1 - z2) / ca
    constexpr double k3 = DIR * 0.86602540378443864676 * ca;   // i DIR sin(2pi/3) ca
    const double2 t2 = cfma(-0.5 * ca, p, z0);
    out[0] = cfma(ca, p, z0);
    out[8] = make_double2(fma(-k3, q.y, t2.x), fma(k3, q.x, t2.y));
    out[16] = make_double2(fma(k3, q.y, t2.x), fma(-k3, q.x, t2.y));
  } else {
    double2 z[3] = {z0, twc<24, e1, DIR>(y1), twc<24, e2, DIR>(y2)};
    DFT<3, DIR>::run(z);
    out[0] = z[0], out[8] = z[1], out[16] = z[2];
  }
}

template <int DIR>
struct DFT<24, DIR> {
  static __device__ __forceinline__ void run(double2* x) {
    double2 y[3][8];  // y[b][ka]: DFT8 over a of x[3a + b]
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double2 q[8] = {x[b], x[3 + b], x[6 + b], x[9 + b], x[12 + b], x[15 + b], x[18 + b], x[21 + b]};
      DFT<8, DIR>::run(q);
#pragma unroll
      for (int k = 0; k < 8; ++k) y[b][k] = q[k];
    }
    sfor<8>([&](auto K) HC_INL {
      constexpr int ka = K;
      dft3_tw24<DIR, ka>(y[0][ka], y[1][ka], y[2][ka], x + ka);
    });
  }
};
#endif

// ---------------------------------------------------------------- block FFT --
template <int... Rs>
struct Radices {
  static constexpr int P = sizeof...(Rs);
  static constexpr int R[P] = {Rs...};
  static constexpr int N = (Rs * ... * 1);
};

template <class RL, int T_>
struct FFTCfg {
  static constexpr int N = RL::N;
  static constexpr int P = RL::P;
  static constexpr int T = T_;
  static constexpr int R(int i) { return RL::R[i]; }
  static constexpr int Ns(int i) {  // sub-sequence length before pass i (Ns(P) = 1)
    int v = 1;
    for (int k = i; k < P; ++k) v *= RL::R[k];
    return v;
  }
  static constexpr int Rprod(int i) {
    int v = 1;
    for (int k = 0; k < i; ++k) v *= RL::R[k];
    return v;
  }
  static constexpr int NB(int i) { return N / RL::R[i]; }                // butterflies in pass i
  static constexpr int C(int i) { return (NB(i) + T - 1) / T; }          // butterflies per thread
  static constexpr int E_calc() {
    int e = 0;
    for (int i = 0; i < P; ++i) e = (C(i) * RL::R[i] > e) ? C(i) * RL::R[i] : e;
    return e;
  }
  static constexpr int E = E_calc();                                     // registers (complex) per thread
  static constexpr int St(int i) { return Ns(i) + ((Ns(i) % 2 == 0) ? 1 : 0); }  // padded row (odd)
  static constexpr int X_calc() {
    int x = N;
    for (int i = 1; i < P; ++i) x = (Rprod(i) * St(i) > x) ? Rprod(i) * St(i) : x;
    return x;
  }
  static constexpr int XS = X_calc();                                    // exchange buffer (complex)
  // middle-pass twiddle tables (passes 1..P-2), staged in shared memory:
  //   MT[MTo(i) + (k-1) * Ns(i+1) + b] = omega_{Ns(i)}^{b k},  1 <= k < R_i,  b < Ns(i+1)
  static constexpr int MTo(int i) {
    int o = 0;
    for (int j = 1; j < i; ++j) o += (RL::R[j] - 1) * Ns(j + 1);
    return o;
  }
  static constexpr int MT = (P > 2) ? MTo(P - 1) : 0;
  static constexpr int ES = C(P - 1) * RL::R[P - 1];                     // last-pass values per thread
};

// Barrier objects of the block FFTs.  operator() is a full barrier (read-after-write between
// an exchange's stores and loads).  The write-after-read hazard (an exchange's loads against
// the next stores into the same buffer) goes through war_arrive() after the loads and
// war_wait() before the next stores: a plain barrier in war_arrive() here, a split barrier in
// SplitSync (kernels.cuh) so that the butterflies between the two overlap the wait.
// Whole-CTA barrier (column-tile kernels, whose line groups interleave within warps).
struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
  __device__ __forceinline__ void war_arrive() const { __syncthreads(); }
  __device__ __forceinline__ void war_wait() const {}
};

// Group barrier over NT threads (named barrier id; NT must be a multiple of 32).
struct GroupSync {
  int id, nt;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nt) : "memory");
  }
  __device__ __forceinline__ void war_arrive() const { (*this)(); }
  __device__ __forceinline__ void war_wait() const {}
};

// Pass-0 twiddles come from a per-butterfly source p0(beta, t0, w): output k of the pass-0
// DFT is multiplied by t0 * w^k (w = omega_N^b; t0 folds the residue pre-twiddle
// zeta_qm^{v b} of the padded transform, or 1).  Passes 1..P-2 read shared-memory tables mt
// (FFTCfg::MT layout); the last pass has no twiddle.
template <int DIR, int R, class P0>
__device__ __forceinline__ void pass0_twiddle(double2* y, int beta, const P0& p0) {
  double2 t, w;
  p0(beta, t, w);
  sfor<R>([&](auto Ki) HC_INL {
    constexpr int k = Ki;
    y[k] = mul_tw<DIR>(y[k], t);
    if constexpr (k + 1 < R) t = cmul(t, w);
  });
}

// Forward FFT: v holds pass-0 inputs (v[c*R0 + a] = x[Ns1*a + b], b = tid + c*T).
// On return v holds the last pass outputs: v[c*R + k] = X[beta + Rprod(P-1)*k], beta = tid + c*T.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// hook() runs right after the last shared-memory exchange (X is free from then on), before the
// last pass's arithmetic -- used to start the next TMA copy into X early.
// XSTR: element stride of the exchange buffer (1, or G when G line groups interleave their
// buffers element by element -- column-tile kernels, kernels.cuh)
// hook0() runs after the first exchange (P > 2: before the last one).
template <class Cfg, class Sync, class P0, class Hook = NoHook, int XSTR = 1, class Hook0 = NoHook>
__device__ __forceinline__ void fft_forward(double2 (&v)[Cfg::E], double2* X, const double2* mt, int tid,
                                            const Sync& sync, const P0& p0, const Hook& hook = Hook(),
                                            const Hook0& hook0 = Hook0()) {
  constexpr int P = Cfg::P, T = Cfg::T;
  static_assert(P >= 2, "radix plans have at least two passes");
  sfor<P>([&](auto I) HC_INL {
    constexpr int i = I;
    constexpr int R = Cfg::R(i), C = Cfg::C(i), NB = Cfg::NB(i), Ns1 = Cfg::Ns(i + 1), Rp = Cfg::Rprod(i);
    sfor<C>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (NB % T == 0 || beta < NB) {
        DFT<R, +1>::run(v + c * R);
        if constexpr (i == 0) {
          pass0_twiddle<+1, R>(v + c * R, beta, p0);
        } else if constexpr (i < P - 1) {
          const int b = beta % Ns1;
          sfor<R - 1>([&](auto Ki) HC_INL {
            constexpr int k = Ki + 1;
            v[c * R + k] = cmul(v[c * R + k], mt[Cfg::MTo(i) + (k - 1) * Ns1 + b]);
          });
        }
      }
    });
    if constexpr (i < P - 1) {
      constexpr int St = Cfg::St(i + 1);
      sync.war_wait();
      sfor<C>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        const int beta = tid + c * T;
        if (NB % T == 0 || beta < NB) {
          const int K = beta / Ns1, b = beta % Ns1;
          sfor<R>([&](auto Ki) HC_INL { X[((K + Rp * Ki) * St + b) * XSTR] = v[c * R + Ki]; });
        }
      });
      sync();
      constexpr int R2 = Cfg::R(i + 1), C2 = Cfg::C(i + 1), NB2 = Cfg::NB(i + 1), Ns2 = Cfg::Ns(i + 2);
      sfor<C2>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        const int beta = tid + c * T;
        if (NB2 % T == 0 || beta < NB2) {
          const int K = beta / Ns2, b = beta % Ns2;
          sfor<R2>([&](auto Ai) HC_INL { v[c * R2 + Ai] = X[(K * St + Ns2 * Ai + b) * XSTR]; });
        }
      });
      sync.war_arrive();
      if constexpr (i == 0) hook0();
      if constexpr (i == P - 2) hook();
    }
  });
}

// Two independent forward FFTs interleaved pass by pass (v through X, w through Y): half the
// barrier phases of two separate transforms, and the butterflies of one stream overlap the
// shared-memory traffic of the other.  hook() runs after the last exchange (X, Y free).
template <class Cfg, class Sync, class P0, class Hook = NoHook>
__device__ __forceinline__ void fft_forward_pair(double2 (&v)[Cfg::E], double2 (&w)[Cfg::E], double2* X, double2* Y,
                                                 const double2* mt, int tid, const Sync& sync, const P0& p0,
                                                 const Hook& hook = Hook()) {
  constexpr int P = Cfg::P, T = Cfg::T;
  static_assert(P >= 2, "radix plans have at least two passes");
  sfor<P>([&](auto I) HC_INL {
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
        } else if constexpr (i < P - 1) {
          const int b = beta % Ns1;
          sfor<R - 1>([&](auto Ki) HC_INL {
            constexpr int k = Ki + 1;
            const double2 tw = mt[Cfg::MTo(i) + (k - 1) * Ns1 + b];
            v[c * R + k] = cmul(v[c * R + k], tw);
            w[c * R + k] = cmul(w[c * R + k], tw);
          });
        }
      }
    });
    if constexpr (i < P - 1) {
      constexpr int St = Cfg::St(i + 1);
      sfor<C>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        const int beta = tid + c * T;
        if (NB % T == 0 || beta < NB) {
          const int K = beta / Ns1, b = beta % Ns1;
          sfor<R>([&](auto Ki) HC_INL {
            X[(K + Rp * Ki) * St + b] = v[c * R + Ki];
            Y[(K + Rp * Ki) * St + b] = w[c * R + Ki];
          });
        }
      });
      sync();
      constexpr int R2 = Cfg::R(i + 1), C2 = Cfg::C(i + 1), NB2 = Cfg::NB(i + 1), Ns2 = Cfg::Ns(i + 2);
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
      if constexpr (i == P - 2) hook();
    }
  });
}

// Inverse FFT (unnormalised, DIR = -1), from the last-pass layout left by fft_forward to the
// pass-0 layout (v[c*R0 + a] = x[Ns1*a + b]); pass-0 twiddles are the conjugates of p0's.
template <class Cfg, class Sync, class P0, class Hook = NoHook, int XSTR = 1>
__device__ __forceinline__ void fft_inverse(double2 (&v)[Cfg::E], double2* X, const double2* mt, int tid,
                                            const Sync& sync, const P0& p0, const Hook& hook = Hook()) {
  constexpr int P = Cfg::P, T = Cfg::T;
  sfor<P>([&](auto Iv) HC_INL {
    constexpr int i = P - 1 - Iv;
    constexpr int R = Cfg::R(i), C = Cfg::C(i), NB = Cfg::NB(i), Ns1 = Cfg::Ns(i + 1);
    sfor<C>([&](auto Ci) HC_INL {
      constexpr int c = Ci;
      const int beta = tid + c * T;
      if (NB % T == 0 || beta < NB) {
        if constexpr (i == 0) {
          pass0_twiddle<-1, R>(v + c * R, beta, p0);
        } else if constexpr (i < P - 1) {
          const int b = beta % Ns1;
          sfor<R - 1>([&](auto Ki) HC_INL {
            constexpr int k = Ki + 1;
            v[c * R + k] = cmulc(v[c * R + k], mt[Cfg::MTo(i) + (k - 1) * Ns1 + b]);
          });
        }
        DFT<R, -1>::run(v + c * R);
      }
    });
    if constexpr (i > 0) {
      constexpr int St = Cfg::St(i);
      sync.war_wait();
      sfor<C>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        const int beta = tid + c * T;
        if (NB % T == 0 || beta < NB) {
          const int K = beta / Ns1, b = beta % Ns1;
          sfor<R>([&](auto Ai) HC_INL { X[(K * St + Ns1 * Ai + b) * XSTR] = v[c * R + Ai]; });
        }
      });
      sync();
      constexpr int R0 = Cfg::R(i - 1), C0 = Cfg::C(i - 1), NB0 = Cfg::NB(i - 1), Rp0 = Cfg::Rprod(i - 1);
      constexpr int Ns0 = Cfg::Ns(i);
      sfor<C0>([&](auto Ci) HC_INL {
        constexpr int c = Ci;
        const int beta = tid + c * T;
        if (NB0 % T == 0 || beta < NB0) {
          const int K = beta / Ns0, b = beta % Ns0;
          sfor<R0>([&](auto Ki) HC_INL { v[c * R0 + Ki] = X[((K + Rp0 * Ki) * St + b) * XSTR]; });
        }
      });
      sync.war_arrive();
      if constexpr (i == 1) hook();
    }
  });
}

}  // namespace hc
