// block_io.cuh — per-symmetry residue-block pre/post-processing shared by every kernel.
//
// Unified form of the paper's padded FFTs.  For an axis with parameters (L, M, m, p, q, n)
// let B be the residue-block length (blockLength(), proj/src/plan.cpp:26-29) so that
// q m = n B in every regime.  Residue block v of the qm-point padded transform is
//     F_{v + n k} = sum_s zeta_B^{k s} W_s,   W_s = sum_{j == s (mod B)} zeta_qm^{v j} f_j,
// the B-point DFT of the pre-twiddled input folded modulo B:
//   * complex, p <= 2 : Alg. forward1/forward2, W_s = w_{r,s};
//   * complex, p > 2  : Alg. forwardInner -- the p-point DFTs over t are
//                       the first radix-p stage of the pm-point DFT, k = p l + u;
//   * centered        : Eqs. forCent/wDef, logical j in [-H, L-H);
//   * Hermitian       : Eq. wHerDef; W is Hermitian so the B-point DFT is
//                       real and is computed as a complex-to-real transform through one
//                       B/2-point complex FFT (Z'_k packing below).
// The inverse of residue v is h_j += zeta_qm^{-v j} w_{j mod B}, w = unnormalised inverse
// B-point DFT of the product (Eqs. invStan/invInner).
#pragma once
#include "fft_device.cuh"

namespace hc {

enum : int { SYM_COMPLEX = 0, SYM_CENTERED = 1, SYM_HERMITIAN = 2 };

// Line addressing: line l starts at (l / nin) * d_out + (l % nin) * d_in (complex elements);
// element j of the line is at start + j * es.
struct Lines {
  long long count, nin, d_out, d_in, es;
  __device__ __forceinline__ long long base(long long l) const { return (l / nin) * d_out + (l % nin) * d_in; }
};

struct AxisDev {
  int sym;
  int L;   // logical length
  int S;   // stored length (L, or ceil(L/2) for Hermitian)
  int B;   // residue block length
  int Bc;  // complex FFT length (B, or B/2 for Hermitian)
  int n;   // residue blocks
  int qm;  // padded length q*m = n*B
  int H;   // centered origin floor(L/2)
  int pe;  // reference-order interleave: p (complex inner), p/2 (centered/Hermitian inner), else 1
  int m;
  const double2* tw;  // zeta_Bc^e, e < Bc                      (direct-sum kernels)
  const double2* zq;  // zeta_qm^e, e < qm                      (direct-sum kernels)
  // radix kernels: per-axis tables built on the host for the kernel's pass-0 split
  // s = Ns1 a + b (no runtime modulo on the device); see hconv_lib.cu build_tables()
  const double2* tab;
  int ns1, nu, nc;      // Ns1, rows of U (2 R0 + 1), rows of Cv
  int oMT, oU, oC, oA, oZ, oH, oBl, oBh;
  int tabn;             // entries staged in shared memory (>= the middle-pass tables)
  int tabfull;          // entries the kernel reads (all staged when tabn >= tabfull)
};

// ---- table accessors (radix kernels) ----
//  A[b]     = omega_Bc^b            b < Ns1
//  Z[v][b]  = zeta_qm^{v b}         b < Ns1
//  U[v][a]  = zeta_qm^{v Ns1 a}     a < 2 R0 + 1
//  Cv[v][t] = zeta_qm^{v t B}       t < nc
//  Hh[v]    = zeta_qm^{v Bc}        (Hermitian)
//  Bl[b]    = zeta_B^b, Bh[a] = zeta_B^{Ns1 a}   (Hermitian packing)
//  MT       = middle-pass twiddles (FFTCfg::MT layout)
// order in memory: MT U C A Z H Bl Bh -- the kernel stages the longest prefix that fits
// tb: the tables as the kernel reads them -- the shared-memory copy when everything was
// staged (a.tabn >= a.tabfull), else the global copy (the middle-pass tables MT are always
// read from shared memory, see kernels.cuh).
__device__ __forceinline__ double2 tget(const AxisDev& a, const double2* tb, int i) { return tb[i]; }
__device__ __forceinline__ double2 tA(const AxisDev& a, const double2* tb, int b) { return tget(a, tb, a.oA + b); }
__device__ __forceinline__ double2 tZ(const AxisDev& a, const double2* tb, int v, int b) { return tget(a, tb, a.oZ + v * a.ns1 + b); }
__device__ __forceinline__ double2 tU(const AxisDev& a, const double2* tb, int v, int i) { return tget(a, tb, a.oU + v * a.nu + i); }
__device__ __forceinline__ double2 tC(const AxisDev& a, const double2* tb, int v, int t) { return tget(a, tb, a.oC + v * a.nc + t); }
__device__ __forceinline__ double2 tH(const AxisDev& a, const double2* tb, int v) { return tget(a, tb, a.oH + v); }
__device__ __forceinline__ double2 tBl(const AxisDev& a, const double2* tb, int b) { return tget(a, tb, a.oBl + b); }
__device__ __forceinline__ double2 tBh(const AxisDev& a, const double2* tb, int i) { return tget(a, tb, a.oBh + i); }

// zeta_qm^e for |e| < 2^31 (32-bit reduction: exponents are v*j with v < n, |j| < 2B)
__device__ __forceinline__ double2 zpow(const AxisDev& a, int e) {
  e %= a.qm;
  if (e < 0) e += a.qm;
  return __ldg(a.zq + e);
}

// W_s for complex / centered data (s in [0, B)).
template <int SYM>
__device__ __forceinline__ double2 load_W(const AxisDev& a, const double2* __restrict__ f, long long es, int s, int v) {
  double2 acc = make_double2(0.0, 0.0);
  if constexpr (SYM == SYM_COMPLEX) {
    for (int j = s; j < a.L; j += a.B) acc = cadd(acc, v ? cmul(f[(long long)j * es], zpow(a, v * j)) : f[(long long)j * es]);
  } else {
    // logical j = s (stored s + H) and j = s - B (stored s - B + H)
    if (s < a.L - a.H) acc = v ? cmul(f[(long long)(s + a.H) * es], zpow(a, v * s)) : f[(long long)(s + a.H) * es];
    const int st2 = s - a.B + a.H;
    if (st2 >= 0) {
      const double2 x = f[(long long)st2 * es];
      acc = cadd(acc, v ? cmul(x, zpow(a, v * (s - a.B))) : x);
    }
  }
  return acc;
}

// Hermitian W_s, s in [0, B/2]: logical j = s (f_s) and j = s - B (conj f_{B-s}).
__device__ __forceinline__ double2 load_WH(const AxisDev& a, const double2* __restrict__ f, long long es, int s, int v) {
  double2 acc = make_double2(0.0, 0.0);
  if (s < a.S) acc = v ? cmul(f[(long long)s * es], zpow(a, v * s)) : f[(long long)s * es];
  const int r = a.B - s;
  if (r > 0 && r < a.S) {
    const double2 x = cconj(f[(long long)r * es]);
    acc = cadd(acc, v ? cmul(x, zpow(a, v * (s - a.B))) : x);
  }
  return acc;
}

// Packed complex-to-real input: Z'_k = (W_k + conj W_{Bc-k}) + i zeta_B^k (W_k - conj W_{Bc-k}),
// so that the Bc-point forward DFT of Z' is z_l = V_{2l} + i V_{2l+1}.
__device__ __forceinline__ double2 load_Zp(const AxisDev& a, const double2* __restrict__ f, long long es, int k, int v) {
  const double2 wk = load_WH(a, f, es, k, v);
  const double2 wm = cconj(load_WH(a, f, es, a.Bc - k, v));
  const double2 e = cadd(wk, wm);
  const double2 o = cmul(csub(wk, wm), __ldg(a.zq + (long long)k * a.n));  // zeta_B^k = zeta_qm^{k n}
  return make_double2(e.x - o.y, e.y + o.x);                                 // e + i o
}

// value of block index s in pass-0 order for the given symmetry
template <int SYM>
__device__ __forceinline__ double2 load_in(const AxisDev& a, const double2* __restrict__ f, long long es, int s, int v) {
  if constexpr (SYM == SYM_HERMITIAN) return load_Zp(a, f, es, s, v);
  else return load_W<SYM>(a, f, es, s, v);
}

// Destination of residue contributions: dst[j] = ((acc ? acc[j] : 0) + val) * scale.
// Final outputs are written with the streaming (evict-first) hint so that the L2-resident
// residue accumulators of the persistent CTAs are not pushed out to HBM.
struct Emit {
  double2* dst;
  long long des;
  const double2* acc;
  long long aes;
  double scale;
  bool stream = false;
  __device__ __forceinline__ void operator()(long long j, double2 val) const {
    put(j, val, acc ? acc[j * aes] : make_double2(0.0, 0.0));
  }
  // store with an already-loaded accumulator value (zero when acc == nullptr)
  __device__ __forceinline__ void put(long long j, double2 val, double2 accv) const {
    if (acc) val = cadd(val, accv);
    if (scale != 1.0) val = cscale(val, scale);
    if (stream) __stcs(dst + j * des, val);
    else dst[j * des] = val;
  }
};

// Complex / centered inverse post-processing of block element s (natural order).
template <int SYM>
__device__ __forceinline__ void store_w(const AxisDev& a, const Emit& em, int s, int v, double2 w) {
  if constexpr (SYM == SYM_COMPLEX) {
    for (int j = s; j < a.L; j += a.B) em(j, v ? cmulc(w, zpow(a, v * j)) : w);
  } else {
    if (s < a.L - a.H) em(s + a.H, v ? cmulc(w, zpow(a, v * s)) : w);
    const int st2 = s - a.B + a.H;
    if (st2 >= 0) em(st2, v ? cmulc(w, zpow(a, v * (s - a.B))) : w);
  }
}

// Hermitian inverse post-processing: Z (natural order, Bc values, shared memory) holds the
// Bc-point inverse DFT of the packed product; output stored index j in [0, S).
__device__ __forceinline__ double2 herm_w(const AxisDev& a, const double2* Z, int j, int v) {
  const bool hi = j > a.Bc;
  const int k = hi ? a.B - j : j;
  const double2 zk = Z[k == a.Bc ? 0 : k];
  const double2 zm = cconj(Z[k == 0 ? 0 : a.Bc - k]);
  const double2 e = cscale(cadd(zk, zm), 0.5);
  const double2 d = cscale(csub(zk, zm), 0.5);
  const double2 o = make_double2(d.y, -d.x);                              // d / i
  double2 w = cadd(e, cmulc(o, __ldg(a.zq + (long long)k * a.n)));         // e + zeta_B^{-k} o
  if (hi) w = cconj(w);
  return v ? cmulc(w, zpow(a, v * j)) : w;
}

// ------------------------------------------------------------- radix kernels --
// pass-0 element (a, b), s = Ns1 a + b, of residue v, WITHOUT the factor zeta_qm^{v b}
// (folded into the pass-0 output twiddle t0 = Z[v][b]):  x = zeta_qm^{v Ns1 a} * sum_t ...
template <int SYM>
__device__ __forceinline__ double2 load_fast(const AxisDev& a, const double2* tb, const double2* __restrict__ f,
                                             long long es, int s, int v, int ia) {
  double2 x;
  if constexpr (SYM == SYM_COMPLEX) {
    x = s < a.L ? f[(long long)s * es] : make_double2(0.0, 0.0);
    int t = 1;
    for (int j = s + a.B; j < a.L; j += a.B, ++t) x = cadd(x, v ? cmul(f[(long long)j * es], tC(a, tb, v, t)) : f[(long long)j * es]);
  } else {
    x = s < a.L - a.H ? f[(long long)(s + a.H) * es] : make_double2(0.0, 0.0);
    const int st2 = s - a.B + a.H;  // logical s - B
    if (st2 >= 0) x = cadd(x, v ? cmulc(f[(long long)st2 * es], tC(a, tb, v, 1)) : f[(long long)st2 * es]);
  }
  return v ? cmul(x, tU(a, tb, v, ia)) : x;
}

// Hermitian W_s (s in [0, Bc]) with the full factor zeta_qm^{v s} = zs (zeta_qm^{-v B} = conj Cv[v][1]).
__device__ __forceinline__ double2 load_WH_fast(const AxisDev& a, const double2* tb, const double2* __restrict__ f,
                                                long long es, int s, int v, double2 zs) {
  double2 x = s < a.S ? f[(long long)s * es] : make_double2(0.0, 0.0);
  const int r = a.B - s;
  if (r > 0 && r < a.S) x = cadd(x, v ? cmulc(cconj(f[(long long)r * es]), tC(a, tb, v, 1)) : cconj(f[(long long)r * es]));
  return v ? cmul(x, zs) : x;
}

// Hermitian packed input Z'_k, k = Ns1 a + b < Bc (no folding into the pass-0 twiddle).
__device__ __forceinline__ double2 load_Zp_fast(const AxisDev& a, const double2* tb, const double2* __restrict__ f,
                                                long long es, int k, int v, int ia, int b) {
  double2 zk = make_double2(1.0, 0.0), zm = zk;
  if (v) {
    zk = cmul(tZ(a, tb, v, b), tU(a, tb, v, ia));   // zeta_qm^{v k}
    zm = cmulc(tH(a, tb, v), zk);               // zeta_qm^{v (Bc - k)}
  }
  const double2 wk = load_WH_fast(a, tb, f, es, k, v, zk);
  const double2 wm = cconj(load_WH_fast(a, tb, f, es, a.Bc - k, v, zm));
  const double2 e = cadd(wk, wm);
  const double2 o = cmul(csub(wk, wm), cmul(tBh(a, tb, ia), tBl(a, tb, b)));  // zeta_B^k
  return make_double2(e.x - o.y, e.y + o.x);
}

// inverse post-processing of pass-0 element s = Ns1 a + b (complex / centered); w already
// carries conj(Z[v][b]) from the inverse pass-0 twiddle.
template <int SYM>
__device__ __forceinline__ void store_fast(const AxisDev& a, const double2* tb, const Emit& em, int s, int v, int ia,
                                           double2 w) {
  if (v) w = cmulc(w, tU(a, tb, v, ia));
  if constexpr (SYM == SYM_COMPLEX) {
    if (s < a.L) em(s, w);
    int t = 1;
    for (int j = s + a.B; j < a.L; j += a.B, ++t) em(j, v ? cmulc(w, tC(a, tb, v, t)) : w);
  } else {
    if (s < a.L - a.H) em(s + a.H, w);
    const int st2 = s - a.B + a.H;
    if (st2 >= 0) em(st2, v ? cmul(w, tC(a, tb, v, 1)) : w);
  }
}

// Hermitian output j in [0, S) from Z (natural order, shared memory); NS1 = Ns1 of the kernel.
template <int NS1>
__device__ __forceinline__ double2 herm_w_fast(const AxisDev& a, const double2* tb, const double2* Z, int j, int v) {
  const bool hi = j > a.Bc;
  const int k = hi ? a.B - j : j;
  const double2 zk = Z[k == a.Bc ? 0 : k];
  const double2 zm = cconj(Z[k == 0 ? 0 : a.Bc - k]);
  const double2 e = cscale(cadd(zk, zm), 0.5);
  const double2 d = cscale(csub(zk, zm), 0.5);
  const double2 o = make_double2(d.y, -d.x);                                   // d / i
  double2 w = cadd(e, cmulc(o, cmul(tBh(a, tb, k / NS1), tBl(a, tb, k % NS1))));        // e + zeta_B^{-k} o
  if (hi) w = cconj(w);
  return v ? cmulc(w, cmul(tZ(a, tb, v, j % NS1), tU(a, tb, v, j / NS1))) : w;
}

// Hermitian post-processing by quads (radix kernels): one (Z_k, Z_{Bc-k}) pair gives
// w_k, w_{Bc-k} and, by Hermitian symmetry, w_{B-k} = conj w_k and w_{Bc+k} = conj w_{Bc-k}
// (E_{Bc-k} = conj E_k, O_{Bc-k} = conj O_k, zeta_B^{-(Bc-k)} = -zeta_B^k).  The accumulator
// values of a quad are loaded before any of its stores.  Bc is even for every radix plan.
template <int NS1>
__device__ __forceinline__ void herm_store_quads(const AxisDev& a, const double2* tb, const Emit& em,
                                                 const double2* Z, int v, int tid, int T) {
  const int Bc = a.Bc, B = a.B, S = a.S, half = Bc / 2;
  const double2 one = make_double2(1.0, 0.0);
  const double2 zBc = v ? tH(a, tb, v) : one;     // zeta_qm^{v Bc}
  const double2 zB = v ? tC(a, tb, v, 1) : one;   // zeta_qm^{v B}
  if (S <= half) {
    // heavily padded lines: every stored output is a quad's first element w_k (the other three
    // lie beyond the data), so only w_k is formed
    for (int k = tid; k < S; k += T) {
      const double2 accv = em.acc ? em.acc[k * em.aes] : make_double2(0.0, 0.0);
      const double2 zk = Z[k];
      const double2 zm = cconj(Z[k == 0 ? 0 : Bc - k]);
      const double2 e = cscale(cadd(zk, zm), 0.5);
      const double2 d = cscale(csub(zk, zm), 0.5);
      const double2 o = make_double2(d.y, -d.x);
      double2 wk = cadd(e, cmulc(o, cmul(tBh(a, tb, k / NS1), tBl(a, tb, k % NS1))));
      if (v) wk = cmulc(wk, cmul(tZ(a, tb, v, k % NS1), tU(a, tb, v, k / NS1)));
      em.put(k, wk, accv);
    }
    return;
  }
  for (int k = tid; k <= half; k += T) {
    int j[4] = {k, B - k, Bc - k, Bc + k};
    bool ok[4] = {k < S, k > 0 && B - k < S, Bc - k != k && Bc - k < S, k > 0 && k != half && Bc + k < S};
    double2 acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = (ok[u] && em.acc) ? em.acc[j[u] * em.aes] : make_double2(0.0, 0.0);
    const double2 zk = Z[k];
    const double2 zm = cconj(Z[k == 0 ? 0 : Bc - k]);
    const double2 e = cscale(cadd(zk, zm), 0.5);
    const double2 d = cscale(csub(zk, zm), 0.5);
    const double2 o = make_double2(d.y, -d.x);                         // d / i
    const double2 tB = cmul(tBh(a, tb, k / NS1), tBl(a, tb, k % NS1));  // zeta_B^k
    const double2 wk = cadd(e, cmulc(o, tB));                          // e + zeta_B^{-k} o
    const double2 wm = csub(cconj(e), cmul(tB, cconj(o)));             // conj e - zeta_B^k conj o
    double2 w[4] = {wk, cconj(wk), wm, cconj(wm)};
    if (v) {
      const double2 zvk = cmul(tZ(a, tb, v, k % NS1), tU(a, tb, v, k / NS1));  // zeta_qm^{v k}
      w[0] = cmulc(w[0], zvk);                  // zeta^{-v k}
      w[1] = cmulc(cmul(w[1], zvk), zB);        // zeta^{-v (B - k)}
      w[2] = cmulc(cmul(w[2], zvk), zBc);       // zeta^{-v (Bc - k)}
      w[3] = cmulc(cmulc(w[3], zvk), zBc);      // zeta^{-v (Bc + k)}
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (ok[u]) em.put(j[u], w[u], acc[u]);
  }
}

// reference order of block value with natural index k' (SPEC pfft-* output: F[u m + l] with
// k' = pe*l + u for inner regimes, F[l] otherwise)
__device__ __forceinline__ long long ref_index(const AxisDev& a, long long kp) {
  if (a.pe <= 1) return kp;
  return (kp % a.pe) * a.m + kp / a.pe;
}

}  // namespace hc
