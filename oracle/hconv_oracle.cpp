// hconv_oracle.cpp — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// CPU restatement of the hybrid-dealiased convolution of arXiv 2303.17510, used
// only as (1) the parity checker of the CUDA path in tests/ and smoke(), and
// (2) the CPU baseline arm of bench.py.  Nothing in the product package links,
// loads or calls this file.
//
// Every routine restates the reference (paths relative to /root/reference):
//   plan        proj/src/plan.cpp:26-99        (deriveParams, root, RootTable, workMemoryWords)
//   forward1    PAPER.md:315-327  backward1    PAPER.md:332-341  (Eqs. forStan/invStan :129-138)
//   forward2    PAPER.md:349-361  backward2    PAPER.md:366-379  -- erratum: the t=1 chunk uses
//               zeta_qm^{-s r} (Eq. invStan :135-138), not zeta_qm^{-(s-m) r} as printed at :375
//   forwardInner / backwardInner PAPER.md:690-749 (Eq. invInner :677-681)
//   forward2C / backward2C       PAPER.md:438-473 (one residue of length m)
//   forwardInnerC/backwardInnerC PAPER.md:1173-1241
//   forward2H / backward2H
//   forwardInnerH/backwardInnerH PAPER.md:1249-1318 -- erratum: the even-m loop runs t < p/2
//               (PAPER.md:1312 prints t = 0..p/2, which indexes W out of range)
//   Appendix algorithms read outside the stored window: such reads are zero, such
//   writes are dropped.
//   forward_conjugate_pair
//   convolve / convolveX         PAPER.md:188-262 -- erratum: inner branch n = ceil(M/(pm))
//               (plan.cpp:52), not ceil(M/m) as printed at :203
//   convolve_nd
//   direct_convolution / padded_dft_slice / naive_dft
// The FFTs underneath are an in-house mixed-radix FFT with exact (integer-reduced)
// twiddles; the reference uses FFTW 3.3.10 via FFTW++ (PAPER.md:891-892,921-922), which
// is absent from /root/reference and from this image.
//
// Parity pinning: the plan functions are checked against the reference's own plan.cpp
// compiled into oracle/_ref/ (oracle/Makefile); the arithmetic is checked against the
// SPEC known-answer examples (tests/golden/spec_kats.json) and naive padded DFTs.
#include "../include/hconv.h"
#include "../paper_2303_17510_b200/csrc/slab.hpp"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <memory>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

using cd = std::complex<double>;

namespace orc {

static thread_local std::string g_err;

static size_t cq(size_t a, size_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- plan ------
// proj/src/plan.cpp:35-64
struct Params {
  size_t L = 1, M = 1, m = 1, p = 1, q = 1, n = 1;
  int sym = HCONV_COMPLEX;
  int regime = HCONV_P1;
};

static Params derive(size_t L, size_t M, size_t m, int sym) {
  if (L == 0) throw std::invalid_argument("deriveParams: L must be positive");
  if (m == 0) throw std::invalid_argument("deriveParams: m must be positive");
  if (M < L) throw std::invalid_argument("deriveParams: M must satisfy M >= L");
  if (sym < 0 || sym > 2) throw std::invalid_argument("deriveParams: bad symmetry");
  Params pp;
  pp.L = L; pp.M = M; pp.m = m; pp.sym = sym;
  if (sym == HCONV_COMPLEX) {
    pp.p = cq(L, m);
    if (pp.p <= 2) { pp.n = cq(M, m); pp.q = pp.n; }
    else { pp.n = cq(M, pp.p * m); pp.q = pp.n * pp.p; }
    pp.regime = pp.p == 1 ? HCONV_P1 : (pp.p == 2 ? HCONV_P2 : HCONV_INNER);
  } else {
    pp.p = 2 * cq(L, 2 * m);
    pp.n = cq(2 * M, pp.p * m);
    pp.q = pp.n * pp.p / 2;
    pp.regime = pp.p == 2 ? HCONV_P2 : HCONV_INNER;
  }
  return pp;
}

static Params from_abi(const hconv_params* a) {
  Params pp = derive(a->L, a->M, a->m, a->symmetry);
  return pp;
}

// Hermitian data: stored non-negative indices 0..ceil(L/2)-1 (logical support |j| < ceil(L/2)).
static size_t stored_len(const Params& pp) { return pp.sym == HCONV_HERMITIAN ? cq(pp.L, 2) : pp.L; }
static size_t block_len(const Params& pp) {  // plan.cpp:26-29
  if (pp.regime != HCONV_INNER) return pp.m;
  return pp.sym == HCONV_COMPLEX ? pp.p * pp.m : (pp.p / 2) * pp.m;
}

// plan.cpp:66-73 (evaluated in long double, then rounded)
static cd root(size_t N, int64_t k) {
  if (N == 0) throw std::invalid_argument("root: N must be positive");
  int64_t r = k % (int64_t)N;
  if (r < 0) r += (int64_t)N;
  if (r == 0) return {1.0, 0.0};
  const long double twopi = 6.283185307179586476925286766559005768L;
  long double a = twopi * (long double)r / (long double)N;
  return {(double)cosl(a), (double)sinl(a)};
}

// plan.hpp:84-106 RootTable
struct Roots {
  size_t N;
  std::vector<cd> z;
  explicit Roots(size_t n) : N(n), z(n) {
    if (n == 0) throw std::invalid_argument("RootTable: modulus must be positive");
    for (size_t k = 0; k < n; ++k) z[k] = root(n, (int64_t)k);
  }
  cd operator()(int64_t k) const {
    int64_t r = k % (int64_t)N;
    if (r < 0) r += (int64_t)N;
    return z[(size_t)r];
  }
};

// ----------------------------------------------------------------- FFT ------
// Unnormalised DFT y_k = sum_j zeta_N^{sign*j*k} x_j (PAPER.md:115-118 sign convention).
static void naive_dft(const cd* x, cd* y, size_t N, int sign) {
  std::vector<cd> out(N);
  for (size_t k = 0; k < N; ++k) {
    cd s = 0;
    for (size_t j = 0; j < N; ++j) s += x[j] * root(N, (int64_t)sign * (int64_t)((j * k) % N));
    out[k] = s;
  }
  std::copy(out.begin(), out.end(), y);
}

// Mixed-radix recursive decimation-in-time FFT with an exact twiddle table.
struct FFT {
  size_t N;
  int sign;
  std::vector<cd> tw;  // zeta_N^{sign*k}
  std::vector<size_t> fac;
  FFT(size_t n, int s) : N(n), sign(s), tw(n) {
    for (size_t k = 0; k < n; ++k) tw[k] = root(n, (int64_t)s * (int64_t)k);
    size_t r = n;
    for (size_t f : {4, 2, 3, 5, 7}) while (r % f == 0 && r > 1) { fac.push_back(f); r /= f; }
    for (size_t f = 11; r > 1; f += 2) while (r % f == 0) { fac.push_back(f); r /= f; }
  }
  void rec(const cd* in, size_t is, cd* out, size_t n, size_t ts, size_t fi) const {
    if (n == 1) { out[0] = in[0]; return; }
    const size_t r = fac[fi], m = n / r;
    for (size_t j = 0; j < r; ++j) rec(in + j * is, is * r, out + j * m, m, ts * r, fi + 1);
    cd t[64];
    std::vector<cd> big;
    cd* tp = t;
    if (r > 64) { big.resize(r); tp = big.data(); }
    for (size_t k = 0; k < m; ++k) {
      for (size_t j = 0; j < r; ++j) tp[j] = out[j * m + k] * tw[(j * k * ts) % N];
      for (size_t s = 0; s < r; ++s) {
        cd acc = 0;
        for (size_t j = 0; j < r; ++j) acc += tp[j] * tw[((j * s) % r) * (N / r)];
        out[k + s * m] = acc;
      }
    }
  }
  void exec(const cd* in, cd* out) const {  // out may not alias in
    rec(in, 1, out, N, 1, 0);
  }
};

static void fft(const cd* x, cd* y, size_t N, int sign) {
  if (N <= 16) { naive_dft(x, y, N, sign); return; }
  FFT f(N, sign);
  std::vector<cd> tmp(x, x + N);
  f.exec(tmp.data(), y);
}

// complex-to-real: V_l = sum_{s<m} zeta_m^{l s} W_s with W_{m-s} = conj(W_s); input W_0..W_{e-1}
static void crfft(const cd* W, double* V, size_t m) {
  const size_t e = m / 2 + 1;
  std::vector<cd> full(m), out(m);
  for (size_t s = 0; s < m; ++s) full[s] = s < e ? W[s] : std::conj(W[m - s]);
  if (m % 2 == 0) full[m / 2] = cd(W[m / 2].real(), 0.0);
  full[0] = cd(W[0].real(), 0.0);
  fft(full.data(), out.data(), m, +1);
  for (size_t l = 0; l < m; ++l) V[l] = out[l].real();
}
// real-to-complex (inverse sign): W_s = sum_l zeta_m^{-s l} V_l, s < e
static void rcfft(const double* V, cd* W, size_t m) {
  const size_t e = m / 2 + 1;
  std::vector<cd> full(m), out(m);
  for (size_t l = 0; l < m; ++l) full[l] = V[l];
  fft(full.data(), out.data(), m, -1);
  for (size_t s = 0; s < e; ++s) W[s] = out[s];
}

// ---------------------------------------------------- padded FFT kernels ----
// Guarded accessors: reads outside the stored window are zero.
struct In {
  const cd* f;
  size_t n;
  cd operator[](int64_t j) const { return (j >= 0 && (size_t)j < n) ? f[j] : cd(0); }
};
struct Out {
  cd* v;
  size_t n;
  void set(int64_t j, cd x) const { if (j >= 0 && (size_t)j < n) v[j] = x; }
};

// forward1
static void forward1(const Params& P, const cd* f, size_t r, cd* F) {
  const size_t L = P.L, m = P.m, qm = P.q * P.m;
  std::vector<cd> W(m, 0.0);
  for (size_t s = 0; s < L; ++s) W[s] = root(qm, (int64_t)(r * s)) * f[s];
  fft(W.data(), F, m, +1);
}
// backward1
static void backward1(const Params& P, const cd* F, size_t r, cd* V) {
  const size_t L = P.L, m = P.m, qm = P.q * P.m;
  std::vector<cd> W(m);
  fft(F, W.data(), m, -1);
  for (size_t s = 0; s < L; ++s) V[s] = root(qm, -(int64_t)(r * s)) * W[s];
}
// forward2
static void forward2(const Params& P, const cd* f, size_t r, cd* F) {
  const size_t L = P.L, m = P.m, qm = P.q * P.m;
  std::vector<cd> W(m, 0.0);
  for (size_t s = 0; s + m < L; ++s)
    W[s] = root(qm, (int64_t)(r * s)) * f[s] + root(qm, (int64_t)(r * (m + s))) * f[m + s];
  for (size_t s = (L > m ? L - m : 0); s < m; ++s) W[s] = s < L ? root(qm, (int64_t)(r * s)) * f[s] : cd(0);
  fft(W.data(), F, m, +1);
}
// backward2, PAPER.md:366-379 with the Eq. invStan exponent (erratum at :375)
static void backward2(const Params& P, const cd* F, size_t r, cd* V) {
  const size_t L = P.L, m = P.m, qm = P.q * P.m;
  std::vector<cd> W(m);
  fft(F, W.data(), m, -1);
  for (size_t s = 0; s < m && s < L; ++s) V[s] = root(qm, -(int64_t)(s * r)) * W[s];
  for (size_t s = m; s < L; ++s) V[s] = root(qm, -(int64_t)(s * r)) * W[s - m];
}
// forwardInner
static void forwardInner(const Params& P, const cd* f, size_t v, cd* F) {
  const size_t L = P.L, m = P.m, q = P.q, p = P.p, n = P.n, qm = q * m;
  std::vector<cd> W(p * m, 0.0);
  for (size_t t = 0; t + 1 < p; ++t)
    for (size_t s = 0; s < m; ++s) W[t * m + s] = root(q, (int64_t)(v * t)) * f[t * m + s];
  const size_t t0 = p - 1;
  for (size_t s = 0; t0 * m + s < L; ++s) W[t0 * m + s] = root(q, (int64_t)(v * t0)) * f[t0 * m + s];
  std::vector<cd> col(p), ocol(p);
  for (size_t s = 0; s < m; ++s) {
    for (size_t t = 0; t < p; ++t) col[t] = W[t * m + s];
    fft(col.data(), ocol.data(), p, +1);
    for (size_t u = 0; u < p; ++u) W[u * m + s] = ocol[u];
  }
  for (size_t u = 0; u < p; ++u) {
    for (size_t s = 0; s < m; ++s) W[u * m + s] *= root(qm, (int64_t)((u * n + v) * s));
    fft(W.data() + u * m, F + u * m, m, +1);
  }
}
// backwardInner
static void backwardInner(const Params& P, const cd* F, size_t v, cd* V) {
  const size_t L = P.L, m = P.m, q = P.q, p = P.p, n = P.n, qm = q * m;
  std::vector<cd> W(p * m);
  for (size_t u = 0; u < p; ++u) fft(F + u * m, W.data() + u * m, m, -1);
  for (size_t u = 0; u < p; ++u)
    for (size_t s = 0; s < m; ++s) W[u * m + s] *= root(qm, -(int64_t)(s * (u * n + v)));
  std::vector<cd> col(p), ocol(p);
  for (size_t s = 0; s < m; ++s) {
    for (size_t u = 0; u < p; ++u) col[u] = W[u * m + s];
    fft(col.data(), ocol.data(), p, -1);
    for (size_t t = 0; t < p; ++t) W[t * m + s] = ocol[t];
  }
  for (size_t t = 0; t < p; ++t)
    for (size_t s = 0; s < m && t * m + s < L; ++s) V[t * m + s] = root(q, -(int64_t)(t * v)) * W[t * m + s];
}
// forward2C, PAPER.md:438-454 (stored[j] = logical[j - H])
static void forward2C(const Params& P, const cd* fs, size_t r, cd* F) {
  const int64_t L = P.L, m = P.m, H = P.L / 2, qm = P.q * P.m;
  In f{fs, P.L};
  std::vector<cd> W(m, 0.0);
  for (int64_t s = 0; s < m - H; ++s) W[s] = root(qm, r * s) * f[H + s];
  for (int64_t s = std::max<int64_t>(m - H, 0); s < L - H; ++s)
    W[s] = root(qm, (int64_t)r * (s - m)) * f[H + s - m] + root(qm, (int64_t)r * s) * f[H + s];
  for (int64_t s = L - H; s < m; ++s) W[s] = root(qm, (int64_t)r * (s - m)) * f[H + s - m];
  fft(W.data(), F, m, +1);
}
// backward2C, PAPER.md:459-472 (input: this residue's block of length m)
static void backward2C(const Params& P, const cd* F, size_t r, cd* Vs) {
  const int64_t L = P.L, m = P.m, H = P.L / 2, qm = P.q * P.m;
  std::vector<cd> W(m);
  fft(F, W.data(), m, -1);
  Out V{Vs, P.L};
  for (int64_t s = std::max<int64_t>(m - H, 0); s < m; ++s) V.set(H + s - m, root(qm, -(int64_t)r * (s - m)) * W[s]);
  for (int64_t s = 0; s < L - H; ++s) V.set(H + s, root(qm, -(int64_t)r * s) * W[s]);
}
// forwardInnerC, PAPER.md:1173-1202 (delta_t = Kronecker delta_{t,0})
static void forwardInnerC(const Params& P, const cd* fs, size_t v, cd* Fout) {
  const int64_t L = P.L, m = P.m, q = P.q, n = P.n, qm = P.q * P.m;
  const int64_t H = L / 2, ph = cq(L, 2 * m), m0 = ph * m - H, m1 = L - H - (ph - 1) * m;
  In f{fs, P.L};
  std::vector<cd> W(ph * m, 0.0);
  for (int64_t s = 0; s < m0 && s < m; ++s) W[s] = f[H + s];
  for (int64_t t = 0; t < ph; ++t) {
    const int64_t m2 = (t == ph - 1) ? m1 : m;
    for (int64_t s = (t == 0 ? m0 : 0); s < m2; ++s)
      W[t * m + s] = root(q, (int64_t)v * (t - ph)) * f[(t - ph) * m + H + s] + root(q, (int64_t)v * t) * f[t * m + H + s];
  }
  for (int64_t s = std::max<int64_t>(m1, 0); s < m; ++s) W[(ph - 1) * m + s] = root(q, -(int64_t)v) * f[-m + H + s];
  std::vector<cd> col(ph), ocol(ph);
  for (int64_t s = 0; s < m; ++s) {
    for (int64_t t = 0; t < ph; ++t) col[t] = W[t * m + s];
    fft(col.data(), ocol.data(), ph, +1);
    for (int64_t u = 0; u < ph; ++u) W[u * m + s] = ocol[u];
  }
  for (int64_t u = 0; u < ph; ++u) {
    for (int64_t s = 1; s < m; ++s) W[u * m + s] *= root(qm, (u * n + (int64_t)v) * s);
    fft(W.data() + u * m, Fout + u * m, m, +1);
  }
}
// backwardInnerC
static void backwardInnerC(const Params& P, const cd* F, size_t v, cd* Vs) {
  const int64_t L = P.L, m = P.m, q = P.q, n = P.n, qm = P.q * P.m;
  const int64_t H = L / 2, ph = cq(L, 2 * m), m0 = ph * m - H, m1 = L - H - (ph - 1) * m;
  std::vector<cd> W(ph * m);
  for (int64_t u = 0; u < ph; ++u) {
    fft(F + u * m, W.data() + u * m, m, -1);
    for (int64_t s = 1; s < m; ++s) W[u * m + s] *= root(qm, -(u * n + (int64_t)v) * s);
  }
  std::vector<cd> col(ph), ocol(ph);
  for (int64_t s = 0; s < m; ++s) {
    for (int64_t u = 0; u < ph; ++u) col[u] = W[u * m + s];
    fft(col.data(), ocol.data(), ph, -1);
    for (int64_t t = 0; t < ph; ++t) W[t * m + s] = ocol[t];
  }
  Out V{Vs, P.L};
  for (int64_t s = 0; s < m0 && s < m; ++s) V.set(H + s, W[s]);
  for (int64_t t = 0; t < ph; ++t) {
    const int64_t m2 = (t == ph - 1) ? m1 : m;
    for (int64_t s = (t == 0 ? m0 : 0); s < m2; ++s) {
      V.set((t - ph) * m + H + s, root(q, -(int64_t)v * (t - ph)) * W[t * m + s]);
      V.set(t * m + H + s, root(q, -(int64_t)v * t) * W[t * m + s]);
    }
  }
  for (int64_t s = std::max<int64_t>(m1, 0); s < m; ++s) V.set(-m + H + s, root(q, (int64_t)v) * W[(ph - 1) * m + s]);
}
// forward2H, PAPER.md:514-527 (f stores logical 0..Ht-1, Ht = ceil(L/2))
static void forward2H(const Params& P, const cd* fs, size_t r, double* V) {
  const int64_t m = P.m, Ht = cq(P.L, 2), e = m / 2 + 1, qm = P.q * P.m;
  In f{fs, (size_t)Ht};
  std::vector<cd> W(std::max<int64_t>(e, m - Ht + 1) + 1, 0.0);
  for (int64_t s = 0; s <= m - Ht; ++s) W[s] = root(qm, (int64_t)r * s) * f[s];
  for (int64_t s = std::max<int64_t>(m - Ht + 1, 0); s < e; ++s)
    W[s] = root(qm, (int64_t)r * s) * f[s] + root(qm, (int64_t)r * (s - m)) * std::conj(f[m - s]);
  crfft(W.data(), V, m);
}
// backward2H, PAPER.md:534-549 (F: this residue's m real values)
static void backward2H(const Params& P, const double* F, size_t r, cd* Vs) {
  const int64_t m = P.m, Ht = cq(P.L, 2), e = m / 2 + 1, q = P.q, qm = P.q * P.m;
  std::vector<cd> W(e);
  rcfft(F, W.data(), m);
  Out V{Vs, (size_t)Ht};
  for (int64_t s = 0; s <= m - e; ++s) V.set(s, root(qm, -(int64_t)r * s) * W[s]);
  for (int64_t s = std::max<int64_t>(m - Ht + 1, 0); s <= m - e; ++s) V.set(m - s, root(qm, -(int64_t)r * (m - s)) * std::conj(W[s]));
  if (m % 2 == 0) V.set(e - 1, root(2 * q, -(int64_t)r) * W[e - 1]);
}
// forwardInnerH
static void forwardInnerH(const Params& P, const cd* fs, size_t v, double* Vout) {
  const int64_t L = P.L, m = P.m, q = P.q, qm = P.q * P.m;
  const int64_t Ht = cq(L, 2), e = m / 2 + 1, ph = cq(L, 2 * m), n = q / ph;
  const int64_t m0 = std::min<int64_t>(ph * m - Ht + 1, e);
  In f{fs, (size_t)Ht};
  std::vector<cd> W(ph * e, 0.0);
  for (int64_t s = 0; s < m0; ++s) W[s] = f[s];
  for (int64_t t = 0; t < ph; ++t)
    for (int64_t s = (t == 0 ? m0 : 0); s < e; ++s)
      W[t * e + s] = root(q, (int64_t)v * (t - ph)) * std::conj(f[(ph - t) * m - s]) + root(q, (int64_t)v * t) * f[t * m + s];
  std::vector<cd> col(ph), ocol(ph);
  for (int64_t s = 0; s < e; ++s) {
    for (int64_t t = 0; t < ph; ++t) col[t] = W[t * e + s];
    fft(col.data(), ocol.data(), ph, +1);
    for (int64_t u = 0; u < ph; ++u) W[u * e + s] = ocol[u];
  }
  for (int64_t u = 0; u < ph; ++u) {
    for (int64_t s = 1; s < e; ++s) W[u * e + s] *= root(qm, (u * n + (int64_t)v) * s);
    crfft(W.data() + u * e, Vout + u * m, m);
  }
}
// backwardInnerH, PAPER.md:1282-1316 (even-m loop t < p/2, erratum at :1312)
static void backwardInnerH(const Params& P, const double* F, size_t v, cd* Vs) {
  const int64_t L = P.L, m = P.m, q = P.q, qm = P.q * P.m;
  const int64_t Ht = cq(L, 2), e = m / 2 + 1, ph = cq(L, 2 * m), n = q / ph;
  const int64_t m0 = std::min<int64_t>(ph * m - Ht + 1, e);
  std::vector<cd> W(ph * e);
  for (int64_t u = 0; u < ph; ++u) {
    rcfft(F + u * m, W.data() + u * e, m);
    for (int64_t s = 1; s < e; ++s) W[u * e + s] *= root(qm, -(u * n + (int64_t)v) * s);
  }
  std::vector<cd> col(ph), ocol(ph);
  for (int64_t s = 0; s < e; ++s) {
    for (int64_t u = 0; u < ph; ++u) col[u] = W[u * e + s];
    fft(col.data(), ocol.data(), ph, -1);
    for (int64_t t = 0; t < ph; ++t) W[t * e + s] = ocol[t];
  }
  Out V{Vs, (size_t)Ht};
  for (int64_t s = 1; s < m0; ++s) V.set(s, W[s]);
  for (int64_t t = 0; t < ph; ++t) {
    V.set(t * m, root(q, -(int64_t)v * t) * W[t * e]);
    for (int64_t s = (t == 0 ? m0 - 1 : 0) + 1; s <= m - e; ++s) {
      V.set(t * m + s, root(q, -(int64_t)v * t) * W[t * e + s]);
      V.set((ph - t) * m - s, root(q, -(int64_t)v * (ph - t)) * std::conj(W[t * e + s]));
    }
  }
  if (m % 2 == 0)
    for (int64_t t = 0; t < ph; ++t) V.set(t * m + e - 1, root(q, -(int64_t)v * t) * W[e * (t + 1) - 1]);
}

// ---- dispatch (Alg. convolve / convolveX kernel selection)
// Complex data in cd; Hermitian spectral blocks are real and carried in cd.real().
static void forward(const Params& P, const cd* f, size_t r, cd* F) {
  const size_t bl = block_len(P);
  if (P.sym == HCONV_COMPLEX) {
    if (P.regime == HCONV_P1) forward1(P, f, r, F);
    else if (P.regime == HCONV_P2) forward2(P, f, r, F);
    else forwardInner(P, f, r, F);
  } else if (P.sym == HCONV_CENTERED) {
    if (P.regime == HCONV_P2) forward2C(P, f, r, F); else forwardInnerC(P, f, r, F);
  } else {
    std::vector<double> R(bl);
    if (P.regime == HCONV_P2) forward2H(P, f, r, R.data()); else forwardInnerH(P, f, r, R.data());
    for (size_t i = 0; i < bl; ++i) F[i] = cd(R[i], 0.0);
  }
}
// returns the residue contribution on the stored window (length stored_len)
static void backward(const Params& P, const cd* F, size_t r, cd* V) {
  const size_t bl = block_len(P);
  std::fill(V, V + stored_len(P), cd(0));
  if (P.sym == HCONV_COMPLEX) {
    if (P.regime == HCONV_P1) backward1(P, F, r, V);
    else if (P.regime == HCONV_P2) backward2(P, F, r, V);
    else backwardInner(P, F, r, V);
  } else if (P.sym == HCONV_CENTERED) {
    if (P.regime == HCONV_P2) backward2C(P, F, r, V); else backwardInnerC(P, F, r, V);
  } else {
    std::vector<double> R(bl);
    for (size_t i = 0; i < bl; ++i) R[i] = F[i].real();
    if (P.regime == HCONV_P2) backward2H(P, R.data(), r, V); else backwardInnerH(P, R.data(), r, V);
  }
}

// blocks v and n-v from one Re/Im split (complex inner form).
static void forward_conjugate_pair(const Params& P, const cd* f, size_t v, cd* Fv, cd* Fnv) {
  const size_t L = P.L, m = P.m, q = P.q, p = P.p, n = P.n, qm = q * m;
  if (v == 0 || 2 * v == n) throw std::invalid_argument("forward_conjugate_pair: self-paired residue");
  std::vector<cd> Wa(p * m, 0.0), Wb(p * m, 0.0);
  for (size_t t = 0; t < p; ++t)
    for (size_t s = 0; s < m; ++s) {
      const size_t j = t * m + s;
      if (j >= L) continue;
      Wa[j] = root(q, (int64_t)(v * t)) * f[j].real();              // A_{s,t,v}
      Wb[j] = cd(0, 1) * root(q, (int64_t)(v * t)) * f[j].imag();   // B_{s,t,v}
    }
  std::vector<cd> c1(p), c2(p), o1(p), o2(p), W1(p * m), W2(p * m);
  for (size_t s = 0; s < m; ++s) {
    for (size_t t = 0; t < p; ++t) {
      c1[t] = Wa[t * m + s] + Wb[t * m + s];
      c2[t] = std::conj(Wa[t * m + s]) - std::conj(Wb[t * m + s]);
    }
    fft(c1.data(), o1.data(), p, +1);
    fft(c2.data(), o2.data(), p, +1);
    for (size_t u = 0; u < p; ++u) { W1[u * m + s] = o1[u]; W2[u * m + s] = o2[u]; }
  }
  for (size_t u = 0; u < p; ++u) {
    for (size_t s = 0; s < m; ++s) {
      W1[u * m + s] *= root(qm, (int64_t)((u * n + v) * s));
      W2[u * m + s] *= root(qm, (int64_t)(u * n) * (int64_t)s - (int64_t)(v * s));
    }
    fft(W1.data() + u * m, Fv + u * m, m, +1);
    fft(W2.data() + u * m, Fnv + u * m, m, +1);
  }
}

// ------------------------------------------------------------- drivers ------
// MultOperator: builtin_mult_product(A) or a user callback
// (include/hconv.h hconv_mult_fn), applied in place to the max(A, B) transformed blocks F[i] of
// one residue.  Hermitian residues are real: the callback
// sees float64 values.
struct Mult {
  size_t A = 2, B = 1;
  int kind = HCONV_MULT_PRODUCT;
  hconv_mult_fn fn = nullptr;
  void* user = nullptr;
  size_t W() const { return std::max(A, B); }
};
static void apply_mult(const Mult& mu, bool real, std::vector<std::vector<cd>>& F, size_t bl) {
  if (mu.kind == HCONV_MULT_PRODUCT) {
    for (size_t a = 1; a < mu.A; ++a) {
      if (real)
        for (size_t i = 0; i < bl; ++i) F[0][i] = cd(F[0][i].real() * F[a][i].real(), 0.0);
      else
        for (size_t i = 0; i < bl; ++i) F[0][i] *= F[a][i];
    }
    return;
  }
  std::vector<void*> ptrs(mu.W());
  std::vector<std::vector<double>> R;
  if (real) {
    R.assign(mu.W(), std::vector<double>(bl, 0.0));
    for (size_t a = 0; a < mu.A; ++a)
      for (size_t i = 0; i < bl; ++i) R[a][i] = F[a][i].real();
    for (size_t w = 0; w < mu.W(); ++w) ptrs[w] = R[w].data();
  } else {
    for (size_t w = 0; w < mu.W(); ++w) ptrs[w] = F[w].data();
  }
  const int rc = mu.fn(ptrs.data(), mu.A, mu.B, bl, real ? 1 : 0, mu.user, nullptr);
  if (rc != 0) throw std::invalid_argument("multiplication operator callback returned " + std::to_string(rc));
  if (real)
    for (size_t b = 0; b < mu.B; ++b)
      for (size_t i = 0; i < bl; ++i) F[b][i] = cd(R[b][i], 0.0);
}

// Alg. convolve / convolveX: the A forward transforms of each residue,
// mult, the B backward transforms accumulated into h_b, then f_b <- h_b / (qm).
// in[a]: stored-length sequences; out[b] (stored length) may alias in[b].
static void conv1d(const Params& P, const Mult& mu, const cd* const* in, cd* const* out) {
  const size_t bl = block_len(P), Ls = stored_len(P), qm = P.q * P.m;
  std::vector<std::vector<cd>> h(mu.B, std::vector<cd>(Ls, 0.0)), F(mu.W(), std::vector<cd>(bl));
  std::vector<cd> V(Ls);
  for (size_t r = 0; r < P.n; ++r) {
    for (size_t a = 0; a < mu.A; ++a) forward(P, in[a], r, F[a].data());
    apply_mult(mu, P.sym == HCONV_HERMITIAN, F, bl);
    for (size_t b = 0; b < mu.B; ++b) {
      backward(P, F[b].data(), r, V.data());
      for (size_t j = 0; j < Ls; ++j) h[b][j] += V[j];
    }
  }
  const double s = 1.0 / (double)qm;
  for (size_t b = 0; b < mu.B; ++b)
    for (size_t j = 0; j < Ls; ++j) out[b][j] = h[b][j] * s;
}

struct AxisP {
  Params P;
  size_t stored;
};

// convolve_nd: for each outer residue, forward the outer axis on every
// inner column, convolve each spectral line recursively, inverse the outer axis and accumulate.
// arrays are row-major with extents stored[level..d-1].
static void convnd_rec(const std::vector<AxisP>& ax, size_t level, const Mult& mu, const std::vector<const cd*>& in,
                       const std::vector<cd*>& out, bool parallel) {
  const size_t d = ax.size(), A = mu.A, Bo = mu.B;
  if (level == d - 1) { conv1d(ax[level].P, mu, in.data(), out.data()); return; }
  const Params& P = ax[level].P;
  const size_t Lx = ax[level].stored, bl = block_len(P), qm = P.q * P.m;
  size_t inner = 1;
  for (size_t k = level + 1; k < d; ++k) inner *= ax[k].stored;
  std::vector<std::vector<cd>> h(Bo, std::vector<cd>(Lx * inner, 0.0));
  std::vector<std::vector<cd>> F(A, std::vector<cd>(bl * inner));
  std::vector<std::vector<cd>> R(Bo, std::vector<cd>(bl * inner));
  for (size_t r = 0; r < P.n; ++r) {
    for (size_t a = 0; a < A; ++a) {
#pragma omp parallel for schedule(dynamic, 16) if (parallel)
      for (size_t c = 0; c < inner; ++c) {
        std::vector<cd> col(Lx), Fc(bl);
        for (size_t x = 0; x < Lx; ++x) col[x] = in[a][x * inner + c];
        forward(P, col.data(), r, Fc.data());
        for (size_t l = 0; l < bl; ++l) F[a][l * inner + c] = Fc[l];
      }
    }
#pragma omp parallel for schedule(dynamic, 1) if (parallel)
    for (size_t l = 0; l < bl; ++l) {
      std::vector<const cd*> sub(A);
      std::vector<cd*> subo(Bo);
      for (size_t a = 0; a < A; ++a) sub[a] = F[a].data() + l * inner;
      for (size_t b = 0; b < Bo; ++b) subo[b] = R[b].data() + l * inner;
      convnd_rec(ax, level + 1, mu, sub, subo, false);
    }
    for (size_t b = 0; b < Bo; ++b) {
#pragma omp parallel for schedule(dynamic, 16) if (parallel)
      for (size_t c = 0; c < inner; ++c) {
        std::vector<cd> Fc(bl), V(Lx);
        for (size_t l = 0; l < bl; ++l) Fc[l] = R[b][l * inner + c];
        backward(P, Fc.data(), r, V.data());
        for (size_t x = 0; x < Lx; ++x) h[b][x * inner + c] += V[x];
      }
    }
  }
  const double s = 1.0 / (double)qm;
  for (size_t b = 0; b < Bo; ++b)
    for (size_t i = 0; i < Lx * inner; ++i) out[b][i] = h[b][i] * s;
}

// ---------------------------------------------------- brute-force oracles ---
// Logical index window of a stored axis.
struct Win { int64_t lo, n; };  // stored index i <-> logical lo + i
static Win window(int sym, size_t L) {
  if (sym == HCONV_COMPLEX) return {0, (int64_t)L};
  if (sym == HCONV_CENTERED) return {-(int64_t)(L / 2), (int64_t)L};
  return {0, (int64_t)cq(L, 2)};
}
// direct_convolution: exact nested-sum linear convolution of the A=2
// inputs, on logical indices (Hermitian axes symmetrised jointly), truncated to the stored
// window.  dims <= 3, syms[k] per axis, L[k] logical lengths.
static void direct_conv(int dims, const int* syms, const size_t* Ls, const cd* f, const cd* g, cd* out) {
  // full logical extents
  int64_t lo[3] = {0, 0, 0}, n[3] = {1, 1, 1}, sn[3] = {1, 1, 1};
  bool herm = false;
  for (int k = 0; k < dims; ++k) {
    Win w = window(syms[k], Ls[k]);
    sn[k] = w.n;
    if (syms[k] == HCONV_HERMITIAN) { herm = true; lo[k] = -(w.n - 1); n[k] = 2 * w.n - 1; }
    else { lo[k] = w.lo; n[k] = w.n; }
  }
  const int64_t tot = n[0] * n[1] * n[2];
  std::vector<cd> F(tot, 0.0), G(tot, 0.0);
  auto lin = [&](int64_t a, int64_t b, int64_t c) { return (a * n[1] + b) * n[2] + c; };
  auto slin = [&](int64_t a, int64_t b, int64_t c) { return (a * sn[1] + b) * sn[2] + c; };
  const int64_t D0 = dims > 0 ? 1 : 0; (void)D0;
  // embed stored values
  for (int64_t i0 = 0; i0 < sn[0]; ++i0)
    for (int64_t i1 = 0; i1 < sn[1]; ++i1)
      for (int64_t i2 = 0; i2 < sn[2]; ++i2) {
        int64_t s[3] = {i0, i1, i2};
        int64_t idx[3];
        for (int k = 0; k < 3; ++k) {
          const Win w = k < dims ? window(syms[k], Ls[k]) : Win{0, 1};
          idx[k] = w.lo + s[k] - lo[k];
        }
        F[lin(idx[0], idx[1], idx[2])] = f[slin(i0, i1, i2)];
        G[lin(idx[0], idx[1], idx[2])] = g[slin(i0, i1, i2)];
      }
  if (herm) {  // f(-x) = conj f(x) for the points not stored (innermost Hermitian axis < 0)
    for (int64_t a = 0; a < n[0]; ++a)
      for (int64_t b = 0; b < n[1]; ++b)
        for (int64_t c = 0; c < n[2]; ++c) {
          int64_t x[3] = {lo[0] + a, lo[1] + b, lo[2] + c};
          const int ki = dims - 1;
          if (x[ki] >= 0) continue;
          int64_t y[3], ok = 1;
          for (int k = 0; k < 3; ++k) {
            y[k] = (k < dims ? -x[k] : x[k]) - lo[k];
            if (y[k] < 0 || y[k] >= n[k]) ok = 0;
          }
          if (ok) {
            F[lin(a, b, c)] = std::conj(F[lin(y[0], y[1], y[2])]);
            G[lin(a, b, c)] = std::conj(G[lin(y[0], y[1], y[2])]);
          }
        }
  }
  // output on the stored window
  for (int64_t o0 = 0; o0 < sn[0]; ++o0)
    for (int64_t o1 = 0; o1 < sn[1]; ++o1)
      for (int64_t o2 = 0; o2 < sn[2]; ++o2) {
        int64_t o[3] = {o0, o1, o2}, kx[3];
        for (int k = 0; k < 3; ++k) {
          const Win w = k < dims ? window(syms[k], Ls[k]) : Win{0, 1};
          kx[k] = w.lo + o[k];  // logical output index
        }
        cd acc = 0;
        for (int64_t a = 0; a < n[0]; ++a) {
          const int64_t j0 = kx[0] - (lo[0] + a) - lo[0];
          if (j0 < 0 || j0 >= n[0]) continue;
          for (int64_t b = 0; b < n[1]; ++b) {
            const int64_t j1 = kx[1] - (lo[1] + b) - lo[1];
            if (j1 < 0 || j1 >= n[1]) continue;
            for (int64_t c = 0; c < n[2]; ++c) {
              const int64_t j2 = kx[2] - (lo[2] + c) - lo[2];
              if (j2 < 0 || j2 >= n[2]) continue;
              acc += F[lin(a, b, c)] * G[lin(j0, j1, j2)];
            }
          }
        }
        out[slin(o0, o1, o2)] = acc;
      }
}

// padded_dft_slice: naive qm-point DFT of the (zero-padded / centered /
// symmetrised) input, sliced by k = q*l + u*n + r.  Output layout as forward().
static void padded_dft_slice(const Params& P, const cd* f, size_t r, cd* F) {
  const size_t qm = P.q * P.m, bl = block_len(P);
  const Win w = window(P.sym, P.L);
  const size_t nblk = (P.regime == HCONV_INNER) ? (P.sym == HCONV_COMPLEX ? P.p : P.p / 2) : 1;
  for (size_t u = 0; u < nblk; ++u)
    for (size_t l = 0; l < P.m; ++l) {
      const size_t k = P.q * l + u * P.n + r;
      cd acc = 0;
      if (P.sym == HCONV_HERMITIAN) {
        for (int64_t j = -(w.n - 1); j <= w.n - 1; ++j) {
          const cd v = j >= 0 ? f[j] : std::conj(f[-j]);
          acc += root(qm, (int64_t)((k % qm)) * j) * v;
        }
      } else {
        for (int64_t i = 0; i < w.n; ++i) acc += root(qm, (int64_t)(k % qm) * (w.lo + i)) * f[i];
      }
      F[u * P.m + l] = P.sym == HCONV_HERMITIAN ? cd(acc.real(), 0.0) : acc;
    }
  (void)bl;
}

// enforce f(-x,-y,0) = conj f(x,y,0) on the innermost-index-0 hyperplane
// of a [Lx][Ly][Kz] (or [Lx][Kz]) centered/centered/Hermitian array.
static void symmetrize_boundary(int dims, const size_t* Ls, cd* f) {
  const size_t Kz = cq(Ls[dims - 1], 2);
  if (dims == 2) {
    const int64_t Lx = Ls[0], Hx = Lx / 2;
    for (int64_t x = -Hx; x < Lx - Hx; ++x) {
      const int64_t xm = -x;
      if (xm < -Hx || xm >= Lx - Hx) { f[(x + Hx) * Kz] = 0; continue; }
      if (x < 0) f[(x + Hx) * Kz] = std::conj(f[(xm + Hx) * Kz]);
      if (x == 0) f[Hx * Kz] = cd(f[Hx * Kz].real(), 0.0);
    }
    return;
  }
  const int64_t Lx = Ls[0], Ly = Ls[1], Hx = Lx / 2, Hy = Ly / 2;
  auto at = [&](int64_t x, int64_t y) -> cd& { return f[((x + Hx) * Ly + (y + Hy)) * Kz]; };
  for (int64_t x = -Hx; x < Lx - Hx; ++x)
    for (int64_t y = -Hy; y < Ly - Hy; ++y) {
      const int64_t xm = -x, ym = -y;
      const bool in = xm >= -Hx && xm < Lx - Hx && ym >= -Hy && ym < Ly - Hy;
      if (!in) { at(x, y) = 0; continue; }
      if (y < 0 || (y == 0 && x < 0)) at(x, y) = std::conj(at(xm, ym));
      if (x == 0 && y == 0) at(0, 0) = cd(at(0, 0).real(), 0.0);
    }
}

}  // namespace orc

// ------------------------------------------------------------ C ABI ---------
using namespace orc;

template <class F>
static hconv_status guarded(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return HCONV_INVALID_ARG;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HCONV_INTERNAL;
  }
  return HCONV_OK;
}

static void to_abi(const Params& P, hconv_params* o) {
  o->L = P.L; o->M = P.M; o->m = P.m; o->p = P.p; o->q = P.q; o->n = P.n;
  o->D = 1; o->C = 1; o->S = 1; o->inplace = 0; o->symmetry = P.sym; o->regime = P.regime;
}

extern "C" {

const char* hconv_backend(void) { return "oracle-cpu"; }
const char* hconv_last_error(void) { return g_err.c_str(); }

hconv_status hconv_derive_params(size_t L, size_t M, size_t m, int sym, hconv_params* out) {
  if (!out) { g_err = "null output"; return HCONV_INVALID_ARG; }
  return guarded([&] { to_abi(derive(L, M, m, sym), out); });
}
size_t hconv_block_length(const hconv_params* pp) {
  try { return block_len(from_abi(pp)); } catch (...) { return 0; }
}
// plan.cpp:31-33 (the reference's storage convention; the data convolved per copy is
// stored_len() = ceil(L/2) values for Hermitian data, the extra entry lies outside the support)
size_t hconv_stored_length(const hconv_params* pp) {
  try {
    const Params P = from_abi(pp);
    return P.sym == HCONV_HERMITIAN ? cq(P.L, 2) + 1 : P.L;
  } catch (...) { return 0; }
}
size_t hconv_padded_length(const hconv_params* pp) { return pp->q * pp->m; }
hconv_status hconv_root(size_t N, int64_t k, double* re, double* im) {
  return guarded([&] {
    cd z = root(N, k);
    *re = z.real(); *im = z.imag();
  });
}
hconv_status hconv_work_memory_words(const hconv_params* pp, size_t A, size_t B, size_t d, size_t L,
                                     uint64_t* iw, double* ew) {
  if (A == 0 || B == 0) { g_err = "workMemoryWords: A and B must be positive"; return HCONV_INVALID_ARG; }
  if (d < 1 || d > 3) { g_err = "workMemoryWords: d must be 1, 2, or 3"; return HCONV_INVALID_ARG; }
  uint64_t imp = (uint64_t)(A + B) * pp->p * pp->m;
  for (size_t i = 1; i < d; ++i) imp *= L;
  double ex = (double)std::max(A, B);
  for (size_t i = 0; i < d; ++i) ex *= (double)pp->q / (double)pp->p * (double)L;
  *iw = imp; *ew = ex;
  return HCONV_OK;
}
hconv_status hconv_root_table(size_t N, double* out) {
  return guarded([&] {
    Roots t(N);
    for (size_t k = 0; k < N; ++k) { out[2 * k] = t.z[k].real(); out[2 * k + 1] = t.z[k].imag(); }
  });
}
const char* hconv_symmetry_name(int s) {
  switch (s) { case HCONV_COMPLEX: return "complex"; case HCONV_CENTERED: return "centered"; case HCONV_HERMITIAN: return "hermitian"; }
  return "?";
}
hconv_status hconv_symmetry_from_name(const char* n, int* s) {
  std::string x(n ? n : "");
  if (x == "complex") *s = HCONV_COMPLEX;
  else if (x == "centered") *s = HCONV_CENTERED;
  else if (x == "hermitian") *s = HCONV_HERMITIAN;
  else { g_err = "unknown symmetry: " + x; return HCONV_INVALID_ARG; }
  return HCONV_OK;
}

hconv_status hconv_pfft_forward(const hconv_params* pp, const void* f, size_t dist, size_t residue, void* F,
                                void* /*stream*/) {
  return guarded([&] {
    Params P = from_abi(pp);
    if (residue >= P.n) throw std::invalid_argument("residue out of range");
    const size_t Ls = stored_len(P), bl = block_len(P), C = pp->C ? pp->C : 1, S = pp->S ? pp->S : 1;
    const cd* fin = (const cd*)f;
#pragma omp parallel for schedule(dynamic, 4)
    for (size_t c = 0; c < C; ++c) {
      std::vector<cd> x(Ls), y(bl);
      for (size_t j = 0; j < Ls; ++j) x[j] = fin[c * dist + j * S];
      forward(P, x.data(), residue, y.data());
      if (P.sym == HCONV_HERMITIAN) {
        double* o = (double*)F + c * bl;
        for (size_t i = 0; i < bl; ++i) o[i] = y[i].real();
      } else {
        std::copy(y.begin(), y.end(), (cd*)F + c * bl);
      }
    }
  });
}
hconv_status hconv_pfft_backward(const hconv_params* pp, const void* F, size_t residue, void* h, size_t dist,
                                 int accumulate, void* /*stream*/) {
  return guarded([&] {
    Params P = from_abi(pp);
    if (residue >= P.n) throw std::invalid_argument("residue out of range");
    const size_t Ls = stored_len(P), bl = block_len(P), C = pp->C ? pp->C : 1, S = pp->S ? pp->S : 1;
    cd* hout = (cd*)h;
#pragma omp parallel for schedule(dynamic, 4)
    for (size_t c = 0; c < C; ++c) {
      std::vector<cd> x(bl), V(Ls);
      if (P.sym == HCONV_HERMITIAN) {
        const double* in = (const double*)F + c * bl;
        for (size_t i = 0; i < bl; ++i) x[i] = in[i];
      } else {
        std::copy((const cd*)F + c * bl, (const cd*)F + (c + 1) * bl, x.begin());
      }
      backward(P, x.data(), residue, V.data());
      for (size_t j = 0; j < Ls; ++j) {
        cd& o = hout[c * dist + j * S];
        o = accumulate ? o + V[j] : V[j];
      }
    }
  });
}

// two-level line batches (include/hconv.h hconv_lines): line l starts at
// (l / nin) * d_out + (l % nin) * d_in, values at stride es
hconv_status hconv_pfft_forward_pair(const hconv_params* pp, const void* f, size_t dist, size_t residue, void* Fv,
                                     void* Fnv, void* /*stream*/) {
  return guarded([&] {
    Params P = from_abi(pp);
    if (P.sym != HCONV_COMPLEX) throw std::runtime_error("forward_conjugate_pair: complex data only");
    if (residue >= P.n) throw std::invalid_argument("residue out of range");
    const size_t Ls = stored_len(P), bl = block_len(P), C = pp->C;
    for (size_t c = 0; c < C; ++c) {
      std::vector<cd> x(Ls);
      for (size_t j = 0; j < Ls; ++j) x[j] = ((const cd*)f)[c * dist + j * pp->S];
      forward_conjugate_pair(P, x.data(), residue, (cd*)Fv + c * bl, (cd*)Fnv + c * bl);
    }
  });
}
static size_t line_base(const hconv_lines& L, size_t l) { return (l / L.nin) * L.d_out + (l % L.nin) * L.d_in; }
static void check_lines(const hconv_lines* a, const hconv_lines* b) {
  if (!a || !b) throw std::invalid_argument("null line batch");
  if (a->nin == 0 || a->es == 0 || b->nin == 0 || b->es == 0) throw std::invalid_argument("line batch: nin and es must be positive");
  if (a->count != b->count) throw std::invalid_argument("line batches differ in count");
}
// natural block order of the CUDA library: the block in the kernels' order.  The oracle's blocks
// are in the reference order F[u m + l]; for p <= 2 (one chunk) the two coincide, and the
// drivers that use the _lines entry points only need a pointwise-consistent order between the
// forward and the backward of the same residue, which the oracle keeps by using its own order
// on both sides.
hconv_status hconv_pfft_forward_lines(const hconv_params* pp, const void* f, const hconv_lines* in, size_t residue,
                                      void* F, const hconv_lines* out, void* /*stream*/) {
  return guarded([&] {
    Params P = from_abi(pp);
    if (residue >= P.n) throw std::invalid_argument("residue out of range");
    check_lines(in, out);
    const size_t Ls = stored_len(P), bl = block_len(P);
#pragma omp parallel for schedule(dynamic, 4)
    for (size_t l = 0; l < in->count; ++l) {
      std::vector<cd> x(Ls), y(bl);
      const cd* src = (const cd*)f + line_base(*in, l);
      for (size_t j = 0; j < Ls; ++j) x[j] = src[j * in->es];
      forward(P, x.data(), residue, y.data());
      const size_t ob = line_base(*out, l);
      if (P.sym == HCONV_HERMITIAN)
        for (size_t i = 0; i < bl; ++i) ((double*)F)[ob + i * out->es] = y[i].real();
      else
        for (size_t i = 0; i < bl; ++i) ((cd*)F)[ob + i * out->es] = y[i];
    }
  });
}
hconv_status hconv_pfft_backward_lines(const hconv_params* pp, const void* F, const hconv_lines* in, size_t residue,
                                       void* h, const hconv_lines* out, int accumulate, double scale, void* /*stream*/) {
  return guarded([&] {
    Params P = from_abi(pp);
    if (residue >= P.n) throw std::invalid_argument("residue out of range");
    check_lines(in, out);
    const size_t Ls = stored_len(P), bl = block_len(P);
#pragma omp parallel for schedule(dynamic, 4)
    for (size_t l = 0; l < in->count; ++l) {
      std::vector<cd> x(bl), V(Ls);
      const size_t ib = line_base(*in, l);
      for (size_t i = 0; i < bl; ++i)
        x[i] = P.sym == HCONV_HERMITIAN ? cd(((const double*)F)[ib + i * in->es], 0.0) : ((const cd*)F)[ib + i * in->es];
      backward(P, x.data(), residue, V.data());
      cd* dst = (cd*)h + line_base(*out, l);
      for (size_t j = 0; j < Ls; ++j) {
        cd& o = dst[j * out->es];
        o = ((accumulate ? o : cd(0.0)) + V[j]) * scale;
      }
    }
  });
}

struct OracleSlab;
struct OracleSlabDel {
  void operator()(OracleSlab* s) const;
};
struct hconv_plan {
  hconv_desc d;
  std::vector<AxisP> ax;
  std::unique_ptr<OracleSlab, OracleSlabDel> slab;
};

// ---- x-slab decomposition (hconv_desc.slab): the product's driver (slab.hpp) over host buffers
// and the oracle's padded FFTs, so the CPU tests (gloo, several processes) check the product's
// index arithmetic and schedule against the oracle's own single-process convolve_nd.  The
// reference has no distributed code; nothing here restates it.
struct OracleSlabOps {
  OracleSlab* st = nullptr;
  void* alloc(size_t elems) { return new cd[elems](); }
  void free(void* p) { delete[] (cd*)p; }
  void fwd(size_t r, const void* f, void* F);
  void bwd(size_t r, const void* W, void* h, bool acc, double scale);
  void inner(size_t count, void* const* T);
  void copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows, bool) {
    for (size_t i = 0; i < rows; ++i) std::copy((const cd*)src + i * spitch, (const cd*)src + i * spitch + width, (cd*)dst + i * dpitch);
  }
  void exchange(const void* send, const size_t* sc, const size_t* sd, void* recv, const size_t* rc, const size_t* rd);
  void comm_after_compute() {}
  void mark_comm(size_t) {}
  void compute_after_comm(size_t) {}
};
struct OracleSlab {
  hconv_slab cfg{};
  hslab::Geometry g;
  hconv_params py{};
  hconv_plan* inner = nullptr;
  OracleSlabOps ops;
  std::unique_ptr<hslab::Driver<OracleSlabOps>> drv;
  ~OracleSlab();
};
static void slab_check(hconv_status st, const char* what) {
  if (st != HCONV_OK) throw std::invalid_argument(std::string(what) + ": " + g_err);
}
void OracleSlabOps::fwd(size_t r, const void* f, void* F) {
  const hslab::Geometry& g = st->g;
  const size_t nxz = g.nx() * g.Z;
  const hconv_lines lin{nxz, g.Z, g.Ly * g.Z, 1, g.Z}, lspec{nxz, nxz, 0, 1, nxz};
  if (nxz) slab_check(hconv_pfft_forward_lines(&st->py, f, &lin, r, F, &lspec, nullptr), "slab forward");
}
void OracleSlabOps::bwd(size_t r, const void* W, void* h, bool acc, double scale) {
  const hslab::Geometry& g = st->g;
  const size_t nxz = g.nx() * g.Z;
  const hconv_lines lin{nxz, g.Z, g.Ly * g.Z, 1, g.Z}, lspec{nxz, nxz, 0, 1, nxz};
  if (nxz) slab_check(hconv_pfft_backward_lines(&st->py, W, &lspec, r, h, &lin, acc ? 1 : 0, scale, nullptr), "slab backward");
}
void OracleSlabOps::inner(size_t count, void* const* T) {
  hconv_plan* P = st->inner;
  const size_t keep = P->d.C;
  P->d.C = count;
  const hconv_status rc = hconv_convolve(P, (const void* const*)T, T, nullptr);
  P->d.C = keep;
  slab_check(rc, "slab subconvolution");
}
void OracleSlabOps::exchange(const void* send, const size_t* sc, const size_t* sd, void* recv, const size_t* rc,
                             const size_t* rd) {
  const hslab::Geometry& g = st->g;
  if (!st->cfg.exchange) {  // one rank: the only segment is its own
    std::copy((const cd*)send + sd[0], (const cd*)send + sd[0] + sc[0], (cd*)recv + rd[0]);
    return;
  }
  (void)g;
  const int r = st->cfg.exchange(send, sc, sd, recv, rc, rd, st->cfg.exchange_user, nullptr);
  if (r != 0) throw std::runtime_error("slab exchange callback returned " + std::to_string(r));
}
OracleSlab::~OracleSlab() {
  drv.reset();
  if (inner) hconv_plan_destroy(inner);
}
void OracleSlabDel::operator()(OracleSlab* s) const { delete s; }

static void build_slab(hconv_plan* p) {
  const hconv_desc* desc = &p->d;
  const hconv_slab& cfg = *desc->slab;
  const int d = desc->dims;
  if (d < 2) throw std::invalid_argument("slab decomposition is for 2D and 3D convolutions");
  if (d == 2 && p->ax[1].P.sym == HCONV_HERMITIAN) throw std::invalid_argument("2D Hermitian slabs are not supported");
  if (desc->C > 1) throw std::invalid_argument("slab plans convolve one global array (C must be 0 or 1)");
  if (cfg.nranks < 1 || cfg.rank < 0 || cfg.rank >= cfg.nranks) throw std::invalid_argument("slab: bad rank / nranks");
  if (cfg.nranks > 1 && !cfg.exchange) throw std::invalid_argument("the oracle exchanges through the callback only");
  for (int k = 0; k < d; ++k)
    if (desc->axis[k].m == 0) throw std::invalid_argument("slab plans need every m (tune on one rank, broadcast)");
  auto st = std::unique_ptr<OracleSlab, OracleSlabDel>(new OracleSlab());
  st->cfg = cfg;
  to_abi(p->ax[1].P, &st->py);
  const Params& Py = p->ax[1].P;
  st->g = hslab::make_geometry(cfg.rank, cfg.nranks, p->ax[0].stored, p->ax[1].stored, d == 3 ? p->ax[2].stored : 1,
                               block_len(Py), Py.n, 1.0 / (double)(Py.q * Py.m), cfg.chunks);
  hconv_desc in{};
  in.dims = d - 1;
  in.axis[0] = desc->axis[0];
  in.axis[0].symmetry = p->ax[0].P.sym;
  if (d == 3) {
    in.axis[1] = desc->axis[2];
    in.axis[1].symmetry = p->ax[2].P.sym;
  }
  in.A = desc->A;
  in.B = desc->B;
  in.mult = desc->mult;
  in.C = std::max<size_t>(1, st->g.max_chunk());
  in.mult_fn = desc->mult_fn;
  in.mult_user = desc->mult_user;
  slab_check(hconv_plan_create(&in, &st->inner), "slab inner plan");
  st->ops.st = st.get();
  st->drv = std::make_unique<hslab::Driver<OracleSlabOps>>(st->g, desc->A, desc->B, st->ops);
  p->slab = std::move(st);
  p->d.slab = nullptr;
}
static void slab_convolve(hconv_plan* p, const void* const* in, void* const* out) {
  OracleSlab& S = *p->slab;
  const size_t n = S.g.nx() * S.g.Ly * S.g.Z;
  std::vector<std::vector<cd>> acc(p->d.B, std::vector<cd>(std::max<size_t>(1, n)));
  std::vector<void*> ap(p->d.B);
  for (size_t b = 0; b < p->d.B; ++b) ap[b] = acc[b].data();
  S.drv->run(in, ap.data());
  for (size_t b = 0; b < p->d.B; ++b) std::copy(acc[b].begin(), acc[b].begin() + n, (cd*)out[b]);
}

hconv_status hconv_plan_create(const hconv_desc* desc, hconv_plan** out) {
  return guarded([&] {
    if (!desc || !out) throw std::invalid_argument("null argument");
    if (desc->dims < 1 || desc->dims > 3) throw std::invalid_argument("dims must be 1, 2 or 3");
    if (desc->mult == HCONV_MULT_PRODUCT) {
      if (desc->A < 2 || desc->B != 1) throw std::invalid_argument("builtin_mult_product needs A >= 2 and B == 1");
    } else if (desc->mult == HCONV_MULT_CALLBACK) {
      if (!desc->mult_fn) throw std::invalid_argument("HCONV_MULT_CALLBACK without mult_fn");
      if (desc->A < 1 || desc->B < 1) throw std::invalid_argument("multiplication operator arity: A >= 1, B >= 1");
    } else {
      throw std::invalid_argument("unknown multiplication operator");
    }
    auto* p = new hconv_plan();
    p->d = *desc;
    const bool herm = desc->axis[desc->dims - 1].symmetry == HCONV_HERMITIAN;
    for (int k = 0; k < desc->dims; ++k) {
      hconv_axis a = desc->axis[k];
      int sym = a.symmetry;
      if (herm && k < desc->dims - 1) sym = HCONV_CENTERED;
      size_t m = a.m;
      if (m == 0) m = a.M;  // oracle has no timer: explicit candidate
      AxisP ap{derive(a.L, a.M, m, sym), 0};
      ap.stored = stored_len(ap.P);
      p->ax.push_back(ap);
    }
    if (desc->dims == 1 && desc->dist != 0 && desc->dist < p->ax[0].stored) {
      delete p;
      throw std::invalid_argument("dist smaller than the data length: copies would overlap");
    }
    if (desc->slab) {
      try {
        build_slab(p);
      } catch (...) {
        delete p;
        throw;
      }
    }
    *out = p;
  });
}
hconv_status hconv_plan_params(const hconv_plan* p, int axis, hconv_params* o) {
  if (!p || axis < 0 || axis >= (int)p->ax.size()) { g_err = "bad axis"; return HCONV_INVALID_ARG; }
  to_abi(p->ax[axis].P, o);
  return HCONV_OK;
}
size_t hconv_plan_workspace_bytes(const hconv_plan*) { return 0; }
hconv_status hconv_plan_slab(const hconv_plan* p, size_t* x0, size_t* nx) {
  return guarded([&] {
    if (!p || !x0 || !nx) throw std::invalid_argument("null argument");
    if (!p->slab) throw std::invalid_argument("not a slab plan");
    *x0 = p->slab->g.xs[p->slab->g.rank].lo;
    *nx = p->slab->g.nx();
  });
}
hconv_status hconv_convolve(hconv_plan* p, const void* const* in, void* const* out, void* /*stream*/) {
  return guarded([&] {
    if (!p || !in || !out) throw std::invalid_argument("null argument");
    Mult mu;
    mu.A = p->d.A; mu.B = p->d.B; mu.kind = p->d.mult; mu.fn = p->d.mult_fn; mu.user = p->d.mult_user;
    const size_t A = mu.A, Bo = mu.B;
    const bool empty = p->slab && p->slab->g.nx() == 0;  // a slab rank without rows: empty arrays
    for (size_t a = 0; a < A; ++a) if (!in[a] && !empty) throw std::invalid_argument("null input array");
    for (size_t b = 0; b < Bo; ++b) if (!out[b] && !empty) throw std::invalid_argument("null output array");
    // a user callback is not assumed thread-safe: the oracle calls it from one thread
    const bool par = mu.kind == HCONV_MULT_PRODUCT;
    if (p->slab) {
      slab_convolve(p, in, out);
    } else if (p->d.dims == 1) {
      const size_t Ls = p->ax[0].stored, dist = p->d.dist ? p->d.dist : Ls, C = p->d.C ? p->d.C : 1;
      std::vector<std::vector<cd>> res(Bo, std::vector<cd>(C * Ls));
      std::string err;
#pragma omp parallel for schedule(dynamic, 1) if (par)
      for (size_t c = 0; c < C; ++c) {
        std::vector<const cd*> ins(A);
        std::vector<cd*> outs(Bo);
        for (size_t a = 0; a < A; ++a) ins[a] = (const cd*)in[a] + c * dist;
        for (size_t b = 0; b < Bo; ++b) outs[b] = res[b].data() + c * Ls;
        try {
          conv1d(p->ax[0].P, mu, ins.data(), outs.data());
        } catch (const std::exception& e) {
#pragma omp critical
          err = e.what();
        }
      }
      if (!err.empty()) throw std::invalid_argument(err);
      for (size_t b = 0; b < Bo; ++b)
        for (size_t c = 0; c < C; ++c)
          std::copy(res[b].begin() + c * Ls, res[b].begin() + (c + 1) * Ls, (cd*)out[b] + c * dist);
    } else {
      if (p->d.dist != 0) throw std::invalid_argument("N-D copies are contiguous arrays: dist must be 0");
      size_t tot = 1;
      for (auto& a : p->ax) tot *= a.stored;
      const size_t C = p->d.C ? p->d.C : 1;
      for (size_t c = 0; c < C; ++c) {  // a batch of C contiguous arrays
        std::vector<const cd*> ins(A);
        for (size_t a = 0; a < A; ++a) ins[a] = (const cd*)in[a] + c * tot;
        std::vector<std::vector<cd>> res(Bo, std::vector<cd>(tot));
        std::vector<cd*> outs(Bo);
        for (size_t b = 0; b < Bo; ++b) outs[b] = res[b].data();
        convnd_rec(p->ax, 0, mu, ins, outs, par);
        for (size_t b = 0; b < Bo; ++b) std::copy(res[b].begin(), res[b].end(), (cd*)out[b] + c * tot);
      }
    }
  });
}

// host arrays already: the oracle's convolve is synchronous on host memory
hconv_status hconv_convolve_host(hconv_plan* p, const void* const* in, void* const* out) {
  return hconv_convolve(p, in, out, nullptr);
}
hconv_status hconv_plan_destroy(hconv_plan* p) { delete p; return HCONV_OK; }

// ---- oracle-only entry points (tests and bench cpu_baseline) ----
int oracle_naive_dft(const double* x, size_t N, int sign, double* y) {
  try { naive_dft((const cd*)x, (cd*)y, N, sign); } catch (...) { return 1; }
  return 0;
}
int oracle_fft(const double* x, size_t N, int sign, double* y) {
  try { fft((const cd*)x, (cd*)y, N, sign); } catch (...) { return 1; }
  return 0;
}
int oracle_padded_dft_slice(const hconv_params* pp, const double* f, size_t r, double* F) {
  try { padded_dft_slice(from_abi(pp), (const cd*)f, r, (cd*)F); } catch (const std::exception& e) { g_err = e.what(); return 1; }
  return 0;
}
int oracle_forward(const hconv_params* pp, const double* f, size_t r, double* F) {
  try { forward(from_abi(pp), (const cd*)f, r, (cd*)F); } catch (const std::exception& e) { g_err = e.what(); return 1; }
  return 0;
}
int oracle_backward(const hconv_params* pp, const double* F, size_t r, double* V) {
  try { backward(from_abi(pp), (const cd*)F, r, (cd*)V); } catch (const std::exception& e) { g_err = e.what(); return 1; }
  return 0;
}
int oracle_forward_conjugate_pair(const hconv_params* pp, const double* f, size_t v, double* Fv, double* Fnv) {
  try { forward_conjugate_pair(from_abi(pp), (const cd*)f, v, (cd*)Fv, (cd*)Fnv); } catch (const std::exception& e) { g_err = e.what(); return 1; }
  return 0;
}
int oracle_direct_convolution(int dims, const int* syms, const size_t* Ls, const double* f, const double* g, double* out) {
  try {
    double macs = 1;  // stored outputs x full logical input points
    for (int k = 0; k < dims; ++k) macs *= (double)Ls[k] * (double)Ls[k];
    if (macs > 2e9) throw std::invalid_argument("direct_convolution: guard exceeded (SPEC.md:588)");
    direct_conv(dims, syms, Ls, (const cd*)f, (const cd*)g, (cd*)out);
  } catch (const std::exception& e) { g_err = e.what(); return 1; }
  return 0;
}
int oracle_symmetrize_boundary(int dims, const size_t* Ls, double* f) {
  try { symmetrize_boundary(dims, Ls, (cd*)f); } catch (const std::exception& e) { g_err = e.what(); return 1; }
  return 0;
}
int oracle_set_threads(int n) { if (n > 0) omp_set_num_threads(n); return omp_get_max_threads(); }

// Counter-based synthetic inputs: value = 2u - 1 with
// u = (mix(seed*phi + (a<<56 | comp<<55 | idx)) >> 11) * 2^-53, mix = splitmix64 finaliser.
static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
void oracle_fill_uniform(uint64_t seed, uint64_t a, uint64_t first_index, size_t count, double* out) {
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < count; ++i) {
    const uint64_t idx = first_index + i;
    for (uint64_t comp = 0; comp < 2; ++comp) {
      const uint64_t z = mix64(seed * 0x9E3779B97F4A7C15ull + ((a << 56) | (comp << 55) | idx));
      out[2 * i + comp] = 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
    }
  }
}

}  // extern "C"
