// plan.hpp — host plan module of the B200 path: hybrid-padding parameters, roots of unity,
// work-memory estimate.  Same contract and formulas as the reference's only compiled module
// (/root/reference/proj/include/hconv/plan.hpp:10-108, proj/src/plan.cpp:1-101); written
// from the formulas, validated against the reference compiled in oracle/_ref/.
#pragma once
#include <complex>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace hb {

using Complex = std::complex<double>;

inline size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }

enum class Symmetry { Complex = 0, Centered = 1, Hermitian = 2 };  // plan.hpp:17
enum class Regime { P1 = 0, P2 = 1, Inner = 2 };                   // plan.hpp:20

const char* name(Symmetry s);                   // plan.cpp:10-17
Symmetry symmetryFromName(const std::string&);  // plan.cpp:19-24

// plan.hpp:39-62.  q*m >= M always; n residue blocks of blockLength() values each, with
// q*m == n*blockLength() in every regime (the identity the GPU kernels are built on).
struct PlanParams {
  size_t L = 1, M = 1, m = 1, p = 1, q = 1, n = 1, D = 1, C = 1, S = 1;
  bool inplace = false;
  Symmetry symmetry = Symmetry::Complex;
  Regime regime = Regime::P1;

  size_t blockLength() const;                    // plan.cpp:26-29
  size_t paddedLength() const { return q * m; }  // plan.hpp:56
  size_t storedLength() const;                   // plan.cpp:31-33 (ceil(L/2)+1 for Hermitian)
  // values the kernels read/write per copy: L, or ceil(L/2) for Hermitian (non-negative
  // logical indices 0..ceil(L/2)-1; the reference's extra stored entry is outside the support)
  size_t dataLength() const;
  // reference-order interleave of inner-regime blocks (F[u m + l] = F_{q l + u n + v})
  size_t interleave() const;
};

// plan.cpp:35-64; throws std::invalid_argument on L == 0, m == 0, M < L
PlanParams deriveParams(size_t L, size_t M, size_t m, Symmetry sym);

// plan.cpp:66-73: zeta_N^k = exp(2 pi i k / N), k reduced mod N; long-double evaluation
Complex root(size_t N, int64_t k);

struct WorkEstimate {
  uint64_t implicitWords;
  double explicitWords;
};
// plan.cpp:75-89
WorkEstimate workMemoryWords(const PlanParams& pp, size_t A, size_t B, size_t d, size_t L);

// plan.hpp:84-106 / plan.cpp:91-99
class RootTable {
 public:
  RootTable() = default;
  explicit RootTable(size_t modulus);
  size_t modulus() const { return N_; }
  Complex operator()(int64_t k) const {
    int64_t r = k % static_cast<int64_t>(N_);
    if (r < 0) r += static_cast<int64_t>(N_);
    return z_[static_cast<size_t>(r)];
  }
  Complex at(uint64_t a, uint64_t b) const { return z_[(a % N_) * (b % N_) % N_]; }
  const std::vector<Complex>& values() const { return z_; }

 private:
  size_t N_ = 0;
  std::vector<Complex> z_;
};

}  // namespace hb
