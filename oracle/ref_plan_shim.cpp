// ref_plan_shim.cpp — TEST INFRASTRUCTURE.  C-ABI shim around the reference's own
// plan module, compiled FROM /root/reference/proj/src/plan.cpp where it lies (nothing
// copied) into oracle/_ref/libplanref.so by oracle/Makefile.  Used only to pin the
// oracle's and the product's plan restatements (tests/test_plan.py) and to generate
// tests/golden/plan_ref.json (tests/golden/make_plan_golden.py).
#include <string>  // plan.hpp:28 uses std::string without including <string>
#include <cstdint>
#include <stdexcept>
#include "hconv/plan.hpp"

extern "C" {
// fields: L M m p q n D C S inplace symmetry regime ; returns 0 or 1 (invalid_argument)
int ref_derive_params(size_t L, size_t M, size_t m, int sym, uint64_t* out12) {
  try {
    hconv::PlanParams pp = hconv::deriveParams(L, M, m, static_cast<hconv::Symmetry>(sym));
    const uint64_t v[12] = {pp.L, pp.M, pp.m, pp.p, pp.q, pp.n, pp.D, pp.C, pp.S, (uint64_t)pp.inplace,
                            (uint64_t)pp.kind.symmetry, (uint64_t)pp.kind.regime};
    for (int i = 0; i < 12; ++i) out12[i] = v[i];
    return 0;
  } catch (const std::invalid_argument&) { return 1; }
}
int ref_lengths(size_t L, size_t M, size_t m, int sym, uint64_t* out3) {
  try {
    hconv::PlanParams pp = hconv::deriveParams(L, M, m, static_cast<hconv::Symmetry>(sym));
    out3[0] = pp.blockLength(); out3[1] = pp.storedLength(); out3[2] = pp.paddedLength();
    return 0;
  } catch (const std::invalid_argument&) { return 1; }
}
int ref_root(size_t N, int64_t k, double* re, double* im) {
  try { auto z = hconv::root(N, k); *re = z.real(); *im = z.imag(); return 0; }
  catch (const std::invalid_argument&) { return 1; }
}
int ref_work_memory_words(size_t L, size_t M, size_t m, int sym, size_t A, size_t B, size_t d, size_t Lw,
                          uint64_t* implicit_words, double* explicit_words) {
  try {
    hconv::PlanParams pp = hconv::deriveParams(L, M, m, static_cast<hconv::Symmetry>(sym));
    auto w = hconv::workMemoryWords(pp, A, B, d, Lw);
    *implicit_words = w.implicitWords; *explicit_words = w.explicitWords;
    return 0;
  } catch (const std::invalid_argument&) { return 1; }
}
int ref_root_table(size_t N, int64_t k_lo, size_t count, double* out) {
  try {
    hconv::RootTable t(N);
    for (size_t i = 0; i < count; ++i) { auto z = t(k_lo + (int64_t)i); out[2 * i] = z.real(); out[2 * i + 1] = z.imag(); }
    return 0;
  } catch (const std::invalid_argument&) { return 1; }
}
int ref_root_table_at(size_t N, uint64_t a, uint64_t b, double* re, double* im) {
  try { hconv::RootTable t(N); auto z = t.at(a, b); *re = z.real(); *im = z.imag(); return 0; }
  catch (const std::invalid_argument&) { return 1; }
}
const char* ref_symmetry_name(int s) { return hconv::name(static_cast<hconv::Symmetry>(s)); }
int ref_symmetry_from_name(const char* n, int* s) {
  try { *s = (int)hconv::symmetryFromName(n); return 0; } catch (const std::invalid_argument&) { return 1; }
}
}
