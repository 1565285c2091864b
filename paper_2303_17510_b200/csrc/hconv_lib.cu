// hconv_lib.cu — host side of libhconv_cuda.so: the C ABI of include/hconv.h, plan objects,
// kernel selection, the device-timed m/p/q planner and the N-D decomposition driver.
//
// Reference interfaces (paths relative to /root/reference):
//   plan module          proj/include/hconv/plan.hpp:10-108, proj/src/plan.cpp:1-101
//   Conv1dPlan/convolve  SPEC.md:400-423, Algs. convolve/convolveX PAPER.md:188-262
//   ConvPlanND
//   tune_1d / tune_nd    SPEC.md:518-572, PAPER.md:894-914 (device events replace the CPU clock)
#include <cuda_runtime.h>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled (bound through the runtime)
#include <dlfcn.h>
#include <sys/file.h>
#include <nccl.h>  // types only: the functions are bound at run time (nccl() below)

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/hconv.h"
#include "../../include/hconv_ext.h"
#include "plan.hpp"
#include "registry.cuh"
#include "slab.hpp"

namespace hc {
// each symmetry's table comes from two translation units (a: blocks up to 3072 points, b: the rest)
void registry_sym0_a(KernelEntry* out, int* count);
void registry_sym0_b(KernelEntry* out, int* count);
void registry_sym1_a(KernelEntry* out, int* count);
void registry_sym1_b(KernelEntry* out, int* count);
void registry_sym2_a(KernelEntry* out, int* count);
void registry_sym2_b(KernelEntry* out, int* count);
// in-place two-residue convolution kernel (conv_ip.cuh, inst_ip.cu), by complex FFT length
const void* conv_ip_fn(int sym, int Bc);
size_t conv_ip_smem_bytes(int Bc, int tabn);
void conv_ip_radices(int Bc, int* P, int* R, int* mt);
int conv_ip_threads(int Bc);
int conv_ip_residues(int Bc);
void conv_ip_launch(int Bc, const ConvArgs& a, int grid, size_t smem, cudaStream_t s);
}  // namespace hc

using hc::KernelEntry;

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Diagnostics switches, read once from the environment (HCONV_*; tools/README.md).  None of
// them is needed in production: the defaults are the measured-best choices.
struct Diag {
  bool poison, no_stage, no_pp, pp2, same_line, no_tmacc, trace, no_cols, no_cols_pp, no_cols_tma, no_cols_tma1, sync_mult;
  bool no_ip;       // HCONV_NO_IP=1: never the in-place two-residue kernel (conv_ip.cuh)
  bool fake_timer;  // planner test hook: every candidate times 1 ms
  int dbg;
  double general_block_mb, nd_block_mb;
  long long host_chunks;
  Diag() {
    auto on = [](const char* n) { const char* v = std::getenv(n); return v && v[0] == '1'; };
    auto num = [](const char* n, double d) { const char* v = std::getenv(n); return v ? std::atof(v) : d; };
    poison = on("HCONV_POISON");
    no_stage = on("HCONV_NO_STAGE");
    no_pp = on("HCONV_NO_PP");
    no_ip = on("HCONV_NO_IP");
    pp2 = !(std::getenv("HCONV_PP2") && std::getenv("HCONV_PP2")[0] == '0');
    same_line = on("HCONV_DEBUG_SAME_LINE");
    no_tmacc = on("HCONV_NO_TMACC");
    trace = on("HCONV_TRACE");
    no_cols = on("HCONV_NO_COLS");
    no_cols_pp = on("HCONV_NO_COLS_PP");
    no_cols_tma = on("HCONV_NO_COLS_TMA");
    no_cols_tma1 = on("HCONV_NO_COLS_TMA1");
    sync_mult = on("HCONV_SYNC_MULT");
    fake_timer = on("HCONV_PLAN_FAKE_TIMER");
    dbg = (int)num("HCONV_DBG", 0);
    general_block_mb = num("HCONV_GENERAL_BLOCK_MB", 256.0);
    nd_block_mb = num("HCONV_ND_BLOCK_MB", 0.0);
    host_chunks = (long long)num("HCONV_HOST_CHUNKS", 8);
  }
};
const Diag& diag() {
  static const Diag d;
  return d;
}

// HCONV_POISON=1 (diagnostics): fill every scratch / work allocation with NaN so that a read
// before write shows up in the results instead of reading zeros from fresh pages
void poison(void* p, size_t bytes) {
  if (diag().poison) CK(cudaMemset(p, 0xff, bytes));
}

// Sets the plan's device for the duration of an ABI call and restores the caller's current
// device on every exit path (the library must not change e.g. torch's current device).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    int cur = 0;
    CK(cudaGetDevice(&cur));
    if (cur != d) {
      CK(cudaSetDevice(d));
      prev = cur;
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

template <class F>
hconv_status guarded(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return HCONV_INVALID_ARG;
  } catch (const Unsupported& e) {
    g_err = e.what();
    return HCONV_UNSUPPORTED;
  } catch (const CudaError& e) {
    g_err = e.what();
    return HCONV_CUDA_ERROR;
  } catch (const NcclError& e) {
    g_err = e.what();
    return HCONV_NCCL_ERROR;
  } catch (const std::bad_alloc& e) {
    g_err = "host allocation failed";
    return HCONV_ALLOC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HCONV_INTERNAL;
  }
  return HCONV_OK;
}

// ------------------------------------------------------------ registry ------
struct Registry {
  KernelEntry e[3][32];
  int n[3] = {0, 0, 0};
  Registry() {
    n[0] = n[1] = n[2] = 0;
    hc::registry_sym0_a(e[0], &n[0]);
    hc::registry_sym0_b(e[0], &n[0]);
    hc::registry_sym1_a(e[1], &n[1]);
    hc::registry_sym1_b(e[1], &n[1]);
    hc::registry_sym2_a(e[2], &n[2]);
    hc::registry_sym2_b(e[2], &n[2]);
  }
};
const Registry& registry() {
  static Registry r;
  return r;
}

// kernel for (symmetry, complex FFT length); naive entry for small non-radix lengths
const KernelEntry* find_kernel(int sym, int Bc, bool allow_naive = true) {
  const Registry& r = registry();
  const KernelEntry* naive = nullptr;
  for (int i = 0; i < r.n[sym]; ++i) {
    if (r.e[sym][i].naive) naive = &r.e[sym][i];
    else if (r.e[sym][i].Bc == Bc) return &r.e[sym][i];
  }
  if (allow_naive && naive && Bc <= hc::kNaiveMax) return naive;
  return nullptr;
}

struct DevInfo {
  int sms = 0;
  std::string name;
};
DevInfo dev_info() {
  int d = 0;
  CK(cudaGetDevice(&d));
  static std::mutex mu;
  static std::map<int, DevInfo> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(d);
  if (it != cache.end()) return it->second;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, d));
  DevInfo di{prop.multiProcessorCount, prop.name};
  cache[d] = di;
  return di;
}

// one-time per (function, device) attribute setting and occupancy query
int occupancy(const void* fn, int threads, size_t smem) {
  int d = 0;
  CK(cudaGetDevice(&d));
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(fn, d, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  // the attribute is per function: only ever raise it (launches with less smem stay valid)
  static std::map<std::pair<const void*, int>, size_t> attr;
  size_t& cur = attr[std::make_pair(fn, d)];
  if (smem > cur) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
  }
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem));
  if (nb < 1) throw Unsupported("kernel does not fit on an SM");
  cache[key] = nb;
  return nb;
}

// ------------------------------------------------------- device tables ------
struct DevTable {
  double2* ptr = nullptr;
};
// zeta_N^e, e < N, computed on the host with exact integer reduction (plan.cpp:66-73,91-99)
const double2* root_table(size_t N) {
  int d = 0;
  CK(cudaGetDevice(&d));
  static std::mutex mu;
  static std::map<std::pair<int, size_t>, DevTable> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(d, N);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second.ptr;
  std::vector<double2> h(N);
  for (size_t k = 0; k < N; ++k) {
    const hb::Complex z = hb::root(N, (int64_t)k);
    h[k] = make_double2(z.real(), z.imag());
  }
  DevTable t;
  CK(cudaMalloc(&t.ptr, N * sizeof(double2)));
  CK(cudaMemcpy(t.ptr, h.data(), N * sizeof(double2), cudaMemcpyHostToDevice));
  cache[key] = t;
  return t.ptr;
}

// ----------------------------------------------------------- axis plans -----
struct AxisPlan {
  hb::PlanParams pp;  // the caller's parameters (m, p, q, n, blockLength as the reference derives them)
  int split = 1;      // r > 1: block B executes as r sub-blocks B/r (dev.B = B/r, dev.n = r n; make_axis)
  hc::AxisDev dev{};
  hc::AxisDev dev_ip{};  // the same axis with the tables of the in-place kernel's radix plan (ip_fn set)
  const void* ip_fn = nullptr;
  const KernelEntry* k = nullptr;
  size_t data = 0;  // values per line (dataLength)
  int tab_full = 0; // table entries the radix kernels use (dev.tabn = the staged prefix)
};

hb::Symmetry to_sym(int s) {
  if (s < 0 || s > 2) throw std::invalid_argument("bad symmetry");
  return static_cast<hb::Symmetry>(s);
}

int complex_len(const hb::PlanParams& pp) {
  const size_t B = pp.blockLength();
  if (pp.symmetry == hb::Symmetry::Hermitian && B % 2 == 0) return (int)(B / 2);
  return (int)B;
}

// Per-axis tables of the radix kernels (block_io.cuh "table accessors"): every exponent is
// reduced exactly in 64-bit integers on the host, so the device never computes a modulo.
// (P, R, mt): the radix plan the tables serve -- the registry entry's, or the in-place kernel's
void build_tables(AxisPlan& ap, hc::AxisDev& a, int P, const int* R, int mt) {
  const int R0 = R[0], ns1 = a.Bc / R0, n = a.n;
  const long long qm = a.qm, B = a.B, Bc = a.Bc;
  const int nu = 2 * R0 + 1;
  const int nc = std::max<int>(2, (int)((a.L + B - 1) / B) + 1);
  a.ns1 = ns1;
  a.nu = nu;
  a.nc = nc;
  // order: MT U C A Z H Bl Bh (block_io.cuh); the kernels stage the prefix that fits.  The
  // residue-indexed tables U C Z H omit row v = 0 (every kernel skips those factors at v = 0):
  // their offsets point one row before the first stored row.
  a.oMT = 0;
  const int rU = mt, rC = rU + (n - 1) * nu, rA = rC + (n - 1) * nc, rZ = rA + ns1, rH = rZ + (n - 1) * ns1;
  a.oU = rU - nu;
  a.oC = rC - nc;
  a.oA = rA;
  a.oZ = rZ - ns1;
  a.oH = rH - 1;
  a.oBl = rH + (n - 1);
  a.oBh = a.oBl + ns1;
  ap.tab_full = a.sym == hc::SYM_HERMITIAN ? a.oBh + R0 + 1 : rH;
  a.tabn = ap.tab_full;
  a.tabfull = ap.tab_full;
  const int total = a.oBh + R0 + 1;
  auto key = std::make_tuple((int)a.Bc, a.qm, a.B, a.n, nc, P, R[0], R[1], R[2], R[3]);
  int d = 0;
  CK(cudaGetDevice(&d));
  static std::mutex mu;
  static std::map<std::pair<int, decltype(key)>, double2*> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto ck = std::make_pair(d, key);
  auto it = cache.find(ck);
  if (it != cache.end()) {
    a.tab = it->second;
    return;
  }
  std::vector<double2> h(total);
  auto z = [](long long N, long long e) {
    e %= N;
    if (e < 0) e += N;
    const hb::Complex c = hb::root((size_t)N, e);
    return make_double2(c.real(), c.imag());
  };
  for (int b = 0; b < ns1; ++b) h[a.oA + b] = z(Bc, b);
  for (int v = 1; v < n; ++v) {
    for (int b = 0; b < ns1; ++b) h[a.oZ + v * ns1 + b] = z(qm, (long long)v * b);
    for (int i = 0; i < nu; ++i) h[a.oU + v * nu + i] = z(qm, (long long)v * ns1 * i);
    for (int t = 0; t < nc; ++t) h[a.oC + v * nc + t] = z(qm, (long long)v * t * B);
    h[a.oH + v] = z(qm, (long long)v * Bc);
  }
  for (int b = 0; b < ns1; ++b) h[a.oBl + b] = z(B, b);
  for (int i = 0; i <= R0; ++i) h[a.oBh + i] = z(B, (long long)ns1 * i);
  // middle passes 1..P-2: omega_{Ns_i}^{b k}
  int o = a.oMT;
  for (int i = 1; i + 1 < P; ++i) {
    long long Nsi = 1, Nsi1 = 1;
    for (int j = i; j < P; ++j) Nsi *= R[j];
    Nsi1 = Nsi / R[i];
    for (int kk = 1; kk < R[i]; ++kk)
      for (long long b = 0; b < Nsi1; ++b) h[o++] = z(Nsi, b * kk);
  }
  if (o != mt) throw std::logic_error("table size mismatch");
  double2* dp = nullptr;
  CK(cudaMalloc(&dp, (size_t)total * sizeof(double2)));
  CK(cudaMemcpy(dp, h.data(), (size_t)total * sizeof(double2), cudaMemcpyHostToDevice));
  cache[ck] = dp;
  a.tab = dp;
}

// Blocks longer than the largest single-kernel FFT.  Residue block v of the qm-point padded
// transform, F_{v + n k} (k < B), splits by k = t + r k'' into r sub-blocks of B' = B / r:
// F_{(v + n t) + (r n) k''} -- residue v + n t of the same qm-point transform with blocks of B'
// (the unified form of block_io.cuh holds for any block length dividing qm).  So a block of B
// executes as r sub-blocks: a radix-r decimation-in-frequency first stage followed by B'-point
// block FFTs, i.e. the same launches as the hybrid plan (m = B', q = r q).  This is how the
// explicit candidate m >= M (p = q = 1) runs beyond 6144 complex points.
// Complex data fold any number of chunks; centered / Hermitian blocks fold at most two, so
// B' >= L / 2 there.  Returns r (1 when B has a kernel), 0 when no split works.
int split_factor(const hb::PlanParams& pp, bool allow_naive) {
  const int sym = (int)pp.symmetry;
  const size_t B = pp.blockLength();
  if (find_kernel(sym, complex_len(pp), allow_naive)) return 1;
  for (size_t r = 2; r <= 64 && B / r >= 64; ++r) {
    if (B % r) continue;
    const size_t Bs = B / r;
    if (pp.symmetry == hb::Symmetry::Hermitian && Bs % 2) continue;
    if (pp.symmetry != hb::Symmetry::Complex && 2 * Bs < pp.L) continue;
    const int Bc = (int)(pp.symmetry == hb::Symmetry::Hermitian ? Bs / 2 : Bs);
    if (const KernelEntry* k = find_kernel(sym, Bc, false); k && !k->naive) return (int)r;
  }
  return 0;
}

// Build the device view of one axis; throws Unsupported if no kernel covers the block.
AxisPlan make_axis(const hb::PlanParams& pp, bool allow_naive = true) {
  AxisPlan ap;
  ap.pp = pp;
  ap.data = pp.dataLength();
  const size_t qm = pp.paddedLength();
  if (qm != pp.n * pp.blockLength()) throw std::logic_error("qm != n B");
  if (qm > (size_t)INT32_MAX / 4) throw Unsupported("padded length too large");
  const int sym = (int)pp.symmetry;
  const int r = split_factor(pp, allow_naive);
  if (r == 0)
    throw Unsupported("no kernel for block length " + std::to_string(pp.blockLength()) + " (" + hb::name(pp.symmetry) + ")");
  ap.split = r;
  const size_t B = pp.blockLength() / (size_t)r;
  const int Bc = (int)(pp.symmetry == hb::Symmetry::Hermitian && B % 2 == 0 ? B / 2 : B);
  ap.k = find_kernel(sym, Bc, allow_naive);
  hc::AxisDev& a = ap.dev;
  a.sym = sym;
  a.L = (int)pp.L;
  a.S = (int)pp.dataLength();
  a.B = (int)B;
  a.Bc = Bc;
  a.n = (int)pp.n * r;
  a.qm = (int)qm;
  a.H = (int)(pp.L / 2);
  a.pe = r == 1 ? (int)pp.interleave() : 1;
  a.m = (int)pp.m;
  a.tw = root_table((size_t)Bc);
  a.zq = root_table(qm);
  if (!ap.k->naive) {
    build_tables(ap, ap.dev, ap.k->P, ap.k->R, ap.k->mt);
    if (r == 1 && (ap.ip_fn = hc::conv_ip_fn(sym, Bc))) {
      int P = 0, R[4] = {0, 0, 0, 0}, mt = 0;
      hc::conv_ip_radices(Bc, &P, R, &mt);
      ap.dev_ip = ap.dev;
      const int full = ap.tab_full;
      build_tables(ap, ap.dev_ip, P, R, mt);
      ap.tab_full = full;  // (the registry plan's; dev_ip.tabfull is the in-place kernel's)
    }
  }
  return ap;
}

size_t smem_conv(const AxisPlan& ap) { return ap.k->naive ? ap.k->smem_conv * ap.dev.Bc : ap.k->smem_conv; }
constexpr size_t kSmemCap = 232448 - 1024;  // opt-in max per block on B200, minus static shared (mbarriers)
// staged table prefix: everything if it fits next to `group_elems` per group, else at least MT
int staged_tabn(const AxisPlan& ap, size_t group_elems) {
  const size_t groups = (size_t)ap.k->G * group_elems;
  const size_t room = kSmemCap / sizeof(double2) > groups ? kSmemCap / sizeof(double2) - groups : 0;
  return (int)std::max<size_t>((size_t)ap.k->mt, std::min<size_t>((size_t)ap.tab_full, room));
}
size_t smem_fwd(const AxisPlan& ap, int* tabn, bool bwd = false) {
  if (ap.k->naive) return (bwd ? ap.k->smem_bwd : ap.k->smem_fwd) * ap.dev.Bc;
  *tabn = staged_tabn(ap, ap.k->xs);
  return (size_t)(*tabn + (size_t)ap.k->G * ap.k->xs) * sizeof(double2);
}

int grid_for(const void* fn, const KernelEntry* k, size_t smem, long long items) {
  const int nb = occupancy(fn, k->T * k->G, smem);
  const long long need = (items + k->G - 1) / k->G;
  const long long cap = (long long)nb * dev_info().sms;
  return (int)std::max<long long>(1, std::min(need, cap));
}

// ------------------------------------------------------------- launches -----
struct Scratch {
  double2* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) CK(cudaFree(p));
    p = nullptr;
    bytes = 0;
    CK(cudaMalloc(&p, b));
    poison(p, b);
    bytes = b;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};


// Staging decision of the radix conv kernel (kernels.cuh): 1 = lines copied by TMA into the
// exchange buffer, 2 = into a separate buffer, 0 = direct global loads (strided lines, or the
// line does not fit).  HCONV_NO_STAGE=1 disables staging (A/B measurements).
struct ConvLayout {
  int stage = 0, gs = 0, in_off = 0, tabn = 0;
  size_t smem = 0;
};
ConvLayout conv_layout(const AxisPlan& ap, const hc::Lines& lin) {
  ConvLayout c;
  const KernelEntry* k = ap.k;
  if (k->naive) {
    c.smem = smem_conv(ap);
    return c;
  }
  const bool off = diag().no_stage;
  const int S = ap.dev.S;
  c.gs = k->xs + k->stash;
  const bool no_pp = diag().no_pp;
  // (the ping-pong kernel reads every table from shared memory: all of them must fit)
  if (!off && !no_pp && lin.es == 1 && S <= k->xs &&
      (size_t)(ap.tab_full + (size_t)k->G * 2 * k->xs) * sizeof(double2) <= kSmemCap) {
    c.stage = 3;  // ping-pong: X (f, its exchanges, stashed F) and Y (g, its and the inverse's exchanges)
    c.gs = 2 * k->xs;
    c.tabn = staged_tabn(ap, c.gs);
    c.smem = (size_t)(c.tabn + (size_t)k->G * c.gs) * sizeof(double2);
    return c;
  }
  if (!off && lin.es == 1) {
    if (S <= k->xs) {
      c.stage = 1;
    } else if ((size_t)(k->mt + (size_t)k->G * (c.gs + std::max(S, ap.dev.Bc))) * sizeof(double2) <= kSmemCap) {
      // (the Hermitian packing writes Z'_k, k < Bc, into the staged line in place)
      c.stage = 2;
      c.in_off = c.gs;
      c.gs += std::max(S, ap.dev.Bc);
    }
  }
  c.tabn = staged_tabn(ap, c.gs);
  c.smem = (size_t)(c.tabn + (size_t)k->G * c.gs) * sizeof(double2);
  if (c.smem > kSmemCap) throw Unsupported("shared-memory budget exceeded");
  return c;
}

void launch_conv(const AxisPlan& ap, const hc::Lines& lin, const double2* f, const double2* g, double2* out,
                 Scratch& scratch, cudaStream_t s) {
  if (lin.count == 0) return;
  const ConvLayout cl = conv_layout(ap, lin);
  // the paired ping-pong kernel where it exists (complex, L <= B; registry) -- HCONV_PP2=0 disables it
  const bool pp2_on = diag().pp2;
  const bool pp2 = pp2_on && cl.stage == 3 && ap.k->convpp2 && ap.dev.L <= ap.dev.B;
  // the in-place two-residue kernel where it exists (complex unit-stride lines, L <= B, n = 2, every table staged)
  if (!diag().no_ip && cl.stage == 3 && ap.ip_fn && ap.dev.L <= ap.dev.B && ap.dev.n == hc::conv_ip_residues(ap.dev.Bc) &&
      !diag().trace && !diag().dbg) {
    hc::ConvArgs a{ap.dev_ip, lin, f, g, out, nullptr, 3, 0, 0, nullptr, 0};
    a.ax.tabn = ap.dev_ip.tabfull;
    const size_t smem = hc::conv_ip_smem_bytes(ap.dev.Bc, a.ax.tabn);
    if (smem <= kSmemCap) {
      const int nb = occupancy(ap.ip_fn, hc::conv_ip_threads(ap.dev.Bc), smem);
      const int grid = (int)std::max<long long>(1, std::min<long long>(lin.count, (long long)nb * dev_info().sms));
      if (diag().same_line) a.lin.d_out = 0;
      hc::conv_ip_launch(ap.dev.Bc, a, grid, smem, s);
      CK(cudaGetLastError());
      return;
    }
  }
  const void* fn = pp2 ? ap.k->convpp2_fn : cl.stage == 3 ? ap.k->convpp_fn : ap.k->conv_fn;
  const int grid = grid_for(fn, ap.k, cl.smem, lin.count);
  // per-group accumulator slots: only residue loops with more than one block use them
  if (ap.dev.n > 1) scratch.ensure((size_t)grid * ap.k->G * ap.dev.S * sizeof(double2));
  hc::ConvArgs a{ap.dev, lin, f, g, out, scratch.p, cl.stage, cl.gs, cl.in_off, nullptr, 0};
  a.dbg = diag().dbg;
  // HCONV_DEBUG_SAME_LINE=1: every line reads/writes line 0 (L2-resident timing of the kernel
  // body without HBM; diagnostics only, results are meaningless)
  if (diag().same_line) a.lin.d_out = 0;
  a.ax.tabn = cl.tabn;
  // the single-buffer Hermitian kernel keeps its accumulator in TMEM when its CTA owns the SM
  const bool no_tmacc = diag().no_tmacc;
  a.tm_acc = (!no_tmacc && cl.stage != 3 && ap.dev.sym == hc::SYM_HERMITIAN && cl.smem > 116 * 1024) ? 1 : 0;
  // HCONV_TRACE=1: phase timestamps (clock64) of CTA 0, printed to stderr (diagnostics)
  const bool trace = diag().trace;
  unsigned long long* tbuf = nullptr;
  if (trace && !ap.k->naive) {
    CK(cudaMalloc(&tbuf, 256 * sizeof(unsigned long long)));
    CK(cudaMemset(tbuf, 0, 256 * sizeof(unsigned long long)));
    a.trace = tbuf;
  }
  if (pp2) ap.k->convpp2(a, grid, cl.smem, s);
  else if (cl.stage == 3) ap.k->convpp(a, grid, cl.smem, s);
  else ap.k->conv(a, grid, cl.smem, s);
  CK(cudaGetLastError());
  if (tbuf) {
    unsigned long long h[256];
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(h, tbuf, sizeof h, cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "[hconv trace %s grid %d]", ap.k->radix, grid);
    for (int i = 1; i < 256 && h[i]; ++i) std::fprintf(stderr, " %llu", h[i] - h[i - 1]);
    std::fprintf(stderr, "\n");
    cudaFree(tbuf);
  }
}

// Column-tile variants for strided outer-axis lines (complex / centered radix kernels).
bool use_cols(const AxisPlan& ap, const hc::Lines& lin) {
  const bool off = diag().no_cols;
  return !off && !ap.k->naive && ap.k->fwdc && lin.es > 1;
}
int cols_tabn(const AxisPlan& ap) {
  const size_t groups = (size_t)ap.k->gc * ap.k->xs;
  const size_t room = kSmemCap / sizeof(double2) > groups ? kSmemCap / sizeof(double2) - groups : 0;
  return (int)std::max<size_t>((size_t)ap.k->mt, std::min<size_t>((size_t)ap.tab_full, room));
}
int grid_cols(const void* fn, const KernelEntry* k, size_t smem, long long items, int gc = 0) {
  if (gc == 0) gc = k->gc;
  const int nb = occupancy(fn, k->T * gc, smem);
  const long long need = (items + gc - 1) / gc;
  return (int)std::max<long long>(1, std::min(need, (long long)nb * dev_info().sms));
}

// Pipelined column tiles (k_pfft_*_cols_pp): two tile buffers of gc x max(xs, rows) values plus
// at least the middle-pass tables must fit; returns the staged table prefix (0 = does not fit).
int cols_pp_tabn(const AxisPlan& ap, int rows, size_t* smem) {
  const bool off = diag().no_cols_pp;
  // only at the unpipelined kernel's tile width: narrower tiles cost more in DRAM row efficiency
  // than the pipelining recovers (c4 outer 4096-point columns, 2 -> 1 column per tile: 0.54 -> 0.69 ms)
  if (off || !ap.k->fwdcp || ap.k->gcp != ap.k->gc) return 0;
  const size_t bufs = 2 * (size_t)ap.k->gcp * (size_t)std::max(ap.k->xs, rows);
  if ((bufs + (size_t)ap.k->mt) * sizeof(double2) > kSmemCap) return 0;
  const size_t room = kSmemCap / sizeof(double2) - bufs;
  const int tabn = (int)std::max<size_t>((size_t)ap.k->mt, std::min<size_t>((size_t)ap.tab_full, room));
  *smem = (tabn + bufs) * sizeof(double2);
  return tabn;
}

// ------------------------------------------------- tensor-map column tiles ----
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
  }();
  return fn;
}
// 3D map {2 nin float64, rows, count / nin} of a two-level line batch with unit inner distance,
// box {2 gc, box_rows, 1}; false when the batch does not have that shape.
bool tile_map(CUtensorMap* map, const void* base, const hc::Lines& l, int rows, int gc, int box_rows) {
  auto enc = encode_tiled();
  if (!enc || l.d_in != 1 || l.nin % gc || l.count % l.nin || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  const unsigned long long outer = (unsigned long long)(l.count / l.nin);
  cuuint64_t dims[3] = {(cuuint64_t)(2 * l.nin), (cuuint64_t)rows, (cuuint64_t)outer};
  const unsigned long long rs = (unsigned long long)l.es * 16ull;
  const unsigned long long os = outer > 1 ? (unsigned long long)l.d_out * 16ull : rs * (unsigned long long)rows;
  if (rs % 16 || os % 16 || rs >= (1ull << 40) || os >= (1ull << 40) || rs == 0 || os == 0) return false;
  cuuint64_t strides[2] = {rs, os};
  cuuint32_t box[3] = {(cuuint32_t)(2 * gc), (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// smem of the TMA column kernels: tables + two 128-byte-aligned tile buffers of *bufn values
// (every box row a tensor copy writes or reads lies inside its buffer); 0 = does not fit
int cols_tma_tabn(const AxisPlan& ap, int rows_in, int box_in, int rows_out, int box_out, size_t* smem, int* bufn) {
  if (diag().no_cols_tma || !ap.k->fwdct || ap.k->gcp != ap.k->gc) return 0;
  const int rin = (rows_in + box_in - 1) / box_in * box_in, rout = (rows_out + box_out - 1) / box_out * box_out;
  const size_t per = ((size_t)ap.k->gcp * (size_t)std::max({ap.k->xs, rows_in, rin, rout}) + 7) & ~(size_t)7;
  const size_t bufs = 2 * per;
  if ((bufs + (size_t)ap.k->mt + 8) * sizeof(double2) > kSmemCap) return 0;
  const size_t room = kSmemCap / sizeof(double2) - bufs - 8;
  const int tabn = (int)std::max<size_t>((size_t)ap.k->mt, std::min<size_t>((size_t)ap.tab_full, room));
  *smem = ((size_t)tabn + 8 + bufs) * sizeof(double2);  // + 128 B: the kernel aligns the buffers
  *bufn = (int)per;
  return tabn;
}
int box_rows_for(int rows) { return rows >= 256 ? 256 : ((rows + 7) / 8) * 8; }
// smem of the one-buffer TMA column kernels (k_pfft_*_cols_tma1, gc columns per tile): tables, the
// 128-byte-aligned exchange / block buffer X of *bufn values and, for the forward pass, the input
// staging area of the data rows behind it; 0 = does not fit or not instantiated
int cols_tma1_tabn(const AxisPlan& ap, bool fwd, int rows_in, int box_in, int rows_out, int box_out, size_t* smem,
                   int* bufn, int* nb_stage = nullptr) {
  if (diag().no_cols_tma || diag().no_cols_tma1 || !ap.k->fwdc1) return 0;
  const int rin = (rows_in + box_in - 1) / box_in * box_in, rout = (rows_out + box_out - 1) / box_out * box_out;
  const size_t gc = (size_t)ap.k->gc, cap = kSmemCap / sizeof(double2);
  const size_t x = (gc * (size_t)std::max({ap.k->xs, rout, fwd ? 0 : rin}) + 7) & ~(size_t)7;
  size_t in = fwd ? (gc * (size_t)rin + 7) & ~(size_t)7 : 0;
  if (x + in + (size_t)ap.k->mt + 8 > cap) return 0;
  if (!fwd) {
    // inverse: stage as many leading boxes as fit next to X and every table (at least one box
    // stays for the late load into X, so both barriers complete every tile)
    const size_t tabs = std::max<size_t>((size_t)ap.k->mt, (size_t)ap.tab_full);
    const size_t box = gc * (size_t)box_in;
    const size_t room = cap > x + tabs + 8 ? cap - x - tabs - 8 : 0;
    const size_t nb = std::min<size_t>(room / box, (size_t)(rin / box_in) - 1);
    in = nb * box;
    if (nb_stage) *nb_stage = (int)nb;
  }
  const size_t room = cap - x - in - 8;
  const int tabn = (int)std::max<size_t>((size_t)ap.k->mt, std::min<size_t>((size_t)ap.tab_full, room));
  *smem = ((size_t)tabn + 8 + x + in) * sizeof(double2);  // + 128 B: the kernel aligns the buffers
  *bufn = (int)x;
  return tabn;
}
int stage_boxes_limit() {  // HCONV_TMA1_STAGE=k caps the staged boxes of the inverse (diagnostics)
  static const int v = [] {
    const char* e = std::getenv("HCONV_TMA1_STAGE");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}

void launch_fwd(const AxisPlan& ap, const hc::Lines& lin, const hc::Lines& lout, const double2* f, void* F, int v,
                int ref_order, cudaStream_t s) {
  if (lin.count == 0) return;
  if (use_cols(ap, lin) && !ref_order) {
    const int rows = (int)ap.data, bi = box_rows_for(rows), bo = box_rows_for(ap.dev.Bc);
    size_t smt = 0;
    int bufn = 0;
    const int tt = cols_tma_tabn(ap, rows, bi, ap.dev.Bc, bo, &smt, &bufn);
    CUtensorMap mi, mo;
    if (tt > 0 && lout.count % ap.k->gcp == 0 && lout.nin == lin.nin && tile_map(&mi, f, lin, rows, ap.k->gcp, bi) &&
        tile_map(&mo, F, lout, ap.dev.Bc, ap.k->gcp, bo)) {
      const int grid = grid_cols(ap.k->fwdct_fn, ap.k, smt, lin.count, ap.k->gcp);
      hc::FwdArgs a{ap.dev, lin, lout, f, F, v, ref_order};
      a.ax.tabn = tt;
      const hc::TileMaps tm{(int)lin.nin, rows, bi, bo, bufn};
      ap.k->fwdct(a, tm, mi, mo, grid, smt, s);
      CK(cudaGetLastError());
      return;
    }
  }
  if (use_cols(ap, lin) && !ref_order) {
    // blocks without room for two full-width tile buffers: one buffer plus the staged data rows
    const int rows = (int)ap.data, bi = box_rows_for(rows), bo = box_rows_for(ap.dev.Bc);
    size_t smt = 0;
    int bufn = 0;
    const int tt = cols_tma1_tabn(ap, true, rows, bi, ap.dev.Bc, bo, &smt, &bufn);
    CUtensorMap mi, mo;
    if (tt > 0 && lin.count % ap.k->gc == 0 && lout.count % ap.k->gc == 0 && lout.nin == lin.nin &&
        tile_map(&mi, f, lin, rows, ap.k->gc, bi) && tile_map(&mo, F, lout, ap.dev.Bc, ap.k->gc, bo)) {
      const int grid = grid_cols(ap.k->fwdc1_fn, ap.k, smt, lin.count, ap.k->gc);
      hc::FwdArgs a{ap.dev, lin, lout, f, F, v, ref_order};
      a.ax.tabn = tt;
      const hc::TileMaps tm{(int)lin.nin, rows, bi, bo, bufn};
      ap.k->fwdc1(a, tm, mi, mo, grid, smt, s);
      CK(cudaGetLastError());
      return;
    }
  }
  size_t smpp = 0;
  int tpp = 0;
  if (use_cols(ap, lin) && !ref_order && (tpp = cols_pp_tabn(ap, (int)ap.data, &smpp)) > 0) {
    const int grid = grid_cols(ap.k->fwdcp_fn, ap.k, smpp, lin.count, ap.k->gcp);
    hc::FwdArgs a{ap.dev, lin, lout, f, F, v, ref_order};
    a.ax.tabn = tpp;
    ap.k->fwdcp(a, grid, smpp, s);
    CK(cudaGetLastError());
    return;
  }
  if (use_cols(ap, lin)) {
    const int tabn = cols_tabn(ap);
    const size_t sm = (size_t)(tabn + (size_t)ap.k->gc * ap.k->xs) * sizeof(double2);
    const int grid = grid_cols(ap.k->fwdc_fn, ap.k, sm, lin.count);
    hc::FwdArgs a{ap.dev, lin, lout, f, F, v, ref_order};
    a.ax.tabn = tabn;
    ap.k->fwdc(a, grid, sm, s);
    CK(cudaGetLastError());
    return;
  }
  int tabn = 0;
  const size_t sm = smem_fwd(ap, &tabn);
  const int grid = grid_for(ap.k->fwd_fn, ap.k, sm, lin.count);
  hc::FwdArgs a{ap.dev, lin, lout, f, F, v, ref_order};
  a.ax.tabn = tabn;
  ap.k->fwd(a, grid, sm, s);
  CK(cudaGetLastError());
}

void launch_bwd(const AxisPlan& ap, const hc::Lines& lin, const hc::Lines& lout, const void* F, double2* dst,
                const double2* acc, double scale, int v, int ref_order, cudaStream_t s) {
  if (lin.count == 0) return;
  if (use_cols(ap, lout) && !ref_order) {
    const int rows = ap.dev.Bc, bi = box_rows_for(rows);
    size_t smt = 0;
    int bufn = 0;
    const int tt = cols_tma_tabn(ap, rows, bi, rows, bi, &smt, &bufn);
    CUtensorMap mi;
    if (tt > 0 && lout.count % ap.k->gcp == 0 && tile_map(&mi, F, lin, rows, ap.k->gcp, bi)) {
      const int grid = grid_cols(ap.k->bwdct_fn, ap.k, smt, lin.count, ap.k->gcp);
      hc::BwdArgs a{ap.dev, lin, lout, F, dst, acc, scale, v, ref_order};
      a.ax.tabn = tt;
      const hc::TileMaps tm{(int)lin.nin, rows, bi, bi, bufn};
      ap.k->bwdct(a, tm, mi, grid, smt, s);
      CK(cudaGetLastError());
      return;
    }
  }
  if (use_cols(ap, lout) && !ref_order) {
    const int rows = ap.dev.Bc, bi = box_rows_for(rows);
    size_t smt = 0;
    int bufn = 0;
    int nbs = 0;
    int tt = cols_tma1_tabn(ap, false, rows, bi, rows, bi, &smt, &bufn, &nbs);
    if (tt > 0 && stage_boxes_limit() >= 0 && stage_boxes_limit() < nbs) {
      smt -= (size_t)(nbs - stage_boxes_limit()) * ap.k->gc * bi * sizeof(double2);
      nbs = stage_boxes_limit();
    }
    CUtensorMap mi;
    if (tt > 0 && lin.count % ap.k->gc == 0 && lout.count % ap.k->gc == 0 && tile_map(&mi, F, lin, rows, ap.k->gc, bi)) {
      const int grid = grid_cols(ap.k->bwdc1_fn, ap.k, smt, lin.count, ap.k->gc);
      hc::BwdArgs a{ap.dev, lin, lout, F, dst, acc, scale, v, ref_order};
      a.ax.tabn = tt;
      const hc::TileMaps tm{(int)lin.nin, rows, bi, bi, bufn, nbs};
      ap.k->bwdc1(a, tm, mi, grid, smt, s);
      CK(cudaGetLastError());
      return;
    }
  }
  size_t smpp = 0;
  int tpp = 0;
  if (use_cols(ap, lout) && !ref_order && (tpp = cols_pp_tabn(ap, ap.dev.Bc, &smpp)) > 0) {
    const int grid = grid_cols(ap.k->bwdcp_fn, ap.k, smpp, lin.count, ap.k->gcp);
    hc::BwdArgs a{ap.dev, lin, lout, F, dst, acc, scale, v, ref_order};
    a.ax.tabn = tpp;
    ap.k->bwdcp(a, grid, smpp, s);
    CK(cudaGetLastError());
    return;
  }
  if (use_cols(ap, lout)) {
    const int tabn = cols_tabn(ap);
    const size_t sm = (size_t)(tabn + (size_t)ap.k->gc * ap.k->xs) * sizeof(double2);
    const int grid = grid_cols(ap.k->bwdc_fn, ap.k, sm, lin.count);
    hc::BwdArgs a{ap.dev, lin, lout, F, dst, acc, scale, v, ref_order};
    a.ax.tabn = tabn;
    ap.k->bwdc(a, grid, sm, s);
    CK(cudaGetLastError());
    return;
  }
  int tabn = 0;
  const size_t sm = smem_fwd(ap, &tabn, true);
  const int grid = grid_for(ap.k->bwd_fn, ap.k, sm, lin.count);
  hc::BwdArgs a{ap.dev, lin, lout, F, dst, acc, scale, v, ref_order};
  a.ax.tabn = tabn;
  ap.k->bwd(a, grid, sm, s);
  CK(cudaGetLastError());
}

// Residue v of the CALLER's plan (public residue-level entry points): with a split block the r
// sub-blocks v + n t interleave as k = t + r k'' in the caller's block (natural order, which is
// the reference order whenever p <= 2).
void residue_fwd(const AxisPlan& ap, const hc::Lines& lin, const hc::Lines& lout, const double2* f, void* F, int v,
                 int ref_order, cudaStream_t s) {
  if (ap.split == 1) {
    launch_fwd(ap, lin, lout, f, F, v, ref_order, s);
    return;
  }
  if (ref_order && ap.pp.interleave() > 1) throw Unsupported("reference block order of a split inner block");
  const int r = ap.split;
  const size_t esz = ap.dev.sym == hc::SYM_HERMITIAN ? sizeof(double) : sizeof(double2);
  hc::Lines lo = lout;
  lo.es *= r;
  for (int t = 0; t < r; ++t)
    launch_fwd(ap, lin, lo, f, (char*)F + (size_t)t * (size_t)lout.es * esz, v + (int)ap.pp.n * t, 0, s);
}
void residue_bwd(const AxisPlan& ap, const hc::Lines& lin, const hc::Lines& lout, const void* F, double2* dst,
                 const double2* acc, double scale, int v, int ref_order, cudaStream_t s) {
  if (ap.split == 1) {
    launch_bwd(ap, lin, lout, F, dst, acc, scale, v, ref_order, s);
    return;
  }
  if (ref_order && ap.pp.interleave() > 1) throw Unsupported("reference block order of a split inner block");
  const int r = ap.split;
  const size_t esz = ap.dev.sym == hc::SYM_HERMITIAN ? sizeof(double) : sizeof(double2);
  hc::Lines li = lin;
  li.es *= r;
  for (int t = 0; t < r; ++t)
    launch_bwd(ap, li, lout, (const char*)F + (size_t)t * (size_t)lin.es * esz, dst, t == 0 ? acc : dst,
               t == r - 1 ? scale : 1.0, v + (int)ap.pp.n * t, 0, s);
}

// ------------------------------------------------ conjugate-pair forward ----
// forward_conjugate_pair, complex data: one pass over the
// input forms A_j = zeta_qm^{v j} Re f_j and B_j = i zeta_qm^{v j} Im f_j once and folds both
// pre-twiddled sequences, W^{(v)} = sum (A + B) and W^{(-v)} = sum (conj A - conj B), modulo B.
// Their B-point DFTs (the radix kernels, residue 0 of a plain B-point plan) are the blocks
// F_{v + n k'} and F_{-v + n k'} (PAPER.md's F_{q l + u n + v} and F_{q l + u n - v},
// k' = p l + u), written in the reference order u m + l.  On the GPU the trick saves a read of
// f and one twiddle per point, not FP64 work (an FMA complex multiply costs the same 4 DFMA/DMUL
// as the A/B split), so the fused convolution kernels do not use it.
__global__ void k_pair_fold(const double2* f, long long dist, long long S, long long C, int L, int B, int qm, int v,
                            const double2* zq, double2* Wv, double2* Wn) {
  const long long total = C * (long long)B;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long c = i / B;
    const int s = (int)(i % B);
    double2 a = make_double2(0.0, 0.0), b = make_double2(0.0, 0.0);
    for (int j = s; j < L; j += B) {
      const double2 x = f[c * dist + (long long)j * S];
      const double2 w = zq[(int)(((long long)v * j) % qm)];
      const double2 A = make_double2(w.x * x.x, w.y * x.x);    // zeta^{vj} Re f_j
      const double2 Bi = make_double2(-w.y * x.y, w.x * x.y);  // i zeta^{vj} Im f_j
      a = make_double2(a.x + A.x + Bi.x, a.y + A.y + Bi.y);
      b = make_double2(b.x + A.x - Bi.x, b.y - A.y + Bi.y);    // conj A - conj B
    }
    Wv[i] = a;
    Wn[i] = b;
  }
}
__global__ void k_pair_order(const double2* X, long long C, int B, int pe, int m, double2* Fv, double2* Fn) {
  const long long total = C * (long long)B;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long c = i / B;
    const int k = (int)(i % B);
    const long long o = c * B + (pe > 1 ? (long long)(k % pe) * m + k / pe : k);
    Fv[o] = X[i];
    Fn[o] = X[total + i];
  }
}

// --------------------------------------------------------- synthetic data ---
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void k_fill_uniform(unsigned long long seed, unsigned long long a, unsigned long long first, long long n,
                               double2* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long idx = first + (unsigned long long)i;
    double v[2];
    for (unsigned long long comp = 0; comp < 2; ++comp) {
      const unsigned long long z = mix64(seed * 0x9E3779B97F4A7C15ull + ((a << 56) | (comp << 55) | idx));
      v[comp] = 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
    }
    out[i] = make_double2(v[0], v[1]);
  }
}

// ------------------------------------------------------------- planner ------
bool smooth7(size_t m) {
  for (size_t f : {2, 3, 5, 7})
    while (m % f == 0) m /= f;
  return m == 1;
}

struct Candidate {
  size_t m;
  hb::PlanParams pp;
  double ms = 0;
  size_t exec_B = 0, exec_n = 0;  // the device work: block length and block count after any split
  bool explicit_ = false;         // the explicit dealiasing candidate (q = 1, m >= M)
};

// Candidate m values: 7-smooth sizes whose block length has a kernel, directly
// or split into sub-blocks (make_axis; the direct-sum kernel only for blocks of at most 64
// points).  Distinct m with the same device work -- the same (sub-)block length and block count
// -- are one class (the p-point pre-DFTs are the first radix stage of the block FFT, block_io.cuh;
// a split block is a radix-r first stage), timed once and labelled by its member with the fewest
// chunks p (then the smaller m).  Timing ties between classes keep the smaller m.
// The explicit candidate (q = 1, the smallest such m >= M) is always in the list;
// when its device work is another class's, it carries that class's time.
std::vector<Candidate> plan_candidates(hb::Symmetry sym, size_t L, size_t M) {
  // split blocks (r sub-blocks) enter the scan only as the explicit candidate, or when no block
  // has a kernel of its own (complex L > 12288), and then at most 8-way and the 8 smallest
  // amounts of device work: a many-way split is the hybrid plan of its sub-block, labelled worse
  std::map<std::pair<size_t, size_t>, Candidate> cls, split_cls;
  Candidate expl{0, {}, 0};
  const size_t mmax = 4 * M + 8;
  for (size_t m = 1; m <= mmax; ++m) {
    if (!smooth7(m)) continue;
    hb::PlanParams pp = hb::deriveParams(L, M, m, sym);
    const int r = split_factor(pp, complex_len(pp) <= 64);
    if (r == 0) continue;
    Candidate c{m, pp, 0, pp.blockLength() / (size_t)r, pp.n * (size_t)r, false};
    if (pp.q == 1 && m >= M && expl.m == 0) {
      expl = c;
      expl.explicit_ = true;
    }
    if (r > 8) continue;
    auto& into = r == 1 ? cls : split_cls;
    auto key = std::make_pair(c.exec_B, c.exec_n);
    auto it = into.find(key);
    if (it == into.end() || pp.p < it->second.pp.p) into[key] = c;
  }
  if (cls.empty()) {
    std::vector<Candidate> sp;
    for (auto& kv : split_cls) sp.push_back(kv.second);
    std::sort(sp.begin(), sp.end(), [](const Candidate& a, const Candidate& b) {
      return a.exec_B * a.exec_n < b.exec_B * b.exec_n || (a.exec_B * a.exec_n == b.exec_B * b.exec_n && a.m < b.m);
    });
    for (size_t i = 0; i < sp.size() && i < 8; ++i) cls[{sp[i].exec_B, sp[i].exec_n}] = sp[i];
  }
  std::vector<Candidate> out;
  bool have_expl = false;
  for (auto& kv : cls) {
    if (expl.m && kv.second.m == expl.m) {
      kv.second.explicit_ = true;
      have_expl = true;
    }
    out.push_back(kv.second);
  }
  if (expl.m && !have_expl) out.push_back(expl);  // shares a hybrid class's device work
  std::sort(out.begin(), out.end(), [](const Candidate& a, const Candidate& b) { return a.m < b.m; });
  return out;
}

// Planner cache: a line-oriented text file (HCONV_PLAN_CACHE), one record per
// line, comma-separated: the key fields (kind, L, M, A, B, C, S, placement) plus the device and
// its SM clock (timings are only comparable on the same device at the same clocks),
// then the choice (m, D, placement) and the median in nanoseconds.  Advisory locking (flock):
// shared while reading, exclusive while appending; the last record of a key wins.
std::string cache_device() {
  int d = 0, khz = 0;
  CK(cudaGetDevice(&d));
  CK(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, d));
  std::string n = dev_info().name;
  std::replace(n.begin(), n.end(), ',', ' ');
  return n + "," + std::to_string(khz / 1000);
}
std::string plan_cache_key(const std::string& kind, size_t L, size_t M, size_t A, size_t B, long long C) {
  return kind + "," + std::to_string(L) + "," + std::to_string(M) + "," + std::to_string(A) + "," +
         std::to_string(B) + "," + std::to_string(C) + ",1,out-of-place," + cache_device();
}

struct PlannerCache {
  std::mutex mu;
  std::map<std::string, std::pair<size_t, double>> mem;  // key -> (m, median ns)
  bool loaded = false;
  std::string path() const {
    const char* p = std::getenv("HCONV_PLAN_CACHE");
    return p ? std::string(p) : std::string();
  }
  static constexpr int kKeyFields = 10;  // kind L M A B C S placement device clock
  void load() {
    if (loaded) return;
    loaded = true;
    const std::string p = path();
    if (p.empty()) return;
    FILE* f = std::fopen(p.c_str(), "r");
    if (!f) return;
    flock(fileno(f), LOCK_SH);
    char line[2048];
    while (std::fgets(line, sizeof line, f)) {
      std::string s(line);
      while (!s.empty() && (s.back() == '\n' || s.back() == '\r')) s.pop_back();
      std::vector<std::string> fl;
      size_t st = 0;
      for (size_t i = 0; i <= s.size(); ++i)
        if (i == s.size() || s[i] == ',') {
          fl.push_back(s.substr(st, i - st));
          st = i + 1;
        }
      if ((int)fl.size() != kKeyFields + 4) continue;  // + m, D, placement, median_ns
      std::string key = fl[0];
      for (int i = 1; i < kKeyFields; ++i) key += "," + fl[i];
      mem[key] = {std::strtoull(fl[kKeyFields].c_str(), nullptr, 10), std::strtod(fl[kKeyFields + 3].c_str(), nullptr)};
    }
    flock(fileno(f), LOCK_UN);
    std::fclose(f);
  }
  void store(const std::string& key, size_t m, double ns) {
    mem[key] = {m, ns};
    const std::string p = path();
    if (p.empty()) return;
    if (FILE* f = std::fopen(p.c_str(), "a")) {
      flock(fileno(f), LOCK_EX);
      std::fprintf(f, "%s,%zu,1,out-of-place,%.0f\n", key.c_str(), m, ns);
      std::fflush(f);
      flock(fileno(f), LOCK_UN);
      std::fclose(f);
    }
  }
};
PlannerCache& planner_cache() {
  static PlannerCache c;
  return c;
}

struct PlanReport {
  std::vector<Candidate> timed;
  bool cached = false;
};

// timed candidate lists of this process, by planner key (a cache hit still knows the ranking)
std::map<std::string, std::vector<Candidate>>& ranked_memo() {
  static std::map<std::string, std::vector<Candidate>> m;
  return m;
}

// tune_1d on the device: median of 5 timed runs after one warm-up, CUDA events,
// over the plan's own batch (capped by memory: three arrays of at most 2 GiB together).
// The candidates are timed with the fused binary-product convolution; for a general operator
// (whose residue loop runs the same padded FFTs through work blocks) that timing is the proxy,
// while tune_nd times the plan's own operator.
size_t tune_axis(hb::Symmetry sym, size_t L, size_t M, long long lines, PlanReport* rep) {
  auto& cache = planner_cache();
  {
    const size_t data = hb::deriveParams(L, M, 1, sym).dataLength();
    const long long cap = std::max<long long>(1, (long long)((size_t(2) << 30) / (3 * 16 * data)));
    lines = std::max<long long>(1, std::min(lines, cap));
  }
  const std::string key = plan_cache_key(hb::name(sym), L, M, 2, 1, lines);
  {
    std::lock_guard<std::mutex> lk(cache.mu);
    cache.load();
    auto it = cache.mem.find(key);
    if (it != cache.mem.end()) {
      if (rep) {
        rep->cached = true;
        auto jt = ranked_memo().find(key);
        if (jt != ranked_memo().end()) rep->timed = jt->second;
      }
      return it->second.first;
    }
  }
  std::vector<Candidate> cands = plan_candidates(sym, L, M);
  if (cands.empty()) throw Unsupported("planner: no candidate m has a kernel for L=" + std::to_string(L));
  const size_t data = hb::deriveParams(L, M, 1, sym).dataLength();
  const size_t elems = (size_t)lines * data;
  double2 *f = nullptr, *g = nullptr, *o = nullptr;
  CK(cudaMalloc(&f, elems * sizeof(double2)));
  CK(cudaMalloc(&g, elems * sizeof(double2)));
  CK(cudaMalloc(&o, elems * sizeof(double2)));
  k_fill_uniform<<<256, 256>>>(7, 0, 0, (long long)elems, f);
  k_fill_uniform<<<256, 256>>>(7, 1, 0, (long long)elems, g);
  CK(cudaGetLastError());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  Scratch scratch;
  const hc::Lines lin{lines, 1, (long long)data, 0, 1};
  size_t best = 0;
  double best_ms = 1e30;
  std::map<std::pair<size_t, size_t>, double> class_ms;  // device work already timed
  for (auto& c : cands) {
    auto cit = class_ms.find({c.exec_B, c.exec_n});
    if (cit != class_ms.end()) {  // the explicit candidate sharing a hybrid class's launches
      c.ms = cit->second;
      continue;
    }
    AxisPlan ap = make_axis(c.pp);
    launch_conv(ap, lin, f, g, o, scratch, 0);
    std::vector<double> t;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      launch_conv(ap, lin, f, g, o, scratch, 0);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    c.ms = diag().fake_timer ? 1.0 : t[2];
    class_ms[{c.exec_B, c.exec_n}] = c.ms;
    if (c.ms < best_ms * (1 - 1e-9)) {  // strict improvement; ties keep the smaller m
      best_ms = c.ms;
      best = c.m;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  scratch.release();
  cudaFree(f);
  cudaFree(g);
  cudaFree(o);
  if (rep) rep->timed = cands;
  std::lock_guard<std::mutex> lk(cache.mu);
  ranked_memo()[key] = cands;
  cache.store(key, best, best_ms * 1e6);
  return best;
}

}  // namespace

// ------------------------------------------------------------------ plan ----
// Device side of hconv_convolve_host: three streams (host->device, compute, device->host),
// three slots of input/output chunks, created on first use.
struct HostPipe {
  static constexpr int kSlots = 3;
  cudaStream_t st[3] = {nullptr, nullptr, nullptr};  // h2d, compute, d2h
  cudaEvent_t loaded[kSlots] = {}, done[kSlots] = {}, drained[kSlots] = {};
  std::vector<double2*> buf[kSlots];  // per slot: max(A, B) arrays (inputs, then outputs in place)
  size_t elems = 0;                   // per buffer
  int nslots = 0;                     // slots allocated
  size_t width = 0;                   // buffers per slot
  bool ready = false;
  void init() {
    if (ready) return;
    for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (int k = 0; k < kSlots; ++k) {
      CK(cudaEventCreateWithFlags(&loaded[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&drained[k], cudaEventDisableTiming));
    }
    ready = true;
  }
  void ensure(size_t n, int slots, size_t w) {
    if (n <= elems && slots <= nslots && w <= width) return;
    for (auto& sl : buf) {
      for (auto& b : sl)
        if (b) CK(cudaFree(b));
      sl.clear();
    }
    elems = 0;
    nslots = 0;
    width = 0;
    for (int k = 0; k < slots; ++k) {
      buf[k].assign(w, nullptr);
      for (auto& b : buf[k]) {
        CK(cudaMalloc(&b, n * sizeof(double2)));
        poison(b, n * sizeof(double2));
      }
    }
    elems = n;
    nslots = slots;
    width = w;
  }
  ~HostPipe() {
    for (auto& sl : buf)
      for (auto& b : sl)
        if (b) cudaFree(b);
    if (!ready) return;
    for (int k = 0; k < kSlots; ++k) {
      cudaEventDestroy(loaded[k]);
      cudaEventDestroy(done[k]);
      cudaEventDestroy(drained[k]);
    }
    for (auto& s : st) cudaStreamDestroy(s);
  }
};

namespace {
struct SlabState;
void destroy_slab(SlabState* s);
struct SlabDel {
  void operator()(SlabState* s) const { destroy_slab(s); }
};
}  // namespace

struct hconv_plan {
  hconv_desc d{};
  std::unique_ptr<SlabState, SlabDel> slab;  // x-slab decomposition over G ranks (slab.hpp)
  int device = 0;
  std::vector<AxisPlan> ax;
  Scratch scratch;                    // conv1d accumulator slots
  Scratch gwork, gacc;                // general operators: work blocks and accumulators
  std::vector<double2*> buffers;      // N-D work / accumulator buffers
  std::vector<long long> chunk;               // per level: arrays processed per pass (L2 blocking)
  PlanReport report;
  HostPipe host;                      // hconv_convolve_host
  size_t W() const { return std::max(d.A, d.B); }
  // the fused kernels compute the binary product; every other operator runs the general loop
  bool fused() const { return d.mult == HCONV_MULT_PRODUCT && d.A == 2 && d.B == 1; }
  ~hconv_plan() {
    gwork.release();
    gacc.release();
    scratch.release();
    for (double2* b : buffers)
      if (b) cudaFree(b);
  }
};

namespace {

// N-D: arrays at a level are contiguous with extents data[level..d-1].
size_t inner_elems(const hconv_plan* P, int level) {
  size_t x = 1;
  for (size_t k = level + 1; k < P->ax.size(); ++k) x *= P->ax[k].data;
  return x;
}

// buffers layout: for level l < d-1: max(A, B) work buffers, then B accumulators
double2* level_work(hconv_plan* P, int level, int a) { return P->buffers[level * (P->W() + P->d.B) + a]; }
double2* level_acc(hconv_plan* P, int level, int b) { return P->buffers[level * (P->W() + P->d.B) + P->W() + b]; }

// ------------------------------------------------- general multiplication operators ----
// builtin_mult_product(A) for A != 2: F_0 <- F_0 F_1 ... F_{A-1}, pointwise
constexpr size_t kMaxArity = 16;
struct BlockPtrs {
  void* p[kMaxArity];
};
__global__ void k_mult_product(BlockPtrs F, int A, long long count, int real) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += stride) {
    if (real) {
      double acc = ((const double*)F.p[0])[i];
      for (int a = 1; a < A; ++a) acc *= ((const double*)F.p[a])[i];
      ((double*)F.p[0])[i] = acc;
    } else {
      double2 acc = ((const double2*)F.p[0])[i];
      for (int a = 1; a < A; ++a) acc = hc::cmul(acc, ((const double2*)F.p[a])[i]);
      ((double2*)F.p[0])[i] = acc;
    }
  }
}

// example operator (hconv_ext.h hconv_example_mult(0)): F0 F0, F0 F1, F1 F1
__global__ void k_mult_pairs(double2* F0, double2* F1, double2* F2, long long count, int real) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += stride) {
    if (real) {
      const double a = ((const double*)F0)[i], b = ((const double*)F1)[i];
      ((double*)F0)[i] = a * a;
      ((double*)F1)[i] = a * b;
      ((double*)F2)[i] = b * b;
    } else {
      const double2 a = F0[i], b = F1[i];
      F0[i] = hc::cmul(a, a);
      F1[i] = hc::cmul(a, b);
      F2[i] = hc::cmul(b, b);
    }
  }
}
int example_mult_pairs(void* const* F, size_t A, size_t B, size_t count, int real, void*, void* stream) {
  if (A != 2 || B != 3) return 1;
  const int blocks = (int)std::max<size_t>(1, std::min<size_t>((count + 255) / 256, 4096));
  k_mult_pairs<<<blocks, 256, 0, (cudaStream_t)stream>>>((double2*)F[0], (double2*)F[1], (double2*)F[2],
                                                           (long long)count, real);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

// MultOperator.apply on one residue's transformed blocks, in place
void apply_mult(const hconv_plan* P, double2* const* F, long long count, bool real, cudaStream_t s) {
  if (P->d.mult == HCONV_MULT_PRODUCT) {
    BlockPtrs b{};
    for (size_t a = 0; a < P->d.A; ++a) b.p[a] = F[a];
    const int blocks = (int)std::max<long long>(1, std::min<long long>((count + 255) / 256, 8LL * dev_info().sms));
    k_mult_product<<<blocks, 256, 0, s>>>(b, (int)P->d.A, count, real ? 1 : 0);
    CK(cudaGetLastError());
    return;
  }
  void* ptrs[kMaxArity];
  for (size_t a = 0; a < P->W(); ++a) ptrs[a] = F[a];
  const bool dsync = diag().sync_mult;
  if (dsync) CK(cudaDeviceSynchronize());
  const int rc = P->d.mult_fn(ptrs, P->d.A, P->d.B, (size_t)count, real ? 1 : 0, P->d.mult_user, s);
  if (dsync) CK(cudaDeviceSynchronize());
  if (rc != 0) throw std::invalid_argument("multiplication operator callback returned " + std::to_string(rc));
}

// Alg. convolve / convolveX for a general operator over C lines of `dist`
// elements: per chunk of lines and residue v, the A forward padded FFTs into work blocks
// (natural block order), mult, and the B backward padded FFTs accumulated in separate buffers
// (the last residue scales by 1/qm and writes out[b], which may alias an input: every input
// line of the chunk has been transformed by then).  Chunks keep the work blocks L2-resident.
void conv1d_general(hconv_plan* P, const AxisPlan& ap, long long C, long long dist, const double2* const* in,
                    double2* const* out, cudaStream_t s) {
  if (C == 0) return;
  const size_t A = P->d.A, Bo = P->d.B, W = P->W();
  const long long Bl = ap.dev.B, S = (long long)ap.data, n = ap.dev.n;
  const bool real = ap.dev.sym == hc::SYM_HERMITIAN;
  // work blocks per pass: HCONV_GENERAL_BLOCK_MB (default 256 MB of blocks and accumulators)
  const double block_mb = diag().general_block_mb;
  const long long per_line = (long long)(W * Bl + (n > 1 ? Bo * dist : 0)) * (long long)sizeof(double2);
  const long long chunk = std::max<long long>(1, std::min<long long>(C, (long long)(block_mb * 1048576.0 / per_line)));
  const long long acc_elems = (chunk - 1) * dist + S;
  P->gwork.ensure((size_t)(W * chunk * Bl) * sizeof(double2));
  if (n > 1) P->gacc.ensure((size_t)(Bo * acc_elems) * sizeof(double2));
  std::vector<double2*> work(W), acc(Bo, nullptr);
  for (size_t w = 0; w < W; ++w) work[w] = P->gwork.p + w * chunk * Bl;
  if (n > 1)
    for (size_t b = 0; b < Bo; ++b) acc[b] = P->gacc.p + b * acc_elems;
  const double scale = 1.0 / (double)ap.dev.qm;
  for (long long c0 = 0; c0 < C; c0 += chunk) {
    const long long cnt = std::min(chunk, C - c0);
    const hc::Lines lin{cnt, 1, dist, 0, 1};  // data lines of the chunk
    const hc::Lines wl{cnt, 1, Bl, 0, 1};     // work blocks (complex128, or float64 when real)
    for (long long v = 0; v < n; ++v) {
      for (size_t a = 0; a < A; ++a) launch_fwd(ap, lin, wl, in[a] + c0 * dist, work[a], (int)v, 0, s);
      apply_mult(P, work.data(), cnt * Bl, real, s);
      const bool first = v == 0, last = v == n - 1;
      for (size_t b = 0; b < Bo; ++b)
        launch_bwd(ap, wl, lin, work[b], last ? out[b] + c0 * dist : acc[b], first ? nullptr : acc[b],
                   last ? scale : 1.0, (int)v, 0, s);
    }
  }
}

// 1D convolution of C lines: the fused kernel for the binary product, else the general loop
void conv1d(hconv_plan* P, const AxisPlan& ap, long long C, long long dist, const double2* const* in,
            double2* const* out, cudaStream_t s) {
  if (P->fused()) {
    const hc::Lines lin{C, 1, dist, 0, 1};
    launch_conv(ap, lin, in[0], in[1], out[0], P->scratch, s);
  } else {
    conv1d_general(P, ap, C, dist, in, out, s);
  }
}

// convolve_nd as grid-wide passes: for each outer residue v, forward the
// outer axis of every column into work buffers, convolve the spectral lines recursively
// (in place into work[0]), inverse the outer axis and accumulate (one normalisation per axis).
void nd_level(hconv_plan* P, int level, long long NB, const double2* const* in, double2* const* out, cudaStream_t s) {
  const int d = (int)P->ax.size();
  const AxisPlan& ap = P->ax[level];
  const long long inner = (long long)inner_elems(P, level);
  const long long Lx = (long long)ap.data, asz = Lx * inner;
  if (level == d - 1) {
    conv1d(P, ap, NB, asz, in, out, s);
    return;
  }
  // L2 blocking: below the top level the NB arrays (spectral planes of the parent axis) are
  // processed `chunk` at a time, so this level's work buffers are reused while L2-resident
  const long long chunk = std::max<long long>(1, P->chunk[level]);
  for (long long c0 = 0; c0 < NB; c0 += chunk) {
    const long long nb = std::min(chunk, NB - c0);
    std::vector<const double2*> inc(P->d.A);
    for (size_t a = 0; a < P->d.A; ++a) inc[a] = in[a] + c0 * asz;
    const long long B = ap.dev.B, n = ap.dev.n;
    const hc::Lines cols{nb * inner, inner, asz, 1, inner};       // columns of the input arrays
    const hc::Lines wcols{nb * inner, inner, B * inner, 1, inner};  // columns of the work arrays
    std::vector<const double2*> sub(P->d.A);
    std::vector<double2*> subo(P->d.B);  // the subconvolutions write their B outputs in place
    for (size_t a = 0; a < P->d.A; ++a) sub[a] = level_work(P, level, (int)a);
    for (size_t b = 0; b < P->d.B; ++b) subo[b] = level_work(P, level, (int)b);
    const double scale = 1.0 / (double)ap.dev.qm;
    for (int v = 0; v < n; ++v) {
      for (size_t a = 0; a < P->d.A; ++a) launch_fwd(ap, cols, wcols, inc[a], level_work(P, level, (int)a), v, 0, s);
      nd_level(P, level + 1, nb * B, sub.data(), subo.data(), s);
      const bool first = v == 0, last = v == n - 1;
      for (size_t b = 0; b < P->d.B; ++b) {
        double2* acc = level_acc(P, level, (int)b);
        double2* dst = last ? out[b] + c0 * asz : acc;
        const double2* accsrc = first ? nullptr : acc;
        launch_bwd(ap, wcols, cols, level_work(P, level, (int)b), dst, accsrc, last ? scale : 1.0, v, 0, s);
      }
    }
  }
}

// ------------------------------------------------------------ NCCL binding ---
// Bound at run time to the libnccl.so.2 the process already has (torch's), else the system one:
// the library itself has no link-time NCCL dependency (single-GPU users never load it).
struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string why;
};
const Nccl& nccl() {
  static const Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      r.why = std::string("libnccl.so.2 not found: ") + (dlerror() ? dlerror() : "");
      return r;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    r.GetUniqueId = (decltype(r.GetUniqueId))sym("ncclGetUniqueId");
    r.CommInitRank = (decltype(r.CommInitRank))sym("ncclCommInitRank");
    r.CommDestroy = (decltype(r.CommDestroy))sym("ncclCommDestroy");
    r.GroupStart = (decltype(r.GroupStart))sym("ncclGroupStart");
    r.GroupEnd = (decltype(r.GroupEnd))sym("ncclGroupEnd");
    r.Send = (decltype(r.Send))sym("ncclSend");
    r.Recv = (decltype(r.Recv))sym("ncclRecv");
    r.GetErrorString = (decltype(r.GetErrorString))sym("ncclGetErrorString");
    if (!r.GetUniqueId || !r.CommInitRank || !r.CommDestroy || !r.GroupStart || !r.GroupEnd || !r.Send || !r.Recv)
      r.why = "libnccl.so.2 lacks a required symbol";
    return r;
  }();
  if (!n.why.empty()) throw NcclError(n.why);
  return n;
}
#define NC(x)                                                                                       \
  do {                                                                                              \
    ncclResult_t r_ = (x);                                                                          \
    if (r_ != ncclSuccess)                                                                          \
      throw NcclError(std::string(#x) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r_) : "error")); \
  } while (0)

// ------------------------------------------------------------ slab plans ----
// hconv_desc.slab != NULL: the x-slab decomposition of slab.hpp with device buffers, the y-axis
// padded FFT kernels (k-major spectral layout), an inner (d-1)-D plan of this library for the
// subconvolutions of one chunk of k-lines, and the exchange on a plan-owned stream.
struct CudaSlabOps {
  SlabState* st = nullptr;
  cudaStream_t s = nullptr;  // the caller's (compute) stream of the current hconv_convolve
  void* alloc(size_t elems);
  void free(void* p) {
    if (p) cudaFree(p);
  }
  void fwd(size_t r, const void* f, void* F);
  void bwd(size_t r, const void* W, void* h, bool acc, double scale);
  void inner(size_t count, void* const* T);
  void copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows, bool on_comm);
  void exchange(const void* send, const size_t* sc, const size_t* sd, void* recv, const size_t* rc, const size_t* rd);
  void comm_after_compute();
  void mark_comm(size_t tag);
  void compute_after_comm(size_t tag);
};

struct SlabState {
  hconv_slab cfg{};
  hslab::Geometry g;
  AxisPlan ay;                     // the outer (y) axis
  hconv_plan* inner = nullptr;     // (d-1)-D subconvolutions of max_chunk copies
  cudaStream_t sc = nullptr;       // communication stream
  std::vector<cudaEvent_t> ev;     // per chunk: forward exchange done (comm -> compute)
  cudaEvent_t ev_c = nullptr, ev_m = nullptr;  // compute -> comm, comm -> compute (all)
  CudaSlabOps ops;
  std::unique_ptr<hslab::Driver<CudaSlabOps>> drv;
  std::vector<double2*> acc;       // accumulators for outputs that alias inputs (lazily)
  ~SlabState() {
    drv.reset();
    for (double2* a : acc)
      if (a) cudaFree(a);
    if (inner) hconv_plan_destroy(inner);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (ev_c) cudaEventDestroy(ev_c);
    if (ev_m) cudaEventDestroy(ev_m);
    if (sc) cudaStreamDestroy(sc);
  }
};
void destroy_slab(SlabState* s) { delete s; }

void* CudaSlabOps::alloc(size_t elems) {
  void* p = nullptr;
  CK(cudaMalloc(&p, elems * sizeof(double2)));
  poison(p, elems * sizeof(double2));
  return p;
}
// y-lines (x, z) of the x-slab [nx][Ly][Z] <-> the same lines k-major F[k][x][z]
void CudaSlabOps::fwd(size_t r, const void* f, void* F) {
  const hslab::Geometry& g = st->g;
  const long long nxz = (long long)(g.nx() * g.Z), Z = (long long)g.Z;
  // (the spectrum's lines described with the same inner extent as the slab's, Z columns per x row:
  // the tensor-map column tiles need matching tile coordinates on both sides)
  const hc::Lines lin{nxz, Z, (long long)g.Ly * Z, 1, Z}, lspec{nxz, Z, Z, 1, nxz};
  launch_fwd(st->ay, lin, lspec, (const double2*)f, F, (int)r, 0, s);
}
void CudaSlabOps::bwd(size_t r, const void* W, void* h, bool acc, double scale) {
  const hslab::Geometry& g = st->g;
  const long long nxz = (long long)(g.nx() * g.Z), Z = (long long)g.Z;
  const hc::Lines lin{nxz, Z, (long long)g.Ly * Z, 1, Z}, lspec{nxz, Z, Z, 1, nxz};
  launch_bwd(st->ay, lspec, lin, W, (double2*)h, acc ? (const double2*)h : nullptr, scale, (int)r, 0, s);
}
void CudaSlabOps::inner(size_t count, void* const* T) {
  hconv_plan* P = st->inner;
  std::vector<const double2*> in(P->d.A);
  std::vector<double2*> out(P->d.B);
  for (size_t a = 0; a < P->d.A; ++a) in[a] = (const double2*)T[a];
  for (size_t b = 0; b < P->d.B; ++b) out[b] = (double2*)T[b];
  if (P->d.dims == 1) conv1d(P, P->ax[0], (long long)count, (long long)P->ax[0].data, in.data(), out.data(), s);
  else nd_level(P, 0, (long long)count, in.data(), out.data(), s);
}
void CudaSlabOps::copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                         bool on_comm) {
  if (!rows || !width) return;
  CK(cudaMemcpy2DAsync(dst, dpitch * sizeof(double2), src, spitch * sizeof(double2), width * sizeof(double2), rows,
                       cudaMemcpyDeviceToDevice, on_comm ? st->sc : s));
}
void CudaSlabOps::exchange(const void* send, const size_t* sc, const size_t* sd, void* recv, const size_t* rc,
                           const size_t* rd) {
  const hslab::Geometry& g = st->g;
  const int me = g.rank;
  auto sp = [&](size_t off) { return (const char*)send + off * sizeof(double2); };
  auto rp = [&](size_t off) { return (char*)recv + off * sizeof(double2); };
  if (st->cfg.nccl_comm || !st->cfg.exchange) {
    // this rank's own segment is a device copy on the communication stream
    if (sc[me]) CK(cudaMemcpyAsync(rp(rd[me]), sp(sd[me]), sc[me] * sizeof(double2), cudaMemcpyDeviceToDevice, st->sc));
    if (!st->cfg.nccl_comm) return;  // one rank, no communicator: the copy was the exchange
    const Nccl& n = nccl();
    ncclComm_t comm = (ncclComm_t)st->cfg.nccl_comm;
    NC(n.GroupStart());
    for (int h = 0; h < g.G; ++h) {
      if (h == me) continue;
      if (sc[h]) NC(n.Send(sp(sd[h]), 2 * sc[h], ncclFloat64, h, comm, st->sc));
      if (rc[h]) NC(n.Recv(rp(rd[h]), 2 * rc[h], ncclFloat64, h, comm, st->sc));
    }
    NC(n.GroupEnd());
    return;
  }
  const int r = st->cfg.exchange(send, sc, sd, recv, rc, rd, st->cfg.exchange_user, st->sc);
  if (r != 0) throw NcclError("slab exchange callback returned " + std::to_string(r));
}
void CudaSlabOps::comm_after_compute() {
  CK(cudaEventRecord(st->ev_c, s));
  CK(cudaStreamWaitEvent(st->sc, st->ev_c, 0));
}
void CudaSlabOps::mark_comm(size_t tag) { CK(cudaEventRecord(st->ev[tag], st->sc)); }
void CudaSlabOps::compute_after_comm(size_t tag) {
  if (tag == (size_t)-1) {
    CK(cudaEventRecord(st->ev_m, st->sc));
    CK(cudaStreamWaitEvent(s, st->ev_m, 0));
  } else {
    CK(cudaStreamWaitEvent(s, st->ev[tag], 0));
  }
}

// Slab plan: axis plans for parameter reports, the y kernels, the inner plan, the buffers.
void build_slab(hconv_plan* P, const std::vector<hb::Symmetry>& syms, const std::vector<size_t>& data) {
  const hconv_desc* desc = &P->d;
  const hconv_slab& cfg = *desc->slab;
  const int d = desc->dims;
  if (d < 2) throw std::invalid_argument("slab decomposition is for 2D and 3D convolutions");
  if (d == 2 && syms[1] == hb::Symmetry::Hermitian)
    throw Unsupported("2D Hermitian slabs need the outer axis sharded (three transposes)");
  if (desc->C > 1) throw std::invalid_argument("slab plans convolve one global array (C must be 0 or 1)");
  if (cfg.nranks < 1 || cfg.rank < 0 || cfg.rank >= cfg.nranks) throw std::invalid_argument("slab: bad rank / nranks");
  if (cfg.nranks > 1 && !cfg.nccl_comm && !cfg.exchange)
    throw std::invalid_argument("slab over several ranks needs nccl_comm or an exchange callback");
  for (int k = 0; k < d; ++k)
    if (desc->axis[k].m == 0) throw std::invalid_argument("slab plans need every m (tune on one rank, broadcast)");
  P->ax.clear();
  for (int k = 0; k < d; ++k) P->ax.push_back(make_axis(hb::deriveParams(desc->axis[k].L, desc->axis[k].M, desc->axis[k].m, syms[k])));
  auto st = std::unique_ptr<SlabState, SlabDel>(new SlabState());
  st->cfg = cfg;
  st->ay = P->ax[1];
  const AxisPlan& ay = st->ay;
  st->g = hslab::make_geometry(cfg.rank, cfg.nranks, data[0], data[1], d == 3 ? data[2] : 1, (size_t)ay.dev.B,
                               (size_t)ay.dev.n, 1.0 / (double)ay.dev.qm, cfg.chunks);
  hconv_desc in{};
  in.dims = d - 1;
  in.axis[0] = desc->axis[0];
  in.axis[0].symmetry = (int)syms[0];
  if (d == 3) {
    in.axis[1] = desc->axis[2];
    in.axis[1].symmetry = (int)syms[2];
  }
  in.A = desc->A;
  in.B = desc->B;
  in.mult = desc->mult;
  in.C = std::max<size_t>(1, st->g.max_chunk());
  in.device = desc->device;
  in.mult_fn = desc->mult_fn;
  in.mult_user = desc->mult_user;
  const hconv_status rc = hconv_plan_create(&in, &st->inner);
  if (rc != HCONV_OK) {
    const std::string why = "slab inner plan: " + g_err;
    if (rc == HCONV_UNSUPPORTED) throw Unsupported(why);
    if (rc == HCONV_CUDA_ERROR) throw CudaError(why);
    throw std::invalid_argument(why);
  }
  CK(cudaStreamCreateWithFlags(&st->sc, cudaStreamNonBlocking));
  st->ev.resize(st->g.nchunks);
  for (auto& e : st->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&st->ev_c, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&st->ev_m, cudaEventDisableTiming));
  st->ops.st = st.get();
  st->drv = std::make_unique<hslab::Driver<CudaSlabOps>>(st->g, desc->A, desc->B, st->ops);
  st->acc.assign(desc->B, nullptr);
  P->slab = std::move(st);
}

void slab_convolve(hconv_plan* P, const double2* const* in, double2* const* out, cudaStream_t s) {
  SlabState& S = *P->slab;
  const hslab::Geometry& g = S.g;
  const size_t n = g.nx() * g.Ly * g.Z;
  std::vector<void*> acc(P->d.B);
  for (size_t b = 0; b < P->d.B; ++b) {
    bool alias = false;
    for (size_t a = 0; a < P->d.A; ++a) alias |= (const void*)out[b] == (const void*)in[a];
    if (alias) {
      if (!S.acc[b]) S.acc[b] = (double2*)S.ops.alloc(std::max<size_t>(1, n));
      acc[b] = S.acc[b];
    } else {
      acc[b] = out[b];
    }
  }
  S.ops.s = s;
  std::vector<const void*> ins(in, in + P->d.A);
  S.drv->run(ins.data(), acc.data());
  for (size_t b = 0; b < P->d.B; ++b)
    if (acc[b] != (void*)out[b] && n) CK(cudaMemcpyAsync(out[b], acc[b], n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  CK(cudaGetLastError());
}

void check_desc(const hconv_desc* d) {
  if (!d) throw std::invalid_argument("null descriptor");
  if (d->dims < 1 || d->dims > 3) throw std::invalid_argument("dims must be 1, 2 or 3");
  if (d->mult == HCONV_MULT_PRODUCT) {
    // builtin_mult_product(A): B = 1, A >= 2
    if (d->A < 2 || d->B != 1) throw std::invalid_argument("builtin_mult_product needs A >= 2 and B == 1");
  } else if (d->mult == HCONV_MULT_CALLBACK) {
    if (!d->mult_fn) throw std::invalid_argument("HCONV_MULT_CALLBACK without mult_fn");
    if (d->A < 1 || d->B < 1) throw std::invalid_argument("multiplication operator arity: A >= 1, B >= 1");
  } else {
    throw std::invalid_argument("unknown multiplication operator");
  }
  if (std::max(d->A, d->B) > kMaxArity) throw Unsupported("operator arity above 16");
  if (d->dims > 1 && d->dist != 0) throw std::invalid_argument("N-D copies are contiguous arrays: dist must be 0");
}

// Build the axis plans for chosen subtransform sizes and allocate the N-D work buffers.
void build_plan(hconv_plan* P, const std::vector<size_t>& ms, const std::vector<hb::Symmetry>& syms) {
  const hconv_desc* desc = &P->d;
  const int d = desc->dims;
  for (double2* b : P->buffers)
    if (b) cudaFree(b);
  P->buffers.clear();
  P->ax.clear();
  for (int k = 0; k < d; ++k) P->ax.push_back(make_axis(hb::deriveParams(desc->axis[k].L, desc->axis[k].M, ms[k], syms[k])));
  if (d == 1) {
    P->ax[0].pp.C = desc->C ? desc->C : 1;
    return;
  }
  // level l processes `chunk[l]` arrays per pass: all of them at the top level, and below it
  // as many as keep this level's buffers within HCONV_ND_BLOCK_MB (0 = all of them)
  // (B200, c5: chunks of 96 MB 13.7 ms, 1 GB 11.8 ms, unchunked 11.6 ms -- the small per-chunk
  // launches lose more to tails than L2 residency saves -- so blocking is off by default)
  const double block_mb = diag().nd_block_mb;
  P->chunk.assign(d, 1);
  long long NB = (long long)(desc->C ? desc->C : 1);  // arrays at the top level (a batch of N-D arrays)
  for (int l = 0; l < d - 1; ++l) {
    const long long inner = (long long)inner_elems(P, l);
    const long long per = (long long)(P->W() * P->ax[l].dev.B + desc->B * P->ax[l].data) * inner * (long long)sizeof(double2);
    long long ch = NB;
    if (l > 0 && block_mb > 0) ch = std::max<long long>(1, std::min<long long>(NB, (long long)(block_mb * 1048576.0 / per)));
    if (l > 0 && (desc->flags & HCONV_FLAG_MIN_MEMORY)) ch = 1;  // one reused buffer per outer plane
    P->chunk[l] = ch;
    const long long work = ch * P->ax[l].dev.B * inner, acc = ch * (long long)P->ax[l].data * inner;
    for (size_t a = 0; a < P->W(); ++a) {
      double2* b = nullptr;
      CK(cudaMalloc(&b, (size_t)work * sizeof(double2)));
      poison(b, (size_t)work * sizeof(double2));
      P->buffers.push_back(b);
    }
    for (size_t b_ = 0; b_ < desc->B; ++b_) {
      double2* b = nullptr;
      CK(cudaMalloc(&b, (size_t)acc * sizeof(double2)));
      poison(b, (size_t)acc * sizeof(double2));
      P->buffers.push_back(b);
    }
    NB = ch * P->ax[l].dev.B;
  }
}

// N-D planning (tune_nd).  Each axis is first tuned independently with 1D
// convolutions; on the GPU the number of outer residue blocks multiplies
// full passes over the volume, so the best per-axis candidates (top 2 by 1D time, plus the
// fewest-residue candidate) are then timed together on the real N-D convolution.
std::vector<size_t> tune_nd(hconv_plan* P, const std::vector<hb::Symmetry>& syms, const std::vector<size_t>& data) {
  const hconv_desc* desc = &P->d;
  const int d = desc->dims;
  // one record per axis: kind "nd<k>:<sym L M m of every axis>" (the joint choice depends on all)
  std::string sig;
  for (int k = 0; k < d; ++k)
    sig += std::string(k ? "/" : "") + hb::name(syms[k]) + ":" + std::to_string(desc->axis[k].L) + ":" +
           std::to_string(desc->axis[k].M) + ":" + std::to_string(desc->axis[k].m);
  auto axis_key = [&](int k) {
    return plan_cache_key("nd" + std::to_string(k) + ":" + sig, desc->axis[k].L, desc->axis[k].M, desc->A, desc->B,
                          (long long)(desc->C ? desc->C : 1));
  };
  auto& cache = planner_cache();
  {
    std::lock_guard<std::mutex> lk(cache.mu);
    cache.load();
    auto it = cache.mem.find(axis_key(0));
    if (it != cache.mem.end()) {
      std::vector<size_t> ms(d);
      bool ok = true;
      for (int k = 0; k < d; ++k) {
        auto jt = cache.mem.find(axis_key(k));
        if (jt == cache.mem.end()) ok = false;
        else ms[k] = jt->second.first;
      }
      if (ok) {
        P->report.cached = true;
        return ms;
      }
    }
  }
  std::vector<std::vector<size_t>> options(d);
  for (int k = 0; k < d; ++k) {
    const hconv_axis& a = desc->axis[k];
    if (a.m) {
      options[k] = {a.m};
      continue;
    }
    long long lines = 1;
    for (int j = 0; j < d; ++j)
      if (j != k) lines *= (long long)data[j];
    PlanReport r;
    const size_t best = tune_axis(syms[k], a.L, a.M, lines, &r);
    options[k].push_back(best);
    if (!r.timed.empty()) {
      std::vector<Candidate> c = r.timed;
      std::sort(c.begin(), c.end(), [](const Candidate& x, const Candidate& y) { return x.ms < y.ms; });
      for (size_t i = 0; i < c.size() && options[k].size() < 2; ++i)
        if (c[i].m != best) options[k].push_back(c[i].m);
      const Candidate* fewest = &c[0];
      for (const auto& x : c)
        if (x.pp.n < fewest->pp.n || (x.pp.n == fewest->pp.n && x.ms < fewest->ms)) fewest = &x;
      if (std::find(options[k].begin(), options[k].end(), fewest->m) == options[k].end()) options[k].push_back(fewest->m);
    }
    if (r.timed.empty()) {  // planner cache from an earlier process: add the fewest-residue class
      auto c = plan_candidates(syms[k], a.L, a.M);
      if (!c.empty()) {
        const Candidate* fewest = &c[0];
        for (const auto& x : c)
          if (x.pp.n < fewest->pp.n) fewest = &x;
        if (fewest->m != best) options[k].push_back(fewest->m);
      }
    }
    for (const auto& x : r.timed) P->report.timed.push_back(x);
  }
  size_t total = 1;
  for (auto& o : options) total *= o.size();
  std::vector<size_t> best(d);
  for (int k = 0; k < d; ++k) best[k] = options[k][0];
  double best_nd_ms = 0.0;
  if (total > 1) {
    size_t elems = 1;
    for (size_t x : data) elems *= x;
    // A synthetic inputs and B outputs (the operator of the plan is the one timed)
    std::vector<double2*> arrs(desc->A + desc->B, nullptr);
    for (size_t i = 0; i < arrs.size(); ++i) {
      CK(cudaMalloc(&arrs[i], elems * sizeof(double2)));
      if (i < desc->A) k_fill_uniform<<<256, 256>>>(7, i, 0, (long long)elems, arrs[i]);
    }
    CK(cudaGetLastError());
    const double2* const* ins = arrs.data();
    double2* const* outs = arrs.data() + desc->A;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double best_ms = 1e30;
    std::vector<size_t> ms(d);
    for (size_t c = 0; c < total; ++c) {
      size_t rem = c;
      for (int k = d - 1; k >= 0; --k) {
        ms[k] = options[k][rem % options[k].size()];
        rem /= options[k].size();
      }
      build_plan(P, ms, syms);
      nd_level(P, 0, 1, ins, outs, 0);
      double t = 1e30;
      for (int r = 0; r < 3; ++r) {
        CK(cudaEventRecord(e0));
        nd_level(P, 0, 1, ins, outs, 0);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float x = 0;
        CK(cudaEventElapsedTime(&x, e0, e1));
        t = std::min<double>(t, x);
      }
      if (diag().fake_timer) t = 1.0;
      if (std::getenv("HCONV_PLAN_VERBOSE")) {
        std::fprintf(stderr, "[hconv tune_nd]");
        for (int k = 0; k < d; ++k) std::fprintf(stderr, " m%d=%zu", k, ms[k]);
        std::fprintf(stderr, " %.3f ms\n", t);
      }
      if (t < best_ms * (1 - 1e-9)) {
        best_ms = t;
        best = ms;
      }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (double2* a : arrs) cudaFree(a);
    best_nd_ms = best_ms;
  }
  std::lock_guard<std::mutex> lk(cache.mu);
  for (int k = 0; k < d; ++k) cache.store(axis_key(k), best[k], best_nd_ms * 1e6);
  return best;
}

}  // namespace

extern "C" {

const char* hconv_backend(void) { return "cuda-sm_100a"; }
const char* hconv_last_error(void) { return g_err.c_str(); }

static void to_abi(const hb::PlanParams& pp, hconv_params* o) {
  o->L = pp.L; o->M = pp.M; o->m = pp.m; o->p = pp.p; o->q = pp.q; o->n = pp.n;
  o->D = pp.D; o->C = pp.C; o->S = pp.S; o->inplace = pp.inplace ? 1 : 0;
  o->symmetry = (int)pp.symmetry; o->regime = (int)pp.regime;
}
static hb::PlanParams from_abi(const hconv_params* a) {
  if (!a) throw std::invalid_argument("null params");
  hb::PlanParams pp = hb::deriveParams(a->L, a->M, a->m, to_sym(a->symmetry));
  pp.C = a->C ? a->C : 1;
  pp.S = a->S ? a->S : 1;
  pp.D = a->D ? a->D : 1;
  pp.inplace = a->inplace != 0;
  return pp;
}

hconv_status hconv_derive_params(size_t L, size_t M, size_t m, int sym, hconv_params* out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null output");
    to_abi(hb::deriveParams(L, M, m, to_sym(sym)), out);
  });
}
size_t hconv_block_length(const hconv_params* pp) {
  try { return from_abi(pp).blockLength(); } catch (...) { return 0; }
}
size_t hconv_stored_length(const hconv_params* pp) {
  try { return from_abi(pp).storedLength(); } catch (...) { return 0; }
}
size_t hconv_padded_length(const hconv_params* pp) {
  try { return from_abi(pp).paddedLength(); } catch (...) { return 0; }
}
hconv_status hconv_root(size_t N, int64_t k, double* re, double* im) {
  return guarded([&] {
    const hb::Complex z = hb::root(N, k);
    *re = z.real();
    *im = z.imag();
  });
}
hconv_status hconv_work_memory_words(const hconv_params* pp, size_t A, size_t B, size_t d, size_t L, uint64_t* iw,
                                     double* ew) {
  return guarded([&] {
    const hb::WorkEstimate w = hb::workMemoryWords(from_abi(pp), A, B, d, L);
    *iw = w.implicitWords;
    *ew = w.explicitWords;
  });
}
hconv_status hconv_root_table(size_t N, double* out) {
  return guarded([&] {
    hb::RootTable t(N);
    for (size_t k = 0; k < N; ++k) {
      out[2 * k] = t.values()[k].real();
      out[2 * k + 1] = t.values()[k].imag();
    }
  });
}
const char* hconv_symmetry_name(int s) {
  if (s < 0 || s > 2) return "?";
  return hb::name(static_cast<hb::Symmetry>(s));
}
hconv_status hconv_symmetry_from_name(const char* n, int* s) {
  return guarded([&] { *s = (int)hb::symmetryFromName(n ? n : ""); });
}

hconv_status hconv_pfft_forward(const hconv_params* pp, const void* f, size_t dist, size_t residue, void* F,
                                void* stream) {
  return guarded([&] {
    const hb::PlanParams p = from_abi(pp);
    if (residue >= p.n) throw std::invalid_argument("residue out of range");
    AxisPlan ap = make_axis(p);
    const long long bl = (long long)p.blockLength();
    const hc::Lines lin{(long long)p.C, 1, (long long)dist, 0, (long long)p.S};
    const hc::Lines lout{(long long)p.C, 1, bl, 0, 1};
    residue_fwd(ap, lin, lout, (const double2*)f, F, (int)residue, 1, (cudaStream_t)stream);
  });
}
hconv_status hconv_pfft_backward(const hconv_params* pp, const void* F, size_t residue, void* h, size_t dist,
                                 int accumulate, void* stream) {
  return guarded([&] {
    const hb::PlanParams p = from_abi(pp);
    if (residue >= p.n) throw std::invalid_argument("residue out of range");
    AxisPlan ap = make_axis(p);
    const long long bl = (long long)p.blockLength();
    const hc::Lines lin{(long long)p.C, 1, bl, 0, 1};
    const hc::Lines lout{(long long)p.C, 1, (long long)dist, 0, (long long)p.S};
    residue_bwd(ap, lin, lout, F, (double2*)h, accumulate ? (const double2*)h : nullptr, 1.0, (int)residue, 1,
                (cudaStream_t)stream);
  });
}

hconv_status hconv_pfft_forward_pair(const hconv_params* pp, const void* f, size_t dist, size_t residue, void* Fv,
                                     void* Fnv, void* stream) {
  return guarded([&] {
    const hb::PlanParams p = from_abi(pp);
    if (p.symmetry != hb::Symmetry::Complex) throw Unsupported("forward_conjugate_pair: complex data only (PAPER.md:795-809)");
    if (residue >= p.n) throw std::invalid_argument("residue out of range");
    if (residue == 0 || 2 * residue == p.n) throw std::invalid_argument("forward_conjugate_pair: self-paired residue");
    const long long C = (long long)p.C, B = (long long)p.blockLength();
    cudaStream_t s = (cudaStream_t)stream;
    if (C == 0) return;
    double2* W = nullptr;  // [Wv | Wn] then the transformed [Xv | Xn]
    CK(cudaMallocAsync(&W, (size_t)(4 * C * B) * sizeof(double2), s));
    const double2* zq = root_table(p.paddedLength());
    const int blocks = (int)std::max<long long>(1, std::min<long long>((C * B + 255) / 256, 8LL * dev_info().sms));
    k_pair_fold<<<blocks, 256, 0, s>>>((const double2*)f, (long long)dist, (long long)p.S, C, (int)p.L, (int)B,
                                       (int)p.paddedLength(), (int)residue, zq, W, W + C * B);
    CK(cudaGetLastError());
    // plain B-point DFTs of the 2C folded lines: residue 0 of the (L = B, M = B, m = B) plan
    const AxisPlan plain = make_axis(hb::deriveParams((size_t)B, (size_t)B, (size_t)B, hb::Symmetry::Complex));
    const hc::Lines lin{2 * C, 1, B, 0, 1};
    residue_fwd(plain, lin, lin, W, W + 2 * C * B, 0, 0, s);
    k_pair_order<<<blocks, 256, 0, s>>>(W + 2 * C * B, C, (int)B, (int)p.interleave(), (int)p.m, (double2*)Fv,
                                        (double2*)Fnv);
    CK(cudaGetLastError());
    CK(cudaFreeAsync(W, s));
  });
}

static hc::Lines to_lines(const hconv_lines* l) {
  if (!l) throw std::invalid_argument("null line batch");
  if (l->nin == 0 || l->es == 0) throw std::invalid_argument("line batch: nin and es must be positive");
  return hc::Lines{(long long)l->count, (long long)l->nin, (long long)l->d_out, (long long)l->d_in, (long long)l->es};
}
hconv_status hconv_pfft_forward_lines(const hconv_params* pp, const void* f, const hconv_lines* in, size_t residue,
                                      void* F, const hconv_lines* out, void* stream) {
  return guarded([&] {
    const hb::PlanParams p = from_abi(pp);
    if (residue >= p.n) throw std::invalid_argument("residue out of range");
    const hc::Lines lin = to_lines(in), lout = to_lines(out);
    if (lin.count != lout.count) throw std::invalid_argument("line batches differ in count");
    AxisPlan ap = make_axis(p);
    residue_fwd(ap, lin, lout, (const double2*)f, F, (int)residue, 0, (cudaStream_t)stream);
  });
}
hconv_status hconv_pfft_backward_lines(const hconv_params* pp, const void* F, const hconv_lines* in, size_t residue,
                                       void* h, const hconv_lines* out, int accumulate, double scale, void* stream) {
  return guarded([&] {
    const hb::PlanParams p = from_abi(pp);
    if (residue >= p.n) throw std::invalid_argument("residue out of range");
    const hc::Lines lin = to_lines(in), lout = to_lines(out);
    if (lin.count != lout.count) throw std::invalid_argument("line batches differ in count");
    AxisPlan ap = make_axis(p);
    residue_bwd(ap, lin, lout, F, (double2*)h, accumulate ? (const double2*)h : nullptr, scale, (int)residue, 0,
                (cudaStream_t)stream);
  });
}

hconv_status hconv_plan_create(const hconv_desc* desc, hconv_plan** out) {
  return guarded([&] {
    check_desc(desc);
    if (!out) throw std::invalid_argument("null output");
    const DeviceGuard dg(desc->device);
    auto P = std::make_unique<hconv_plan>();
    P->d = *desc;
    P->device = desc->device;
    const int d = desc->dims;
    const bool herm = desc->axis[d - 1].symmetry == HCONV_HERMITIAN;
    std::vector<size_t> data(d), ms(d);
    std::vector<hb::Symmetry> syms(d);
    bool tune = false;
    for (int k = 0; k < d; ++k) {
      int s = desc->axis[k].symmetry;
      if (herm && k < d - 1) s = HCONV_CENTERED;  // outer axes of a Hermitian convolution
      syms[k] = to_sym(s);
      data[k] = hb::deriveParams(desc->axis[k].L, desc->axis[k].M, 1, syms[k]).dataLength();
      ms[k] = desc->axis[k].m;
      tune |= ms[k] == 0;
    }
    if (desc->slab) {
      build_slab(P.get(), syms, data);
      P->d.slab = nullptr;  // the configuration lives in P->slab (the caller's struct may go)
      *out = P.release();
      return;
    }
    if (tune) {
      if (d == 1) {
        const long long lines = (long long)(desc->C ? desc->C : 1);
        ms[0] = tune_axis(syms[0], desc->axis[0].L, desc->axis[0].M, lines, &P->report);
      } else {
        ms = tune_nd(P.get(), syms, data);
      }
    }
    if (d == 1 && desc->dist != 0 && desc->dist < data[0])
      throw std::invalid_argument("dist smaller than the data length: copies would overlap");
    build_plan(P.get(), ms, syms);
    *out = P.release();
  });
}

hconv_status hconv_plan_slab(const hconv_plan* p, size_t* x0, size_t* nx) {
  return guarded([&] {
    if (!p || !x0 || !nx) throw std::invalid_argument("null argument");
    if (!p->slab) throw std::invalid_argument("not a slab plan");
    *x0 = p->slab->g.xs[p->slab->g.rank].lo;
    *nx = p->slab->g.nx();
  });
}

hconv_status hconv_nccl_unique_id(void* id128) {
  return guarded([&] {
    if (!id128) throw std::invalid_argument("null argument");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    NC(nccl().GetUniqueId(&id));
    std::memcpy(id128, &id, sizeof(id));
  });
}
hconv_status hconv_nccl_comm_init(const void* id128, int nranks, int rank, int device, void** comm) {
  return guarded([&] {
    if (!id128 || !comm) throw std::invalid_argument("null argument");
    const DeviceGuard dg(device);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t c = nullptr;
    NC(nccl().CommInitRank(&c, nranks, id, rank));
    *comm = c;
  });
}
hconv_status hconv_nccl_comm_destroy(void* comm) {
  return guarded([&] {
    if (comm) NC(nccl().CommDestroy((ncclComm_t)comm));
  });
}

hconv_status hconv_plan_params(const hconv_plan* p, int axis, hconv_params* o) {
  return guarded([&] {
    if (!p || !o || axis < 0 || axis >= (int)p->ax.size()) throw std::invalid_argument("bad axis");
    to_abi(p->ax[axis].pp, o);
  });
}

size_t hconv_plan_workspace_bytes(const hconv_plan* p) {
  if (!p) return 0;
  if (p->slab) return p->slab->drv->buffer_elems() * sizeof(double2) + hconv_plan_workspace_bytes(p->slab->inner);
  size_t b = p->scratch.bytes;
  const int d = p->d.dims;
  for (int l = 0; l + 1 < d; ++l) {
    size_t inner = 1;
    for (int k = l + 1; k < d; ++k) inner *= p->ax[k].data;
    b += (size_t)p->chunk[l] * (p->ax[l].dev.B * p->W() + p->ax[l].data * p->d.B) * inner * sizeof(double2);
  }
  return b + p->gwork.bytes + p->gacc.bytes;
}

// in[A] / out[B] pointer arrays of a call, null-checked
static void io_arrays(const hconv_plan* p, const void* const* in, void* const* out, std::vector<const double2*>& ins,
                      std::vector<double2*>& outs) {
  if (!p || !in || !out) throw std::invalid_argument("null argument");
  // a slab rank may hold no rows (G > L_x): its (empty) arrays may be null
  const bool empty = p->slab && p->slab->g.nx() == 0;
  for (size_t a = 0; a < p->d.A; ++a) {
    if (!in[a] && !empty) throw std::invalid_argument("null input array");
    ins.push_back((const double2*)in[a]);
  }
  for (size_t b = 0; b < p->d.B; ++b) {
    if (!out[b] && !empty) throw std::invalid_argument("null output array");
    outs.push_back((double2*)out[b]);
  }
}

hconv_status hconv_convolve(hconv_plan* p, const void* const* in, void* const* out, void* stream) {
  return guarded([&] {
    std::vector<const double2*> ins;
    std::vector<double2*> outs;
    io_arrays(p, in, out, ins, outs);
    const DeviceGuard dg(p->device);
    cudaStream_t s = (cudaStream_t)stream;
    if (p->slab) {
      slab_convolve(p, ins.data(), outs.data(), s);
    } else if (p->d.dims == 1) {
      const AxisPlan& ap = p->ax[0];
      const long long dist = (long long)(p->d.dist ? p->d.dist : ap.data);
      conv1d(p, ap, (long long)(p->d.C ? p->d.C : 1), dist, ins.data(), outs.data(), s);
    } else {
      nd_level(p, 0, (long long)(p->d.C ? p->d.C : 1), ins.data(), outs.data(), s);
    }
  });
}

hconv_status hconv_convolve_host(hconv_plan* p, const void* const* in, void* const* out) {
  return guarded([&] {
    std::vector<const double2*> hin_;
    std::vector<double2*> hout_;
    io_arrays(p, in, out, hin_, hout_);
    if (p->slab) throw std::invalid_argument("slab plans take device slabs (hconv_convolve)");
    const DeviceGuard dg(p->device);
    HostPipe& hp = p->host;
    hp.init();
    const size_t A = p->d.A, Bo = p->d.B, W = p->W();
    auto hin = [&](size_t a) { return (const char*)hin_[a]; };
    auto hout = [&](size_t b) { return (char*)hout_[b]; };
    if (p->d.dims == 1) {
      const AxisPlan& ap = p->ax[0];
      const long long C = (long long)(p->d.C ? p->d.C : 1), S = (long long)ap.data;
      const long long dist = (long long)(p->d.dist ? p->d.dist : ap.data);
      const long long want = diag().host_chunks;
      const long long nch = std::max<long long>(1, std::min<long long>(C, want));
      const long long per = (C + nch - 1) / nch;
      hp.ensure((size_t)((per - 1) * dist + S), (int)std::min<long long>(nch, HostPipe::kSlots), W);
      int slot = 0;
      for (long long c0 = 0; c0 < C; c0 += per, slot = (slot + 1) % HostPipe::kSlots) {
        const long long cnt = std::min(per, C - c0);
        const size_t off = (size_t)(c0 * dist) * sizeof(double2);
        double2* const* b = hp.buf[slot].data();
        // slot reuse: its previous chunk has been copied back
        CK(cudaStreamWaitEvent(hp.st[0], hp.drained[slot], 0));
        // rows only (the gaps between rows at distance dist are neither read nor written)
        const size_t pitch = (size_t)dist * sizeof(double2), width = (size_t)S * sizeof(double2);
        const bool rows = dist != S;
        for (size_t a = 0; a < A; ++a) {
          if (rows) CK(cudaMemcpy2DAsync(b[a], pitch, hin(a) + off, pitch, width, (size_t)cnt, cudaMemcpyHostToDevice, hp.st[0]));
          else CK(cudaMemcpyAsync(b[a], hin(a) + off, width * (size_t)cnt, cudaMemcpyHostToDevice, hp.st[0]));
        }
        CK(cudaEventRecord(hp.loaded[slot], hp.st[0]));
        CK(cudaStreamWaitEvent(hp.st[1], hp.loaded[slot], 0));
        conv1d(p, ap, cnt, dist, b, b, hp.st[1]);  // in place: outputs in the first B buffers
        CK(cudaEventRecord(hp.done[slot], hp.st[1]));
        CK(cudaStreamWaitEvent(hp.st[2], hp.done[slot], 0));
        for (size_t o = 0; o < Bo; ++o) {
          if (rows) CK(cudaMemcpy2DAsync(hout(o) + off, pitch, b[o], pitch, width, (size_t)cnt, cudaMemcpyDeviceToHost, hp.st[2]));
          else CK(cudaMemcpyAsync(hout(o) + off, b[o], width * (size_t)cnt, cudaMemcpyDeviceToHost, hp.st[2]));
        }
        CK(cudaEventRecord(hp.drained[slot], hp.st[2]));
      }
      CK(cudaStreamSynchronize(hp.st[2]));
    } else {
      const long long C = (long long)(p->d.C ? p->d.C : 1);
      size_t n = (size_t)C;
      for (const AxisPlan& ap : p->ax) n *= ap.data;
      hp.ensure(n, 1, W);
      double2* const* b = hp.buf[0].data();
      for (size_t a = 0; a < A; ++a) CK(cudaMemcpyAsync(b[a], hin(a), n * sizeof(double2), cudaMemcpyHostToDevice, hp.st[1]));
      nd_level(p, 0, C, b, b, hp.st[1]);
      for (size_t o = 0; o < Bo; ++o) CK(cudaMemcpyAsync(hout(o), b[o], n * sizeof(double2), cudaMemcpyDeviceToHost, hp.st[1]));
      CK(cudaStreamSynchronize(hp.st[1]));
    }
  });
}

hconv_status hconv_plan_destroy(hconv_plan* p) {
  delete p;
  return HCONV_OK;
}

// ---- utilities outside the reference API (bench / tests) ----
hconv_status hconv_util_fill_uniform(uint64_t seed, uint64_t a, uint64_t first_index, size_t count, void* out,
                                     void* stream) {
  return guarded([&] {
    if (count == 0) return;
    const int blocks = (int)std::min<size_t>((count + 255) / 256, 4096);
    k_fill_uniform<<<blocks, 256, 0, (cudaStream_t)stream>>>(seed, a, first_index, (long long)count, (double2*)out);
    CK(cudaGetLastError());
  });
}

// planner report: up to cap candidates as (m, p, q, n, block, median ms); returns the count
int hconv_plan_report(const hconv_plan* p, double* out, int cap) {
  if (!p) return 0;
  int k = 0;
  for (const auto& c : p->report.timed) {
    if (k >= cap) break;
    double* r = out + 7 * k++;
    r[0] = (double)c.m; r[1] = (double)c.pp.p; r[2] = (double)c.pp.q; r[3] = (double)c.pp.n;
    r[4] = (double)c.pp.blockLength(); r[5] = c.ms; r[6] = c.explicit_ ? 1.0 : 0.0;
  }
  return p->report.cached ? -k - 1 : k;
}

hconv_mult_fn hconv_example_mult(int which) { return which == 0 ? example_mult_pairs : nullptr; }

// kernel description for a plan axis: threads per line group, groups per CTA, radix plan
const char* hconv_plan_kernel(const hconv_plan* p, int axis) {
  if (!p || axis < 0 || axis >= (int)p->ax.size()) return "";
  const AxisPlan& ap = p->ax[axis];
  // 1D plans whose unit-stride lines run the in-place two-residue kernel (launch_conv)
  if (p->ax.size() == 1 && ap.ip_fn && !diag().no_ip && ap.dev.L <= ap.dev.B && ap.dev.n == hc::conv_ip_residues(ap.dev.Bc))
    return "16x24x16 in place, two residues";
  return ap.k->radix;
}

}  // extern "C"
