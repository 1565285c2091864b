// naive.cuh — direct-sum (O(B^2)) residue kernels for block sizes without a radix plan
// (small or non-7-smooth m used by the parity grids).  Same pre/post-processing as the
// radix kernels (block_io.cuh); the B-point DFT is a shared-memory direct sum.  The planner
// only selects these for blocks of at most kNaiveMax points.
#pragma once
#include "kernels.cuh"

namespace hc {

constexpr int kNaiveT = 128;
constexpr int kNaiveMax = 2048;

// Hermitian blocks of odd length B cannot use the B/2 packing: the naive path then runs the
// full B-point transform of the Hermitian W (Bc == B) and keeps the real part.
template <int SYM>
__device__ __forceinline__ double2 load_naive(const AxisDev& a, const double2* f, long long es, int s, int v) {
  if constexpr (SYM == SYM_HERMITIAN) {
    if (a.Bc == a.B) return load_WH(a, f, es, s, v);
  }
  return load_in<SYM>(a, f, es, s, v);
}
__device__ __forceinline__ double2 herm_naive(const AxisDev& a, const double2* W, int j, int v) {
  if (a.Bc != a.B) return herm_w(a, W, j, v);
  return v ? cmulc(W[j], zpow(a, v * j)) : W[j];
}

template <int DIR>
__device__ __forceinline__ double2 dft_at(const double2* X, const double2* __restrict__ tw, int Bc, int k) {
  double2 acc = make_double2(0.0, 0.0);
  int e = 0;
  for (int s = 0; s < Bc; ++s) {
    acc = cadd(acc, mul_tw<DIR>(X[s], __ldg(tw + e)));
    e += k;
    if (e >= Bc) e -= Bc;
  }
  return acc;
}

template <int SYM>
__global__ void __launch_bounds__(kNaiveT) k_conv1d_naive(ConvArgs p) {
  extern __shared__ double2 smem[];
  const AxisDev& a = p.ax;
  const int Bc = a.Bc, tid = threadIdx.x;
  double2 *W = smem, *F = smem + Bc, *Y = smem + 2 * Bc;
  double2* slot = p.scratch + (long long)blockIdx.x * a.S;
  for (long long item = blockIdx.x; item < p.lin.count; item += gridDim.x) {
    const long long base = p.lin.base(item), es = p.lin.es;
    for (int res = 0; res < a.n; ++res) {
      for (int s = tid; s < Bc; s += kNaiveT) W[s] = load_naive<SYM>(a, p.f + base, es, s, res);
      __syncthreads();
      for (int k = tid; k < Bc; k += kNaiveT) F[k] = dft_at<+1>(W, a.tw, Bc, k);
      __syncthreads();
      for (int s = tid; s < Bc; s += kNaiveT) W[s] = load_naive<SYM>(a, p.g + base, es, s, res);
      __syncthreads();
      for (int k = tid; k < Bc; k += kNaiveT) {
        const double2 G = dft_at<+1>(W, a.tw, Bc, k), Fk = F[k];
        Y[k] = SYM != SYM_HERMITIAN ? cmul(G, Fk)
               : (Bc == a.B ? make_double2(G.x * Fk.x, 0.0) : make_double2(G.x * Fk.x, G.y * Fk.y));
      }
      __syncthreads();
      for (int s = tid; s < Bc; s += kNaiveT) W[s] = dft_at<-1>(Y, a.tw, Bc, s);
      __syncthreads();
      const bool last = res == a.n - 1;
      const Emit em = last ? Emit{p.out + base, es, res > 0 ? slot : nullptr, 1, 1.0 / (double)a.qm}
                           : Emit{slot, 1, res > 0 ? slot : nullptr, 1, 1.0};
      if constexpr (SYM == SYM_HERMITIAN) {
        for (int j = tid; j < a.S; j += kNaiveT) em(j, herm_naive(a, W, j, res));
      } else {
        for (int s = tid; s < Bc; s += kNaiveT) store_w<SYM>(a, em, s, res, W[s]);
      }
      __syncthreads();
    }
  }
}

template <int SYM>
__global__ void __launch_bounds__(kNaiveT) k_pfft_fwd_naive(FwdArgs p) {
  extern __shared__ double2 smem[];
  const AxisDev& a = p.ax;
  const int Bc = a.Bc, tid = threadIdx.x;
  double2* W = smem;
  for (long long item = blockIdx.x; item < p.lin.count; item += gridDim.x) {
    for (int s = tid; s < Bc; s += kNaiveT) W[s] = load_naive<SYM>(a, p.f + p.lin.base(item), p.lin.es, s, p.v);
    __syncthreads();
    const long long ob = p.lout.base(item), oes = p.lout.es;
    for (int k = tid; k < Bc; k += kNaiveT) {
      const double2 val = dft_at<+1>(W, a.tw, Bc, k);
      if constexpr (SYM == SYM_HERMITIAN) {
        double* F = (double*)p.F;
        if (Bc == a.B) {
          F[ob + (p.ref_order ? ref_index(a, k) : k) * oes] = val.x;
        } else {
          F[ob + (p.ref_order ? ref_index(a, 2 * k) : 2 * k) * oes] = val.x;
          F[ob + (p.ref_order ? ref_index(a, 2 * k + 1) : 2 * k + 1) * oes] = val.y;
        }
      } else {
        ((double2*)p.F)[ob + (p.ref_order ? ref_index(a, k) : k) * oes] = val;
      }
    }
    __syncthreads();
  }
}

template <int SYM>
__global__ void __launch_bounds__(kNaiveT) k_pfft_bwd_naive(BwdArgs p) {
  extern __shared__ double2 smem[];
  const AxisDev& a = p.ax;
  const int Bc = a.Bc, tid = threadIdx.x;
  double2 *Y = smem, *W = smem + Bc;
  for (long long item = blockIdx.x; item < p.lin.count; item += gridDim.x) {
    const long long ib = p.lin.base(item), ies = p.lin.es;
    for (int k = tid; k < Bc; k += kNaiveT) {
      if constexpr (SYM == SYM_HERMITIAN) {
        const double* F = (const double*)p.F;
        Y[k] = Bc == a.B ? make_double2(F[ib + (p.ref_order ? ref_index(a, k) : k) * ies], 0.0)
                         : make_double2(F[ib + (p.ref_order ? ref_index(a, 2 * k) : 2 * k) * ies],
                                        F[ib + (p.ref_order ? ref_index(a, 2 * k + 1) : 2 * k + 1) * ies]);
      } else {
        Y[k] = ((const double2*)p.F)[ib + (p.ref_order ? ref_index(a, k) : k) * ies];
      }
    }
    __syncthreads();
    for (int s = tid; s < Bc; s += kNaiveT) W[s] = dft_at<-1>(Y, a.tw, Bc, s);
    __syncthreads();
    const long long ob = p.lout.base(item);
    const Emit em{p.dst + ob, p.lout.es, p.acc ? p.acc + ob : nullptr, p.lout.es, p.scale};
    if constexpr (SYM == SYM_HERMITIAN) {
      for (int j = tid; j < a.S; j += kNaiveT) em(j, herm_naive(a, W, j, p.v));
    } else {
      for (int s = tid; s < Bc; s += kNaiveT) store_w<SYM>(a, em, s, p.v, W[s]);
    }
    __syncthreads();
  }
}

}  // namespace hc
