// Elementwise median over the D family estimates (median_reduce,
// estimators.cpp:117-138): even D averages the two middle order statistics,
// which is the value std::sort + middle pick yields for finite inputs.
// Shared by median_kernel (spectral.cu) and the fused tail of the cluster
// estimator (spectral_cluster.cu); `ld` loads one value (plain, or an
// L2-coherent load for estimates written earlier in the same kernel).
#pragma once

#include <math_constants.h>

namespace fcs {

// Finite values, D <= N: all D values in registers (fully unrolled, padded
// with +inf) and the order statistics by rank counting. Returns false (caller
// falls back) on a non-finite input.
template <int N, typename Ld>
__device__ __forceinline__ bool median_regs(const double* col, int D, int len, double* res, Ld ld) {
  double v[N];
  bool finite = true;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    v[k] = k < D ? ld(col + static_cast<size_t>(k) * len) : CUDART_INF;
    if (k < D) finite &= isfinite(v[k]);
  }
  if (!finite) return false;
  const int m1 = (D - 1) / 2, m2 = D / 2;  // equal for odd D
  double lo = 0.0, hi = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    int less = 0, eq = 0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      less += v[j] < v[k];
      eq += v[j] == v[k];
    }
    if (k < D) {
      if (less <= m1 && m1 < less + eq) lo = v[k];
      if (less <= m2 && m2 < less + eq) hi = v[k];
    }
  }
  *res = (D & 1) ? hi : 0.5 * (lo + hi);
  return true;
}

// Median of col[0], col[len], ..., col[(D - 1) len].
template <typename Ld>
__device__ __forceinline__ double median_col(const double* col, int D, int len, Ld ld) {
  double r;
  bool ok = false;
  switch (D) {  // exact register counts for the common family counts
#define FCS_MEDIAN_CASE(n) \
  case n: ok = median_regs<n>(col, D, len, &r, ld); break;
    FCS_MEDIAN_CASE(1) FCS_MEDIAN_CASE(2) FCS_MEDIAN_CASE(3) FCS_MEDIAN_CASE(4)
    FCS_MEDIAN_CASE(5) FCS_MEDIAN_CASE(6) FCS_MEDIAN_CASE(7) FCS_MEDIAN_CASE(8)
    FCS_MEDIAN_CASE(9) FCS_MEDIAN_CASE(10) FCS_MEDIAN_CASE(11) FCS_MEDIAN_CASE(12)
    FCS_MEDIAN_CASE(13) FCS_MEDIAN_CASE(14) FCS_MEDIAN_CASE(15) FCS_MEDIAN_CASE(16)
#undef FCS_MEDIAN_CASE
    default: break;
  }
  if (ok) return r;
  if (D > 64) {
    // rank selection without storage (O(D^2)): x_k is the m-th order
    // statistic iff #less <= m < #less + #equal (std::sort order for finite values)
    auto order_stat = [&](int m) {
      for (int k = 0; k < D; ++k) {
        const double x = ld(col + static_cast<size_t>(k) * len);
        int less = 0, eq = 0;
        for (int j = 0; j < D; ++j) {
          const double y = ld(col + static_cast<size_t>(j) * len);
          less += y < x;
          eq += y == x;
        }
        if (less <= m && m < less + eq) return x;
      }
      return ld(col);  // non-finite input: no consistent order
    };
    return (D & 1) ? order_stat(D / 2) : 0.5 * (order_stat(D / 2 - 1) + order_stat(D / 2));
  }
  double v[64];
  for (int d = 0; d < D; ++d) {
    const double x = ld(col + static_cast<size_t>(d) * len);
    int k = d;
    while (k > 0 && v[k - 1] > x) {
      v[k] = v[k - 1];
      --k;
    }
    v[k] = x;
  }
  return (D & 1) ? v[D / 2] : 0.5 * (v[D / 2 - 1] + v[D / 2]);
}

// median_col for D <= 16 with at most a 16-entry local array (the
// non-finite fallback): for kernels whose stack frame must stay small
// (the fused tails of the one-CTA estimators share SMs with the cluster
// kernel; median_col's 64-entry sort array doubled the one-CTA kernel's
// stack and broke that co-residency — measured).
template <typename Ld>
__device__ __forceinline__ double median_col16(const double* col, int D, int len, Ld ld) {
  double r;
  bool ok = false;
  switch (D) {
#define FCS_MEDIAN_CASE(n) \
  case n: ok = median_regs<n>(col, D, len, &r, ld); break;
    FCS_MEDIAN_CASE(1) FCS_MEDIAN_CASE(2) FCS_MEDIAN_CASE(3) FCS_MEDIAN_CASE(4)
    FCS_MEDIAN_CASE(5) FCS_MEDIAN_CASE(6) FCS_MEDIAN_CASE(7) FCS_MEDIAN_CASE(8)
    FCS_MEDIAN_CASE(9) FCS_MEDIAN_CASE(10) FCS_MEDIAN_CASE(11) FCS_MEDIAN_CASE(12)
    FCS_MEDIAN_CASE(13) FCS_MEDIAN_CASE(14) FCS_MEDIAN_CASE(15) FCS_MEDIAN_CASE(16)
#undef FCS_MEDIAN_CASE
    default: break;
  }
  if (ok) return r;
  double v[16];  // the same insertion sort as median_col's fallback
  for (int d = 0; d < D; ++d) {
    const double x = ld(col + static_cast<size_t>(d) * len);
    int k = d;
    while (k > 0 && v[k - 1] > x) {
      v[k] = v[k - 1];
      --k;
    }
    v[k] = x;
  }
  return (D & 1) ? v[D / 2] : 0.5 * (v[D / 2 - 1] + v[D / 2]);
}

}  // namespace fcs
