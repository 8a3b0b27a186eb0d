// Fused estimator tail for kernels with one CTA per (vector, family) item
// (iuv1_kernel in spectral.cu, corr_z_kernel in correlate.cu): the last CTA of
// vector `bvec` to finish (per-vector arrival counter, `arrivals` CTAs per
// vector) takes the median over the D families (median_reduce,
// estimators.cpp:117-138) and, by mode, normalises the row (the rtpm restart
// step, cpd.cpp:253-257) or applies the refinement update (cpd.cpp:266-270) —
// the single-CTA form of the cluster estimator's IuvTail (spectral_cluster.cu).
#pragma once

#include "fft.cuh"
#include "median.cuh"

namespace fcs {

// D <= 16 (callers fall back to the separate median kernels beyond).
// est: per-family values, vector-major (bvec * D + d) * nt + i, nt = nf (the
// row) or 1 (mode 4, one contraction value per family). Call from every
// thread of the CTA after its estimates are written; returns immediately
// unless this CTA is the vector's last arrival.
// `red`: caller's shared scratch of kThreads / 32 + 1 doubles (no static
// shared memory here: the one-CTA estimator's co-residency with the cluster
// kernel on the same SMs depends on its exact footprint).
template <int kThreads>
__device__ __forceinline__ void estimator_tail(const IuvTail& tail, const double* est, int bvec,
                                               int D, int nt, int arrivals, double* red) {
  volatile int* last = reinterpret_cast<volatile int*>(red + kThreads / 32);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int old = atomicAdd(tail.cnt + bvec, 1);
    const int is_last = old == arrivals - 1;
    if (is_last) tail.cnt[bvec] = 0;  // every CTA of bvec has arrived: ready for the next launch
    *last = is_last;
  }
  __syncthreads();
  if (!*last) return;
  __threadfence();
  if (tail.mode == 3 && *reinterpret_cast<volatile int*>(tail.stopped)) return;
  const double* col0 = est + static_cast<size_t>(bvec) * D * nt;
  double* ob = tail.out + static_cast<size_t>(bvec) * nt;
  double acc = 0.0;
  for (int i = threadIdx.x; i < nt; i += kThreads) {
    const double m = median_col16(col0 + i, D, nt, [](const double* p) { return __ldcg(p); });
    ob[i] = m;
    acc += m * m;
  }
  if (tail.mode == 1 || tail.mode == 4) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  double tot = 0.0;
#pragma unroll
  for (int k = 0; k < kThreads / 32; ++k) tot += red[k];
  const double nv = sqrt(tot);
  if (tail.mode == 2) {
    for (int i = threadIdx.x; i < nt; i += kThreads) ob[i] = nv < 1e-150 ? 0.0 : ob[i] / nv;
  } else {
    if (nv < 1e-150) {
      if (threadIdx.x == 0) *tail.stopped = 1;
      return;
    }
    for (int i = threadIdx.x; i < nt; i += kThreads) tail.best[i] = ob[i] / nv;
  }
}

}  // namespace fcs
