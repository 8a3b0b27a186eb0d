// Spectral FCS kernels (K2-K9): CP-form FCS, batched linear convolution,
// and the sketched-contraction estimators T(I,a,b) / T(u,v,w) with the D
// families batched per launch, all built on the shared-memory FFT of fft.cuh.
//
// One CTA owns one (item, family) transform; every real sequence is count-
// sketched straight into the CTA's shared FFT buffer (K2 fused into the FFT
// prologue), and products / sums over rank happen in the frequency domain
// (K4) so each output needs a single inverse transform (K5).
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdlib>

#include <math_constants.h>

#include "fft.cuh"
#include "median.cuh"

namespace fcs {

namespace {

__device__ __forceinline__ int tid() { return threadIdx.x; }

// Shared memory carve-up: twiddles, then one or two P-slot FFT buffers, then a
// 32-double reduction scratch.
struct Smem {
  double2* tw;
  double2* buf;
  double2* buf2;  // second buffer (two-buffer kernels only)
  double* red;
};

__device__ __forceinline__ Smem carve(const FftPlan& pl, int nbuf = 1) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem s;
  s.tw = reinterpret_cast<double2*>(smem_raw);
  s.buf = s.tw + table_slots(pl, false);  // no frequency -> slot table here
  s.buf2 = nbuf > 1 ? s.buf + pl.P : nullptr;
  s.red = reinterpret_cast<double*>(s.buf + static_cast<size_t>(nbuf) * pl.P);
  return s;
}

// Count sketch of vec[0..I) under a packed pair, scattered into the packed
// real buffer (cs_sketch, sketch.cpp:105-116: zeros skipped).
__device__ void scatter_cs(double2* buf, const double* __restrict__ vec, int I,
                           const uint32_t* __restrict__ tab) {
  for (int i = tid(); i < I; i += blockDim.x) {
    const double v = vec[i];
    if (v != 0.0) {
      const uint32_t e = __ldg(tab + i);
      atomicAdd(&packed_real(buf, e & 0x7fffffffu), (e >> 31) ? -v : v);
    }
  }
}

// Count sketch then the length-M real transform -> half spectrum in slot order.
// zeroed: the caller already cleared buf (fused into its last read of it) and
// synchronised.
__device__ void rfft_of_cs(const Smem& sm, double2* buf, const FftPlan& pl,
                           const double* __restrict__ vec, int I,
                           const uint32_t* __restrict__ tab, bool zeroed = false) {
  if (!zeroed) {
    zero_slots(buf, pl.P);
    __syncthreads();
  }
  scatter_cs(buf, vec, I, tab);
  cp_async_wait_all();  // twiddles of load_twiddles_async (no-op otherwise)
  __syncthreads();
  fft_forward_post(buf, pl, sm.tw);
  __syncthreads();
}

// Two count sketches transformed together (sm.buf <- a, sm.buf2 <- b).
__device__ void rfft_of_cs2(const Smem& sm, const FftPlan& pl, const double* __restrict__ va,
                            int Ia, const uint32_t* __restrict__ ta,
                            const double* __restrict__ vb, int Ib,
                            const uint32_t* __restrict__ tb) {
  zero_slots(sm.buf, pl.P);
  zero_slots(sm.buf2, pl.P);
  __syncthreads();
  scatter_cs(sm.buf, va, Ia, ta);
  scatter_cs(sm.buf2, vb, Ib, tb);
  __syncthreads();
  fft_forward2_post(sm.buf, sm.buf2, pl, sm.tw);
  __syncthreads();
}

// Zero-padded real x[0..len) -> half spectrum (dft, fft.cpp:42-51).
__device__ void rfft_of_real(const Smem& sm, const FftPlan& pl, const double* __restrict__ x,
                             int len) {
  for (int s = tid(); s < pl.P; s += blockDim.x) {
    const int t = 2 * s;
    sm.buf[swz(s)] = make_double2(t < len ? x[t] : 0.0, t + 1 < len ? x[t + 1] : 0.0);
  }
  __syncthreads();
  fft_forward_post(sm.buf, pl, sm.tw);
  __syncthreads();
}

// Half spectrum already in sm.buf -> natural-order real sequence scaled by P
// (caller divides by P; idft_real's 1/n, fft.cpp:61-66).
__device__ void irfft_in_place(const Smem& sm, const FftPlan& pl) {
  __syncthreads();
  fft_inverse_pre(sm.buf, pl, sm.tw);
}

__device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < static_cast<int>(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

}  // namespace

// --------------------------------------------------------------- kernels
__global__ void __launch_bounds__(kFftThreads) spec_from_real_kernel(FftPlan pl, const double* x,
                                                                     size_t ldx, int len,
                                                                     double2* spec) {
  const Smem sm = carve(pl);
  load_twiddles(sm.tw, pl, false);
  __syncthreads();
  rfft_of_real(sm, pl, x + blockIdx.x * ldx, len);
  double2* o = spec + static_cast<size_t>(blockIdx.x) * pl.P;
  for (int s = tid(); s < pl.P; s += blockDim.x) o[s] = sm.buf[swz(s)];
}

__global__ void __launch_bounds__(kFftThreads) real_from_spec_kernel(FftPlan pl,
                                                                     const double2* spec,
                                                                     double* out, size_t ldo,
                                                                     int out_len, int accumulate) {
  const Smem sm = carve(pl);
  load_twiddles(sm.tw, pl, false);
  const double2* in = spec + static_cast<size_t>(blockIdx.x) * pl.P;
  for (int s = tid(); s < pl.P; s += blockDim.x) sm.buf[swz(s)] = in[s];
  irfft_in_place(sm, pl);
  const double inv = 1.0 / pl.P;
  double* o = out + blockIdx.x * ldo;
  for (int t = tid(); t < out_len; t += blockDim.x) {
    const double v = packed_real(sm.buf, t) * inv;
    o[t] = accumulate ? o[t] + v : v;
  }
}

// K2-K4: per (rank r, family d) the product of the mode spectra times w_r.
__global__ void __launch_bounds__(kFftThreads) cp_rank_kernel(FftPlan pl, CpArgs a,
                                                              const uint32_t* __restrict__ packed,
                                                              double2* __restrict__ Q) {
  const Smem sm = carve(pl, 2);
  load_twiddles(sm.tw, pl, false);
  const int rl = blockIdx.x, d = blockIdx.y;
  const int r = a.r_begin + rl;
  const double w = a.weights[r];
  double2* q = Q + (static_cast<size_t>(d) * a.r_count + rl) * pl.P;
  const uint32_t* tab = packed + static_cast<size_t>(d) * a.fam_stride;
  if (w == 0.0) return;  // convolved_cp_sketch skips zero weights (sketch.cpp:75)
  auto col = [&](int n) { return a.factors[n] + static_cast<size_t>(r) * a.dims[n]; };
  // modes 0 and 1 together, then the product accumulates in sm.buf and every
  // further mode is transformed in sm.buf2
  int n = 1;
  if (a.order >= 2) {
    __syncthreads();
    rfft_of_cs2(sm, pl, col(0), a.dims[0], tab + a.tab_off[0], col(1), a.dims[1],
                tab + a.tab_off[1]);
    for (int s = tid(); s < pl.P; s += blockDim.x)
      sm.buf[swz(s)] = hmul(sm.buf[swz(s)], sm.buf2[swz(s)], s == 0);
    n = 2;
  } else {
    __syncthreads();
    rfft_of_cs(sm, sm.buf, pl, col(0), a.dims[0], tab + a.tab_off[0]);
  }
  for (; n < a.order; ++n) {
    __syncthreads();
    rfft_of_cs(sm, sm.buf2, pl, col(n), a.dims[n], tab + a.tab_off[n]);
    for (int s = tid(); s < pl.P; s += blockDim.x)
      sm.buf[swz(s)] = hmul(sm.buf[swz(s)], sm.buf2[swz(s)], s == 0);
  }
  __syncthreads();
  for (int s = tid(); s < pl.P; s += blockDim.x) q[s] = cscale(sm.buf[swz(s)], w);
}

// K2-K4, one-buffer form: the product over modes accumulates in the item's Q
// slot (each thread re-reads only the slots it wrote, L2-resident), so shared
// memory is one buffer plus the tables and two CTAs fit per SM — fewer waves
// when the (rank, family) items are several times the SM count (config 2:
// 500 items of P = 6144).
__global__ void __launch_bounds__(kFftThreads, 2) cp_rank1_kernel(FftPlan pl, CpArgs a,
                                                                  const uint32_t* __restrict__ packed,
                                                                  double2* __restrict__ Q) {
  const Smem sm = carve(pl, 1);
  load_twiddles_async(sm.tw, pl);
  const int rl = blockIdx.x, d = blockIdx.y;
  const int r = a.r_begin + rl;
  const double w = a.weights[r];
  double2* q = Q + (static_cast<size_t>(d) * a.r_count + rl) * pl.P;
  const uint32_t* tab = packed + static_cast<size_t>(d) * a.fam_stride;
  if (w == 0.0) return;  // convolved_cp_sketch skips zero weights (sketch.cpp:75)
  for (int n = 0; n < a.order; ++n) {
    __syncthreads();
    rfft_of_cs(sm, sm.buf, pl, a.factors[n] + static_cast<size_t>(r) * a.dims[n], a.dims[n],
               tab + a.tab_off[n], n > 0);
    const bool last = n + 1 == a.order;
    for (int s = tid(); s < pl.P; s += blockDim.x) {
      double2 v = sm.buf[swz(s)];
      if (!last) sm.buf[swz(s)] = make_double2(0.0, 0.0);  // cleared for the next mode
      if (n > 0) v = hmul(q[s], v, s == 0);
      q[s] = last ? cscale(v, w) : v;
    }
  }
}

// K4: fixed-order sum over ranks, parallel over (slot, family): acc[d][s] =
// sum_{r: w_r != 0} Q[d][r][s] (convolved_cp_sketch sums per rank, sketch.cpp:73-84;
// here in the frequency domain by linearity).
__global__ void cp_rank_sum_kernel(const double2* __restrict__ Q, const double* __restrict__ weights,
                                   int r_begin, int r_count, int P, double2* __restrict__ acc) {
  // 32 slots x 8 rank lanes: lane y sums ranks y, y + 8, ... (several loads in
  // flight per slot), then the 8 lane sums are added in lane order — a fixed order
  __shared__ double2 red[8][32];
  const int s = blockIdx.x * 32 + threadIdx.x;
  const int d = blockIdx.y;
  double2 a = make_double2(0.0, 0.0);
  if (s < P) {
    const double2* q = Q + static_cast<size_t>(d) * r_count * P + s;
    for (int rl = threadIdx.y; rl < r_count; rl += 8) {
      if (weights[r_begin + rl] == 0.0) continue;
      a = cadd(a, q[static_cast<size_t>(rl) * P]);
    }
  }
  red[threadIdx.y][threadIdx.x] = a;
  __syncthreads();
  if (threadIdx.y == 0 && s < P) {
    double2 t = red[0][threadIdx.x];
#pragma unroll
    for (int y = 1; y < 8; ++y) t = cadd(t, red[y][threadIdx.x]);
    acc[static_cast<size_t>(d) * P + s] = t;
  }
}

// K5: one inverse transform per family, first J~ values into out.
__global__ void __launch_bounds__(2 * kFftThreads, 1) cp_sum_kernel(FftPlan pl,
                                                             const double2* __restrict__ acc,
                                                             double* out, int jt, int accumulate) {
  const Smem sm = carve(pl);
  load_twiddles(sm.tw, pl, false);
  const int d = blockIdx.x;
  const double2* a = acc + static_cast<size_t>(d) * pl.P;
  for (int s = tid(); s < pl.P; s += blockDim.x) sm.buf[swz(s)] = a[s];
  irfft_in_place(sm, pl);
  const double inv = 1.0 / pl.P;
  double* o = out + static_cast<size_t>(d) * jt;
  for (int t = tid(); t < jt; t += blockDim.x) {
    const double v = packed_real(sm.buf, t) * inv;
    o[t] = accumulate ? o[t] + v : v;
  }
}

// Linear convolution of row pairs: out[b] = a[b] (*) b[b] (fft_convolve, fft.cpp:75-84).
__global__ void __launch_bounds__(kFftThreads) conv_kernel(FftPlan pl, const double* a, int la,
                                                           size_t lda, const double* b, int lb,
                                                           size_t ldb, double2* scratch,
                                                           double* out, size_t ldo) {
  const Smem sm = carve(pl);
  load_twiddles(sm.tw, pl, false);
  __syncthreads();
  const int item = blockIdx.x;
  double2* scr = scratch + static_cast<size_t>(item) * pl.P;
  rfft_of_real(sm, pl, a + item * lda, la);
  for (int s = tid(); s < pl.P; s += blockDim.x) scr[s] = sm.buf[swz(s)];
  __syncthreads();
  rfft_of_real(sm, pl, b + item * ldb, lb);
  for (int s = tid(); s < pl.P; s += blockDim.x) sm.buf[swz(s)] = hmul(scr[s], sm.buf[swz(s)], s == 0);
  irfft_in_place(sm, pl);
  const double inv = 1.0 / pl.P;
  const int lo = la + lb - 1;
  double* o = out + item * ldo;
  for (int t = tid(); t < lo; t += blockDim.x) o[t] = packed_real(sm.buf, t) * inv;
}

// K6: z = IFFT(S_d conj(F cs_a) conj(F cs_b)); est = s_f(i) z[h_f(i)]
// (iuv_spectral, estimators.cpp:66-90). Grid (batch, D).
__global__ void __launch_bounds__(kFftThreads) iuv_kernel(FftPlan pl, EngArgs e, const double* A,
                                                          const double* B, int c1, int c2, int f,
                                                          double2* scratch, double* est) {
  (void)scratch;
  const Smem sm = carve(pl, 2);
  load_twiddles(sm.tw, pl, false);
  __syncthreads();
  const int b = blockIdx.x, d = blockIdx.y;
  const size_t item = static_cast<size_t>(b) * e.D + d;
  const uint32_t* tab = e.packed + static_cast<size_t>(d) * e.fam_stride;
  const double2* S = e.spec + static_cast<size_t>(d) * pl.P;
  rfft_of_cs2(sm, pl, A + static_cast<size_t>(b) * e.dims[c1], e.dims[c1], tab + e.tab_off[c1],
              B + static_cast<size_t>(b) * e.dims[c2], e.dims[c2], tab + e.tab_off[c2]);
  constexpr int kU = 6;  // S loads of kU slots in flight
  for (int s0 = tid(); s0 < pl.P; s0 += kU * blockDim.x) {
    double2 sv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int s = s0 + u * blockDim.x;
      if (s < pl.P) sv[u] = __ldg(S + s);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int s = s0 + u * blockDim.x;
      if (s >= pl.P) continue;
      const bool z = s == 0;
      const double2 ab = hmul(sm.buf[swz(s)], sm.buf2[swz(s)], z);
      sm.buf[swz(s)] = hmul(sv[u], hconj(ab, z), z);
    }
  }
  irfft_in_place(sm, pl);
  const double inv = 1.0 / pl.P;
  const int nf = e.dims[f];
  const uint32_t* tf = tab + e.tab_off[f];
  double* o = est + item * nf;
  for (int i = tid(); i < nf; i += blockDim.x) {
    const uint32_t t = __ldg(tf + i);
    const double z = packed_real(sm.buf, t & 0x7fffffffu) * inv;
    o[i] = (t >> 31) ? -z : z;
  }
}

// K6, one-buffer form: F cs_a goes through a global scratch slot instead of a
// second shared buffer, halving shared memory so two CTAs fit per SM. Used when
// the batch is slightly above one wave of the two-buffer kernel (config 3:
// 15 x 10 = 150 items on 148 SMs), where it removes the nearly empty second wave.
// wdot != nullptr: T(u, v, w) by linearity — est[item] = <w_b, T_d(u, v, I)>
// instead of the free-mode vector (the uvw estimate, one transform fewer than
// uvw_kernel's three forward ones).
__global__ void __launch_bounds__(kFftThreads, 2) iuv1_kernel(FftPlan pl, EngArgs e, const double* A,
                                                           const double* B, int c1, int c2, int f,
                                                           double2* scratch, double* est,
                                                           const double* wdot = nullptr) {
  const Smem sm = carve(pl, 1);
  load_twiddles_async(sm.tw, pl);
  const int b = blockIdx.x, d = blockIdx.y;
  const size_t item = static_cast<size_t>(b) * e.D + d;
  const uint32_t* tab = e.packed + static_cast<size_t>(d) * e.fam_stride;
  const double2* S = e.spec + static_cast<size_t>(d) * pl.P;
  double2* scr = scratch + item * pl.P;
  rfft_of_cs(sm, sm.buf, pl, A + static_cast<size_t>(b) * e.dims[c1], e.dims[c1],
             tab + e.tab_off[c1]);
  for (int s = tid(); s < pl.P; s += blockDim.x) {
    scr[s] = sm.buf[swz(s)];
    sm.buf[swz(s)] = make_double2(0.0, 0.0);  // cleared for cs_b
  }
  __syncthreads();
  rfft_of_cs(sm, sm.buf, pl, B + static_cast<size_t>(b) * e.dims[c2], e.dims[c2],
             tab + e.tab_off[c2], true);
  // kU slots per thread per step with their scr / S loads (L2) in flight together
  constexpr int kU = 4;
  for (int s0 = tid(); s0 < pl.P; s0 += kU * blockDim.x) {
    double2 fa[kU], sv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int s = s0 + u * blockDim.x;
      if (s < pl.P) {
        fa[u] = __ldcg(scr + s);
        sv[u] = __ldg(S + s);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int s = s0 + u * blockDim.x;
      if (s >= pl.P) continue;
      const bool z = s == 0;
      const double2 ab = hmul(fa[u], sm.buf[swz(s)], z);
      sm.buf[swz(s)] = hmul(sv[u], hconj(ab, z), z);
    }
  }
  irfft_in_place(sm, pl);
  const double inv = 1.0 / pl.P;
  const int nf = e.dims[f];
  const uint32_t* tf = tab + e.tab_off[f];
  if (wdot != nullptr) {
    const double* wv = wdot + static_cast<size_t>(b) * nf;
    double acc = 0.0;
    for (int i = tid(); i < nf; i += blockDim.x) {
      const uint32_t t = __ldg(tf + i);
      const double z = packed_real(sm.buf, t & 0x7fffffffu) * inv;
      acc += wv[i] * ((t >> 31) ? -z : z);
    }
    const double tot = block_sum(acc, sm.red);
    if (tid() == 0) est[item] = tot;
    return;
  }
  double* o = est + item * nf;
  for (int i = tid(); i < nf; i += blockDim.x) {
    const uint32_t t = __ldg(tf + i);
    const double z = packed_real(sm.buf, t & 0x7fffffffu) * inv;
    o[i] = (t >> 31) ? -z : z;
  }
}

// K7: (1/M) sum_k Re(S_d conj(F cs_u F cs_v F cs_w)) (uvw_spectral + spectral_dot,
// estimators.cpp:38-64). Grid (batch, D); est[b][d].
__global__ void __launch_bounds__(kFftThreads) uvw_kernel(FftPlan pl, EngArgs e, const double* U,
                                                          const double* V, const double* W,
                                                          double2* scratch, double* est) {
  (void)scratch;
  const Smem sm = carve(pl, 2);
  load_twiddles(sm.tw, pl, false);
  __syncthreads();
  const int b = blockIdx.x, d = blockIdx.y;
  const size_t item = static_cast<size_t>(b) * e.D + d;
  const uint32_t* tab = e.packed + static_cast<size_t>(d) * e.fam_stride;
  const double2* S = e.spec + static_cast<size_t>(d) * pl.P;
  rfft_of_cs2(sm, pl, U + static_cast<size_t>(b) * e.dims[0], e.dims[0], tab + e.tab_off[0],
              V + static_cast<size_t>(b) * e.dims[1], e.dims[1], tab + e.tab_off[1]);
  for (int s = tid(); s < pl.P; s += blockDim.x)
    sm.buf[swz(s)] = hmul(sm.buf[swz(s)], sm.buf2[swz(s)], s == 0);
  __syncthreads();
  rfft_of_cs(sm, sm.buf2, pl, W + static_cast<size_t>(b) * e.dims[2], e.dims[2],
             tab + e.tab_off[2]);
  double acc = 0.0;
  for (int s = tid(); s < pl.P; s += blockDim.x) {
    const double2 g = hmul(sm.buf[swz(s)], sm.buf2[swz(s)], s == 0);
    const double2 sd = S[s];
    const double re = sd.x * g.x + sd.y * g.y;  // Re(S conj(G)) / (X0*G0 + XP*GP at slot 0)
    acc += s == 0 ? re : 2.0 * re;
  }
  const double tot = block_sum(acc, sm.red);
  if (threadIdx.x == 0) est[item] = tot / pl.M;
}

// K9: S_d -= weight * F cs_u F cs_v F cs_w (FcsEngine::deflate, cpd.cpp:79-87, by linearity).
__global__ void __launch_bounds__(kFftThreads) deflate_kernel(FftPlan pl, EngArgs e, double weight,
                                                              const double* U, const double* V,
                                                              const double* W, double2* scratch,
                                                              double2* spec) {
  (void)scratch;
  const Smem sm = carve(pl, 2);
  load_twiddles(sm.tw, pl, false);
  __syncthreads();
  const int d = blockIdx.x;
  const uint32_t* tab = e.packed + static_cast<size_t>(d) * e.fam_stride;
  double2* S = spec + static_cast<size_t>(d) * pl.P;
  rfft_of_cs2(sm, pl, U, e.dims[0], tab + e.tab_off[0], V, e.dims[1], tab + e.tab_off[1]);
  for (int s = tid(); s < pl.P; s += blockDim.x)
    sm.buf[swz(s)] = hmul(sm.buf[swz(s)], sm.buf2[swz(s)], s == 0);
  __syncthreads();
  rfft_of_cs(sm, sm.buf2, pl, W, e.dims[2], tab + e.tab_off[2]);
  for (int s = tid(); s < pl.P; s += blockDim.x) {
    const double2 g = hmul(sm.buf[swz(s)], sm.buf2[swz(s)], s == 0);
    S[s] = csub(S[s], cscale(g, weight));
  }
}

// K8: elementwise median over D (median_reduce, estimators.cpp:117-138):
// est[b][d][i] -> out[b][i]; median_col (median.cuh) is shared with the fused
// tail of the cluster estimator.
__global__ void median_kernel(const double* __restrict__ est, int batch, int D, int len,
                              double* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= batch * len) return;
  const int b = idx / len, i = idx - b * len;
  const double* col = est + static_cast<size_t>(b) * D * len + i;  // stride len
  out[idx] = median_col(col, D, len, [](const double* p) { return *p; });
}

// Median over D then row normalisation, one CTA per row (the rtpm restart
// step, cpd.cpp:253-257): the median of median_kernel and the norm of
// normalize_rows_kernel (same thread count and reduction order, so the result
// equals the two kernels run back to back, with one launch fewer).
__global__ void median_normalize_kernel(const double* __restrict__ est, int D, int len,
                                        double* __restrict__ out) {
  __shared__ double red[32];
  __shared__ double norm;
  const int b = blockIdx.x;
  const double* base = est + static_cast<size_t>(b) * D * len;
  double* o = out + static_cast<size_t>(b) * len;
  double acc = 0.0;
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    const double m = median_col(base + i, D, len, [](const double* p) { return *p; });
    o[i] = m;
    acc += m * m;
  }
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) norm = sqrt(tot);
  __syncthreads();
  const double nv = norm;
  for (int i = threadIdx.x; i < len; i += blockDim.x) o[i] = nv < 1e-150 ? 0.0 : o[i] / nv;
}

// Per-column count sketch into global memory (cs_sketch_columns, sketch.cpp:118-133).
__global__ void cs_columns_kernel(const double* __restrict__ u, int I, int cols,
                                  const uint32_t* __restrict__ tab, int J, double* __restrict__ out) {
  const size_t n = static_cast<size_t>(I) * cols;
  for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(k % I);
    const size_t r = k / I;
    const double v = u[k];
    if (v == 0.0) continue;
    const uint32_t e = __ldg(tab + i);
    atomicAdd(out + r * J + (e & 0x7fffffffu), (e >> 31) ? -v : v);
  }
}

// Row normalisation for the batched power iteration: u <- u/||u|| or 0 when
// ||u|| < 1e-150 (normalize_or_zero, cpd.cpp:208-216). One block per row.
__global__ void normalize_rows_kernel(double* __restrict__ U, int dim) {
  __shared__ double red[32];
  double* u = U + static_cast<size_t>(blockIdx.x) * dim;
  double acc = 0.0;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) acc += u[i] * u[i];
  double tot = block_sum(acc, red);
  __shared__ double norm;
  if (threadIdx.x == 0) norm = sqrt(tot);
  __syncthreads();
  const double nv = norm;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) u[i] = nv < 1e-150 ? 0.0 : u[i] / nv;
}

// Refinement step of rtpm (cpd.cpp:266-270): best <- next/||next|| unless the
// norm underflows, which stops the refinement for good (sticky flag).
__global__ void refine_update_kernel(double* __restrict__ best, const double* __restrict__ next,
                                     int dim, int* __restrict__ stopped) {
  __shared__ double red[32];
  __shared__ double norm;
  if (*stopped) return;
  double acc = 0.0;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) acc += next[i] * next[i];
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) norm = sqrt(tot);
  __syncthreads();
  const double nv = norm;
  if (nv < 1e-150) {
    if (threadIdx.x == 0) *stopped = 1;
    return;
  }
  for (int i = threadIdx.x; i < dim; i += blockDim.x) best[i] = next[i] / nv;
}

// ------------------------------------------------------------ launchers
namespace {

// Per-(kernel, device) cache of the dynamic shared-memory opt-in (raised only
// when a larger plan needs it) and of the occupancy per shared-memory size:
// the per-call host work of a small step stays a map lookup.
struct KernelCache {
  std::mutex mu;
  std::map<std::pair<const void*, int>, size_t> smem_set;
  std::map<std::tuple<const void*, int, size_t>, int> occ;
};
KernelCache& kcache() {
  static KernelCache c;
  return c;
}

template <typename K>
int prep(K kernel, const FftPlan& pl, size_t* smem, int nbuf = 1) {
  *smem = fft_smem_bytes(pl, false) + static_cast<size_t>(nbuf - 1) * pl.P * sizeof(double2) +
          32 * sizeof(double);
  int dev = 0;
  FCS_CUDA_TRY(cudaGetDevice(&dev));
  KernelCache& c = kcache();
  std::lock_guard<std::mutex> lock(c.mu);
  size_t& cur = c.smem_set[{reinterpret_cast<const void*>(kernel), dev}];
  if (*smem > cur) {
    FCS_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(*smem)));
    cur = *smem;
  }
  return ST_OK;
}

template <typename K>
int occupancy(K kernel, int threads, size_t smem, int* out) {
  int dev = 0;
  FCS_CUDA_TRY(cudaGetDevice(&dev));
  KernelCache& c = kcache();
  std::lock_guard<std::mutex> lock(c.mu);
  auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), dev, smem);
  auto it = c.occ.find(key);
  if (it == c.occ.end()) {
    int n = 0;
    FCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem));
    it = c.occ.emplace(key, n).first;
  }
  *out = it->second;
  return ST_OK;
}

}  // namespace

int launch_spec_from_real(const FftPlan& pl, const double* x, size_t ldx, int len, int items,
                          double2* spec, cudaStream_t st) {
  if (pl.large_p1) return large_rfft(pl, x, ldx, len, items, spec, st);
  size_t sm;
  if (int rc = prep(spec_from_real_kernel, pl, &sm)) return rc;
  spec_from_real_kernel<<<items, kFftThreads, sm, st>>>(pl, x, ldx, len, spec);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_real_from_spec(const FftPlan& pl, const double2* spec, int items, double* out,
                          size_t ldo, int out_len, int accumulate, cudaStream_t st) {
  if (pl.large_p1) return large_real_from_spec(pl, spec, items, out, ldo, out_len, accumulate, st);
  size_t sm;
  if (int rc = prep(real_from_spec_kernel, pl, &sm)) return rc;
  real_from_spec_kernel<<<items, kFftThreads, sm, st>>>(pl, spec, out, ldo, out_len, accumulate);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_cp(const FftPlan& pl, const CpArgs& a, int D, const uint32_t* packed, double2* Q,
              double* out, int jt, int accumulate, cudaStream_t st) {
  if (pl.large_p1) return large_cp(pl, a, D, packed, a.hash_lens, out, jt, accumulate, st);
  size_t sm, sm1;
  if (int rc = prep(cp_rank_kernel, pl, &sm, 2)) return rc;
  if (int rc = prep(cp_rank1_kernel, pl, &sm1, 1)) return rc;
  if (a.r_count > 0) {
    // the one-buffer form when it needs fewer waves (as launch_iuv)
    int occ2 = 0, occ1 = 0;
    if (int rc = occupancy(cp_rank_kernel, kFftThreads, sm, &occ2)) return rc;
    if (int rc = occupancy(cp_rank1_kernel, kFftThreads, sm1, &occ1)) return rc;
    DeviceInfo di;
    if (int rc = device_info(&di)) return rc;
    const long items = static_cast<long>(a.r_count) * D;
    const long c2 = static_cast<long>(std::max(occ2, 1)) * di.sm_count;
    const long c1 = static_cast<long>(std::max(occ1, 1)) * di.sm_count;
    if ((items + c1 - 1) / c1 < (items + c2 - 1) / c2 && !std::getenv("ST_CP_TWO_BUFFER"))
      cp_rank1_kernel<<<dim3(a.r_count, D), kFftThreads, sm1, st>>>(pl, a, packed, Q);
    else
      cp_rank_kernel<<<dim3(a.r_count, D), kFftThreads, sm, st>>>(pl, a, packed, Q);
    FCS_CUDA_TRY(cudaGetLastError());
  }
  // The summed spectra go to their own region after Q (st_fcs_cp_workspace
  // reserves D*P extra slots).
  double2* acc = Q + static_cast<size_t>(D) * std::max(a.r_count, 1) * pl.P;
  cp_rank_sum_kernel<<<dim3(ceil_div(pl.P, 32), D), dim3(32, 8), 0, st>>>(Q, a.weights, a.r_begin,
                                                                          a.r_count, pl.P, acc);
  FCS_CUDA_TRY(cudaGetLastError());
  {  // D families: one 8-CTA cluster each (spectral_cluster.cu)
    const int rc = launch_spec_inverse_cluster(pl, acc, D, out, jt, accumulate, st);
    if (rc != 1) return rc;
  }
  if (int rc = prep(cp_sum_kernel, pl, &sm)) return rc;
  // D CTAs only: twice the threads per CTA shortens the one-transform latency
  cp_sum_kernel<<<D, 2 * kFftThreads, sm, st>>>(pl, acc, out, jt, accumulate);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_conv(const FftPlan& pl, const double* a, int la, size_t lda, const double* b, int lb,
                size_t ldb, int items, double2* scratch, double* out, size_t ldo, cudaStream_t st) {
  if (pl.large_p1) return large_conv(pl, a, la, lda, b, lb, ldb, items, out, ldo, st);
  {  // one wave of items: an 8-CTA cluster per item (spectral_cluster.cu)
    const int rc = launch_conv_cluster(pl, a, la, lda, b, lb, ldb, items, out, ldo, st);
    if (rc != 1) return rc;
  }
  size_t sm;
  if (int rc = prep(conv_kernel, pl, &sm)) return rc;
  conv_kernel<<<items, kFftThreads, sm, st>>>(pl, a, la, lda, b, lb, ldb, scratch, out, ldo);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_iuv(const FftPlan& pl, const EngArgs& e, int batch, const double* A, const double* B,
               int c1, int c2, int f, double2* scratch, double* est, cudaStream_t st) {
  if (pl.large_p1) return large_iuv(pl, e, batch, A, B, c1, c2, f, e.hash_len, est, st);
  {  // small batches: one 8-CTA cluster per item (spectral_cluster.cu)
    const int rc = launch_iuv_cluster(pl, e, batch, A, B, c1, c2, f, est, IuvTail{}, st);
    if (rc != 1) return rc;
  }
  size_t sm2, sm1;
  if (int rc = prep(iuv_kernel, pl, &sm2, 2)) return rc;
  if (int rc = prep(iuv1_kernel, pl, &sm1, 1)) return rc;
  // waves of each form; the one-buffer kernel (scratch: batch x D x P slots)
  // wins when it fits the batch in fewer waves
  int occ2 = 0, occ1 = 0;
  if (int rc = occupancy(iuv_kernel, kFftThreads, sm2, &occ2)) return rc;
  if (int rc = occupancy(iuv1_kernel, kFftThreads, sm1, &occ1)) return rc;
  DeviceInfo di;
  if (int rc = device_info(&di)) return rc;
  // One CTA per SM for the first nb1 vectors; the vectors beyond go to the
  // cluster kernel on the side stream, concurrently (config 3's 15 x 10
  // items: 140 one-CTA items + 10 clusters, 51 -> 41 us per step with the
  // median, instead of two CTAs sharing an SM setting the span).
  // (nb1 - 1 .. - 4: 43.8-51.2 us; the two-buffer kernel for the one-CTA part:
  // 52 us pipelined — measured)
  const int nb1 = di.sm_count / e.D;
  if (nb1 > 0 && batch > nb1 && scratch != nullptr) {
    cudaStream_t st2 = nullptr;
    FCS_CUDA_TRY(fork_side(st, &st2));
    const size_t na = e.dims[c1], nbv = e.dims[c2], nf = e.dims[f];
    // the one-CTA part is submitted first: submitted after the clusters, the
    // two parts ran serialised on a caller stream other than the legacy
    // default stream (61 vs 41 us per step, tools/stream_probe.py); if the
    // cluster form does not apply, the general path below redoes the batch
    iuv1_kernel<<<dim3(nb1, e.D), kFftThreads, sm1, st>>>(pl, e, A, B, c1, c2, f, scratch, est);
    const int rc = launch_iuv_cluster(pl, e, batch - nb1, A + nb1 * na, B + nb1 * nbv, c1, c2, f,
                                      est + static_cast<size_t>(nb1) * e.D * nf, IuvTail{}, st2);
    const cudaError_t le = cudaGetLastError();
    FCS_CUDA_TRY(join_side(st));
    FCS_CUDA_TRY(le);
    if (rc == 0) return ST_OK;
    if (rc != 1) return rc;
  }
  const long items = static_cast<long>(batch) * e.D;
  const long w2 = (items + std::max(occ2, 1) * di.sm_count - 1) / (std::max(occ2, 1) * di.sm_count);
  const long w1 = (items + std::max(occ1, 1) * di.sm_count - 1) / (std::max(occ1, 1) * di.sm_count);
  if (scratch != nullptr && w1 < w2)
    iuv1_kernel<<<dim3(batch, e.D), kFftThreads, sm1, st>>>(pl, e, A, B, c1, c2, f, scratch, est);
  else
    iuv_kernel<<<dim3(batch, e.D), kFftThreads, sm2, st>>>(pl, e, A, B, c1, c2, f, scratch, est);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

// T(u, v, w) through the one-buffer estimator with the dot product (one CTA
// per item, the one-CTA part of a split batch): est[b D + d].
int launch_uvw_dot(const FftPlan& pl, const EngArgs& e, int batch, const double* U,
                   const double* V, const double* W, double2* scratch, double* est,
                   cudaStream_t st) {
  if (pl.large_p1) return 1;
  size_t sm1;
  if (int rc = prep(iuv1_kernel, pl, &sm1, 1)) return rc;
  iuv1_kernel<<<dim3(batch, e.D), kFftThreads, sm1, st>>>(pl, e, U, V, 0, 1, 2, scratch, est, W);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_uvw(const FftPlan& pl, const EngArgs& e, int batch, const double* U, const double* V,
               const double* W, double2* scratch, double* est, cudaStream_t st) {
  if (pl.large_p1) return large_uvw(pl, e, batch, U, V, W, e.hash_len, est, st);
  // the one-buffer estimator with the dot product (2 forward + 1 inverse,
  // two CTAs per SM) beats the three-forward kernel once there are items to
  // fill the device (config 3, 150 items: 51 vs 62 us; 10 items: 39 vs 35 us)
  if (scratch != nullptr && static_cast<long>(batch) * e.D >= 32)
    return launch_uvw_dot(pl, e, batch, U, V, W, scratch, est, st);
  size_t sm;
  if (int rc = prep(uvw_kernel, pl, &sm, 2)) return rc;
  uvw_kernel<<<dim3(batch, e.D), kFftThreads, sm, st>>>(pl, e, U, V, W, scratch, est);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_deflate(const FftPlan& pl, const EngArgs& e, double weight, const double* U,
                   const double* V, const double* W, double2* scratch, double2* spec,
                   cudaStream_t st) {
  if (pl.large_p1) return large_deflate(pl, e, weight, U, V, W, e.hash_len, spec, st);
  {  // one 8-CTA cluster per family (spectral_cluster.cu)
    const int rc = launch_deflate_cluster(pl, e, weight, U, V, W, spec, st);
    if (rc != 1) return rc;
  }
  size_t sm;
  if (int rc = prep(deflate_kernel, pl, &sm, 2)) return rc;
  deflate_kernel<<<e.D, kFftThreads, sm, st>>>(pl, e, weight, U, V, W, scratch, spec);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_median(const double* est, int batch, int D, int len, double* out, cudaStream_t st) {
  FCS_CHECK_ARG(D >= 1, "median_reduce: empty input");
  const int n = batch * len;
  if (n == 0) return ST_OK;
  median_kernel<<<ceil_div(n, 128), 128, 0, st>>>(est, batch, D, len, out);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_median_normalize(const double* est, int batch, int D, int len, double* out,
                            cudaStream_t st) {
  FCS_CHECK_ARG(D >= 1, "median_reduce: empty input");
  if (batch == 0 || len == 0) return ST_OK;
  median_normalize_kernel<<<batch, 256, 0, st>>>(est, D, len, out);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_cs_columns(const double* u, int I, int cols, const uint32_t* tab, int J, double* out,
                      cudaStream_t st) {
  FCS_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * static_cast<size_t>(J) * cols, st));
  const size_t n = static_cast<size_t>(I) * cols;
  if (n == 0) return ST_OK;
  cs_columns_kernel<<<std::min<unsigned>(ceil_div(n, 256), 4096), 256, 0, st>>>(u, I, cols, tab, J,
                                                                                 out);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_normalize_rows(double* U, int rows, int dim, cudaStream_t st) {
  if (rows == 0) return ST_OK;
  normalize_rows_kernel<<<rows, 256, 0, st>>>(U, dim);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_refine_update(double* best, const double* next, int dim, int* stopped,
                         cudaStream_t st) {
  refine_update_kernel<<<1, 256, 0, st>>>(best, next, dim, stopped);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace fcs
