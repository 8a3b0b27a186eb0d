// Shared-memory fp64 FFT for the spectral FCS paths (sm_100a).
//
// Real sequences of length M (zero-padded sketches) are transformed as
// complex sequences of P = M/2 points (z[j] = x[2j] + i x[2j+1]) with an
// in-place mixed-radix decimation-in-frequency Cooley-Tukey over radices
// {3, 16, 8, 4, 2}: each butterfly reads R slots and writes its results back
// to the same slots, so passes need one barrier and no second buffer, and
// the spectrum comes out in digit-reversed slot order. Every spectrum in the
// library (cached tensor spectra, factor spectra, products) lives in that
// same slot order, so pointwise products never permute; the inverse
// (decimation-in-time, the exact reverse of the forward passes) returns
// natural order. The post / pre pair maps (post_pair / pre_pair, fused into
// the last forward / first inverse pass) convert between the packed P-point
// transform and the Hermitian half spectrum X[0..P] of the length-M real
// transform; slot pos(0) holds the two real bins (X[0], X[P]).
//
// Reference semantics (fft.cpp:42-84): dft zero-pads to n = J~ and the
// inverse is normalised by 1/n. Padding to any M >= J~ leaves every value the
// reference reads unchanged (linear convolution support [0, J~-1]; the
// correlation read z[h] only touches lags < J~; Parseval dot over [0, J~-1]).
#pragma once

#include "common.cuh"

namespace fcs {

constexpr int kFftMaxPasses = 10;
constexpr int kTwLoBits = 6;  // two-level twiddle table: w_M^e = lo[e & 63] * hi[e >> 6]
constexpr int kFftThreads = 256;
constexpr int kMaxFftM = 12288;  // largest supported padded length (P = 6144)

struct FftPlan {
  int M;                       // real transform length (even)
  int P;                       // complex points = M / 2
  int npass;
  int radix[kFftMaxPasses];    // DIF order
  int len[kFftMaxPasses];      // sub-transform length L entering each pass
  unsigned long long rcode;    // radix[p] - 1 in bits 4p..4p+3 (device loops decode this
                               // instead of indexing radix[] / len[], which would copy the
                               // plan to local memory)
  int hi_count;                // entries of the hi table (= M >> kTwLoBits, rounded up)
  const double2* tw;           // device: lo[64] then hi[hi_count]
  const int* f2p;              // device: slot position of frequency k, k in [0, P)
  const uint2* units;          // device: pair units of the last pass (see last_pass_post)
  int nunits;
  int large_p1;                // 0: one-CTA plan; else P = large_p1 * P2 two-level plan
};                             // (spectral_large.cu; npass, tw, f2p unused)

// Two-level plan for M > kMaxFftM: P = P1 * P2 with shared-memory sub-plans
// a (P1-point column transforms) and b (P2-point row transforms).
struct LargeFft {
  int M, P, P1, P2;
  FftPlan a, b;
  const int* p2f_a;  // device: slot -> frequency of plan a
};

// XOR swizzle of 16-byte slots: the low 3 bits (slot within a 128-byte
// wavefront) are XORed with bits 3-5, so stride-1, -8 and -16 slot patterns of
// the butterfly passes land on distinct bank groups.
__device__ __forceinline__ uint32_t swz(uint32_t s) { return s ^ ((s >> 3) & 7u); }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by sign * i
__device__ __forceinline__ double2 cmul_si(double2 a, double sign) { return make_double2(-sign * a.y, sign * a.x); }

// w_M^e = exp(-2 pi i e / M) for 0 <= e < M (forward convention).
__device__ __forceinline__ double2 twiddle(const double2* tw, int hi_off, uint32_t e) {
  return cmul(tw[e & ((1u << kTwLoBits) - 1)], tw[hi_off + (e >> kTwLoBits)]);
}

// x[r] *= w^r, r = 1..R-1, for one butterfly from w = w^1 with powers by a
// product chain instead of R - 1 table lookups (each two shared-memory loads
// and a complex product): w2 = w w, w4 = w2 w2, w8 = w4 w4, then for r < 8
// t_r (at most two products of w, w2, w4) scales x[r] and w8 t_r scales
// x[r + 8], so only a handful of twiddles are live at a time. Relative error
// a few ulp beyond the table's, far inside the fp64 FFT's own error budget.
template <int R, int NB>
__device__ __forceinline__ void apply_twiddles(double2 (*x)[R], double2 w) {
  auto mul = [&](int r, double2 t) {
#pragma unroll
    for (int b = 0; b < NB; ++b) x[b][r] = cmul(x[b][r], t);
  };
  mul(1, w);
  if constexpr (R == 3) mul(2, cmul(w, w));
  if constexpr (R == 9) {
    const double2 w2 = cmul(w, w);
    const double2 w3 = cmul(w2, w);
    const double2 w4 = cmul(w2, w2);
    mul(2, w2);
    mul(3, w3);
    mul(4, w4);
    mul(5, cmul(w4, w));
    mul(6, cmul(w3, w3));
    mul(7, cmul(w4, w3));
    mul(8, cmul(w4, w4));
  }
  if constexpr (R >= 4 && R != 9) {
    const double2 w2 = cmul(w, w);
    const double2 w3 = cmul(w2, w);
    mul(2, w2);
    mul(3, w3);
    if constexpr (R >= 8) {
      const double2 w4 = cmul(w2, w2);
      const double2 w5 = cmul(w4, w);
      const double2 w6 = cmul(w4, w2);
      const double2 w7 = cmul(w4, w3);
      mul(4, w4);
      mul(5, w5);
      mul(6, w6);
      mul(7, w7);
      if constexpr (R == 16) {
        const double2 w8 = cmul(w4, w4);
        mul(8, w8);
        mul(9, cmul(w8, w));
        mul(10, cmul(w8, w2));
        mul(11, cmul(w8, w3));
        mul(12, cmul(w8, w4));
        mul(13, cmul(w8, w5));
        mul(14, cmul(w8, w6));
        mul(15, cmul(w8, w7));
      }
    }
  }
}

// ------------------------------------------------------ in-register DFTs
// cos(2 pi k / 16); sin(2 pi k / 16) = cos16(k - 4). Folds to constants once
// the butterfly loops are unrolled.
__host__ __device__ constexpr double cos16(int k) {
  constexpr double t[16] = {1.0,
                            0.92387953251128675613,
                            0.70710678118654752440,
                            0.38268343236508977173,
                            0.0,
                            -0.38268343236508977173,
                            -0.70710678118654752440,
                            -0.92387953251128675613,
                            -1.0,
                            -0.92387953251128675613,
                            -0.70710678118654752440,
                            -0.38268343236508977173,
                            0.0,
                            0.38268343236508977173,
                            0.70710678118654752440,
                            0.92387953251128675613};
  return t[k & 15];
}

// y[k] = sum_r x[r] exp(sign * 2 pi i r k / R), sign = -1 forward.
template <int R>
struct RegDft {
  static __device__ __forceinline__ void run(double2* x, double sign) {
    constexpr int H = R / 2;
    double2 e[H], o[H];
#pragma unroll
    for (int r = 0; r < H; ++r) {
      e[r] = x[2 * r];
      o[r] = x[2 * r + 1];
    }
    RegDft<H>::run(e, sign);
    RegDft<H>::run(o, sign);
#pragma unroll
    for (int k = 0; k < H; ++k) {
      // w_R^k = exp(sign * 2 pi i k / R) from the 16th-root table
      const int q = k * (16 / R);
      const double2 w = make_double2(cos16(q), sign * cos16(q - 4));
      const double2 t = (k == 0) ? o[k] : cmul(w, o[k]);
      x[k] = cadd(e[k], t);
      x[k + H] = csub(e[k], t);
    }
  }
};

template <>
struct RegDft<1> {
  static __device__ __forceinline__ void run(double2*, double) {}
};

template <>
struct RegDft<2> {
  static __device__ __forceinline__ void run(double2* x, double) {
    const double2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
  }
};

template <>
struct RegDft<4> {
  static __device__ __forceinline__ void run(double2* x, double sign) {
    const double2 s02 = cadd(x[0], x[2]), d02 = csub(x[0], x[2]);
    const double2 s13 = cadd(x[1], x[3]), d13 = cmul_si(csub(x[1], x[3]), sign);
    x[0] = cadd(s02, s13);
    x[2] = csub(s02, s13);
    x[1] = cadd(d02, d13);
    x[3] = csub(d02, d13);
  }
};

template <>
struct RegDft<3> {
  static __device__ __forceinline__ void run(double2* x, double sign) {
    constexpr double kS = 0.86602540378443864676372317075294;  // sqrt(3)/2
    const double2 t = cadd(x[1], x[2]);
    const double2 u = cmul_si(csub(x[1], x[2]), sign * kS);
    const double2 m = make_double2(x[0].x - 0.5 * t.x, x[0].y - 0.5 * t.y);
    x[0] = cadd(x[0], t);
    x[1] = cadd(m, u);
    x[2] = csub(m, u);
  }
};

// 9 = 3 x 3: DFT3 over n1 for each n2 (x[3 n1 + n2]), twiddle w9^{n2 k1},
// DFT3 over n2 for each k1; output y[k1 + 3 k2] in natural order.
template <>
struct RegDft<9> {
  static __device__ __forceinline__ void run(double2* x, double sign) {
    // cos / sin(2 pi k / 9), k = 1, 2, 4
    constexpr double c1 = 0.76604444311897803520, s1 = 0.64278760968653932632;
    constexpr double c2 = 0.17364817766693034885, s2 = 0.98480775301220805936;
    constexpr double c4 = -0.93969262078590838405, s4 = 0.34202014332566873304;
    double2 a[3][3];  // a[n2][k1]
#pragma unroll
    for (int n2 = 0; n2 < 3; ++n2) {
      double2 t[3] = {x[n2], x[3 + n2], x[6 + n2]};
      RegDft<3>::run(t, sign);
#pragma unroll
      for (int k1 = 0; k1 < 3; ++k1) a[n2][k1] = t[k1];
    }
    // w9^{n2 k1}: (1,1) -> w, (1,2) and (2,1) -> w^2, (2,2) -> w^4
    const double2 w1 = make_double2(c1, sign * s1), w2 = make_double2(c2, sign * s2),
                  w4 = make_double2(c4, sign * s4);
    a[1][1] = cmul(a[1][1], w1);
    a[1][2] = cmul(a[1][2], w2);
    a[2][1] = cmul(a[2][1], w2);
    a[2][2] = cmul(a[2][2], w4);
#pragma unroll
    for (int k1 = 0; k1 < 3; ++k1) {
      double2 t[3] = {a[0][k1], a[1][k1], a[2][k1]};
      RegDft<3>::run(t, sign);
#pragma unroll
      for (int k2 = 0; k2 < 3; ++k2) x[k1 + 3 * k2] = t[k2];
    }
  }
};

// R = P Q with n = Q n1 + n2, k = k1 + P k2: DFT_P over n1 for each n2,
// twiddle w_R^{n2 k1}, DFT_Q over n2 for each k1; output y[k1 + P k2] in
// natural order (as RegDft<9>). Twiddles from exact cos/sin of 2 pi m / R.
template <int P, int Q>
__device__ __forceinline__ void reg_dft_pq(double2* x, double sign) {
  constexpr int R = P * Q;
  constexpr double kTwoPi = 6.283185307179586476925286766559;
  double2 a[Q][P];  // a[n2][k1]
#pragma unroll
  for (int n2 = 0; n2 < Q; ++n2) {
    double2 t[P];
#pragma unroll
    for (int n1 = 0; n1 < P; ++n1) t[n1] = x[Q * n1 + n2];
    RegDft<P>::run(t, sign);
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) {
      const int m = (n2 * k1) % R;
      if (m == 0) {
        a[n2][k1] = t[k1];
      } else {
        const double2 w = make_double2(cos(kTwoPi * m / R), sign * sin(kTwoPi * m / R));
        a[n2][k1] = cmul(t[k1], w);
      }
    }
  }
#pragma unroll
  for (int k1 = 0; k1 < P; ++k1) {
    double2 t[Q];
#pragma unroll
    for (int n2 = 0; n2 < Q; ++n2) t[n2] = a[n2][k1];
    RegDft<Q>::run(t, sign);
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) x[k1 + P * k2] = t[k2];
  }
}
template <>
struct RegDft<6> {
  static __device__ __forceinline__ void run(double2* x, double sign) { reg_dft_pq<3, 2>(x, sign); }
};
template <>
struct RegDft<12> {
  static __device__ __forceinline__ void run(double2* x, double sign) { reg_dft_pq<4, 3>(x, sign); }
};

// ----------------------------------------------------- block-wide passes
// One radix-R pass over all butterflies of sub-transforms of length L.
// Forward (DIF): DFT then twiddle w_L^{j r'}; inverse (DIT): conj twiddle then DFT.
template <int R, bool kForward>
__device__ __forceinline__ void fft_pass(double2* buf, const double2* tw, int hi_off, int M, int P,
                                         int L) {
  const int stride = L / R;
  const int nbfly = P / R;
  const uint32_t tw_scale = static_cast<uint32_t>(M / L);  // w_L = w_M^{M/L}
  // b / stride as a multiply-high (stride > 1): exact for every b < P <= 2^13
  const uint32_t magic = 0xffffffffu / static_cast<uint32_t>(stride) + 1u;
  for (int b = threadIdx.x; b < nbfly; b += blockDim.x) {
    const int blk = stride == 1 ? b : static_cast<int>(__umulhi(static_cast<uint32_t>(b), magic));
    const int j = b - blk * stride;
    const int base = blk * L + j;
    double2 x[1][R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[0][r] = buf[swz(base + r * stride)];
    if (kForward) {
      RegDft<R>::run(x[0], -1.0);
      if (j) apply_twiddles<R, 1>(x, twiddle(tw, hi_off, static_cast<uint32_t>(j) * tw_scale));
    } else {
      if (j)
        apply_twiddles<R, 1>(x, cconj(twiddle(tw, hi_off, static_cast<uint32_t>(j) * tw_scale)));
      RegDft<R>::run(x[0], +1.0);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) buf[swz(base + r * stride)] = x[0][r];
  }
}

template <bool kForward>
__device__ __forceinline__ void fft_dispatch(double2* buf, const double2* tw, int hi_off, int M,
                                             int P, int radix, int L) {
  switch (radix) {
    case 16: fft_pass<16, kForward>(buf, tw, hi_off, M, P, L); break;
    case 8: fft_pass<8, kForward>(buf, tw, hi_off, M, P, L); break;
    case 4: fft_pass<4, kForward>(buf, tw, hi_off, M, P, L); break;
    case 9: fft_pass<9, kForward>(buf, tw, hi_off, M, P, L); break;
    case 3: fft_pass<3, kForward>(buf, tw, hi_off, M, P, L); break;
    default: fft_pass<2, kForward>(buf, tw, hi_off, M, P, L); break;
  }
}

__device__ __forceinline__ int pass_radix(const FftPlan& pl, int p) {
  return static_cast<int>((pl.rcode >> (4 * p)) & 15ull) + 1;
}

// Natural-order packed input -> digit-reversed spectrum (unnormalised, e^{-i}).
__device__ __forceinline__ void fft_forward(double2* buf, const FftPlan& pl, const double2* tw) {
  int L = pl.P;
  for (int p = 0; p < pl.npass; ++p) {
    const int R = pass_radix(pl, p);
    fft_dispatch<true>(buf, tw, 1 << kTwLoBits, pl.M, pl.P, R, L);
    __syncthreads();
    L /= R;
  }
}

// Two independent forward transforms in one sweep: the butterflies of b0 and
// b1 at the same position share their twiddles, and because the buffers are
// distinct (__restrict__) the loads of one overlap the arithmetic and stores
// of the other — twice the instruction-level parallelism of fft_pass.
template <int R>
__device__ __forceinline__ void fft_pass2(double2* __restrict__ b0, double2* __restrict__ b1,
                                          const double2* tw, int hi_off, int M, int P, int L) {
  const int stride = L / R;
  const int nbfly = P / R;
  const uint32_t tw_scale = static_cast<uint32_t>(M / L);
  const uint32_t magic = 0xffffffffu / static_cast<uint32_t>(stride) + 1u;
  for (int b = threadIdx.x; b < nbfly; b += blockDim.x) {
    const int blk = stride == 1 ? b : static_cast<int>(__umulhi(static_cast<uint32_t>(b), magic));
    const int j = b - blk * stride;
    const int base = blk * L + j;
    double2 xy[2][R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      xy[0][r] = b0[swz(base + r * stride)];
      xy[1][r] = b1[swz(base + r * stride)];
    }
    RegDft<R>::run(xy[0], -1.0);
    RegDft<R>::run(xy[1], -1.0);
    if (j) apply_twiddles<R, 2>(xy, twiddle(tw, hi_off, static_cast<uint32_t>(j) * tw_scale));
#pragma unroll
    for (int r = 0; r < R; ++r) {
      b0[swz(base + r * stride)] = xy[0][r];
      b1[swz(base + r * stride)] = xy[1][r];
    }
  }
}

// The first `npass` paired forward passes (all of them, or all but the last).
__device__ __forceinline__ void fft_forward2_passes(double2* __restrict__ b0,
                                                    double2* __restrict__ b1, const FftPlan& pl,
                                                    const double2* tw, int npass) {
  const int hi = 1 << kTwLoBits;
  int L = pl.P;
  for (int p = 0; p < npass; ++p) {
    const int R = pass_radix(pl, p);
    switch (R) {
      case 16: fft_pass2<16>(b0, b1, tw, hi, pl.M, pl.P, L); break;
      case 8: fft_pass2<8>(b0, b1, tw, hi, pl.M, pl.P, L); break;
      case 4: fft_pass2<4>(b0, b1, tw, hi, pl.M, pl.P, L); break;
      case 9: fft_pass2<9>(b0, b1, tw, hi, pl.M, pl.P, L); break;
      case 3: fft_pass2<3>(b0, b1, tw, hi, pl.M, pl.P, L); break;
      default: fft_pass2<2>(b0, b1, tw, hi, pl.M, pl.P, L); break;
    }
    __syncthreads();
    L /= R;
  }
}

// Digit-reversed spectrum -> natural order (unnormalised, e^{+i}).
__device__ __forceinline__ void fft_inverse(double2* buf, const FftPlan& pl, const double2* tw) {
  int L = 1;  // len[p] = prod_{q >= p} radix[q]
  for (int p = pl.npass - 1; p >= 0; --p) {
    const int R = pass_radix(pl, p);
    L *= R;
    fft_dispatch<false>(buf, tw, 1 << kTwLoBits, pl.M, pl.P, R, L);
    __syncthreads();
  }
}

// Shared-memory table region, in double2 slots. Layout: twiddles (lo, hi), the last-pass pair units, then (only for kernels
// that index spectra by frequency, spectral_large.cu) the frequency -> slot table.
__host__ __device__ inline int table_slots(const FftPlan& pl, bool with_f2p = true) {
  return (1 << kTwLoBits) + pl.hi_count + (pl.nunits + 1) / 2 + (with_f2p ? (pl.P + 3) / 4 : 0);
}
__device__ __forceinline__ const uint2* smem_units(const double2* tw, const FftPlan& pl) {
  return reinterpret_cast<const uint2*>(tw + (1 << kTwLoBits) + pl.hi_count);
}
__device__ __forceinline__ const int* smem_f2p(const double2* tw, const FftPlan& pl) {
  return reinterpret_cast<const int*>(tw + (1 << kTwLoBits) + pl.hi_count + (pl.nunits + 1) / 2);
}

// The real-transform pair maps on two registers, w = w_M^k:
//   post (r2c): a = Z[k], b = Z[P-k] of the packed P-point spectrum ->
//     a = X[k] = E + w O, b = X[P-k] = conj(E - w O) of the Hermitian half
//     spectrum of the M-point real transform, with E = (Z[k] + conj Z[P-k]) / 2,
//     O = (Z[k] - conj Z[P-k]) / (2i); slot of k = 0 holds (X0, XP).
//   pre (c2r): the inverse map (Z[k] = E + i O, Z[P-k] = conj(E) + i conj(O));
//     after the inverse passes slot j holds P (x[2j] + i x[2j+1]).
// a and b may alias (k = P/2): both formulas then write the same value twice.
__device__ __forceinline__ void post_pair(double2& a, double2& b, double2 w) {
  const double2 e = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
  const double2 o = make_double2(0.5 * (a.y + b.y), -0.5 * (a.x - b.x));
  const double2 wo = cmul(w, o);
  a = cadd(e, wo);
  b = cconj(csub(e, wo));
}
__device__ __forceinline__ void pre_pair(double2& a, double2& b, double2 w) {
  const double2 e = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
  const double2 dif = make_double2(0.5 * (a.x - b.x), 0.5 * (a.y + b.y));
  const double2 o = cmul(dif, cconj(w));
  a = make_double2(e.x - o.y, e.y + o.x);
  b = make_double2(e.x + o.y, -e.y + o.x);
}

// Last DIF pass fused with the r2c post map / first DIT pass fused with the
// c2r pre map.
// The last pass (radix R, stride 1, no twiddles) transforms groups b of R
// consecutive slots; slot b R + r holds frequency k = m(b) + r G (G = P / R).
// The partner P - k of every k in group b sits in the mirror group b' with
// m(b') = G - m(b), at r' = R - 1 - r; groups with m = 0 or 2m = G pair with
// themselves. One thread takes a unit (b, b') — both groups in registers — so
// the (k, P-k) pass needs no extra shared-memory sweep (nor its
// bank-conflicted frequency-order accesses). units[u] = {b | b' << 16, m(b)}
// (fft_plan.cu).
// w_M^{m + rG} for the fused pass (M = 2 R G): w_M^m times the constant
// w_M^{rG} = exp(-i pi r / R) — one table lookup per group instead of R.
template <int R>
__device__ __forceinline__ double2 group_twiddle(double2 wm, int r) {
  if constexpr (R == 2 || R == 4 || R == 8) {
    const int q = r * (8 / R);  // angle pi r / R = 2 pi q / 16
    const double2 c = make_double2(cos16(q), -cos16(q - 4));
    return r == 0 ? wm : cmul(wm, c);
  } else {
    constexpr double kPi = 3.14159265358979323846;
    return r == 0 ? wm : cmul(wm, make_double2(cos(kPi * r / R), -sin(kPi * r / R)));
  }
}

template <int R, bool kForward>
__device__ __forceinline__ void pair_group_pass(double2* buf, const FftPlan& pl,
                                                const double2* tw) {
  const uint2* un = smem_units(tw, pl);
  const int hi_off = 1 << kTwLoBits;
  for (int u = threadIdx.x; u < pl.nunits; u += blockDim.x) {
    const uint2 d = un[u];
    const uint32_t b = d.x & 0xffffu, bp = d.x >> 16, m = d.y;
    double2 x[R], y[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = buf[swz(b * R + r)];
    if (bp != b) {
#pragma unroll
      for (int r = 0; r < R; ++r) y[r] = buf[swz(bp * R + r)];
    }
    if (kForward) RegDft<R>::run(x, -1.0);
    if (bp != b) {
      if (kForward) RegDft<R>::run(y, -1.0);
      const double2 wm = twiddle(tw, hi_off, m);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double2 w = group_twiddle<R>(wm, r);
        if (kForward) post_pair(x[r], y[R - 1 - r], w);
        else pre_pair(x[r], y[R - 1 - r], w);
      }
      if (!kForward) RegDft<R>::run(y, +1.0);
#pragma unroll
      for (int r = 0; r < R; ++r) buf[swz(bp * R + r)] = y[r];
    } else if (m == 0) {  // k = r G: pairs (r, R - r), r = 0 the (X0, XP) slot
      const double2 z = x[0];
      x[0] = kForward ? make_double2(z.x + z.y, z.x - z.y)
                      : make_double2(0.5 * (z.x + z.y), 0.5 * (z.x - z.y));
#pragma unroll
      for (int r = 1; r <= R / 2; ++r) {
        const double2 w = group_twiddle<R>(make_double2(1.0, 0.0), r);
        if (kForward) post_pair(x[r], x[R - r], w);
        else pre_pair(x[r], x[R - r], w);
      }
    } else {  // 2m = G: pairs (r, R - 1 - r)
      const double2 wm = twiddle(tw, hi_off, m);
#pragma unroll
      for (int r = 0; r <= (R - 1) / 2; ++r) {
        const double2 w = group_twiddle<R>(wm, r);
        if (kForward) post_pair(x[r], x[R - 1 - r], w);
        else pre_pair(x[r], x[R - 1 - r], w);
      }
    }
    if (!kForward) RegDft<R>::run(x, +1.0);
#pragma unroll
    for (int r = 0; r < R; ++r) buf[swz(b * R + r)] = x[r];
  }
}

template <bool kForward>
__device__ __forceinline__ void pair_group_dispatch(double2* buf, const FftPlan& pl,
                                                    const double2* tw) {
  switch (pass_radix(pl, pl.npass - 1)) {
    case 8: pair_group_pass<8, kForward>(buf, pl, tw); break;
    case 4: pair_group_pass<4, kForward>(buf, pl, tw); break;
    case 3: pair_group_pass<3, kForward>(buf, pl, tw); break;
    default: pair_group_pass<2, kForward>(buf, pl, tw); break;
  }
}

// fft_forward + the r2c post map (no trailing barrier).
__device__ __forceinline__ void fft_forward_post(double2* buf, const FftPlan& pl,
                                                 const double2* tw) {
  int L = pl.P;
  for (int p = 0; p + 1 < pl.npass; ++p) {
    const int R = pass_radix(pl, p);
    fft_dispatch<true>(buf, tw, 1 << kTwLoBits, pl.M, pl.P, R, L);
    __syncthreads();
    L /= R;
  }
  pair_group_dispatch<true>(buf, pl, tw);
}

// Both buffers: paired forward passes + the r2c post map.
__device__ __forceinline__ void fft_forward2_post(double2* __restrict__ b0,
                                                  double2* __restrict__ b1, const FftPlan& pl,
                                                  const double2* tw) {
  fft_forward2_passes(b0, b1, pl, tw, pl.npass - 1);
  pair_group_dispatch<true>(b0, pl, tw);
  pair_group_dispatch<true>(b1, pl, tw);
}

// The c2r pre map + fft_inverse (ends with a barrier, like fft_inverse).
__device__ __forceinline__ void fft_inverse_pre(double2* buf, const FftPlan& pl,
                                                const double2* tw) {
  pair_group_dispatch<false>(buf, pl, tw);
  __syncthreads();
  int L = pass_radix(pl, pl.npass - 1);
  for (int p = pl.npass - 2; p >= 0; --p) {
    const int R = pass_radix(pl, p);
    L *= R;
    fft_dispatch<false>(buf, tw, 1 << kTwLoBits, pl.M, pl.P, R, L);
    __syncthreads();
  }
}

// Zero the P packed slots.
__device__ __forceinline__ void zero_slots(double2* buf, int P) {
  for (int s = threadIdx.x; s < P; s += blockDim.x) buf[s] = make_double2(0.0, 0.0);
}

// Real value x[t] of a natural-order packed buffer.
__device__ __forceinline__ double& packed_real(double2* buf, uint32_t t) {
  double2& s = buf[swz(t >> 1)];
  return (t & 1u) ? s.y : s.x;
}

// Loads the twiddle table (lo then hi), the last-pass pair units and, with
// with_f2p, the frequency -> slot table into shared memory (table_slots layout).
__device__ __forceinline__ void load_twiddles(double2* sm_tw, const FftPlan& pl,
                                              bool with_f2p = true) {
  const int n = (1 << kTwLoBits) + pl.hi_count;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm_tw[i] = __ldg(pl.tw + i);
  uint2* units = reinterpret_cast<uint2*>(sm_tw + n);
  for (int i = threadIdx.x; i < pl.nunits; i += blockDim.x) units[i] = __ldg(pl.units + i);
  if (!with_f2p) return;
  // P is a multiple of 8: copy the table as int4 with all loads in flight
  int4* f2p = reinterpret_cast<int4*>(sm_tw + n + (pl.nunits + 1) / 2);
  const int4* src = reinterpret_cast<const int4*>(pl.f2p);
  const int n4 = pl.P / 4;
  constexpr int kU = 8;
  for (int i0 = threadIdx.x; i0 < n4; i0 += kU * blockDim.x) {
    int4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + u * blockDim.x < n4) v[u] = __ldg(src + i0 + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + u * blockDim.x < n4) f2p[i0 + u * blockDim.x] = v[u];
  }
}

// load_twiddles without the frequency -> slot table, as asynchronous 16-byte
// global -> shared copies (cp.async): the caller overlaps the latency with
// other work and calls cp_async_wait_all() before the first FFT pass.
__device__ __forceinline__ void load_twiddles_async(double2* sm_tw, const FftPlan& pl) {
  const int n = (1 << kTwLoBits) + pl.hi_count + (pl.nunits + 1) / 2;  // 16-byte chunks
  const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(sm_tw));
  const int ntw = (1 << kTwLoBits) + pl.hi_count;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const void* src = i < ntw ? static_cast<const void*>(pl.tw + i)
                              : static_cast<const void*>(pl.units + 2 * (i - ntw));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * i), "l"(src)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Pointwise helpers on the half-spectrum slot layout (slot 0 holds two reals).
__device__ __forceinline__ double2 hmul(double2 a, double2 b, bool slot0) {
  return slot0 ? make_double2(a.x * b.x, a.y * b.y) : cmul(a, b);
}
__device__ __forceinline__ double2 hconj(double2 a, bool slot0) { return slot0 ? a : cconj(a); }

// Shared-memory bytes a spectral kernel with this plan needs (buffer + twiddles).
inline size_t fft_smem_bytes(const FftPlan& pl, bool with_f2p = true) {
  return static_cast<size_t>(pl.P + table_slots(pl, with_f2p)) * sizeof(double2);
}

// Host: plan for the smallest supported M >= min_len (cached per device):
// one-CTA shared-memory plans up to kMaxFftM, two-level plans beyond.
int get_fft_plan(size_t min_len, FftPlan* out);
int get_large_fft(const FftPlan& pl, LargeFft* out);

// Kernel argument blocks shared by spectral.cu (kernels) and engine.cu (host).
struct CpArgs {
  int order;
  int dims[ST_MAX_ORDER];
  int tab_off[ST_MAX_ORDER];
  int hash_lens[ST_MAX_ORDER];
  int fam_stride;
  const double* factors[ST_MAX_ORDER];  // I_n x R column-major
  const double* weights;
  int r_begin;
  int r_count;
};

struct EngArgs {
  int dims[3];
  int tab_off[3];
  int fam_stride;
  int D;
  int hash_len;            // J of every mode
  const uint32_t* packed;  // D families x 3 modes, packed tables
  const double2* spec;     // D x P cached spectra S_d (slot order)
};

// Fused epilogue of the cluster estimator: the last cluster of vector b to
// finish (per-vector arrival counter) takes the median over the D families
// and, by mode, normalises the row (the rtpm restart step) or applies the
// refinement update (cpd.cpp:266-270).
struct IuvTail {
  int mode = 0;             // 0: estimates only; 1: median -> out; 2: median, row / ||row|| -> out;
                            // 3: median -> out (scratch), best = out / ||out|| unless stopped;
                            // 4: T(u, v, w) = <w, T(u, v, I)> per family, median -> out[b]
  int* cnt = nullptr;       // batch arrival counters, zero between launches
  double* out = nullptr;    // batch x nf
  double* best = nullptr;   // mode 3
  int* stopped = nullptr;   // mode 3: sticky underflow flag
  const double* wvec = nullptr;  // mode 4: batch x dims[2] third vectors
};
// Cluster (8-CTA, DSMEM) form of the iuv estimator for M in {2048, 3072, 4096,
// 8192, 9216} and batches that fit one wave of clusters (spectral_cluster.cu);
// returns 1 without launching otherwise.
int launch_iuv_cluster(const FftPlan& pl, const EngArgs& e, int batch, const double* A,
                       const double* B, int c1, int c2, int f, double* est, const IuvTail& tail,
                       cudaStream_t st);
// Cluster form of the deflation S_d -= weight F(cs_u) F(cs_v) F(cs_w) (D <= 32).
int launch_deflate_cluster(const FftPlan& pl, const EngArgs& e, double weight, const double* U,
                           const double* V, const double* W, double2* spec, cudaStream_t st);
// Cluster form of the per-family inverse of a half spectrum in slot order
// (cp_sum_kernel: out[d][t] (+)= z[t], t < jt).
int launch_spec_inverse_cluster(const FftPlan& pl, const double2* acc, int D, double* out, int jt,
                                int accumulate, cudaStream_t st);
// Cluster form of the row-pair linear convolution (same lengths; one wave).
int launch_conv_cluster(const FftPlan& pl, const double* a, int la, size_t lda, const double* b,
                        int lb, size_t ldb, int items, double* out, size_t ldo, cudaStream_t st);

// Two-level counterparts of the spectral launchers (spectral_large.cu).
// Exact n-point transforms (Bluestein over the library FFTs, spectral_large.cu).
int exact_dft(const double* xr, const double2* xc, size_t ldx, size_t len, size_t n, int items,
              double sign, double2* out, cudaStream_t st);
int exact_idft_real(const double2* spec, size_t n, int items, double* out, int check,
                    cudaStream_t st);
int exact_fft_convolve(const double* const* inputs, const size_t* lens, size_t k, size_t n,
                       double* out, cudaStream_t st);
int exact_precompute_z(const double2* spectrum, size_t n, const double* csa, size_t ja,
                       const double* csb, size_t jb, double* z, cudaStream_t st);
int large_rfft(const FftPlan& pl, const double* x, size_t ldx, int64_t len, int items,
               double2* spec, cudaStream_t st);
int large_irfft(const FftPlan& pl, double2* spec, int items, double* out, size_t ldo,
                int64_t out_len, int accumulate, cudaStream_t st);
int large_real_from_spec(const FftPlan& pl, const double2* spec, int items, double* out,
                         size_t ldo, int out_len, int accumulate, cudaStream_t st);
int large_conv(const FftPlan& pl, const double* a, int la, size_t lda, const double* b, int lb,
               size_t ldb, int items, double* out, size_t ldo, cudaStream_t st);
int large_iuv(const FftPlan& pl, const EngArgs& e, int batch, const double* A, const double* B,
              int c1, int c2, int f, int J, double* est, cudaStream_t st);
int large_uvw(const FftPlan& pl, const EngArgs& e, int batch, const double* U, const double* V,
              const double* W, int J, double* est, cudaStream_t st);
int large_deflate(const FftPlan& pl, const EngArgs& e, double weight, const double* U,
                  const double* V, const double* W, int J, double2* spec, cudaStream_t st);
int large_cp(const FftPlan& pl, const CpArgs& a, int D, const uint32_t* packed, const int* J,
             double* out, int jt, int accumulate, cudaStream_t st);

}  // namespace fcs
