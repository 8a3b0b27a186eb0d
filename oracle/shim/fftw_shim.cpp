// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Exact-length fp64 complex DFT behind the fftw3.h subset in fftw3.h.
// Recursive decimation-in-time Cooley–Tukey over the prime factorisation of
// n when every prime factor is <= 61; otherwise Bluestein's chirp-z through a
// power-of-two transform of length >= 2n-1. Sign convention matches FFTW:
// X[j] = sum_k x[k] exp(sign * 2*pi*i*j*k/n), unnormalised.
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstdint>
#include <vector>

using cd = std::complex<double>;

struct shim_fftw_plan_s {
  int n = 0;
  int sign = -1;
  std::vector<int> factors;      // mixed-radix factors (empty when Bluestein)
  std::vector<cd> twiddle;       // exp(sign*2*pi*i*t/n), t in [0, n)
  // Bluestein state
  int m = 0;                     // power-of-two convolution length
  std::vector<cd> chirp;         // exp(sign*pi*i*k^2/n), k in [0, n)
  std::vector<cd> kernel_hat;    // forward transform of conj(chirp) kernel
  shim_fftw_plan_s* sub_fwd = nullptr;
  shim_fftw_plan_s* sub_bwd = nullptr;
};

namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;

std::vector<int> factorize(int n, int* largest) {
  std::vector<int> f;
  *largest = 1;
  while (n % 4 == 0) { f.push_back(4); n /= 4; *largest = 2 > *largest ? 2 : *largest; }
  for (int p = 2; p * p <= n; ++p) {
    while (n % p == 0) { f.push_back(p); n /= p; if (p > *largest) *largest = p; }
  }
  if (n > 1) { f.push_back(n); if (n > *largest) *largest = n; }
  return f;
}

// out[0..n) = DFT of in[0], in[stride], ... using factors[fi..]
void mixed_radix(const shim_fftw_plan_s* p, const cd* in, std::size_t stride, cd* out, int n,
                 std::size_t fi, std::size_t tw_stride) {
  if (n == 1) {
    out[0] = in[0];
    return;
  }
  const int r = p->factors[fi];
  const int m = n / r;
  for (int q = 0; q < r; ++q) {
    mixed_radix(p, in + q * stride, stride * r, out + q * m, m, fi + 1, tw_stride * r);
  }
  // Butterflies: out'[k + j m] = sum_q out[q m + k] * w_n^{q (k + j m)}.
  std::vector<cd> tmp(static_cast<std::size_t>(r));
  const std::size_t big_n = static_cast<std::size_t>(p->n);
  for (int k = 0; k < m; ++k) {
    for (int q = 0; q < r; ++q) tmp[q] = out[q * m + k];
    for (int j = 0; j < r; ++j) {
      cd acc = 0.0;
      for (int q = 0; q < r; ++q) {
        const std::size_t e =
            (static_cast<std::size_t>(q) * static_cast<std::size_t>(k + j * m) * tw_stride) % big_n;
        acc += tmp[q] * p->twiddle[e];
      }
      out[k + j * m] = acc;
    }
  }
}

void execute(const shim_fftw_plan_s* p, const cd* in, cd* out) {
  if (p->factors.empty() && p->m == 0) {  // n == 1
    out[0] = in[0];
    return;
  }
  if (p->m == 0) {
    std::vector<cd> src(in, in + p->n);  // allow in == out
    mixed_radix(p, src.data(), 1, out, p->n, 0, 1);
    return;
  }
  // Bluestein: X_j = c_j * sum_k (x_k c_k) conj(c_{j-k}).
  std::vector<cd> a(static_cast<std::size_t>(p->m), 0.0), ah(static_cast<std::size_t>(p->m));
  for (int k = 0; k < p->n; ++k) a[k] = in[k] * p->chirp[k];
  execute(p->sub_fwd, a.data(), ah.data());
  for (int t = 0; t < p->m; ++t) ah[t] *= p->kernel_hat[t];
  execute(p->sub_bwd, ah.data(), a.data());
  const double inv_m = 1.0 / static_cast<double>(p->m);
  for (int j = 0; j < p->n; ++j) out[j] = p->chirp[j] * a[j] * inv_m;
}

shim_fftw_plan_s* make_plan(int n, int sign) {
  auto* p = new shim_fftw_plan_s;
  p->n = n;
  p->sign = sign;
  int largest = 1;
  std::vector<int> f = factorize(n, &largest);
  if (n == 1) return p;
  if (largest <= 61) {
    p->factors = f;
    p->twiddle.resize(static_cast<std::size_t>(n));
    for (int t = 0; t < n; ++t) {
      const double ang = sign * kTwoPi * static_cast<double>(t) / n;
      p->twiddle[t] = cd(std::cos(ang), std::sin(ang));
    }
    return p;
  }
  int m = 1;
  while (m < 2 * n - 1) m <<= 1;
  p->m = m;
  p->chirp.resize(static_cast<std::size_t>(n));
  const std::uint64_t two_n = 2ULL * static_cast<std::uint64_t>(n);
  for (int k = 0; k < n; ++k) {
    const std::uint64_t kk = (static_cast<std::uint64_t>(k) * static_cast<std::uint64_t>(k)) % two_n;
    const double ang = sign * kTwoPi * 0.5 * static_cast<double>(kk) / n;
    p->chirp[k] = cd(std::cos(ang), std::sin(ang));
  }
  p->sub_fwd = make_plan(m, -1);
  p->sub_bwd = make_plan(m, +1);
  std::vector<cd> b(static_cast<std::size_t>(m), 0.0);
  b[0] = std::conj(p->chirp[0]);
  for (int t = 1; t < n; ++t) {
    b[t] = std::conj(p->chirp[t]);
    b[m - t] = std::conj(p->chirp[t]);
  }
  p->kernel_hat.resize(static_cast<std::size_t>(m));
  execute(p->sub_fwd, b.data(), p->kernel_hat.data());
  return p;
}

void free_plan(shim_fftw_plan_s* p) {
  if (!p) return;
  free_plan(p->sub_fwd);
  free_plan(p->sub_bwd);
  delete p;
}

}  // namespace

extern "C" fftw_plan fftw_plan_dft_1d(int n, fftw_complex*, fftw_complex*, int sign, unsigned) {
  return make_plan(n, sign);
}

extern "C" void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
  execute(p, reinterpret_cast<const cd*>(in), reinterpret_cast<cd*>(out));
}

extern "C" void fftw_destroy_plan(fftw_plan p) { free_plan(p); }
