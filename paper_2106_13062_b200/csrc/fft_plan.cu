// Host-side FFT plans: padded length choice, radix schedule, twiddle table
// and frequency -> slot map, cached per (device, M).
#include <cmath>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "fft.cuh"

namespace fcs {

namespace {

// Smallest M >= n (M = 2^a 3^b with a >= 4, b <= 2) not above kMaxFftM. a >= 4
// keeps P = M/2 a multiple of 8, which the slot swizzle (groups of 8) needs.
int choose_m(size_t n) {
  int best = 0;
  for (int b3 = 1; b3 <= 9; b3 *= 3) {
    for (long m = 16L * b3; m <= kMaxFftM; m *= 2) {
      if (m >= static_cast<long>(n) && (best == 0 || m < best)) best = static_cast<int>(m);
    }
  }
  return best;
}

// Slot position -> frequency for the DIF schedule (radices in pass order):
// freq(p) = r' + R * freq_sub(p mod (L/R)) with r' = p / (L/R).
int freq_of(int p, const std::vector<int>& radix, size_t level, int L) {
  if (level == radix.size() || L == 1) return 0;
  const int R = radix[level];
  const int sub = L / R;
  return p / sub + R * freq_of(p % sub, radix, level + 1, sub);
}

}  // namespace

// Two-level plan: the smallest P = P1 * P2 >= ceil(min_len / 2) over the
// one-CTA sizes, ties broken toward balanced factors (P1 <= P2).
int large_plan(size_t min_len, FftPlan* out) {
  std::vector<long> sizes;
  for (int b3 = 1; b3 <= 9; b3 *= 3)
    for (long m = 16L * b3; m <= kMaxFftM; m *= 2) sizes.push_back(m / 2);
  const long need = static_cast<long>((min_len + 1) / 2);
  long best = 0, b1 = 0;
  for (long p1 : sizes)
    for (long p2 : sizes) {
      if (p1 > p2 || p1 * p2 < need) continue;
      const long p = p1 * p2;
      if (best == 0 || p < best || (p == best && p2 - p1 < best / b1 - b1)) {
        best = p;
        b1 = p1;
      }
    }
  if (best == 0 || best > (1L << 30))
    return fail(ST_EINVAL, "fft: composed length " + std::to_string(min_len) + " is too large");
  FftPlan pl{};
  pl.M = static_cast<int>(2 * best);
  pl.P = static_cast<int>(best);
  pl.large_p1 = static_cast<int>(b1);
  *out = pl;
  return ST_OK;
}

int get_fft_plan(size_t min_len, FftPlan* out) {
  const int M = choose_m(min_len);
  if (M == 0) return large_plan(min_len, out);
  int dev = 0;
  FCS_CUDA_TRY(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<std::pair<int, int>, FftPlan> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({dev, M});
  if (it != cache.end()) {
    *out = it->second;
    return ST_OK;
  }
  FftPlan pl{};
  pl.M = M;
  pl.P = M / 2;
  // radix schedule: 9s and 3s first, then 16s, then the remainder (16 * 2 as 8 * 4)
  std::vector<int> radix;
  int rem = pl.P;
  while (rem % 9 == 0) {  // 3 * 3 as one radix-9 pass (one shared-memory sweep fewer)
    radix.push_back(9);
    rem /= 9;
  }
  if (rem % 3 == 0) {
    radix.push_back(3);
    rem /= 3;
  }
  while (rem % 16 == 0) {
    radix.push_back(16);
    rem /= 16;
  }
  if (rem == 2 && !radix.empty() && radix.back() == 16) {
    radix.back() = 8;  // 16 * 2 -> 8 * 4: a radix-2 pass has P/2 butterflies
    rem = 4;
  }
  if (rem > 1) radix.push_back(rem);  // 8, 4 or 2
  if (rem == 1 && !radix.empty() && radix.back() == 16) {
    radix.back() = 4;  // the fused last pass (pair_group_pass) holds 2 R values: R <= 8
    radix.push_back(4);
  }
  pl.npass = static_cast<int>(radix.size());
  int L = pl.P;
  for (int p = 0; p < pl.npass; ++p) {
    pl.radix[p] = radix[p];
    pl.len[p] = L;
    pl.rcode |= static_cast<unsigned long long>(radix[p] - 1) << (4 * p);
    L /= radix[p];
  }
  pl.hi_count = (M + (1 << kTwLoBits) - 1) >> kTwLoBits;
  std::vector<double2> tw((1 << kTwLoBits) + pl.hi_count);
  auto root = [M](long e) {
    // exp(-2 pi i e / M), angle reduced exactly in integers first
    const long r = e % M;
    const long double ang = -2.0L * 3.141592653589793238462643383279502884L * r / M;
    return make_double2(static_cast<double>(std::cos(ang)), static_cast<double>(std::sin(ang)));
  };
  for (int e = 0; e < (1 << kTwLoBits); ++e) tw[e] = root(e);
  for (int e = 0; e < pl.hi_count; ++e) tw[(1 << kTwLoBits) + e] = root(static_cast<long>(e) << kTwLoBits);
  std::vector<int> f2p(pl.P);
  for (int p = 0; p < pl.P; ++p) f2p[freq_of(p, radix, 0, pl.P)] = p;
  // pair units of the fused last pass: group b holds k = m(b) + r G; its
  // partner group has m = G - m(b) (self for m = 0 and 2m = G)
  const int R = radix.back(), G = pl.P / R;
  std::vector<int> m_of(G), b_of(G);
  for (int b = 0; b < G; ++b) {
    m_of[b] = freq_of(b * R, radix, 0, pl.P);
    b_of[m_of[b]] = b;
  }
  std::vector<uint2> units;
  for (int b = 0; b < G; ++b) {
    const int m = m_of[b];
    if (m == 0 || 2 * m == G) {
      units.push_back(make_uint2(static_cast<uint32_t>(b) | (static_cast<uint32_t>(b) << 16), m));
    } else if (m < G - m) {
      const int bp = b_of[G - m];
      units.push_back(make_uint2(static_cast<uint32_t>(b) | (static_cast<uint32_t>(bp) << 16), m));
    }
  }
  pl.nunits = static_cast<int>(units.size());
  if (units.size() & 1) units.push_back(make_uint2(0, 0));  // whole 16-byte chunks (async copy)
  double2* dtw = nullptr;
  int* df2p = nullptr;
  FCS_CUDA_TRY(cudaMalloc(&dtw, tw.size() * sizeof(double2)));
  FCS_CUDA_TRY(cudaMalloc(&df2p, f2p.size() * sizeof(int)));
  FCS_CUDA_TRY(cudaMemcpy(dtw, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
  FCS_CUDA_TRY(cudaMemcpy(df2p, f2p.data(), f2p.size() * sizeof(int), cudaMemcpyHostToDevice));
  uint2* dunits = nullptr;
  FCS_CUDA_TRY(cudaMalloc(&dunits, units.size() * sizeof(uint2)));
  FCS_CUDA_TRY(cudaMemcpy(dunits, units.data(), units.size() * sizeof(uint2),
                          cudaMemcpyHostToDevice));
  pl.units = dunits;
  pl.tw = dtw;
  pl.f2p = df2p;
  cache[{dev, M}] = pl;
  *out = pl;
  return ST_OK;
}

}  // namespace fcs
