// Drop-in check: the reference's FcsEngine (cpd.cpp:61-94, built unmodified in
// oracle/_ref) and the GPU-backed GpuFcsEngine, constructed through the same
// factory signature, must agree on every ContractionEngine call (cpd.hpp:21-41)
// and on a power-iteration driver written only against that interface.
// Prints one JSON line; exit 0 iff every comparison is within 1e-9 relative.
#include <sketchtensor/cpd.hpp>
#include <sketchtensor/rng.hpp>

#include <cmath>
#include <cstdio>
#include <limits>
#include <memory>
#include <vector>

#include "gpu_fcs_engine.hpp"

using namespace sketchtensor;

namespace {

double rel_err(const Eigen::VectorXd& g, const Eigen::VectorXd& c) {
  double inf = 0.0, worst = 0.0;
  for (Eigen::Index i = 0; i < c.size(); ++i) inf = std::max(inf, std::abs(c[i]));
  for (Eigen::Index i = 0; i < c.size(); ++i)
    worst = std::max(worst, std::abs(g[i] - c[i]) / (std::abs(c[i]) + inf + 1e-300));
  return worst;
}

Eigen::VectorXd gaussian_vec(SplitMix64& rng, std::size_t n) {
  Eigen::VectorXd v(static_cast<Eigen::Index>(n));
  for (std::size_t i = 0; i < n; ++i) v[static_cast<Eigen::Index>(i)] = rng.next_gaussian();
  return v;
}

// Power iteration with deflation using only the ContractionEngine interface.
std::vector<double> power_method(ContractionEngine& e, std::size_t dim, std::size_t rank,
                                 std::size_t inits, std::size_t iters, std::uint64_t seed) {
  SplitMix64 rng(seed);
  std::vector<double> weights;
  for (std::size_t r = 0; r < rank; ++r) {
    Eigen::VectorXd best;
    double best_value = -std::numeric_limits<double>::infinity();
    for (std::size_t l = 0; l < inits; ++l) {
      Eigen::VectorXd u = gaussian_vec(rng, dim);
      u /= u.norm();
      for (std::size_t it = 0; it < iters; ++it) {
        u = e.iuu(u);
        u /= u.norm();
      }
      const double value = e.uuu(u);
      if (value > best_value) {
        best_value = value;
        best = u;
      }
    }
    const double w = e.uuu(best);
    weights.push_back(w);
    e.deflate(w, best, best, best);
  }
  return weights;
}

}  // namespace

int main() {
  EstimatorConfig cfg;
  cfg.hash_len = 64;
  cfg.sketch_count = 5;
  cfg.seed = 9;
  SplitMix64 rng(77);
  DenseTensor t({40, 30, 20});
  for (std::size_t i = 0; i < t.size(); ++i) t[i] = rng.next_gaussian();
  auto ref = sketchtensor::make_contraction_engine(t, SketchBackend::FCS, cfg);
  auto gpu = sketchtensor_b200::make_contraction_engine(t, SketchBackend::FCS, cfg);
  const Eigen::VectorXd u = gaussian_vec(rng, 40), v = gaussian_vec(rng, 30),
                        w = gaussian_vec(rng, 20);
  double worst = 0.0;
  worst = std::max(worst, rel_err(gpu->iuv(v, w, 0), ref->iuv(v, w, 0)));
  worst = std::max(worst, rel_err(gpu->iuv(u, w, 1), ref->iuv(u, w, 1)));
  worst = std::max(worst, rel_err(gpu->iuv(u, v, 2), ref->iuv(u, v, 2)));
  Eigen::VectorXd a(1), b(1);
  a[0] = gpu->uvw(u, v, w);
  b[0] = ref->uvw(u, v, w);
  worst = std::max(worst, rel_err(a, b));
  ref->deflate(0.5, u, v, w);
  gpu->deflate(0.5, u, v, w);
  worst = std::max(worst, rel_err(gpu->iuv(u, v, 2), ref->iuv(u, v, 2)));
  a[0] = gpu->uvw(u, v, w);
  b[0] = ref->uvw(u, v, w);
  worst = std::max(worst, rel_err(a, b));
  // the TS backend through the same factory (TsEngine, cpd.cpp:96-126)
  auto ref_ts = sketchtensor::make_contraction_engine(t, SketchBackend::TS, cfg);
  auto gpu_ts = sketchtensor_b200::make_contraction_engine(t, SketchBackend::TS, cfg);
  worst = std::max(worst, rel_err(gpu_ts->iuv(v, w, 0), ref_ts->iuv(v, w, 0)));
  worst = std::max(worst, rel_err(gpu_ts->iuv(u, w, 1), ref_ts->iuv(u, w, 1)));
  a[0] = gpu_ts->uvw(u, v, w);
  b[0] = ref_ts->uvw(u, v, w);
  worst = std::max(worst, rel_err(a, b));
  ref_ts->deflate(0.5, u, v, w);
  gpu_ts->deflate(0.5, u, v, w);
  worst = std::max(worst, rel_err(gpu_ts->iuv(u, v, 2), ref_ts->iuv(u, v, 2)));
  // the exact and baseline backends (Plain, HCS, long-pair CS) through the same factory
  EstimatorConfig small = cfg;
  small.hash_len = 12;
  for (SketchBackend bk : {SketchBackend::Plain, SketchBackend::HCS, SketchBackend::CS}) {
    auto r = sketchtensor::make_contraction_engine(t, bk, small);
    auto g = sketchtensor_b200::make_contraction_engine(t, bk, small);
    worst = std::max(worst, rel_err(g->iuv(v, w, 0), r->iuv(v, w, 0)));
    a[0] = g->uvw(u, v, w);
    b[0] = r->uvw(u, v, w);
    worst = std::max(worst, rel_err(a, b));
    r->deflate(0.5, u, v, w);
    g->deflate(0.5, u, v, w);
    worst = std::max(worst, rel_err(g->iuv(u, w, 1), r->iuv(u, w, 1)));
  }
  bool threw = false;
  try {
    gpu->iuv(u, v, 3);
  } catch (const std::invalid_argument&) {
    threw = true;
  }

  // symmetric cube: rank-2 + noise, power method through the interface only
  DenseTensor s({24, 24, 24});
  Eigen::VectorXd p = gaussian_vec(rng, 24), q = gaussian_vec(rng, 24);
  p /= p.norm();
  q /= q.norm();
  for (std::size_t k = 0; k < 24; ++k)
    for (std::size_t j = 0; j < 24; ++j)
      for (std::size_t i = 0; i < 24; ++i)
        s.at({i, j, k}) = 3.0 * p[i] * p[j] * p[k] + 1.5 * q[i] * q[j] * q[k];
  EstimatorConfig c2 = cfg;
  c2.hash_len = 40;
  auto ref2 = sketchtensor::make_contraction_engine(s, SketchBackend::FCS, c2);
  auto gpu2 = sketchtensor_b200::make_contraction_engine(s, SketchBackend::FCS, c2);
  const auto wr = power_method(*ref2, 24, 2, 3, 8, 5);
  const auto wg = power_method(*gpu2, 24, 2, 3, 8, 5);
  Eigen::VectorXd wa(2), wb(2);
  for (int r = 0; r < 2; ++r) {
    wa[r] = wg[r];
    wb[r] = wr[r];
  }
  const double wrel = rel_err(wa, wb);
  const bool ok = worst < 1e-9 && wrel < 1e-8 && threw;
  std::printf(
      "{\"ok\": %s, \"max_rel_err_calls\": %.3e, \"max_rel_err_power_method\": %.3e, "
      "\"invalid_argument_on_bad_mode\": %s, \"weights_ref\": [%.12f, %.12f], "
      "\"weights_gpu\": [%.12f, %.12f]}\n",
      ok ? "true" : "false", worst, wrel, threw ? "true" : "false", wb[0], wb[1], wa[0], wa[1]);
  return ok ? 0 : 1;
}
