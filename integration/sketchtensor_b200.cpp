// libsketchtensor_b200.so — the reference's own free-function API, DEFINED
// over the B200 C-ABI (include/fcs_b200.h).
//
// The reference declares its sketch / estimator / transform entry points in
// proj/include/sketchtensor/{sketch,estimators,fft}.hpp and defines them in
// proj/src/{sketch,estimators,fft}.cpp (CPU, FFTW). This file supplies
// definitions for exactly those declarations, compiled against the
// reference's headers, so a reference build links this library in place of
// the three .cpp files (link-time substitution) and every caller — cpd.cpp's
// engines and rtpm / rtpm_asym / als, user code — runs on the GPU unchanged.
// hashing.cpp, tensor.cpp, rng.cpp and cpd.cpp stay the reference's.
//
// Host work here is argument validation with the reference's exception
// types and messages, host <-> device copies, and assembling the by-value
// results; every sketch, transform, contraction and reduction is a device
// kernel behind the C-ABI. Estimators over spans of precomputed sketches
// build a device engine from the sketches (st_engine_from_sketches, or the
// exact-contraction engine over the HCS / long-pair sketch) and cache it
// under a hash of the sketch contents, since cpd.cpp's engines call them
// thousands of times on unchanged sketches (and mutate HCS / CS sketches in
// place on deflation, which changes the hash).
#include <sketchtensor/estimators.hpp>
#include <sketchtensor/fft.hpp>
#include <sketchtensor/sketch.hpp>

#include <cuda_runtime.h>

#include <algorithm>
#include <complex>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fcs_b200.h"

namespace sketchtensor {

namespace {

// ------------------------------------------------------------ plumbing
void check(int rc) {
  if (rc == ST_OK) return;
  const std::string msg = st_last_error();
  if (rc == ST_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Owned device buffer.
struct Dev {
  void* p = nullptr;
  size_t bytes = 0;
  Dev() = default;
  explicit Dev(size_t n) : bytes(n) {
    if (n) cuda_check(cudaMalloc(&p, n), "cudaMalloc");
  }
  Dev(const void* host, size_t n) : Dev(n) {
    if (n) cuda_check(cudaMemcpy(p, host, n, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  Dev(Dev&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; }
  ~Dev() {
    if (p) cudaFree(p);
  }
  double* d() const { return static_cast<double*>(p); }
  uint32_t* u() const { return static_cast<uint32_t*>(p); }
};

std::vector<double> download(const void* dev, size_t count) {
  std::vector<double> h(count);
  if (count)
    cuda_check(cudaMemcpy(h.data(), dev, count * sizeof(double), cudaMemcpyDeviceToHost),
               "cudaMemcpy D2H");
  return h;
}

Eigen::VectorXd to_vec(const std::vector<double>& h) {
  Eigen::VectorXd v(static_cast<Eigen::Index>(h.size()));
  if (!h.empty()) std::memcpy(v.data(), h.data(), h.size() * sizeof(double));
  return v;
}

// Packed pair / family tables: bucket | (sign < 0) << 31 (fcs_b200.h).
void pack_pair(const HashPair& p, std::vector<uint32_t>& out) {
  for (size_t i = 0; i < p.input_dim(); ++i)
    out.push_back(p.bucket(i) | (p.sign(i) < 0 ? 0x80000000u : 0u));
}
std::vector<uint32_t> pack_family(const HashFamily& f) {
  std::vector<uint32_t> out;
  for (size_t n = 0; n < f.modes(); ++n) pack_pair(f.pair(n), out);
  return out;
}

// require_family_matches / equal_hash_len (sketch.cpp:12-44), same messages.
void require_family_matches(const DenseTensor& t, const HashFamily& family, const char* op) {
  if (t.order() != family.modes())
    throw std::invalid_argument(std::string(op) + ": family order mismatch");
  for (size_t n = 0; n < family.modes(); ++n)
    if (t.shape()[n] != family.pair(n).input_dim())
      throw std::invalid_argument(std::string(op) + ": shape mismatch");
}
void require_family_matches(const CpTensor& cp, const HashFamily& family, const char* op) {
  if (cp.order() != family.modes())
    throw std::invalid_argument(std::string(op) + ": family order mismatch");
  for (size_t n = 0; n < family.modes(); ++n)
    if (static_cast<size_t>(cp.factors[n].rows()) != family.pair(n).input_dim())
      throw std::invalid_argument(std::string(op) + ": shape mismatch");
}
size_t equal_hash_len(const HashFamily& family, const char* op) {
  const size_t len = family.pair(0).hash_len();
  for (size_t n = 1; n < family.modes(); ++n)
    if (family.pair(n).hash_len() != len)
      throw std::invalid_argument(std::string(op) + ": all hash lengths must be equal");
  return len;
}

// A CP tensor on the device: weights, factor matrices (column-major I x R).
struct DevCp {
  Dev w;
  std::vector<Dev> f;
  std::vector<const double*> ptrs;
  std::vector<size_t> dims;
  explicit DevCp(const CpTensor& cp)
      : w(cp.weights.data(), static_cast<size_t>(cp.weights.size()) * sizeof(double)) {
    for (const Eigen::MatrixXd& m : cp.factors) {
      f.emplace_back(m.data(), static_cast<size_t>(m.size()) * sizeof(double));
      dims.push_back(static_cast<size_t>(m.rows()));
    }
    for (const Dev& d : f) ptrs.push_back(d.d());
  }
  size_t rank() const { return w.bytes / sizeof(double); }
};

// ------------------------------------------------- cached device engines
uint64_t mix(uint64_t h, const void* data, size_t bytes) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < bytes; ++i) {  // FNV-1a, 64-bit
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

struct Engine {
  st_engine* e = nullptr;
  std::vector<size_t> dims;
  std::vector<uint32_t> free_tables;  // host copy: pair n's packed table per family (FCS/TS)
  ~Engine() { st_engine_destroy(e); }
};

class EngineCache {
 public:
  template <typename Build>
  std::shared_ptr<Engine> get(uint64_t key, Build&& build) {
    {
      std::lock_guard<std::mutex> lock(mu_);
      for (auto it = lru_.begin(); it != lru_.end(); ++it)
        if (it->first == key) {
          auto hit = it->second;
          lru_.splice(lru_.begin(), lru_, it);
          return hit;
        }
    }
    std::shared_ptr<Engine> e = build();
    std::lock_guard<std::mutex> lock(mu_);
    lru_.emplace_front(key, e);
    if (lru_.size() > kCap) lru_.pop_back();
    return e;
  }

 private:
  static constexpr size_t kCap = 8;
  std::mutex mu_;
  std::list<std::pair<uint64_t, std::shared_ptr<Engine>>> lru_;
};

EngineCache& cache() {
  static EngineCache c;
  return c;
}

// The D families of a span must share dims; FCS/TS engines also need one J.
template <typename Pre>
bool uniform_families(std::span<const Pre> pres, size_t* J) {
  const HashFamily& f0 = pres[0].sketch.family;
  if (f0.modes() != 3) return false;
  *J = f0.pair(0).hash_len();
  for (const Pre& p : pres) {
    const HashFamily& f = p.sketch.family;
    if (f.modes() != 3) return false;
    for (size_t n = 0; n < 3; ++n)
      if (f.pair(n).hash_len() != *J || f.pair(n).input_dim() != f0.pair(n).input_dim())
        return false;
  }
  return true;
}

// FCS / TS engine over the sketches of a span (st_engine_from_sketches).
template <typename Pre>
std::shared_ptr<Engine> sketch_engine(std::span<const Pre> pres, int backend, size_t J) {
  const size_t D = pres.size();
  const size_t len = static_cast<size_t>(pres[0].sketch.values.size());
  const HashFamily& f0 = pres[0].sketch.family;
  const std::vector<size_t> dims = f0.input_dims();
  std::vector<uint32_t> packed;
  std::vector<double> vals;
  vals.reserve(D * len);
  for (const Pre& p : pres) {
    std::vector<uint32_t> t = pack_family(p.sketch.family);
    packed.insert(packed.end(), t.begin(), t.end());
    vals.insert(vals.end(), p.sketch.values.data(), p.sketch.values.data() + len);
  }
  uint64_t key = 0xcbf29ce484222325ull ^ static_cast<uint64_t>(backend);
  key = mix(key, dims.data(), dims.size() * sizeof(size_t));
  key = mix(key, &J, sizeof(J));
  key = mix(key, packed.data(), packed.size() * sizeof(uint32_t));
  key = mix(key, vals.data(), vals.size() * sizeof(double));
  return cache().get(key, [&] {
    auto e = std::make_shared<Engine>();
    e->dims = dims;
    e->free_tables = packed;
    Dev dv(vals.data(), vals.size() * sizeof(double));
    Dev dp(packed.data(), packed.size() * sizeof(uint32_t));
    check(st_engine_from_sketches(&e->e, backend, dv.d(), D, dims.data(), J, dp.u(), nullptr));
    cuda_check(cudaDeviceSynchronize(), "st_engine_from_sketches");
    return e;
  });
}

// Exact-contraction engine over one dense device tensor (the HCS sketch, or
// the long-pair sketch's virtual tensor); `fill` writes it on the device.
template <typename Fill>
std::shared_ptr<Engine> plain_engine(uint64_t key, const std::vector<size_t>& dims, Fill&& fill) {
  return cache().get(key, [&] {
    auto e = std::make_shared<Engine>();
    e->dims = dims;
    Dev t(dims[0] * dims[1] * dims[2] * sizeof(double));
    fill(t.d());
    check(st_engine_create_backend(&e->e, ST_BACKEND_PLAIN, ST_F64, t.d(), dims.data(), 1, 1, 0,
                                   nullptr));
    cuda_check(cudaDeviceSynchronize(), "st_engine_create_backend");
    return e;
  });
}

// One engine call with host vectors.
double engine_uvw(const Engine& e, const Eigen::VectorXd& u, const Eigen::VectorXd& v,
                  const Eigen::VectorXd& w, int median = 1) {
  Dev du(u.data(), u.size() * sizeof(double)), dv(v.data(), v.size() * sizeof(double)),
      dw(w.data(), w.size() * sizeof(double)), out(sizeof(double));
  check(st_engine_uvw(e.e, 1, du.d(), dv.d(), dw.d(), out.d(), median, nullptr));
  return download(out.p, 1)[0];
}
Eigen::VectorXd engine_iuv(const Engine& e, const Eigen::VectorXd& a, const Eigen::VectorXd& b,
                           size_t free_mode, size_t nout) {
  Dev da(a.data(), a.size() * sizeof(double)), db(b.data(), b.size() * sizeof(double)),
      out(nout * sizeof(double));
  check(st_engine_iuv(e.e, 1, da.d(), db.d(), free_mode, out.d(), 1, nullptr));
  return to_vec(download(out.p, nout));
}

// Estimator preconditions (estimators.cpp:16-35), same messages.
void require_order3(const HashFamily& family, const char* op) {
  if (family.modes() != 3) throw std::invalid_argument(std::string(op) + ": order-3 family required");
}
std::pair<size_t, size_t> contracted_modes(size_t free_mode, const char* op) {
  if (free_mode > 2) throw std::invalid_argument(std::string(op) + ": mode out of range");
  return {free_mode == 0 ? 1u : 0u, free_mode == 2 ? 1u : 2u};
}
void require_length(const Eigen::VectorXd& v, const HashPair& pair, const char* op) {
  if (static_cast<size_t>(v.size()) != pair.input_dim())
    throw std::invalid_argument(std::string(op) + ": vector length mismatch");
}

// Device count sketch of a host vector under one pair (cs_sketch's values).
Dev cs_device(const Eigen::VectorXd& x, const HashPair& pair) {
  if (static_cast<size_t>(x.size()) != pair.input_dim())
    throw std::invalid_argument("cs_sketch: input length mismatch");
  std::vector<uint32_t> tab;
  pack_pair(pair, tab);
  Dev dx(x.data(), x.size() * sizeof(double)), dt(tab.data(), tab.size() * sizeof(uint32_t));
  Dev out(pair.hash_len() * sizeof(double));
  check(st_cs_columns(dx.d(), pair.input_dim(), 1, dt.u(), pair.hash_len(), out.d(), nullptr));
  return out;
}

// Device readout out[i] = s(i) src[h(i)] through one pair (host result).
Eigen::VectorXd readout(const double* dsrc, size_t src_len, const HashPair& pair) {
  std::vector<uint32_t> tab;
  pack_pair(pair, tab);
  Dev dt(tab.data(), tab.size() * sizeof(uint32_t)), out(pair.input_dim() * sizeof(double));
  check(st_cs_expand(dsrc, src_len, dt.u(), pair.input_dim(), out.d(), nullptr));
  return to_vec(download(out.p, pair.input_dim()));
}

template <typename Pre, typename Fn>
auto median_over(std::span<const Pre> pres, Fn&& one) {
  if (pres.empty()) throw std::invalid_argument("estimator: no sketches");
  using Result = decltype(one(pres[0]));
  std::vector<Result> results;
  results.reserve(pres.size());
  for (const Pre& pre : pres) results.push_back(one(pre));
  return median_reduce(std::move(results));
}

double dot_device(const Eigen::VectorXd& a, const Eigen::VectorXd& b) {
  Dev da(a.data(), a.size() * sizeof(double)), db(b.data(), b.size() * sizeof(double)),
      out(sizeof(double));
  check(st_sketch_dots(1, static_cast<size_t>(a.size()), da.d(), db.d(), out.d(), nullptr));
  return download(out.p, 1)[0];
}

std::vector<std::complex<double>> to_complex(const std::vector<double>& h) {
  std::vector<std::complex<double>> c(h.size() / 2);
  for (size_t k = 0; k < c.size(); ++k) c[k] = {h[2 * k], h[2 * k + 1]};
  return c;
}

}  // namespace

// =============================================================== sketch.hpp

SketchVec::SketchVec(Eigen::VectorXd v, HashFamily f, SketchKind k)
    : values(std::move(v)), family(std::move(f)), kind(k) {
  const auto len = static_cast<size_t>(values.size());
  const size_t expected =
      kind == SketchKind::FCS ? family.composed_len() : family.pair(0).hash_len();
  if (len != expected) throw std::invalid_argument("SketchVec: length contract violated");
}

SketchTensor::SketchTensor(DenseTensor v, HashFamily f) : values(std::move(v)), family(std::move(f)) {
  if (values.shape() != family.hash_lens())
    throw std::invalid_argument("SketchTensor: shape does not match hash lengths");
}

SketchVec cs_sketch(const Eigen::VectorXd& x, const HashPair& pair) {
  Dev out = cs_device(x, pair);
  return SketchVec(to_vec(download(out.p, pair.hash_len())), HashFamily({pair}), SketchKind::CS);
}

Eigen::MatrixXd cs_sketch_columns(const Eigen::MatrixXd& u, const HashPair& pair) {
  if (static_cast<size_t>(u.rows()) != pair.input_dim())
    throw std::invalid_argument("cs_sketch_columns: input length mismatch");
  const size_t J = pair.hash_len(), R = static_cast<size_t>(u.cols());
  Eigen::MatrixXd out(static_cast<Eigen::Index>(J), u.cols());
  if (R == 0) return out;
  std::vector<uint32_t> tab;
  pack_pair(pair, tab);
  Dev du(u.data(), u.size() * sizeof(double)), dt(tab.data(), tab.size() * sizeof(uint32_t));
  Dev dout(J * R * sizeof(double));
  check(st_cs_columns(du.d(), pair.input_dim(), R, dt.u(), J, dout.d(), nullptr));
  cuda_check(cudaMemcpy(out.data(), dout.p, J * R * sizeof(double), cudaMemcpyDeviceToHost),
             "cudaMemcpy D2H");
  return out;
}

SketchVec ts_sketch(const DenseTensor& t, const HashFamily& family) {
  require_family_matches(t, family, "ts_sketch");
  const size_t J = equal_hash_len(family, "ts_sketch");
  const std::vector<size_t> dims = t.shape(), lens = family.hash_lens();
  const std::vector<uint32_t> packed = pack_family(family);
  Dev dt(t.data().data(), t.size() * sizeof(double));
  Dev dp(packed.data(), packed.size() * sizeof(uint32_t)), out(J * sizeof(double));
  const size_t ws = st_ts_dense_workspace(ST_F64, dims.size(), dims.data(), dims.back(), 1,
                                          lens.data());
  Dev dw(std::max<size_t>(ws, 1));
  check(st_ts_dense(ST_F64, dt.p, dims.size(), dims.data(), 0, dims.back(), 1, dp.u(), lens.data(),
                    out.d(), 0, dw.p, ws, nullptr));
  return SketchVec(to_vec(download(out.p, J)), family, SketchKind::TS);
}

SketchVec ts_sketch(const CpTensor& cp, const HashFamily& family) {
  require_family_matches(cp, family, "ts_sketch");
  const size_t J = equal_hash_len(family, "ts_sketch");
  DevCp d(cp);
  const std::vector<size_t> lens = family.hash_lens();
  const std::vector<uint32_t> packed = pack_family(family);
  Dev dp(packed.data(), packed.size() * sizeof(uint32_t)), out(J * sizeof(double));
  const size_t ws = st_ts_cp_workspace(d.dims.size(), d.dims.data(), d.rank(), 1, lens.data());
  Dev dw(std::max<size_t>(ws, 1));
  check(st_ts_cp(d.w.d(), d.rank(), d.dims.size(), d.dims.data(), d.ptrs.data(), 0, d.rank(), 1,
                 dp.u(), lens.data(), out.d(), 0, dw.p, ws, nullptr));
  return SketchVec(to_vec(download(out.p, J)), family, SketchKind::TS);
}

SketchTensor hcs_sketch(const DenseTensor& t, const HashFamily& family) {
  require_family_matches(t, family, "hcs_sketch");
  const std::vector<size_t> dims = t.shape(), lens = family.hash_lens();
  size_t total = 1;
  for (size_t j : lens) total *= j;
  const std::vector<uint32_t> packed = pack_family(family);
  Dev dt(t.data().data(), t.size() * sizeof(double));
  Dev dp(packed.data(), packed.size() * sizeof(uint32_t)), out(total * sizeof(double));
  const size_t ws = st_hcs_dense_workspace(ST_F64, dims.size(), dims.data(), dims.back(), 1,
                                           lens.data());
  Dev dw(std::max<size_t>(ws, 1));
  check(st_hcs_dense(ST_F64, dt.p, dims.size(), dims.data(), 0, dims.back(), 1, dp.u(),
                     lens.data(), out.d(), 0, dw.p, ws, nullptr));
  return SketchTensor(DenseTensor(lens, download(out.p, total)), family);
}

SketchTensor hcs_sketch(const CpTensor& cp, const HashFamily& family) {
  require_family_matches(cp, family, "hcs_sketch");
  DevCp d(cp);
  const std::vector<size_t> lens = family.hash_lens();
  size_t total = 1;
  for (size_t j : lens) total *= j;
  const std::vector<uint32_t> packed = pack_family(family);
  Dev dp(packed.data(), packed.size() * sizeof(uint32_t)), out(total * sizeof(double));
  const size_t ws = st_hcs_cp_workspace(d.dims.size(), d.dims.data(), d.rank(), 1, lens.data());
  Dev dw(std::max<size_t>(ws, 1));
  check(st_hcs_cp(d.w.d(), d.rank(), d.dims.size(), d.dims.data(), d.ptrs.data(), 1, dp.u(),
                  lens.data(), out.d(), 0, dw.p, ws, nullptr));
  return SketchTensor(DenseTensor(lens, download(out.p, total)), family);
}

SketchVec fcs_sketch(const DenseTensor& t, const HashFamily& family) {
  require_family_matches(t, family, "fcs_sketch");
  const std::vector<size_t> dims = t.shape(), lens = family.hash_lens();
  const std::vector<uint32_t> packed = pack_family(family);
  std::vector<double> out(family.composed_len());
  // host tensor -> chunked H2D overlapped with K1 -> D2H (st_fcs_dense_host_tables)
  check(st_fcs_dense_host_tables(ST_F64, t.data().data(), dims.size(), dims.data(), 0,
                                 dims.back(), 1, packed.data(), lens.data(), out.data()));
  return SketchVec(to_vec(out), family, SketchKind::FCS);
}

SketchVec fcs_sketch(const CpTensor& cp, const HashFamily& family) {
  require_family_matches(cp, family, "fcs_sketch");
  DevCp d(cp);
  const std::vector<size_t> lens = family.hash_lens();
  const size_t jt = family.composed_len();
  const std::vector<uint32_t> packed = pack_family(family);
  Dev dp(packed.data(), packed.size() * sizeof(uint32_t)), out(jt * sizeof(double));
  const size_t ws = st_fcs_cp_workspace(d.dims.size(), d.dims.data(), d.rank(), 1, lens.data());
  Dev dw(std::max<size_t>(ws, 1));
  check(st_fcs_cp(d.w.d(), d.rank(), d.dims.size(), d.dims.data(), d.ptrs.data(), 0, d.rank(), 1,
                  dp.u(), lens.data(), out.d(), 0, dw.p, ws, nullptr));
  return SketchVec(to_vec(download(out.p, jt)), family, SketchKind::FCS);
}

// ================================================================== fft.hpp

std::vector<std::complex<double>> dft(std::span<const double> x, std::size_t n) {
  if (n == 0) throw std::invalid_argument("dft: zero length");
  Dev dx(x.data(), x.size() * sizeof(double)), out(2 * n * sizeof(double));
  check(st_dft(dx.d(), x.size(), n, out.d(), nullptr));
  return to_complex(download(out.p, 2 * n));
}

std::vector<double> idft_real(const std::vector<std::complex<double>>& spectrum) {
  const size_t n = spectrum.size();
  if (n == 0) throw std::invalid_argument("idft_real: zero length");
  Dev ds(spectrum.data(), n * sizeof(std::complex<double>)), out(n * sizeof(double));
  check(st_idft_real(ds.d(), n, out.d(), 1, nullptr));
  return download(out.p, n);
}

std::vector<double> fft_convolve(const std::vector<std::span<const double>>& inputs,
                                 std::size_t n) {
  if (inputs.empty()) throw std::invalid_argument("fft_convolve: no inputs");
  if (n == 0) throw std::invalid_argument("dft: zero length");
  std::vector<Dev> d;
  std::vector<const double*> ptrs;
  std::vector<size_t> lens;
  for (const auto& x : inputs) {
    d.emplace_back(x.data(), x.size() * sizeof(double));
    lens.push_back(x.size());
  }
  for (const Dev& b : d) ptrs.push_back(b.d());
  Dev out(n * sizeof(double));
  check(st_fft_convolve(ptrs.data(), lens.data(), ptrs.size(), n, out.d(), nullptr));
  return download(out.p, n);
}

// =========================================================== estimators.hpp

std::vector<HashFamily> families_for(const std::vector<std::size_t>& dims,
                                     const EstimatorConfig& cfg) {
  if (cfg.hash_len == 0 || cfg.sketch_count == 0)
    throw std::invalid_argument("EstimatorConfig: hash_len and sketch_count must be >= 1");
  std::vector<HashFamily> families;
  families.reserve(cfg.sketch_count);
  for (size_t d = 0; d < cfg.sketch_count; ++d)
    families.emplace_back(dims, cfg.hash_len, family_seed(cfg.seed, d));
  return families;
}

double median_reduce(std::vector<double> values) {
  if (values.empty()) throw std::invalid_argument("median_reduce: empty input");
  std::sort(values.begin(), values.end());
  const size_t n = values.size();
  return n % 2 ? values[n / 2] : 0.5 * (values[n / 2 - 1] + values[n / 2]);
}

Eigen::VectorXd median_reduce(const std::vector<Eigen::VectorXd>& values) {
  if (values.empty()) throw std::invalid_argument("median_reduce: empty input");
  const Eigen::Index len = values[0].size();
  for (const Eigen::VectorXd& v : values)
    if (v.size() != len) throw std::invalid_argument("median_reduce: length mismatch");
  Eigen::VectorXd out(len);
  std::vector<double> column(values.size());
  for (Eigen::Index i = 0; i < len; ++i) {
    for (size_t d = 0; d < values.size(); ++d) column[d] = values[d][i];
    out[i] = median_reduce(column);
  }
  return out;
}

PrecomputedFcs::PrecomputedFcs(SketchVec s) : sketch(std::move(s)) {
  if (sketch.kind != SketchKind::FCS)
    throw std::invalid_argument("PrecomputedFcs: FCS sketch required");
  spectrum = dft(std::span<const double>(sketch.values.data(),
                                         static_cast<size_t>(sketch.values.size())),
                 sketch.family.composed_len());
}

PrecomputedFcs precompute_fcs(const DenseTensor& t, const HashFamily& family) {
  return PrecomputedFcs(fcs_sketch(t, family));
}

Eigen::VectorXd precompute_z(const PrecomputedFcs& pre, const Eigen::VectorXd& a,
                             const Eigen::VectorXd& b, std::size_t free_mode) {
  const HashFamily& family = pre.sketch.family;
  require_order3(family, "precompute_z");
  const size_t n = family.composed_len();
  const auto [c1, c2] = contracted_modes(free_mode, "precompute_z");
  const HashPair &pa = family.pair(c1), &pb = family.pair(c2);
  if (static_cast<size_t>(a.size()) != pa.input_dim() ||
      static_cast<size_t>(b.size()) != pb.input_dim())
    throw std::invalid_argument("cs_sketch: input length mismatch");
  std::vector<uint32_t> ta, tb;
  pack_pair(pa, ta);
  pack_pair(pb, tb);
  Dev ds(pre.spectrum.data(), pre.spectrum.size() * sizeof(std::complex<double>));
  Dev da(a.data(), a.size() * sizeof(double)), db(b.data(), b.size() * sizeof(double));
  Dev dta(ta.data(), ta.size() * sizeof(uint32_t)), dtb(tb.data(), tb.size() * sizeof(uint32_t));
  Dev z(n * sizeof(double));
  check(st_precompute_z(ds.d(), n, da.d(), pa.input_dim(), dta.u(), pa.hash_len(), db.d(),
                        pb.input_dim(), dtb.u(), pb.hash_len(), z.d(), nullptr));
  return to_vec(download(z.p, n));
}

namespace {

// uvw / iuv of one FCS or TS sketch at n points, any family: z through the
// exact-length transforms, the composed-length Parseval sum as a device dot
// of the sketch with the linear convolution of the three count sketches.
template <typename Pre>
double uvw_one(const Pre& pre, const Eigen::VectorXd& u, const Eigen::VectorXd& v,
               const Eigen::VectorXd& w, size_t n) {
  const HashFamily& family = pre.sketch.family;
  Dev cu = cs_device(u, family.pair(0)), cv = cs_device(v, family.pair(1)),
      cw = cs_device(w, family.pair(2));
  const double* ptrs[3] = {cu.d(), cv.d(), cw.d()};
  const size_t lens[3] = {family.pair(0).hash_len(), family.pair(1).hash_len(),
                          family.pair(2).hash_len()};
  Dev conv(n * sizeof(double));
  check(st_fft_convolve(ptrs, lens, 3, n, conv.d(), nullptr));
  Dev sk(pre.sketch.values.data(), n * sizeof(double)), out(sizeof(double));
  check(st_sketch_dots(1, n, sk.d(), conv.d(), out.d(), nullptr));
  return download(out.p, 1)[0];
}

template <typename Pre>
Eigen::VectorXd iuv_one(const Pre& pre, const Eigen::VectorXd& a, const Eigen::VectorXd& b,
                        size_t free_mode, size_t n) {
  const HashFamily& family = pre.sketch.family;
  const auto [c1, c2] = contracted_modes(free_mode, "estimate_iuv");
  const HashPair &pa = family.pair(c1), &pb = family.pair(c2);
  std::vector<uint32_t> ta, tb;
  pack_pair(pa, ta);
  pack_pair(pb, tb);
  Dev ds(pre.spectrum.data(), n * sizeof(std::complex<double>));
  Dev da(a.data(), a.size() * sizeof(double)), db(b.data(), b.size() * sizeof(double));
  Dev dta(ta.data(), ta.size() * sizeof(uint32_t)), dtb(tb.data(), tb.size() * sizeof(uint32_t));
  Dev z(n * sizeof(double));
  check(st_precompute_z(ds.d(), n, da.d(), pa.input_dim(), dta.u(), pa.hash_len(), db.d(),
                        pb.input_dim(), dtb.u(), pb.hash_len(), z.d(), nullptr));
  return readout(z.d(), n, family.pair(free_mode));
}

template <typename Pre>
void check_uvw_args(std::span<const Pre> pres, const Eigen::VectorXd& u, const Eigen::VectorXd& v,
                    const Eigen::VectorXd& w) {
  if (pres.empty()) throw std::invalid_argument("estimator: no sketches");
  for (const Pre& p : pres) {
    require_order3(p.sketch.family, "estimate_uvw");
    require_length(u, p.sketch.family.pair(0), "estimate_uvw");
    require_length(v, p.sketch.family.pair(1), "estimate_uvw");
    require_length(w, p.sketch.family.pair(2), "estimate_uvw");
  }
}

template <typename Pre>
void check_iuv_args(std::span<const Pre> pres, const Eigen::VectorXd& a, const Eigen::VectorXd& b,
                    size_t free_mode) {
  if (pres.empty()) throw std::invalid_argument("estimator: no sketches");
  for (const Pre& p : pres) {
    require_order3(p.sketch.family, "estimate_iuv");
    const auto [c1, c2] = contracted_modes(free_mode, "estimate_iuv");
    require_length(a, p.sketch.family.pair(c1), "estimate_iuv");
    require_length(b, p.sketch.family.pair(c2), "estimate_iuv");
  }
}

// Spectral estimators (FCS at n = J~, TS at n = J): the batched device
// engine when the families share dims and J, else per family.
template <typename Pre>
double spectral_uvw(std::span<const Pre> pres, const Eigen::VectorXd& u, const Eigen::VectorXd& v,
                    const Eigen::VectorXd& w, int backend) {
  check_uvw_args(pres, u, v, w);
  size_t J = 0;
  if (uniform_families(pres, &J))
    return engine_uvw(*sketch_engine(pres, backend, J), u, v, w);
  return median_over(pres, [&](const Pre& pre) {
    return uvw_one(pre, u, v, w, pre.spectrum.size());
  });
}

template <typename Pre>
Eigen::VectorXd spectral_iuv(std::span<const Pre> pres, const Eigen::VectorXd& a,
                             const Eigen::VectorXd& b, size_t free_mode, int backend) {
  check_iuv_args(pres, a, b, free_mode);
  size_t J = 0;
  if (uniform_families(pres, &J))
    return engine_iuv(*sketch_engine(pres, backend, J), a, b, free_mode,
                      pres[0].sketch.family.pair(free_mode).input_dim());
  return median_over(pres, [&](const Pre& pre) {
    return iuv_one(pre, a, b, free_mode, pre.spectrum.size());
  });
}

}  // namespace

double estimate_uvw(std::span<const PrecomputedFcs> pres, const Eigen::VectorXd& u,
                    const Eigen::VectorXd& v, const Eigen::VectorXd& w) {
  return spectral_uvw(pres, u, v, w, ST_BACKEND_FCS);
}

double estimate_uuu(std::span<const PrecomputedFcs> pres, const Eigen::VectorXd& u) {
  return estimate_uvw(pres, u, u, u);
}

Eigen::VectorXd estimate_iuv(std::span<const PrecomputedFcs> pres, const Eigen::VectorXd& a,
                             const Eigen::VectorXd& b, std::size_t free_mode) {
  return spectral_iuv(pres, a, b, free_mode, ST_BACKEND_FCS);
}

Eigen::VectorXd estimate_iuu(std::span<const PrecomputedFcs> pres, const Eigen::VectorXd& u) {
  return estimate_iuv(pres, u, u, 0);
}

double inner_once(const DenseTensor& a, const DenseTensor& b, const HashFamily& family) {
  if (a.shape() != b.shape()) throw std::invalid_argument("inner_once: shape mismatch");
  return dot_device(fcs_sketch(a, family).values, fcs_sketch(b, family).values);
}

double estimate_inner(const DenseTensor& a, const DenseTensor& b, const EstimatorConfig& cfg) {
  if (a.shape() != b.shape()) throw std::invalid_argument("estimate_inner: shape mismatch");
  std::vector<double> estimates;
  for (const HashFamily& family : families_for(a.shape(), cfg))
    estimates.push_back(inner_once(a, b, family));
  return median_reduce(std::move(estimates));
}

PrecomputedTs::PrecomputedTs(SketchVec s) : sketch(std::move(s)) {
  if (sketch.kind != SketchKind::TS) throw std::invalid_argument("PrecomputedTs: TS sketch required");
  spectrum = dft(std::span<const double>(sketch.values.data(),
                                         static_cast<size_t>(sketch.values.size())),
                 static_cast<size_t>(sketch.values.size()));
}

PrecomputedTs precompute_ts(const DenseTensor& t, const HashFamily& family) {
  return PrecomputedTs(ts_sketch(t, family));
}

double estimate_uvw(std::span<const PrecomputedTs> pres, const Eigen::VectorXd& u,
                    const Eigen::VectorXd& v, const Eigen::VectorXd& w) {
  return spectral_uvw(pres, u, v, w, ST_BACKEND_TS);
}

Eigen::VectorXd estimate_iuv(std::span<const PrecomputedTs> pres, const Eigen::VectorXd& a,
                             const Eigen::VectorXd& b, std::size_t free_mode) {
  return spectral_iuv(pres, a, b, free_mode, ST_BACKEND_TS);
}

double inner_once_ts(const DenseTensor& a, const DenseTensor& b, const HashFamily& family) {
  if (a.shape() != b.shape()) throw std::invalid_argument("inner_once_ts: shape mismatch");
  return dot_device(ts_sketch(a, family).values, ts_sketch(b, family).values);
}

PrecomputedHcs precompute_hcs(const DenseTensor& t, const HashFamily& family) {
  return PrecomputedHcs(hcs_sketch(t, family));
}

namespace {
// The exact-contraction engine over one HCS sketch (J_0 x J_1 x J_2).
std::shared_ptr<Engine> hcs_engine(const PrecomputedHcs& pre) {
  const DenseTensor& s = pre.sketch.values;
  uint64_t key = 0x48435345ull;
  key = mix(key, s.shape().data(), s.shape().size() * sizeof(size_t));
  key = mix(key, s.data().data(), s.size() * sizeof(double));
  return plain_engine(key, s.shape(), [&](double* dst) {
    cuda_check(cudaMemcpy(dst, s.data().data(), s.size() * sizeof(double), cudaMemcpyHostToDevice),
               "cudaMemcpy H2D");
  });
}
}  // namespace

double estimate_uvw(std::span<const PrecomputedHcs> pres, const Eigen::VectorXd& u,
                    const Eigen::VectorXd& v, const Eigen::VectorXd& w) {
  return median_over(pres, [&](const PrecomputedHcs& pre) {
    const HashFamily& family = pre.sketch.family;
    require_order3(family, "estimate_uvw");
    // contract3(S, cs_u, cs_v, cs_w) on the device
    Dev cu = cs_device(u, family.pair(0)), cv = cs_device(v, family.pair(1)),
        cw = cs_device(w, family.pair(2)), out(sizeof(double));
    check(st_engine_uvw(hcs_engine(pre)->e, 1, cu.d(), cv.d(), cw.d(), out.d(), 1, nullptr));
    return download(out.p, 1)[0];
  });
}

Eigen::VectorXd estimate_iuv(std::span<const PrecomputedHcs> pres, const Eigen::VectorXd& a,
                             const Eigen::VectorXd& b, std::size_t free_mode) {
  return median_over(pres, [&](const PrecomputedHcs& pre) {
    const HashFamily& family = pre.sketch.family;
    require_order3(family, "estimate_iuv");
    const auto [c1, c2] = contracted_modes(free_mode, "estimate_iuv");
    Dev ca = cs_device(a, family.pair(c1)), cb = cs_device(b, family.pair(c2));
    const size_t jf = family.pair(free_mode).hash_len();
    Dev w(jf * sizeof(double));
    // contract3_free(S, cs_a, cs_b, free_mode), then s_f(i) w[h_f(i)]
    check(st_engine_iuv(hcs_engine(pre)->e, 1, ca.d(), cb.d(), free_mode, w.d(), 1, nullptr));
    return readout(w.d(), jf, family.pair(free_mode));
  });
}

PrecomputedCs::PrecomputedCs(SketchVec s, std::vector<std::size_t> d)
    : sketch(std::move(s)), dims(std::move(d)) {
  size_t total = 1;
  for (size_t dim : dims) total *= dim;
  if (sketch.family.modes() != 1 || sketch.family.pair(0).input_dim() != total)
    throw std::invalid_argument("PrecomputedCs: long pair does not cover the shape");
}

PrecomputedCs precompute_cs(const DenseTensor& t, const HashPair& long_pair) {
  return PrecomputedCs(cs_sketch(Eigen::VectorXd(t.vec()), long_pair), t.shape());
}

namespace {
// The exact-contraction engine over the long pair's virtual tensor
// V[l] = s(l) sk[h(l)] (estimators.cpp:290-350), materialised on the device.
std::shared_ptr<Engine> cs_engine(const PrecomputedCs& pre, const char* op) {
  if (pre.dims.size() != 3) throw std::invalid_argument(std::string(op) + ": order-3 shape required");
  const HashPair& pair = pre.sketch.family.pair(0);
  const Eigen::VectorXd& sk = pre.sketch.values;
  std::vector<uint32_t> tab;
  pack_pair(pair, tab);
  uint64_t key = 0x4353ull;
  key = mix(key, pre.dims.data(), pre.dims.size() * sizeof(size_t));
  key = mix(key, tab.data(), tab.size() * sizeof(uint32_t));
  key = mix(key, sk.data(), sk.size() * sizeof(double));
  return plain_engine(key, pre.dims, [&](double* dst) {
    Dev dsk(sk.data(), sk.size() * sizeof(double)), dt(tab.data(), tab.size() * sizeof(uint32_t));
    check(st_cs_expand(dsk.d(), static_cast<size_t>(sk.size()), dt.u(), tab.size(), dst, nullptr));
    cuda_check(cudaDeviceSynchronize(), "st_cs_expand");
  });
}
}  // namespace

double estimate_uvw(std::span<const PrecomputedCs> pres, const Eigen::VectorXd& u,
                    const Eigen::VectorXd& v, const Eigen::VectorXd& w) {
  return median_over(pres, [&](const PrecomputedCs& pre) {
    auto e = cs_engine(pre, "estimate_uvw");
    if (static_cast<size_t>(u.size()) != pre.dims[0] || static_cast<size_t>(v.size()) != pre.dims[1] ||
        static_cast<size_t>(w.size()) != pre.dims[2])
      throw std::invalid_argument("estimate_uvw: vector length mismatch");
    return engine_uvw(*e, u, v, w, 0);
  });
}

Eigen::VectorXd estimate_iuv(std::span<const PrecomputedCs> pres, const Eigen::VectorXd& a,
                             const Eigen::VectorXd& b, std::size_t free_mode) {
  return median_over(pres, [&](const PrecomputedCs& pre) {
    auto e = cs_engine(pre, "estimate_iuv");
    const auto [c1, c2] = contracted_modes(free_mode, "estimate_iuv");
    if (static_cast<size_t>(a.size()) != pre.dims[c1] || static_cast<size_t>(b.size()) != pre.dims[c2])
      throw std::invalid_argument("estimate_iuv: vector length mismatch");
    return engine_iuv(*e, a, b, free_mode, pre.dims[free_mode]);
  });
}

}  // namespace sketchtensor
