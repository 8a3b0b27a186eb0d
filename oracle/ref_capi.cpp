// ORACLE TEST INFRASTRUCTURE — not product code.
//
// extern "C" wrappers around the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile
// against the from-scratch shims in oracle/shim/). Loaded with ctypes by
// oracle/ref.py; used only by tests/, __graft_entry__.smoke() (never: smoke
// uses the numpy restatement) and bench.py's cpu_baseline / --impl reference
// legs. Every entry returns 0 on success, 1 on std::invalid_argument, 2 on
// std::runtime_error, 3 on anything else; ref_last_error() has the message.
#include <sketchtensor/cpd.hpp>
#include <sketchtensor/estimators.hpp>
#include <sketchtensor/fft.hpp>
#include <sketchtensor/hashing.hpp>
#include <sketchtensor/rng.hpp>
#include <sketchtensor/sketch.hpp>
#include <sketchtensor/tensor.hpp>

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

using namespace sketchtensor;

namespace {
thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

std::vector<std::size_t> to_dims(std::size_t order, const std::size_t* dims) {
  return std::vector<std::size_t>(dims, dims + order);
}

DenseTensor make_tensor(const double* data, std::size_t order, const std::size_t* dims) {
  std::vector<std::size_t> shape = to_dims(order, dims);
  std::size_t total = 1;
  for (std::size_t d : shape) total *= d;
  return DenseTensor(shape, std::vector<double>(data, data + total));
}

// Concatenated per-mode tables -> HashFamily of explicit pairs.
HashFamily make_family(std::size_t order, const std::size_t* dims, const std::uint32_t* buckets,
                       const std::int8_t* signs, const std::size_t* hash_lens) {
  std::vector<HashPair> pairs;
  std::size_t off = 0;
  for (std::size_t n = 0; n < order; ++n) {
    pairs.emplace_back(std::vector<std::uint32_t>(buckets + off, buckets + off + dims[n]),
                       std::vector<std::int8_t>(signs + off, signs + off + dims[n]),
                       hash_lens[n]);
    off += dims[n];
  }
  return HashFamily(std::move(pairs));
}

CpTensor make_cp(const double* weights, std::size_t rank, std::size_t order,
                 const std::size_t* dims, const double* factors) {
  Eigen::VectorXd w(static_cast<Eigen::Index>(rank));
  for (std::size_t r = 0; r < rank; ++r) w[static_cast<Eigen::Index>(r)] = weights[r];
  std::vector<Eigen::MatrixXd> fs;
  std::size_t off = 0;
  for (std::size_t n = 0; n < order; ++n) {
    Eigen::MatrixXd m(static_cast<Eigen::Index>(dims[n]), static_cast<Eigen::Index>(rank));
    std::memcpy(m.data(), factors + off, sizeof(double) * dims[n] * rank);
    off += dims[n] * rank;
    fs.push_back(std::move(m));
  }
  return CpTensor(std::move(w), std::move(fs));
}

void copy_out(const Eigen::VectorXd& v, double* out) {
  std::memcpy(out, v.data(), sizeof(double) * static_cast<std::size_t>(v.size()));
}

Eigen::VectorXd vec_in(const double* p, std::size_t n) {
  return Eigen::VectorXd(Eigen::Map<const Eigen::VectorXd>(p, static_cast<Eigen::Index>(n)));
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// First `count` raw draws of SplitMix64(seed) (rng.hpp:16-21).
void ref_splitmix_draws(std::uint64_t seed, std::size_t count, std::uint64_t* out) {
  SplitMix64 rng(seed);
  for (std::size_t i = 0; i < count; ++i) out[i] = rng.next();
}

std::uint64_t ref_family_seed(std::uint64_t base, std::size_t d) { return family_seed(base, d); }

// n successive SplitMix64(seed).next_gaussian() values (rng.cpp:8-21).
void ref_gaussian(std::uint64_t seed, std::size_t n, double* out) {
  SplitMix64 rng(seed);
  for (std::size_t i = 0; i < n; ++i) out[i] = rng.next_gaussian();
}

// HashPair(I, J, seed) tables (hashing.cpp:10-22).
int ref_hash_pair(std::uint64_t seed, std::size_t input_dim, std::size_t hash_len,
                  std::uint32_t* bucket, std::int8_t* sign) {
  return guarded([&] {
    HashPair p(input_dim, hash_len, seed);
    std::memcpy(bucket, p.bucket_map().data(), sizeof(std::uint32_t) * input_dim);
    std::memcpy(sign, p.sign_map().data(), input_dim);
  });
}

// HashFamily(dims, J, master) tables, concatenated mode-major; returns composed_len.
int ref_hash_family(std::size_t order, const std::size_t* dims, std::size_t hash_len,
                    std::uint64_t master, std::uint32_t* buckets, std::int8_t* signs,
                    std::size_t* composed_len) {
  return guarded([&] {
    HashFamily f(to_dims(order, dims), hash_len, master);
    std::size_t off = 0;
    for (std::size_t n = 0; n < order; ++n) {
      std::memcpy(buckets + off, f.pair(n).bucket_map().data(), sizeof(std::uint32_t) * dims[n]);
      std::memcpy(signs + off, f.pair(n).sign_map().data(), dims[n]);
      off += dims[n];
    }
    *composed_len = f.composed_len();
  });
}

// HashFamily::compose (hashing.cpp:83-98) on an explicit family.
int ref_compose(std::size_t order, const std::size_t* dims, const std::uint32_t* buckets,
                const std::int8_t* signs, const std::size_t* hash_lens,
                const std::size_t* multi_index, std::size_t* bucket, int* sign) {
  return guarded([&] {
    HashFamily f = make_family(order, dims, buckets, signs, hash_lens);
    auto [b, s] = f.compose(std::vector<std::size_t>(multi_index, multi_index + order));
    *bucket = b;
    *sign = s;
  });
}

// materialize_composed_pair (hashing.cpp:100-121).
int ref_materialize(std::size_t order, const std::size_t* dims, const std::uint32_t* buckets,
                    const std::int8_t* signs, const std::size_t* hash_lens,
                    std::uint32_t* out_bucket, std::int8_t* out_sign) {
  return guarded([&] {
    HashPair p = make_family(order, dims, buckets, signs, hash_lens).materialize_composed_pair();
    std::memcpy(out_bucket, p.bucket_map().data(), sizeof(std::uint32_t) * p.input_dim());
    std::memcpy(out_sign, p.sign_map().data(), p.input_dim());
  });
}

// fcs_sketch(DenseTensor, HashFamily) (sketch.cpp:187-201), seeded family.
int ref_fcs_dense(const double* data, std::size_t order, const std::size_t* dims,
                  std::size_t hash_len, std::uint64_t master, double* out) {
  return guarded([&] {
    DenseTensor t = make_tensor(data, order, dims);
    copy_out(fcs_sketch(t, HashFamily(to_dims(order, dims), hash_len, master)).values, out);
  });
}

// fcs_sketch(DenseTensor, HashFamily) with explicit tables (and explicit tensor dims,
// which may differ from the table dims to exercise the shape checks).
int ref_fcs_dense_tables(const double* data, std::size_t order, const std::size_t* dims,
                         std::size_t fam_order, const std::size_t* fam_dims,
                         const std::uint32_t* buckets, const std::int8_t* signs,
                         const std::size_t* hash_lens, double* out) {
  return guarded([&] {
    DenseTensor t = make_tensor(data, order, dims);
    copy_out(fcs_sketch(t, make_family(fam_order, fam_dims, buckets, signs, hash_lens)).values,
             out);
  });
}

// cs_sketch (sketch.cpp:105-116) with an explicit pair.
int ref_cs_sketch(const double* x, std::size_t len, const std::uint32_t* bucket,
                  const std::int8_t* sign, std::size_t input_dim, std::size_t hash_len,
                  double* out) {
  return guarded([&] {
    HashPair p(std::vector<std::uint32_t>(bucket, bucket + input_dim),
               std::vector<std::int8_t>(sign, sign + input_dim), hash_len);
    copy_out(cs_sketch(vec_in(x, len), p).values, out);
  });
}

// cs_sketch_columns (sketch.cpp:118-133); u is rows x cols column-major.
int ref_cs_sketch_columns(const double* u, std::size_t rows, std::size_t cols,
                          const std::uint32_t* bucket, const std::int8_t* sign,
                          std::size_t input_dim, std::size_t hash_len, double* out) {
  return guarded([&] {
    HashPair p(std::vector<std::uint32_t>(bucket, bucket + input_dim),
               std::vector<std::int8_t>(sign, sign + input_dim), hash_len);
    Eigen::MatrixXd m(static_cast<Eigen::Index>(rows), static_cast<Eigen::Index>(cols));
    std::memcpy(m.data(), u, sizeof(double) * rows * cols);
    Eigen::MatrixXd r = cs_sketch_columns(m, p);
    std::memcpy(out, r.data(), sizeof(double) * static_cast<std::size_t>(r.size()));
  });
}

// fcs_sketch(CpTensor, HashFamily) (sketch.cpp:203-207), seeded family.
int ref_fcs_cp(const double* weights, std::size_t rank, std::size_t order,
               const std::size_t* dims, const double* factors, std::size_t hash_len,
               std::uint64_t master, double* out) {
  return guarded([&] {
    CpTensor cp = make_cp(weights, rank, order, dims, factors);
    copy_out(fcs_sketch(cp, HashFamily(to_dims(order, dims), hash_len, master)).values, out);
  });
}

// fcs_sketch(CpTensor, HashFamily) with explicit tables.
int ref_fcs_cp_tables(const double* weights, std::size_t rank, std::size_t order,
                      const std::size_t* dims, const double* factors,
                      const std::uint32_t* buckets, const std::int8_t* signs,
                      const std::size_t* hash_lens, double* out) {
  return guarded([&] {
    CpTensor cp = make_cp(weights, rank, order, dims, factors);
    copy_out(fcs_sketch(cp, make_family(order, dims, buckets, signs, hash_lens)).values, out);
  });
}

// densify (tensor.cpp:86-115).
int ref_densify(const double* weights, std::size_t rank, std::size_t order,
                const std::size_t* dims, const double* factors, double* out) {
  return guarded([&] {
    DenseTensor t = densify(make_cp(weights, rank, order, dims, factors));
    std::memcpy(out, t.data().data(), sizeof(double) * t.size());
  });
}

// kron (tensor.cpp:228-236); a is ra x ca, b is rb x cb, both column-major.
int ref_kron(const double* a, std::size_t ra, std::size_t ca, const double* b, std::size_t rb,
             std::size_t cb, double* out) {
  return guarded([&] {
    Eigen::MatrixXd ma(static_cast<Eigen::Index>(ra), static_cast<Eigen::Index>(ca));
    Eigen::MatrixXd mb(static_cast<Eigen::Index>(rb), static_cast<Eigen::Index>(cb));
    std::memcpy(ma.data(), a, sizeof(double) * ra * ca);
    std::memcpy(mb.data(), b, sizeof(double) * rb * cb);
    Eigen::MatrixXd k = kron(ma, mb);
    std::memcpy(out, k.data(), sizeof(double) * static_cast<std::size_t>(k.size()));
  });
}

// dft (fft.cpp:42-51); out is n interleaved complex values.
int ref_dft(const double* x, std::size_t len, std::size_t n, double* out) {
  return guarded([&] {
    auto s = dft(std::span<const double>(x, len), n);
    std::memcpy(out, s.data(), sizeof(double) * 2 * s.size());
  });
}

// idft_real (fft.cpp:53-73); spec is n interleaved complex values.
int ref_idft_real(const double* spec, std::size_t n, double* out) {
  return guarded([&] {
    std::vector<std::complex<double>> s(n);
    std::memcpy(static_cast<void*>(s.data()), spec, sizeof(double) * 2 * n);
    auto r = idft_real(s);
    std::memcpy(out, r.data(), sizeof(double) * n);
  });
}

// fft_convolve (fft.cpp:75-84) of k real inputs.
int ref_fft_convolve(const double* const* inputs, const std::size_t* lens, std::size_t k,
                     std::size_t n, double* out) {
  return guarded([&] {
    std::vector<std::span<const double>> in;
    for (std::size_t i = 0; i < k; ++i) in.emplace_back(inputs[i], lens[i]);
    auto r = fft_convolve(in, n);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}

// median_reduce scalar (estimators.cpp:117-123).
int ref_median(const double* v, std::size_t n, double* out) {
  return guarded([&] { *out = median_reduce(std::vector<double>(v, v + n)); });
}

// median_reduce vector (estimators.cpp:125-138): count vectors of length len, row-major.
int ref_median_vec(const double* v, std::size_t count, std::size_t len, double* out) {
  return guarded([&] {
    std::vector<Eigen::VectorXd> vs;
    for (std::size_t d = 0; d < count; ++d) vs.push_back(vec_in(v + d * len, len));
    copy_out(median_reduce(vs), out);
  });
}

// Contraction engine (cpd.cpp:220-232) — backend 0 plain, 4 fcs (SketchBackend order).
void* ref_engine_create(const double* data, const std::size_t* dims, std::size_t hash_len,
                        std::size_t sketch_count, std::uint64_t seed, int backend) {
  ContractionEngine* eng = nullptr;
  int rc = guarded([&] {
    DenseTensor t = make_tensor(data, 3, dims);
    EstimatorConfig cfg;
    cfg.hash_len = hash_len;
    cfg.sketch_count = sketch_count;
    cfg.seed = seed;
    eng = make_contraction_engine(t, static_cast<SketchBackend>(backend), cfg).release();
  });
  return rc == 0 ? eng : nullptr;
}

void ref_engine_destroy(void* h) { delete static_cast<ContractionEngine*>(h); }

int ref_engine_iuv(void* h, const double* a, std::size_t la, const double* b, std::size_t lb,
                   std::size_t free_mode, double* out) {
  return guarded([&] {
    copy_out(static_cast<ContractionEngine*>(h)->iuv(vec_in(a, la), vec_in(b, lb), free_mode),
             out);
  });
}

int ref_engine_uvw(void* h, const double* u, std::size_t lu, const double* v, std::size_t lv,
                   const double* w, std::size_t lw, double* out) {
  return guarded([&] {
    *out = static_cast<ContractionEngine*>(h)->uvw(vec_in(u, lu), vec_in(v, lv), vec_in(w, lw));
  });
}

int ref_engine_deflate(void* h, double weight, const double* u, std::size_t lu,
                       const double* v, std::size_t lv, const double* w, std::size_t lw) {
  return guarded([&] {
    static_cast<ContractionEngine*>(h)->deflate(weight, vec_in(u, lu), vec_in(v, lv),
                                                vec_in(w, lw));
  });
}

// rtpm (cpd.cpp:234-277): weights[rank], factor dim x rank column-major.
int ref_rtpm(const double* data, std::size_t dim, std::size_t rank, std::size_t num_inits,
             std::size_t num_iters, int backend, std::size_t hash_len, std::size_t sketch_count,
             std::uint64_t seed, double* weights, double* factor) {
  return guarded([&] {
    const std::size_t dims[3] = {dim, dim, dim};
    DenseTensor t = make_tensor(data, 3, dims);
    RtpmConfig cfg;
    cfg.target_rank = rank;
    cfg.num_inits = num_inits;
    cfg.num_power_iters = num_iters;
    cfg.backend = static_cast<SketchBackend>(backend);
    cfg.estimator.hash_len = hash_len;
    cfg.estimator.sketch_count = sketch_count;
    cfg.estimator.seed = seed;
    CpTensor cp = rtpm(t, cfg);
    copy_out(cp.weights, weights);
    std::memcpy(factor, cp.factors[0].data(), sizeof(double) * dim * rank);
  });
}

// residual_norm (cpd.cpp:385-392) of a symmetric CP (shared factor) against t.
int ref_residual_norm_sym(const double* data, std::size_t dim, const double* weights,
                          std::size_t rank, const double* factor, double* out) {
  return guarded([&] {
    const std::size_t dims[3] = {dim, dim, dim};
    DenseTensor t = make_tensor(data, 3, dims);
    std::vector<double> fs;
    for (int n = 0; n < 3; ++n) fs.insert(fs.end(), factor, factor + dim * rank);
    *out = residual_norm(t, make_cp(weights, rank, 3, dims, fs.data()));
  });
}

}  // extern "C"

// ---------------------------------------------------------------- TS / HCS
extern "C" {

// ts_sketch(DenseTensor, explicit HashFamily) (sketch.cpp:135-149).
int ref_ts_dense_tables(const double* data, std::size_t order, const std::size_t* dims,
                        const std::uint32_t* buckets, const std::int8_t* signs,
                        const std::size_t* hash_lens, double* out) {
  return guarded([&] {
    DenseTensor t = make_tensor(data, order, dims);
    copy_out(ts_sketch(t, make_family(order, dims, buckets, signs, hash_lens)).values, out);
  });
}

// ts_sketch(CpTensor, explicit HashFamily) (sketch.cpp:151-155).
int ref_ts_cp_tables(const double* weights, std::size_t rank, std::size_t order,
                     const std::size_t* dims, const double* factors, const std::uint32_t* buckets,
                     const std::int8_t* signs, const std::size_t* hash_lens, double* out) {
  return guarded([&] {
    CpTensor cp = make_cp(weights, rank, order, dims, factors);
    copy_out(ts_sketch(cp, make_family(order, dims, buckets, signs, hash_lens)).values, out);
  });
}

// hcs_sketch(DenseTensor, explicit HashFamily) (sketch.cpp:157-173); out is prod J (col-major).
int ref_hcs_dense_tables(const double* data, std::size_t order, const std::size_t* dims,
                         const std::uint32_t* buckets, const std::int8_t* signs,
                         const std::size_t* hash_lens, double* out) {
  return guarded([&] {
    DenseTensor t = make_tensor(data, order, dims);
    SketchTensor s = hcs_sketch(t, make_family(order, dims, buckets, signs, hash_lens));
    std::memcpy(out, s.values.data().data(), sizeof(double) * s.values.size());
  });
}

// hcs_sketch(CpTensor, explicit HashFamily) (sketch.cpp:175-185).
int ref_hcs_cp_tables(const double* weights, std::size_t rank, std::size_t order,
                      const std::size_t* dims, const double* factors,
                      const std::uint32_t* buckets, const std::int8_t* signs,
                      const std::size_t* hash_lens, double* out) {
  return guarded([&] {
    CpTensor cp = make_cp(weights, rank, order, dims, factors);
    SketchTensor s = hcs_sketch(cp, make_family(order, dims, buckets, signs, hash_lens));
    std::memcpy(out, s.values.data().data(), sizeof(double) * s.values.size());
  });
}

}  // extern "C"

// ---------------------------------------------------------- CPD drivers
extern "C" {

namespace {
void copy_factors(const CpTensor& cp, double* out) {
  std::size_t off = 0;
  for (const Eigen::MatrixXd& f : cp.factors) {
    std::memcpy(out + off, f.data(), sizeof(double) * f.size());
    off += static_cast<std::size_t>(f.size());
  }
}
}  // namespace

// rtpm_asym (cpd.cpp:279-335); factors packed dims[0] x rank, dims[1] x rank, dims[2] x rank.
int ref_rtpm_asym(const double* data, const std::size_t* dims, std::size_t rank,
                  std::size_t num_inits, std::size_t num_iters, int backend, std::size_t hash_len,
                  std::size_t sketch_count, std::uint64_t seed, double* weights, double* factors) {
  return guarded([&] {
    DenseTensor t = make_tensor(data, 3, dims);
    RtpmConfig cfg;
    cfg.target_rank = rank;
    cfg.num_inits = num_inits;
    cfg.num_power_iters = num_iters;
    cfg.backend = static_cast<SketchBackend>(backend);
    cfg.estimator.hash_len = hash_len;
    cfg.estimator.sketch_count = sketch_count;
    cfg.estimator.seed = seed;
    CpTensor cp = rtpm_asym(t, cfg);
    copy_out(cp.weights, weights);
    copy_factors(cp, factors);
  });
}

// als (cpd.cpp:337-383); same packing.
int ref_als(const double* data, const std::size_t* dims, std::size_t rank, std::size_t max_iters,
            double tol, int backend, std::size_t hash_len, std::size_t sketch_count,
            std::uint64_t seed, double* weights, double* factors) {
  return guarded([&] {
    DenseTensor t = make_tensor(data, 3, dims);
    AlsConfig cfg;
    cfg.target_rank = rank;
    cfg.max_iters = max_iters;
    cfg.tol = tol;
    cfg.backend = static_cast<SketchBackend>(backend);
    cfg.estimator.hash_len = hash_len;
    cfg.estimator.sketch_count = sketch_count;
    cfg.estimator.seed = seed;
    CpTensor cp = als(t, cfg);
    copy_out(cp.weights, weights);
    copy_factors(cp, factors);
  });
}

// residual_norm (cpd.cpp:385-392) of an order-3 CP (packed factors) against t.
int ref_residual_norm(const double* data, const std::size_t* dims, const double* weights,
                      std::size_t rank, const double* factors, double* out) {
  return guarded([&] {
    DenseTensor t = make_tensor(data, 3, dims);
    *out = residual_norm(t, make_cp(weights, rank, 3, dims, factors));
  });
}

}  // extern "C"

// ------------------------------------------------------ inner products
extern "C" {

// estimate_inner (estimators.cpp:198-207).
int ref_estimate_inner(const double* a, const double* b, std::size_t order,
                       const std::size_t* dims, std::size_t hash_len, std::size_t sketch_count,
                       std::uint64_t seed, double* out) {
  return guarded([&] {
    EstimatorConfig cfg;
    cfg.hash_len = hash_len;
    cfg.sketch_count = sketch_count;
    cfg.seed = seed;
    *out = estimate_inner(make_tensor(a, order, dims), make_tensor(b, order, dims), cfg);
  });
}

// inner_once / inner_once_ts (estimators.cpp:193-196, 235-239) with an explicit family.
int ref_inner_once_tables(int ts, const double* a, const double* b, std::size_t order,
                          const std::size_t* dims, const std::uint32_t* buckets,
                          const std::int8_t* signs, const std::size_t* hash_lens, double* out) {
  return guarded([&] {
    HashFamily fam = make_family(order, dims, buckets, signs, hash_lens);
    DenseTensor ta = make_tensor(a, order, dims), tb = make_tensor(b, order, dims);
    *out = ts ? inner_once_ts(ta, tb, fam) : inner_once(ta, tb, fam);
  });
}

}  // extern "C"

extern "C" {
// psnr (cpd.cpp:394-403).
int ref_psnr(const double* a, const double* b, std::size_t order, const std::size_t* dims,
             double* out) {
  return guarded([&] { *out = psnr(make_tensor(a, order, dims), make_tensor(b, order, dims)); });
}
}  // extern "C"

extern "C" {
// mode_unfold (tensor.cpp:117-136): out is dims[mode] x (size / dims[mode]) column-major.
int ref_mode_unfold(const double* data, std::size_t order, const std::size_t* dims,
                    std::size_t mode, double* out) {
  return guarded([&] {
    Eigen::MatrixXd m = mode_unfold(make_tensor(data, order, dims), mode);
    std::memcpy(out, m.data(), sizeof(double) * m.size());
  });
}

// contract_pair (tensor.cpp:238-261): result data (column-major) of size
// prod(a rest) * prod(b rest).
int ref_contract_pair(const double* a, std::size_t oa, const std::size_t* da, const double* b,
                      std::size_t ob, const std::size_t* db, std::size_t ma, std::size_t mb,
                      double* out) {
  return guarded([&] {
    DenseTensor r = contract_pair(make_tensor(a, oa, da), make_tensor(b, ob, db), ma, mb);
    std::memcpy(out, r.data().data(), sizeof(double) * r.size());
  });
}
}  // extern "C"

extern "C" {
// Resident reference tensors for timing (bench.py cpu_baseline / --impl
// reference): the DenseTensor is built once, outside the timed region, so a
// timed call is exactly fcs_sketch(const DenseTensor&, const HashFamily&)
// (sketch.cpp:187-201) plus the HashFamily construction from explicit tables.

// DenseTensor(dims) filled with `count` SplitMix64(seed).next_gaussian()
// draws (rng.cpp:8-21), optionally rounded to float32 and widened back (the
// config-4 input is fp32; the reference API is fp64-only, tensor.hpp:50-51).
void* ref_dense_gaussian(std::uint64_t seed, std::size_t order, const std::size_t* dims,
                         int round_f32) {
  try {
    std::vector<std::size_t> shape = to_dims(order, dims);
    std::size_t total = 1;
    for (std::size_t d : shape) total *= d;
    std::vector<double> v(total);
    SplitMix64 rng(seed);
    for (std::size_t i = 0; i < total; ++i) {
      const double g = rng.next_gaussian();
      v[i] = round_f32 ? static_cast<double>(static_cast<float>(g)) : g;
    }
    return new DenseTensor(std::move(shape), std::move(v));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void* ref_dense_create(const double* data, std::size_t order, const std::size_t* dims) {
  try {
    return new DenseTensor(make_tensor(data, order, dims));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_dense_destroy(void* t) { delete static_cast<DenseTensor*>(t); }

// fcs_sketch(t, HashFamily(explicit pairs)) on a resident tensor.
int ref_fcs_dense_handle(const void* t, std::size_t fam_order, const std::size_t* fam_dims,
                         const std::uint32_t* buckets, const std::int8_t* signs,
                         const std::size_t* hash_lens, double* out) {
  return guarded([&] {
    copy_out(fcs_sketch(*static_cast<const DenseTensor*>(t),
                        make_family(fam_order, fam_dims, buckets, signs, hash_lens))
                 .values,
             out);
  });
}
}  // extern "C"

extern "C" {
// precompute_fcs + precompute_z (estimators.cpp:147-167) on a cubical tensor
// with the family HashFamily({I, I, I}, J, master): the exact n-point
// spectrum (2n doubles) and z (n doubles).
int ref_precompute_z(const double* data, std::size_t dim, std::size_t hash_len,
                     std::uint64_t master, const double* a, const double* b,
                     std::size_t free_mode, double* spectrum, double* z) {
  return guarded([&] {
    const std::size_t dims[3] = {dim, dim, dim};
    DenseTensor t = make_tensor(data, 3, dims);
    const PrecomputedFcs pre = precompute_fcs(t, HashFamily(to_dims(3, dims), hash_len, master));
    for (std::size_t k = 0; k < pre.spectrum.size(); ++k) {
      spectrum[2 * k] = pre.spectrum[k].real();
      spectrum[2 * k + 1] = pre.spectrum[k].imag();
    }
    copy_out(precompute_z(pre, vec_in(a, dim), vec_in(b, dim), free_mode), z);
  });
}
}  // extern "C"

extern "C" {
// estimate_uvw / estimate_iuv over PrecomputedFcs built with families of
// UNEQUAL hash lengths (HashFamily(dims, lens, family_seed(seed, d))): the
// span estimators of estimators.cpp:169-186 outside families_for.
int ref_estimate_mixed(const double* data, const std::size_t* dims, const std::size_t* lens,
                       std::size_t count, std::uint64_t seed, const double* u, const double* v,
                       const double* w, std::size_t free_mode, double* uvw_out, double* iuv_out) {
  return guarded([&] {
    DenseTensor t = make_tensor(data, 3, dims);
    std::vector<PrecomputedFcs> pres;
    for (std::size_t d = 0; d < count; ++d)
      pres.push_back(precompute_fcs(t, HashFamily(to_dims(3, dims), to_dims(3, lens),
                                                  family_seed(seed, d))));
    const Eigen::VectorXd vu = vec_in(u, dims[0]), vv = vec_in(v, dims[1]), vw = vec_in(w, dims[2]);
    *uvw_out = estimate_uvw(std::span<const PrecomputedFcs>(pres), vu, vv, vw);
    const Eigen::VectorXd* in[3] = {&vu, &vv, &vw};
    const std::size_t c1 = free_mode == 0 ? 1 : 0, c2 = free_mode == 2 ? 1 : 2;
    copy_out(estimate_iuv(std::span<const PrecomputedFcs>(pres), *in[c1], *in[c2], free_mode),
             iuv_out);
  });
}
}  // extern "C"
