// Facade driver: the reference's own cpd.cpp / tensor.cpp / hashing.cpp /
// rng.cpp (compiled unmodified from /root/reference/proj/src) linked against
// libsketchtensor_b200.so, which defines sketch.hpp / estimators.hpp /
// fft.hpp over the GPU C-ABI in place of sketch.cpp / estimators.cpp /
// fft.cpp. Each subcommand reads raw fp64 inputs, calls the reference API,
// and writes raw fp64 outputs; tests/test_facade.py compares them with the
// unmodified reference (oracle/_ref) on the same inputs.
//
//   test_facade fcs_dense <t.bin> <J> <D> <seed> <out.bin> <I_0> ... <I_N-1>
//   test_facade fcs_cp <w.bin> <f.bin> <R> <J> <D> <seed> <out.bin> <I_0> ... <I_N-1>
//   test_facade kron <A.bin> <B.bin> <ra> <ca> <rb> <cb> <J> <D> <seed> <out.bin>
//   test_facade rtpm <t.bin> <dim> <rank> <inits> <iters> <backend> <J> <D> <seed> <out.bin>
//   test_facade engine <t.bin> <I0> <I1> <I2> <backend> <J> <D> <seed> <u.bin> <nvec> <out.bin>
//   test_facade fft <x.bin> <len> <n> <out.bin>
//   test_facade z <t.bin> <I> <J> <seed> <a.bin> <b.bin> <free> <out.bin>
//   test_facade sketches <t.bin> <I0> <I1> <I2> <J> <seed> <out.bin>   (cs/ts/hcs, TS/HCS CP)
//   test_facade mixed <t.bin> <I0> <I1> <I2> <J0> <J1> <J2> <D> <seed> <v.bin> <free> <out.bin>
//   test_facade errors
#include <sketchtensor/cpd.hpp>
#include <sketchtensor/estimators.hpp>
#include <sketchtensor/fft.hpp>
#include <sketchtensor/sketch.hpp>
#include <sketchtensor/tensor.hpp>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <stdexcept>
#include <string>
#include <vector>

using namespace sketchtensor;

namespace {

std::vector<double> read_bin(const std::string& path, size_t n) {
  std::vector<double> v(n);
  std::ifstream f(path, std::ios::binary);
  f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(double)));
  if (!f) throw std::runtime_error("cannot read " + path);
  return v;
}

struct Out {
  std::vector<double> v;
  void add(const double* p, size_t n) { v.insert(v.end(), p, p + n); }
  void add(const Eigen::VectorXd& x) { add(x.data(), static_cast<size_t>(x.size())); }
  void add(double x) { v.push_back(x); }
  void write(const std::string& path) const {
    std::ofstream f(path, std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(double)));
  }
};

size_t prod(const std::vector<size_t>& d) {
  size_t p = 1;
  for (size_t x : d) p *= x;
  return p;
}

Eigen::VectorXd vec_at(const std::vector<double>& all, size_t k, size_t n) {
  Eigen::VectorXd v(static_cast<Eigen::Index>(n));
  for (size_t i = 0; i < n; ++i) v[static_cast<Eigen::Index>(i)] = all[k * n + i];
  return v;
}

CpTensor read_cp(const std::string& wp, const std::string& fp, const std::vector<size_t>& dims,
                 size_t R) {
  std::vector<double> w = read_bin(wp, R);
  size_t tot = 0;
  for (size_t d : dims) tot += d * R;
  std::vector<double> f = read_bin(fp, tot);
  Eigen::VectorXd wv(static_cast<Eigen::Index>(R));
  for (size_t r = 0; r < R; ++r) wv[static_cast<Eigen::Index>(r)] = w[r];
  std::vector<Eigen::MatrixXd> fs;
  size_t off = 0;
  for (size_t d : dims) {
    Eigen::MatrixXd m(static_cast<Eigen::Index>(d), static_cast<Eigen::Index>(R));
    for (size_t i = 0; i < d * R; ++i) m.data()[i] = f[off + i];
    off += d * R;
    fs.push_back(std::move(m));
  }
  return CpTensor(std::move(wv), std::move(fs));
}

int run(int argc, char** argv) {
  const std::string cmd = argv[1];
  auto S = [&](int i) { return std::string(argv[i]); };
  auto U = [&](int i) { return static_cast<size_t>(std::strtoull(argv[i], nullptr, 10)); };
  if (cmd == "fcs_dense") {
    std::vector<size_t> dims;
    for (int i = 7; i < argc; ++i) dims.push_back(U(i));
    DenseTensor t(dims, read_bin(S(2), prod(dims)));
    EstimatorConfig cfg{U(3), U(4), U(5)};
    Out o;
    for (const HashFamily& f : families_for(dims, cfg)) o.add(fcs_sketch(t, f).values);
    o.write(S(6));
  } else if (cmd == "fcs_cp") {
    std::vector<size_t> dims;
    for (int i = 9; i < argc; ++i) dims.push_back(U(i));
    const CpTensor cp = read_cp(S(2), S(3), dims, U(4));
    EstimatorConfig cfg{U(5), U(6), U(7)};
    Out o;
    for (const HashFamily& f : families_for(dims, cfg)) o.add(fcs_sketch(cp, f).values);
    o.write(S(8));
  } else if (cmd == "kron") {
    const size_t ra = U(4), ca = U(5), rb = U(6), cb = U(7);
    Eigen::MatrixXd A(static_cast<Eigen::Index>(ra), static_cast<Eigen::Index>(ca));
    Eigen::MatrixXd B(static_cast<Eigen::Index>(rb), static_cast<Eigen::Index>(cb));
    std::vector<double> a = read_bin(S(2), ra * ca), b = read_bin(S(3), rb * cb);
    for (size_t i = 0; i < ra * ca; ++i) A.data()[i] = a[i];
    for (size_t i = 0; i < rb * cb; ++i) B.data()[i] = b[i];
    EstimatorConfig cfg{U(8), U(9), U(10)};
    Out o;
    for (const HashFamily& f : families_for({ra, ca, rb, cb}, cfg)) {
      // FCS(A (x) B) = FCS_{p0,p1}(A) * FCS_{p2,p3}(B)
      const SketchVec sa = fcs_sketch(tensor_from_matrix(A), HashFamily({f.pair(0), f.pair(1)}));
      const SketchVec sb = fcs_sketch(tensor_from_matrix(B), HashFamily({f.pair(2), f.pair(3)}));
      const std::vector<double> c = fft_convolve(
          {std::span<const double>(sa.values.data(), static_cast<size_t>(sa.values.size())),
           std::span<const double>(sb.values.data(), static_cast<size_t>(sb.values.size()))},
          f.composed_len());
      o.add(c.data(), c.size());
    }
    o.write(S(11));
  } else if (cmd == "rtpm") {
    const size_t dim = U(3);
    DenseTensor t({dim, dim, dim}, read_bin(S(2), dim * dim * dim));
    RtpmConfig cfg;
    cfg.target_rank = U(4);
    cfg.num_inits = U(5);
    cfg.num_power_iters = U(6);
    cfg.backend = static_cast<SketchBackend>(U(7));
    cfg.estimator = EstimatorConfig{U(8), U(9), U(10)};
    const CpTensor cp = rtpm(t, cfg);
    Out o;
    o.add(cp.weights);
    o.add(cp.factors[0].data(), static_cast<size_t>(cp.factors[0].size()));
    o.write(S(11));
  } else if (cmd == "engine") {
    const std::vector<size_t> dims = {U(3), U(4), U(5)};
    DenseTensor t(dims, read_bin(S(2), prod(dims)));
    EstimatorConfig cfg{U(7), U(8), U(9)};
    auto e = make_contraction_engine(t, static_cast<SketchBackend>(U(6)), cfg);
    const size_t nvec = U(11);
    // nvec triples (u0: I0, u1: I1, u2: I2)
    const size_t per = dims[0] + dims[1] + dims[2];
    std::vector<double> all = read_bin(S(10), nvec * per);
    Out o;
    auto call_all = [&]() {
      for (size_t k = 0; k < nvec; ++k) {
        Eigen::VectorXd v0(static_cast<Eigen::Index>(dims[0])), v1(static_cast<Eigen::Index>(dims[1])),
            v2(static_cast<Eigen::Index>(dims[2]));
        for (size_t i = 0; i < dims[0]; ++i) v0[static_cast<Eigen::Index>(i)] = all[k * per + i];
        for (size_t i = 0; i < dims[1]; ++i) v1[static_cast<Eigen::Index>(i)] = all[k * per + dims[0] + i];
        for (size_t i = 0; i < dims[2]; ++i)
          v2[static_cast<Eigen::Index>(i)] = all[k * per + dims[0] + dims[1] + i];
        o.add(e->uvw(v0, v1, v2));
        o.add(e->iuv(v1, v2, 0));
        o.add(e->iuv(v0, v2, 1));
        o.add(e->iuv(v0, v1, 2));
      }
    };
    call_all();
    {
      Eigen::VectorXd v0(static_cast<Eigen::Index>(dims[0])), v1(static_cast<Eigen::Index>(dims[1])),
          v2(static_cast<Eigen::Index>(dims[2]));
      for (size_t i = 0; i < dims[0]; ++i) v0[static_cast<Eigen::Index>(i)] = all[i];
      for (size_t i = 0; i < dims[1]; ++i) v1[static_cast<Eigen::Index>(i)] = all[dims[0] + i];
      for (size_t i = 0; i < dims[2]; ++i) v2[static_cast<Eigen::Index>(i)] = all[dims[0] + dims[1] + i];
      e->deflate(0.75, v0, v1, v2);
    }
    call_all();
    o.write(S(12));
  } else if (cmd == "fft") {
    const size_t len = U(3), n = U(4);
    std::vector<double> x = read_bin(S(2), len);
    const auto spec = dft(std::span<const double>(x.data(), len), n);
    Out o;
    for (const auto& c : spec) {
      o.add(c.real());
      o.add(c.imag());
    }
    const std::vector<double> back = idft_real(spec);
    o.add(back.data(), back.size());
    const std::vector<double> conv =
        fft_convolve({std::span<const double>(x.data(), len), std::span<const double>(x.data(), len / 2)}, n);
    o.add(conv.data(), conv.size());
    o.write(S(5));
  } else if (cmd == "z") {
    const size_t I = U(3), J = U(4);
    DenseTensor t({I, I, I}, read_bin(S(2), I * I * I));
    const HashFamily fam({I, I, I}, J, family_seed(U(5), 0));
    const PrecomputedFcs pre = precompute_fcs(t, fam);
    std::vector<double> a = read_bin(S(6), I), b = read_bin(S(7), I);
    Out o;
    for (const auto& c : pre.spectrum) {
      o.add(c.real());
      o.add(c.imag());
    }
    o.add(precompute_z(pre, vec_at(a, 0, I), vec_at(b, 0, I), U(8)));
    o.write(S(9));
  } else if (cmd == "sketches") {
    const std::vector<size_t> dims = {U(3), U(4), U(5)};
    const std::vector<double> tv = read_bin(S(2), prod(dims));
    DenseTensor t(dims, tv);
    const HashFamily fam(dims, U(6), family_seed(U(7), 0));
    Out o;
    o.add(ts_sketch(t, fam).values);
    const SketchTensor h = hcs_sketch(t, fam);
    o.add(h.values.data().data(), h.values.size());
    Eigen::VectorXd x(static_cast<Eigen::Index>(dims[0]));
    for (size_t i = 0; i < dims[0]; ++i) x[static_cast<Eigen::Index>(i)] = tv[i];
    o.add(cs_sketch(x, fam.pair(0)).values);
    // a rank-3 CP tensor from the first entries: TS / HCS / FCS of the CP form
    std::vector<Eigen::MatrixXd> fs;
    size_t off = 0;
    for (size_t d : dims) {
      Eigen::MatrixXd m(static_cast<Eigen::Index>(d), 3);
      for (size_t i = 0; i < d * 3; ++i) m.data()[i] = tv[off + i];
      off += d * 3;
      fs.push_back(std::move(m));
    }
    Eigen::VectorXd w(3);
    w[0] = 1.0;
    w[1] = -0.5;
    w[2] = 2.0;
    const CpTensor cp(w, fs);
    o.add(ts_sketch(cp, fam).values);
    const SketchTensor hc = hcs_sketch(cp, fam);
    o.add(hc.values.data().data(), hc.values.size());
    o.add(fcs_sketch(cp, fam).values);
    const Eigen::MatrixXd cols = cs_sketch_columns(fs[0], fam.pair(0));
    o.add(cols.data(), static_cast<size_t>(cols.size()));
    o.write(S(8));
  } else if (cmd == "mixed") {
    // estimators over PrecomputedFcs of families with unequal hash lengths
    // (the facade's per-family exact path)
    const std::vector<size_t> dims = {U(3), U(4), U(5)}, lens = {U(6), U(7), U(8)};
    DenseTensor t(dims, read_bin(S(2), prod(dims)));
    const size_t D = U(9), free_mode = U(12);
    std::vector<PrecomputedFcs> pres;
    for (size_t d = 0; d < D; ++d)
      pres.push_back(precompute_fcs(t, HashFamily(dims, lens, family_seed(U(10), d))));
    const size_t per = dims[0] + dims[1] + dims[2];
    std::vector<double> all = read_bin(S(11), per);
    Eigen::VectorXd v[3];
    size_t off = 0;
    for (int n = 0; n < 3; ++n) {
      v[n] = Eigen::VectorXd(static_cast<Eigen::Index>(dims[n]));
      for (size_t i = 0; i < dims[n]; ++i) v[n][static_cast<Eigen::Index>(i)] = all[off + i];
      off += dims[n];
    }
    Out o;
    o.add(estimate_uvw(std::span<const PrecomputedFcs>(pres), v[0], v[1], v[2]));
    const size_t c1 = free_mode == 0 ? 1 : 0, c2 = free_mode == 2 ? 1 : 2;
    o.add(estimate_iuv(std::span<const PrecomputedFcs>(pres), v[c1], v[c2], free_mode));
    o.write(S(13));
  } else if (cmd == "errors") {
    auto expect = [](const char* what, const std::function<void()>& fn, bool runtime) {
      try {
        fn();
        std::printf("MISSING %s\n", what);
      } catch (const std::invalid_argument& e) {
        std::printf("%s %s: %s\n", runtime ? "WRONG" : "ok", what, e.what());
      } catch (const std::runtime_error& e) {
        std::printf("%s %s: %s\n", runtime ? "ok" : "WRONG", what, e.what());
      }
    };
    expect("dft zero", [] { dft(std::span<const double>(), 0); }, false);
    expect("idft_real zero", [] { idft_real({}); }, false);
    expect("idft_real not real", [] {
      std::vector<std::complex<double>> s(8);
      s[1] = {1.0, 0.0};  // asymmetric spectrum: complex inverse
      idft_real(s);
    }, true);
    expect("fft_convolve empty", [] { fft_convolve({}, 4); }, false);
    expect("fcs shape", [] {
      DenseTensor t({3, 4});
      fcs_sketch(t, HashFamily({3, 5}, 4, 1));
    }, false);
    expect("fcs order", [] {
      DenseTensor t({3, 4});
      fcs_sketch(t, HashFamily({3, 4, 2}, 4, 1));
    }, false);
    expect("ts unequal", [] {
      DenseTensor t({3, 4});
      ts_sketch(t, HashFamily({3, 4}, std::vector<size_t>{4, 5}, 1));
    }, false);
    expect("cs length", [] { cs_sketch(Eigen::VectorXd(3), HashPair(4, 5, 1)); }, false);
    expect("families zero", [] { families_for({3}, EstimatorConfig{0, 1, 0}); }, false);
    expect("median empty", [] { median_reduce(std::vector<double>{}); }, false);
    expect("precomputed kind", [] {
      PrecomputedFcs p(SketchVec(Eigen::VectorXd::Zero(4), HashFamily({HashPair(3, 4, 1)}), SketchKind::CS));
    }, false);
    expect("estimator empty", [] { estimate_uuu(std::span<const PrecomputedFcs>(), Eigen::VectorXd(3)); },
           false);
    std::printf("median %g %g\n", median_reduce(std::vector<double>{1, 2, 100}),
                median_reduce(std::vector<double>{1, 2, 3, 10}));
  } else {
    std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
    return 2;
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: test_facade <command> ...\n");
    return 2;
  }
  try {
    return run(argc, argv);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
