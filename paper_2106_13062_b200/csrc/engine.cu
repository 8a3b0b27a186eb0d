// Host side of the spectral paths: CP-form FCS, convolution / Kronecker,
// the FCS contraction engine (FcsEngine, cpd.cpp:61-94) and the batched
// robust tensor power method driver (rtpm, cpd.cpp:234-277).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <numbers>
#include <string>
#include <vector>

#include "fft.cuh"

namespace fcs {

int launch_spec_from_real(const FftPlan&, const double*, size_t, int, int, double2*, cudaStream_t);
int launch_real_from_spec(const FftPlan&, const double2*, int, double*, size_t, int, int,
                          cudaStream_t);
int launch_cp(const FftPlan&, const CpArgs&, int, const uint32_t*, double2*, double*, int, int,
              cudaStream_t);
int launch_conv(const FftPlan&, const double*, int, size_t, const double*, int, size_t, int,
                double2*, double*, size_t, cudaStream_t);
int launch_iuv(const FftPlan&, const EngArgs&, int, const double*, const double*, int, int, int,
               double2*, double*, cudaStream_t);
int launch_uvw(const FftPlan&, const EngArgs&, int, const double*, const double*, const double*,
               double2*, double*, cudaStream_t);
int launch_deflate(const FftPlan&, const EngArgs&, double, const double*, const double*,
                   const double*, double2*, double2*, cudaStream_t);
int launch_median(const double*, int, int, int, double*, cudaStream_t);
int launch_cs_columns(const double*, int, int, const uint32_t*, int, double*, cudaStream_t);
int launch_normalize_rows(double*, int, int, cudaStream_t);
int launch_refine_update(double*, const double*, int, int*, cudaStream_t);
int launch_family_tables(size_t, const size_t*, const size_t*, size_t, const uint64_t*,
                         uint32_t*, cudaStream_t);
size_t dense_workspace(int, size_t, const size_t*, size_t, size_t, const size_t*, int kind = 0);
int launch_fcs_dense(int, const void*, size_t, const size_t*, size_t, size_t, size_t,
                     const uint32_t*, const size_t*, double*, int, void*, size_t, cudaStream_t,
                     size_t fam_stride = 0, int kind = 0);

namespace {

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Stream-ordered scratch that only grows.
struct Scratch {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t need, cudaStream_t st) {
    if (need <= bytes) return ST_OK;
    if (p) FCS_CUDA_TRY(cudaFreeAsync(p, st));
    p = nullptr;
    bytes = 0;
    FCS_CUDA_TRY(cudaMallocAsync(&p, need, st));
    bytes = need;
    return ST_OK;
  }
  void release(cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    bytes = 0;
  }
};

// contracted_modes (estimators.cpp:23-29)
void contracted(size_t f, int* c1, int* c2) {
  *c1 = f == 0 ? 1 : 0;
  *c2 = f == 2 ? 1 : 2;
}

// Host SplitMix64 with the Box-Muller spare (rng.hpp:12-48, rng.cpp:8-21).
struct HostRng {
  uint64_t state;
  double spare = 0.0;
  bool has_spare = false;
  explicit HostRng(uint64_t s) : state(s) {}
  uint64_t next() {
    state += kGamma;
    return fmix64(state);
  }
  double gaussian() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    const double u1 = static_cast<double>((next() >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(next() >> 11) * 0x1.0p-53;
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * std::numbers::pi * u2;
    spare = radius * std::sin(angle);
    has_spare = true;
    return radius * std::cos(angle);
  }
};

}  // namespace
}  // namespace fcs

using namespace fcs;

struct st_engine {
  int device = 0;
  size_t dims[3] = {0, 0, 0};
  size_t hash_len = 0;
  size_t D = 0;
  size_t jt = 0;
  FftPlan plan{};
  uint32_t* packed = nullptr;  // D x sum(dims)
  double2* spec = nullptr;     // D x P
  Scratch scratch, est, vec;
  EngArgs args() const {
    EngArgs e{};
    size_t off = 0;
    for (int n = 0; n < 3; ++n) {
      e.dims[n] = static_cast<int>(dims[n]);
      e.tab_off[n] = static_cast<int>(off);
      off += dims[n];
    }
    e.fam_stride = static_cast<int>(off);
    e.D = static_cast<int>(D);
    e.packed = packed;
    e.spec = spec;
    return e;
  }
};

extern "C" {

int st_cs_columns(const double* u, size_t input_dim, size_t cols, const uint32_t* packed_pair,
                  size_t hash_len, double* out, void* stream) {
  FCS_CHECK_ARG(input_dim > 0 && hash_len > 0, "HashPair: dimensions must be positive");
  return launch_cs_columns(u, static_cast<int>(input_dim), static_cast<int>(cols), packed_pair,
                           static_cast<int>(hash_len), out, as_stream(stream));
}

size_t st_fcs_cp_workspace(size_t order, const size_t* dims, size_t rank, size_t sketch_count,
                           const size_t* hash_lens) {
  (void)dims;
  size_t sum_j = 0;
  for (size_t n = 0; n < order; ++n) sum_j += hash_lens[n];
  FftPlan pl;
  if (get_fft_plan(sum_j - order + 1, &pl) != ST_OK) return 0;
  return (std::max<size_t>(1, rank) + 1) * sketch_count * pl.P * sizeof(double2);
}

int st_fcs_cp(const double* weights, size_t rank, size_t order, const size_t* dims,
              const double* const* factors, size_t r_begin, size_t r_count, size_t sketch_count,
              const uint32_t* packed, const size_t* hash_lens, double* out, int accumulate,
              void* workspace, size_t workspace_bytes, void* stream) {
  FCS_CHECK_ARG(order >= 1 && order <= ST_MAX_ORDER, "CpTensor: no factors");
  FCS_CHECK_ARG(sketch_count >= 1, "EstimatorConfig: hash_len and sketch_count must be >= 1");
  FCS_CHECK_ARG(r_begin + r_count <= rank, "st_fcs_cp: rank range out of bounds");
  CpArgs a{};
  a.order = static_cast<int>(order);
  size_t off = 0, sum_j = 0;
  for (size_t n = 0; n < order; ++n) {
    FCS_CHECK_ARG(dims[n] > 0 && hash_lens[n] > 0, "HashPair: dimensions must be positive");
    a.dims[n] = static_cast<int>(dims[n]);
    a.tab_off[n] = static_cast<int>(off);
    a.factors[n] = factors[n];
    off += dims[n];
    sum_j += hash_lens[n];
  }
  a.fam_stride = static_cast<int>(off);
  a.weights = weights;
  a.r_begin = static_cast<int>(r_begin);
  a.r_count = static_cast<int>(r_count);
  const size_t jt = sum_j - order + 1;
  FftPlan pl;
  if (int rc = get_fft_plan(jt, &pl)) return rc;
  const size_t need = (std::max<size_t>(1, r_count) + 1) * sketch_count * pl.P * sizeof(double2);
  FCS_CHECK_ARG(workspace && workspace_bytes >= need, "st_fcs_cp: workspace too small");
  return launch_cp(pl, a, static_cast<int>(sketch_count), packed,
                   static_cast<double2*>(workspace), out, static_cast<int>(jt), accumulate,
                   as_stream(stream));
}

int st_convolve_pairs(const double* a, size_t la, const double* b, size_t lb, size_t batch,
                      double* out, void* stream) {
  FCS_CHECK_ARG(la > 0 && lb > 0, "fft_convolve: no inputs");
  if (batch == 0) return ST_OK;
  FftPlan pl;
  if (int rc = get_fft_plan(la + lb - 1, &pl)) return rc;
  cudaStream_t st = as_stream(stream);
  double2* scr = nullptr;
  FCS_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&scr), batch * pl.P * sizeof(double2), st));
  const int rc = launch_conv(pl, a, static_cast<int>(la), la, b, static_cast<int>(lb), lb,
                             static_cast<int>(batch), scr, out, la + lb - 1, st);
  cudaFreeAsync(scr, st);
  return rc;
}

int st_fcs_kron(const double* a, size_t ra, size_t ca, const double* b, size_t rb, size_t cb,
                size_t sketch_count, const uint32_t* packed, const size_t* hash_lens, double* out,
                void* stream) {
  FCS_CHECK_ARG(ra && ca && rb && cb, "DenseTensor: zero dimension");
  FCS_CHECK_ARG(sketch_count >= 1, "EstimatorConfig: hash_len and sketch_count must be >= 1");
  cudaStream_t st = as_stream(stream);
  const size_t stride = ra + ca + rb + cb;
  const size_t da[2] = {ra, ca}, db[2] = {rb, cb};
  const size_t la = hash_lens[0] + hash_lens[1] - 1, lb = hash_lens[2] + hash_lens[3] - 1;
  const size_t D = sketch_count;
  const size_t wsa = dense_workspace(ST_F64, 2, da, ca, D, hash_lens);
  const size_t wsb = dense_workspace(ST_F64, 2, db, cb, D, hash_lens + 2);
  void* ws = nullptr;
  double *fa = nullptr, *fb = nullptr;
  FCS_CUDA_TRY(cudaMallocAsync(&ws, std::max<size_t>(1, std::max(wsa, wsb)), st));
  FCS_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&fa), D * la * sizeof(double), st));
  FCS_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&fb), D * lb * sizeof(double), st));
  int rc = launch_fcs_dense(ST_F64, a, 2, da, 0, ca, D, packed, hash_lens, fa, 0, ws, wsa, st,
                            stride);
  if (!rc)
    rc = launch_fcs_dense(ST_F64, b, 2, db, 0, cb, D, packed + ra + ca, hash_lens + 2, fb, 0, ws,
                          wsb, st, stride);
  if (!rc) rc = st_convolve_pairs(fa, la, fb, lb, D, out, st);
  cudaFreeAsync(ws, st);
  cudaFreeAsync(fa, st);
  cudaFreeAsync(fb, st);
  return rc;
}

int st_engine_create(st_engine** engine, int dtype, const void* tensor, const size_t* dims,
                     size_t hash_len, size_t sketch_count, uint64_t seed, void* stream) {
  FCS_CHECK_ARG(engine != nullptr, "st_engine_create: null engine pointer");
  FCS_CHECK_ARG(dtype == ST_F32 || dtype == ST_F64, "st_engine_create: unknown dtype");
  FCS_CHECK_ARG(hash_len > 0 && sketch_count > 0,
                "EstimatorConfig: hash_len and sketch_count must be >= 1");
  for (int n = 0; n < 3; ++n) FCS_CHECK_ARG(dims[n] > 0, "DenseTensor: zero dimension");
  cudaStream_t st = as_stream(stream);
  auto* e = new st_engine();
  FCS_CUDA_TRY(cudaGetDevice(&e->device));
  for (int n = 0; n < 3; ++n) e->dims[n] = dims[n];
  e->hash_len = hash_len;
  e->D = sketch_count;
  e->jt = 3 * hash_len - 2;
  int rc = get_fft_plan(e->jt, &e->plan);
  if (rc) {
    delete e;
    return rc;
  }
  const size_t hl[3] = {hash_len, hash_len, hash_len};
  const size_t sum_dims = dims[0] + dims[1] + dims[2];
  std::vector<uint64_t> seeds(sketch_count);
  for (size_t d = 0; d < sketch_count; ++d)  // families_for (estimators.cpp:104-115)
    seeds[d] = splitmix_draw(seed + static_cast<uint64_t>(d), 1);
  double* vals = nullptr;
  void* ws = nullptr;
  const size_t wsb = dense_workspace(dtype, 3, dims, dims[2], sketch_count, hl);
  if (cudaMallocAsync(reinterpret_cast<void**>(&e->packed),
                      sketch_count * sum_dims * sizeof(uint32_t), st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&e->spec),
                      sketch_count * e->plan.P * sizeof(double2), st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&vals), sketch_count * e->jt * sizeof(double), st) !=
          cudaSuccess ||
      cudaMallocAsync(&ws, std::max<size_t>(1, wsb), st) != cudaSuccess) {
    st_engine_destroy(e);
    return fail(ST_ENOMEM, "st_engine_create: device allocation failed");
  }
  rc = launch_family_tables(3, dims, hl, sketch_count, seeds.data(), e->packed, st);
  if (!rc)
    rc = launch_fcs_dense(dtype, tensor, 3, dims, 0, dims[2], sketch_count, e->packed, hl, vals,
                          0, ws, wsb, st, 0);
  if (!rc)
    rc = launch_spec_from_real(e->plan, vals, e->jt, static_cast<int>(e->jt),
                               static_cast<int>(sketch_count), e->spec, st);
  cudaFreeAsync(vals, st);
  cudaFreeAsync(ws, st);
  if (rc) {
    st_engine_destroy(e);
    return rc;
  }
  *engine = e;
  return ST_OK;
}

int st_engine_destroy(st_engine* e) {
  if (!e) return ST_OK;
  cudaDeviceSynchronize();
  if (e->packed) cudaFree(e->packed);
  if (e->spec) cudaFree(e->spec);
  e->scratch.release(nullptr);
  e->est.release(nullptr);
  e->vec.release(nullptr);
  cudaDeviceSynchronize();
  delete e;
  return ST_OK;
}

size_t st_engine_composed_len(const st_engine* e) { return e ? e->jt : 0; }

int st_engine_sketches(st_engine* e, double* out, void* stream) {
  FCS_CHECK_ARG(e != nullptr, "st_engine_sketches: null engine");
  return launch_real_from_spec(e->plan, e->spec, static_cast<int>(e->D), out, e->jt,
                               static_cast<int>(e->jt), 0, as_stream(stream));
}

int st_engine_iuv(st_engine* e, size_t batch, const double* a, const double* b, size_t free_mode,
                  double* out, int median, void* stream) {
  FCS_CHECK_ARG(e != nullptr, "st_engine_iuv: null engine");
  FCS_CHECK_ARG(free_mode <= 2, "estimate_iuv: mode out of range");
  if (batch == 0) return ST_OK;
  cudaStream_t st = as_stream(stream);
  int c1, c2;
  contracted(free_mode, &c1, &c2);
  const size_t nf = e->dims[free_mode];
  if (int rc = e->scratch.ensure(batch * e->D * e->plan.P * sizeof(double2), st)) return rc;
  double* est = out;
  if (median) {
    if (int rc = e->est.ensure(batch * e->D * nf * sizeof(double), st)) return rc;
    est = static_cast<double*>(e->est.p);
  }
  const EngArgs args = e->args();
  if (int rc = launch_iuv(e->plan, args, static_cast<int>(batch), a, b, c1, c2,
                          static_cast<int>(free_mode), static_cast<double2*>(e->scratch.p), est, st))
    return rc;
  if (median)
    return launch_median(est, static_cast<int>(batch), static_cast<int>(e->D),
                         static_cast<int>(nf), out, st);
  return ST_OK;
}

int st_engine_uvw(st_engine* e, size_t batch, const double* u, const double* v, const double* w,
                  double* out, int median, void* stream) {
  FCS_CHECK_ARG(e != nullptr, "st_engine_uvw: null engine");
  if (batch == 0) return ST_OK;
  cudaStream_t st = as_stream(stream);
  if (int rc = e->scratch.ensure(batch * e->D * e->plan.P * sizeof(double2), st)) return rc;
  double* est = out;
  if (median) {
    if (int rc = e->est.ensure(batch * e->D * sizeof(double), st)) return rc;
    est = static_cast<double*>(e->est.p);
  }
  if (int rc = launch_uvw(e->plan, e->args(), static_cast<int>(batch), u, v, w,
                          static_cast<double2*>(e->scratch.p), est, st))
    return rc;
  if (median) return launch_median(est, static_cast<int>(batch), static_cast<int>(e->D), 1, out, st);
  return ST_OK;
}

int st_engine_deflate(st_engine* e, double weight, const double* u, const double* v,
                      const double* w, void* stream) {
  FCS_CHECK_ARG(e != nullptr, "st_engine_deflate: null engine");
  cudaStream_t st = as_stream(stream);
  if (int rc = e->scratch.ensure(e->D * e->plan.P * sizeof(double2), st)) return rc;
  return launch_deflate(e->plan, e->args(), weight, u, v, w, static_cast<double2*>(e->scratch.p),
                        e->spec, st);
}

int st_rtpm(int dtype, const void* tensor, size_t dim, size_t rank, size_t num_inits,
            size_t num_iters, size_t hash_len, size_t sketch_count, uint64_t seed,
            double* weights, double* factor, void* stream) {
  FCS_CHECK_ARG(dim > 0, "DenseTensor: zero dimension");
  FCS_CHECK_ARG(rank > 0 && num_inits > 0 && num_iters > 0,
                "rtpm: rank, inits, and iterations must be >= 1");
  cudaStream_t st = as_stream(stream);
  const size_t dims[3] = {dim, dim, dim};
  st_engine* e = nullptr;
  if (int rc = st_engine_create(&e, dtype, tensor, dims, hash_len, sketch_count, seed, st))
    return rc;
  struct Guard {
    st_engine* e;
    ~Guard() { st_engine_destroy(e); }
  } guard{e};
  const size_t L = num_inits;
  // device: U (L x dim), Y (L x dim), best, next, values, stopped flag
  if (int rc = e->vec.ensure((2 * L + 2) * dim * sizeof(double) + (L + 1) * sizeof(double) + 16, st))
    return rc;
  double* U = static_cast<double*>(e->vec.p);
  double* Y = U + L * dim;
  double* best = Y + L * dim;
  double* next = best + dim;
  double* vals = next + dim;
  int* stopped = reinterpret_cast<int*>(vals + L + 1);
  std::vector<double> hU(L * dim), hvals(L);
  // init_rng = SplitMix64(mix(seed ^ 0x7274706d)) (cpd.cpp:245)
  HostRng rng(splitmix_draw(seed ^ 0x7274706dULL, 1));
  for (size_t r = 0; r < rank; ++r) {
    for (size_t l = 0; l < L; ++l) {  // random_unit (cpd.cpp:199-204), same draw order
      double* u = hU.data() + l * dim;
      double sq = 0.0;
      for (size_t i = 0; i < dim; ++i) {
        u[i] = rng.gaussian();
      }
      for (size_t i = 0; i < dim; ++i) sq += u[i] * u[i];
      const double norm = std::sqrt(sq);
      if (norm > 0)
        for (size_t i = 0; i < dim; ++i) u[i] /= norm;
    }
    FCS_CUDA_TRY(cudaMemcpyAsync(U, hU.data(), L * dim * sizeof(double), cudaMemcpyHostToDevice, st));
    // L restarts advance in lockstep; a row whose norm underflows stays zero,
    // exactly like the reference's early break (iuu(0) = 0).
    for (size_t it = 0; it < num_iters; ++it) {
      if (int rc = st_engine_iuv(e, L, U, U, 0, Y, 1, st)) return rc;
      if (int rc = launch_normalize_rows(Y, static_cast<int>(L), static_cast<int>(dim), st)) return rc;
      std::swap(U, Y);
    }
    if (int rc = st_engine_uvw(e, L, U, U, U, vals, 1, st)) return rc;
    FCS_CUDA_TRY(cudaMemcpyAsync(hvals.data(), vals, L * sizeof(double), cudaMemcpyDeviceToHost, st));
    FCS_CUDA_TRY(cudaStreamSynchronize(st));
    double best_value = -std::numeric_limits<double>::infinity();
    long arg = -1;
    for (size_t l = 0; l < L; ++l) {
      if (hvals[l] > best_value) {  // strict >, first wins (cpd.cpp:260)
        best_value = hvals[l];
        arg = static_cast<long>(l);
      }
    }
    if (arg < 0) return fail(ST_ENUMERIC, "rtpm: no candidate with a finite contraction value");
    FCS_CUDA_TRY(cudaMemcpyAsync(best, U + arg * dim, dim * sizeof(double), cudaMemcpyDeviceToDevice, st));
    FCS_CUDA_TRY(cudaMemsetAsync(stopped, 0, sizeof(int), st));
    for (size_t it = 0; it < num_iters; ++it) {  // refinement (cpd.cpp:266-270)
      if (int rc = st_engine_iuv(e, 1, best, best, 0, next, 1, st)) return rc;
      if (int rc = launch_refine_update(best, next, static_cast<int>(dim), stopped, st)) return rc;
    }
    if (int rc = st_engine_uvw(e, 1, best, best, best, vals, 1, st)) return rc;
    double weight = 0.0;
    FCS_CUDA_TRY(cudaMemcpyAsync(&weight, vals, sizeof(double), cudaMemcpyDeviceToHost, st));
    FCS_CUDA_TRY(cudaMemcpyAsync(factor + r * dim, best, dim * sizeof(double), cudaMemcpyDeviceToHost, st));
    FCS_CUDA_TRY(cudaStreamSynchronize(st));
    weights[r] = weight;
    if (int rc = st_engine_deflate(e, weight, best, best, best, st)) return rc;
  }
  FCS_CUDA_TRY(cudaStreamSynchronize(st));
  return ST_OK;
}

}  // extern "C"
