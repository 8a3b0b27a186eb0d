// Host side of the spectral paths: CP-form FCS, convolution / Kronecker and
// the contraction engine (FcsEngine cpd.cpp:61-94, TsEngine cpd.cpp:96-126).
// The CPD drivers built on the engine live in cpd.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <string>
#include <vector>

#include "engine.cuh"

namespace fcs {

__global__ void ts_extend_kernel(const double* __restrict__ in, int D, int jt, int J,
                                 double* __restrict__ ext, double scale, int accumulate) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<size_t>(D) * jt) return;
  const int d = static_cast<int>(i / jt);
  const int k = static_cast<int>(i - static_cast<size_t>(d) * jt);
  const double* row = in + static_cast<size_t>(d) * jt;
  double acc = 0.0;
  for (int m = k % J; m < jt; m += J) acc += row[m];  // TS bucket (sum h) mod J, sketch.cpp:141
  ext[i] = accumulate ? ext[i] + scale * acc : scale * acc;
}

int launch_ts_extend(const double* in, int D, int jt, int J, double* ext, double scale,
                     int accumulate, cudaStream_t st) {
  const size_t n = static_cast<size_t>(D) * jt;
  if (n == 0) return ST_OK;
  ts_extend_kernel<<<ceil_div(n, 256), 256, 0, st>>>(in, D, jt, J, ext, scale, accumulate);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace fcs

using namespace fcs;

namespace fcs {
static int iuv_fused_ab(st_engine* e, size_t batch, const double* a, const double* b, size_t free_mode,
                 int mode, double* out, double* best, int* stopped, cudaStream_t st,
                 const double* wvec = nullptr) {
  if (is_exact(e) || batch == 0) return 1;
  const bool direct = use_direct(e, batch, free_mode);
  if (e->plan.large_p1 && !direct) return 1;
  int c1, c2;
  contracted(free_mode, &c1, &c2);
  const size_t nf = e->dims[free_mode];
  const size_t had = e->cnt.bytes;
  if (int rc = e->cnt.ensure(std::max<size_t>(batch, 64) * sizeof(int), st)) return rc;
  if (e->cnt.bytes != had) FCS_CUDA_TRY(cudaMemsetAsync(e->cnt.p, 0, e->cnt.bytes, st));
  if (int rc = e->est.ensure(batch * e->D * nf * sizeof(double), st)) return rc;
  IuvTail t;
  t.mode = mode;
  t.cnt = static_cast<int*>(e->cnt.p);
  t.out = out;
  t.best = best;
  t.stopped = stopped;
  t.wvec = wvec;
  if (direct) {  // the time-domain estimator with the same fused tail
    if (e->D > 16) return 1;  // the tail's register median: callers run the separate kernels
    if (int rc = corr_sync(e, st)) return rc;
    return corr_estimate(e, batch, a, b, free_mode, mode == 4 ? wvec : nullptr,
                         static_cast<double*>(e->est.p), st, &t);
  }
  // beyond one wave of clusters the caller's separate kernels run (a tail
  // fused into the split one-CTA + cluster step measured slower: the join
  // directly followed by the next call's fork serialises the two parts,
  // tools/experiments/iuv_fused_median.patch)
  return launch_iuv_cluster(e->plan, e->args(), static_cast<int>(batch), a, b, c1, c2,
                            static_cast<int>(free_mode), static_cast<double*>(e->est.p), t, st);
}

// ST_ENGINE_PATH=spectral|direct sets the initial path of new engines (A/B
// runs of drivers that build their engine internally, e.g. st_rtpm).
int default_path() {
  const char* v = std::getenv("ST_ENGINE_PATH");
  if (!v) return ST_PATH_AUTO;
  const std::string s(v);
  return s == "spectral" ? ST_PATH_SPECTRAL : s == "direct" ? ST_PATH_DIRECT : ST_PATH_AUTO;
}

// Cost rule of the direct path, fitted to the measured A/B of both paths on
// one B200 (profiles/corr_sweep_r02.txt: I^3 tensors, I = 50-400, J =
// 300-4000, D = 10, batches 1 and 15; model times in us). Fq = (2J - 1) I_c2
// multiply-adds of the Hankel product (tensor cores for batches of 2+,
// shared-memory bound for one vector), Fz = I_f I_c1 gathered multiply-adds
// of the readout, per (vector, family) item; M the real transform length. The spectral path costs about
// one transform latency per wave of items (~one item per SM). The direct
// path wins where I is small against J (batch 15: I <= 100 with J >= 1000).
bool use_direct(st_engine* e, size_t batch, size_t free_mode) {
  if (is_exact(e) || batch == 0 || e->tsk == nullptr) return false;
  if (e->path == ST_PATH_SPECTRAL) return false;
  if (!corr_feasible(e, free_mode)) return false;
  if (e->path == ST_PATH_DIRECT) return true;
  if (e->plan.large_p1) return false;  // two-level transforms: not in the fitted range
  int c1, c2;
  contracted(free_mode, &c1, &c2);
  const double J = static_cast<double>(e->hash_len);
  const double Fq = (2 * J - 1) * static_cast<double>(e->dims[c2]);
  const double Fz = static_cast<double>(e->dims[free_mode]) * static_cast<double>(e->dims[c1]);
  const double M = static_cast<double>(e->plan.M);  // real transform length
  const double items = static_cast<double>(batch) * static_cast<double>(e->D);
  if (batch == 1) {
    const double direct = 13.0 + (2.7e-6 * Fq + 6e-5 * Fz) * std::max(1.0, items / 10.0) + 1.5e-3 * J;
    const double spectral = M < 4096 ? 18.5 : 10.4 + 6.5e-4 * M;
    return direct < spectral;
  }
  // the spectral step splits a batch beyond one item per SM between the
  // one-CTA kernel and clusters on a side stream: no whole extra wave
  const double load = std::max(1.0, items / 160.0);
  return 17.0 + (1.7e-5 * Fq + 2.9e-4 * Fz) * items / 150.0 < (17.0 + 2.5e-3 * M) * load;
}

int corr_sync(st_engine* e, cudaStream_t st) {
  if (!e->tsk_stale) return ST_OK;
  if (int rc = launch_real_from_spec(e->plan, e->spec, static_cast<int>(e->D), e->tsk, e->jt,
                                     static_cast<int>(e->jt), 0, st))
    return rc;
  e->tsk_stale = false;
  return ST_OK;
}

int engine_iuv_fused(st_engine* e, size_t batch, const double* a, size_t free_mode, int mode,
                     double* out, double* best, int* stopped, cudaStream_t st) {
  return iuv_fused_ab(e, batch, a, a, free_mode, mode, out, best, stopped, st);
}
}  // namespace fcs

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
  if (pl.large_p1) return 1;  // the two-level path allocates its own scratch
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
    a.hash_lens[n] = static_cast<int>(hash_lens[n]);
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
  const size_t need =
      pl.large_p1 ? 1 : (std::max<size_t>(1, r_count) + 1) * sketch_count * pl.P * sizeof(double2);
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
  FCS_CUDA_TRY(malloc_async(reinterpret_cast<void**>(&scr), batch * pl.P * sizeof(double2), st));
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
  const size_t wa = (std::max<size_t>(1, wsa) + 255) / 256 * 256;
  FCS_CUDA_TRY(malloc_async(&ws, wa + std::max<size_t>(1, wsb), st));
  FCS_CUDA_TRY(malloc_async(reinterpret_cast<void**>(&fa), D * la * sizeof(double), st));
  FCS_CUDA_TRY(malloc_async(reinterpret_cast<void**>(&fb), D * lb * sizeof(double), st));
  // the two operand sketches are independent and each fills ~one wave: B's
  // runs on the side stream (fork / join) concurrently with A's
  cudaStream_t st2 = nullptr;
  FCS_CUDA_TRY(fork_side(st, &st2));
  int rc = launch_fcs_dense(ST_F64, a, 2, da, 0, ca, D, packed, hash_lens, fa, 0, ws, wsa, st,
                            stride);
  const int rcb = launch_fcs_dense(ST_F64, b, 2, db, 0, cb, D, packed + ra + ca, hash_lens + 2, fb,
                                   0, static_cast<char*>(ws) + wa, wsb, st2, stride);
  FCS_CUDA_TRY(join_side(st));  // before anything else on st, whatever the launches returned
  if (!rc) rc = rcb;
  if (!rc) rc = st_convolve_pairs(fa, la, fb, lb, D, out, st);
  cudaFreeAsync(ws, st);
  cudaFreeAsync(fa, st);
  cudaFreeAsync(fb, st);
  return rc;
}

int st_dft(const double* x, size_t len, size_t n, double* out, void* stream) {
  FCS_CHECK_ARG(n > 0, "dft: zero length");
  return exact_dft(x, nullptr, len, len, n, 1, -1.0, reinterpret_cast<double2*>(out),
                   as_stream(stream));
}

int st_idft_real(const double* spectrum, size_t n, double* out, int check, void* stream) {
  FCS_CHECK_ARG(n > 0, "idft_real: zero length");
  return exact_idft_real(reinterpret_cast<const double2*>(spectrum), n, 1, out, check,
                         as_stream(stream));
}

int st_fft_convolve(const double* const* inputs, const size_t* lens, size_t k, size_t n,
                    double* out, void* stream) {
  FCS_CHECK_ARG(k > 0, "fft_convolve: no inputs");
  FCS_CHECK_ARG(n > 0, "dft: zero length");
  return exact_fft_convolve(inputs, lens, k, n, out, as_stream(stream));
}

int st_precompute_z(const double* spectrum, size_t n, const double* a, size_t la,
                    const uint32_t* pair_a, size_t ja, const double* b, size_t lb,
                    const uint32_t* pair_b, size_t jb, double* z, void* stream) {
  FCS_CHECK_ARG(n > 0, "dft: zero length");
  FCS_CHECK_ARG(la > 0 && lb > 0 && ja > 0 && jb > 0, "HashPair: dimensions must be positive");
  cudaStream_t st = as_stream(stream);
  double* cs = nullptr;
  FCS_CUDA_TRY(malloc_async(reinterpret_cast<void**>(&cs), (ja + jb) * sizeof(double), st));
  int rc = launch_cs_columns(a, static_cast<int>(la), 1, pair_a, static_cast<int>(ja), cs, st);
  if (!rc)
    rc = launch_cs_columns(b, static_cast<int>(lb), 1, pair_b, static_cast<int>(jb), cs + ja, st);
  if (!rc)
    rc = exact_precompute_z(reinterpret_cast<const double2*>(spectrum), n, cs, ja, cs + ja, jb, z,
                            st);
  cudaFreeAsync(cs, st);
  return rc;
}

int st_engine_create_backend(st_engine** engine, int backend, int dtype, const void* tensor,
                             const size_t* dims, size_t hash_len, size_t sketch_count,
                             uint64_t seed, void* stream) {
  FCS_CHECK_ARG(engine != nullptr, "st_engine_create: null engine pointer");
  FCS_CHECK_ARG(backend >= ST_BACKEND_PLAIN && backend <= ST_BACKEND_FCS,
                "make_contraction_engine: unknown backend");
  FCS_CHECK_ARG(dtype == ST_F32 || dtype == ST_F64, "st_engine_create: unknown dtype");
  FCS_CHECK_ARG(backend == ST_BACKEND_PLAIN || (hash_len > 0 && sketch_count > 0),
                "EstimatorConfig: hash_len and sketch_count must be >= 1");
  for (int n = 0; n < 3; ++n) FCS_CHECK_ARG(dims[n] > 0, "DenseTensor: zero dimension");
  *engine = nullptr;
  cudaStream_t st = as_stream(stream);
  auto* e = new st_engine();
  FCS_CUDA_TRY(cudaGetDevice(&e->device));
  e->backend = backend;
  e->path = default_path();
  for (int n = 0; n < 3; ++n) e->dims[n] = dims[n];
  e->hash_len = hash_len;
  e->D = sketch_count;
  if (backend == ST_BACKEND_PLAIN || backend == ST_BACKEND_HCS || backend == ST_BACKEND_CS) {
    // engines_exact.cu: Plain holds the tensor (D = 1: exact contractions);
    // HCS the D J^3 sketches (needs the families' tables); CS the D long pairs
    if (backend == ST_BACKEND_PLAIN) e->D = 1;
    const size_t sum_dims = dims[0] + dims[1] + dims[2];
    std::vector<uint64_t> seeds(e->D);
    for (size_t d = 0; d < e->D; ++d)  // families_for / CsEngine seeds (cpd.cpp:162-166)
      seeds[d] = splitmix_draw(seed + static_cast<uint64_t>(d), 1);
    int rc = ST_OK;
    if (backend == ST_BACKEND_HCS) {
      const size_t hl[3] = {hash_len, hash_len, hash_len};
      if (cudaMalloc(reinterpret_cast<void**>(&e->packed), e->D * sum_dims * sizeof(uint32_t)) !=
          cudaSuccess)
        rc = fail(ST_ENOMEM, "st_engine_create: device allocation failed");
      if (!rc) rc = launch_family_tables(3, dims, hl, e->D, seeds.data(), e->packed, st);
    } else if (backend == ST_BACKEND_CS) {
      if (cudaMalloc(reinterpret_cast<void**>(&e->seeds), e->D * sizeof(uint64_t)) != cudaSuccess)
        rc = fail(ST_ENOMEM, "st_engine_create: device allocation failed");
      if (!rc && cudaMemcpy(e->seeds, seeds.data(), e->D * sizeof(uint64_t),
                            cudaMemcpyHostToDevice) != cudaSuccess)
        rc = fail(ST_ECUDA, "st_engine_create: seed upload failed");
    }
    if (!rc) rc = exact_create(e, dtype, tensor, st);
    if (rc) {
      st_engine_destroy(e);
      return rc;
    }
    *engine = e;
    return ST_OK;
  }
  e->jt = 3 * hash_len - 2;
  e->slen = backend == ST_BACKEND_TS ? hash_len : e->jt;
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
  const size_t vbytes = sketch_count * e->jt * sizeof(double);
  bool ok = malloc_async(reinterpret_cast<void**>(&e->packed),
                            sketch_count * sum_dims * sizeof(uint32_t), st) == cudaSuccess &&
            malloc_async(reinterpret_cast<void**>(&e->spec),
                            sketch_count * e->plan.P * sizeof(double2), st) == cudaSuccess &&
            malloc_async(reinterpret_cast<void**>(&vals), vbytes, st) == cudaSuccess &&
            malloc_async(&ws, std::max<size_t>(1, wsb), st) == cudaSuccess;
  if (ok && backend == ST_BACKEND_TS) {
    const double one = 1.0;
    ok = cudaMalloc(reinterpret_cast<void**>(&e->ext), vbytes) == cudaSuccess &&
         cudaMalloc(reinterpret_cast<void**>(&e->one), sizeof(double)) == cudaSuccess &&
         cudaMemcpy(e->one, &one, sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess;
  }
  if (!ok) {
    if (vals) cudaFreeAsync(vals, st);
    if (ws) cudaFreeAsync(ws, st);
    st_engine_destroy(e);
    return fail(ST_ENOMEM, "st_engine_create: device allocation failed");
  }
  rc = launch_family_tables(3, dims, hl, sketch_count, seeds.data(), e->packed, st);
  if (!rc)
    rc = launch_fcs_dense(dtype, tensor, 3, dims, 0, dims[2], sketch_count, e->packed, hl, vals,
                          0, ws, wsb, st, 0);
  const double* src = vals;
  if (!rc && backend == ST_BACKEND_TS) {  // TS = (FCS) mod J, kept as its periodic extension
    rc = launch_ts_extend(vals, static_cast<int>(sketch_count), static_cast<int>(e->jt),
                          static_cast<int>(hash_len), e->ext, 1.0, 0, st);
    src = e->ext;
  }
  if (!rc)
    rc = launch_spec_from_real(e->plan, src, e->jt, static_cast<int>(e->jt),
                               static_cast<int>(sketch_count), e->spec, st);
  if (backend == ST_BACKEND_FCS) {  // the direct estimator's time-domain sketches
    e->tsk = vals;
    e->tsk_own = true;
  } else {
    cudaFreeAsync(vals, st);
    e->tsk = e->ext;
  }
  cudaFreeAsync(ws, st);
  if (rc) {
    st_engine_destroy(e);
    return rc;
  }
  *engine = e;
  return ST_OK;
}

namespace {
// out[l] = s(l) * src[h(l)] for a packed pair (bucket | sign << 31).
__global__ void cs_expand_kernel(const double* __restrict__ src, const uint32_t* __restrict__ pair,
                                 size_t count, double* __restrict__ out) {
  for (size_t l = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; l < count;
       l += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint32_t e = __ldg(pair + l);
    const double v = src[e & 0x7fffffffu];
    out[l] = (e & 0x80000000u) ? -v : v;
  }
}
}  // namespace

int st_cs_expand(const double* src, size_t src_len, const uint32_t* packed_pair, size_t count,
                 double* out, void* stream) {
  FCS_CHECK_ARG(src_len > 0, "HashPair: dimensions must be positive");
  if (count == 0) return ST_OK;
  cs_expand_kernel<<<static_cast<unsigned>(std::min<size_t>(ceil_div(count, 256), 65535)), 256, 0,
                     as_stream(stream)>>>(src, packed_pair, count, out);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

namespace {
// ext[d][k] = ts[d][k mod J], k < jt (the TS engine's periodic extension of a
// given TS sketch; st_engine_create builds it from the FCS instead).
__global__ void ts_periodic_kernel(const double* __restrict__ ts, int D, int J, int jt,
                                   double* __restrict__ ext) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<size_t>(D) * jt) return;
  const int d = static_cast<int>(i / jt);
  const int k = static_cast<int>(i - static_cast<size_t>(d) * jt);
  ext[i] = ts[static_cast<size_t>(d) * J + k % J];
}
}  // namespace

int st_engine_from_sketches(st_engine** engine, int backend, const double* sketches,
                            size_t sketch_count, const size_t* dims, size_t hash_len,
                            const uint32_t* packed, void* stream) {
  FCS_CHECK_ARG(engine != nullptr, "st_engine_create: null engine pointer");
  FCS_CHECK_ARG(backend == ST_BACKEND_FCS || backend == ST_BACKEND_TS,
                "st_engine_from_sketches: FCS or TS backend required");
  FCS_CHECK_ARG(hash_len > 0 && sketch_count > 0,
                "EstimatorConfig: hash_len and sketch_count must be >= 1");
  for (int n = 0; n < 3; ++n) FCS_CHECK_ARG(dims[n] > 0, "DenseTensor: zero dimension");
  *engine = nullptr;
  cudaStream_t st = as_stream(stream);
  auto* e = new st_engine();
  FCS_CUDA_TRY(cudaGetDevice(&e->device));
  e->backend = backend;
  e->path = default_path();
  for (int n = 0; n < 3; ++n) e->dims[n] = dims[n];
  e->hash_len = hash_len;
  e->D = sketch_count;
  e->jt = 3 * hash_len - 2;
  e->slen = backend == ST_BACKEND_TS ? hash_len : e->jt;
  int rc = get_fft_plan(e->jt, &e->plan);
  if (rc) {
    delete e;
    return rc;
  }
  const size_t sum_dims = dims[0] + dims[1] + dims[2];
  const size_t vbytes = sketch_count * e->jt * sizeof(double);
  bool ok = cudaMalloc(reinterpret_cast<void**>(&e->packed),
                       sketch_count * sum_dims * sizeof(uint32_t)) == cudaSuccess &&
            cudaMalloc(reinterpret_cast<void**>(&e->spec),
                       sketch_count * e->plan.P * sizeof(double2)) == cudaSuccess;
  if (ok && backend == ST_BACKEND_TS) {
    const double one = 1.0;
    ok = cudaMalloc(reinterpret_cast<void**>(&e->ext), vbytes) == cudaSuccess &&
         cudaMalloc(reinterpret_cast<void**>(&e->one), sizeof(double)) == cudaSuccess &&
         cudaMemcpy(e->one, &one, sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess;
  }
  if (!ok) {
    st_engine_destroy(e);
    return fail(ST_ENOMEM, "st_engine_create: device allocation failed");
  }
  if (cudaMemcpyAsync(e->packed, packed, sketch_count * sum_dims * sizeof(uint32_t),
                      cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
    st_engine_destroy(e);
    return fail(ST_ECUDA, "st_engine_from_sketches: table copy failed");
  }
  const double* src = sketches;
  if (backend == ST_BACKEND_FCS) {
    if (cudaMalloc(reinterpret_cast<void**>(&e->tsk), vbytes) != cudaSuccess) {
      st_engine_destroy(e);
      return fail(ST_ENOMEM, "st_engine_create: device allocation failed");
    }
    e->tsk_own = true;
    if (cudaMemcpyAsync(e->tsk, sketches, vbytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
      st_engine_destroy(e);
      return fail(ST_ECUDA, "st_engine_from_sketches: sketch copy failed");
    }
  } else {
    e->tsk = e->ext;
  }
  if (backend == ST_BACKEND_TS) {
    const size_t n = sketch_count * e->jt;
    ts_periodic_kernel<<<ceil_div(n, 256), 256, 0, st>>>(
        sketches, static_cast<int>(sketch_count), static_cast<int>(hash_len),
        static_cast<int>(e->jt), e->ext);
    src = e->ext;
  }
  rc = launch_spec_from_real(e->plan, src, e->jt, static_cast<int>(e->jt),
                             static_cast<int>(sketch_count), e->spec, st);
  if (rc) {
    st_engine_destroy(e);
    return rc;
  }
  *engine = e;
  return ST_OK;
}

int st_engine_create(st_engine** engine, int dtype, const void* tensor, const size_t* dims,
                     size_t hash_len, size_t sketch_count, uint64_t seed, void* stream) {
  return st_engine_create_backend(engine, ST_BACKEND_FCS, dtype, tensor, dims, hash_len,
                                  sketch_count, seed, stream);
}

int st_engine_destroy(st_engine* e) {
  if (!e) return ST_OK;
  cudaDeviceSynchronize();
  if (e->packed) cudaFree(e->packed);
  if (e->spec) cudaFree(e->spec);
  if (e->ext) cudaFree(e->ext);
  if (e->one) cudaFree(e->one);
  if (e->dense) cudaFree(e->dense);
  if (e->seeds) cudaFree(e->seeds);
  if (e->tsk && e->tsk_own) cudaFree(e->tsk);
  e->corr.release(nullptr);
  e->scratch.release(nullptr);
  e->est.release(nullptr);
  e->vec.release(nullptr);
  e->vec2.release(nullptr);
  e->cnt.release(nullptr);
  e->est2.release(nullptr);
  cudaDeviceSynchronize();
  delete e;
  return ST_OK;
}

int st_engine_backend(const st_engine* e) { return e ? e->backend : -1; }

size_t st_engine_composed_len(const st_engine* e) { return e ? e->slen : 0; }

int st_engine_sketches(st_engine* e, double* out, void* stream) {
  FCS_CHECK_ARG(e != nullptr, "st_engine_sketches: null engine");
  FCS_CHECK_ARG(e->backend != ST_BACKEND_PLAIN, "st_engine_sketches: the plain engine has no sketches");
  if (e->backend == ST_BACKEND_HCS || e->backend == ST_BACKEND_CS) {
    FCS_CUDA_TRY(cudaMemcpyAsync(out, e->dense, e->D * e->slen * sizeof(double),
                                 cudaMemcpyDeviceToDevice, as_stream(stream)));
    return ST_OK;
  }
  if (e->backend == ST_BACKEND_TS) {
    FCS_CUDA_TRY(cudaMemcpy2DAsync(out, e->slen * sizeof(double), e->ext, e->jt * sizeof(double),
                                   e->slen * sizeof(double), e->D, cudaMemcpyDeviceToDevice,
                                   as_stream(stream)));
    return ST_OK;
  }
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
  if (is_exact(e)) {  // Plain / HCS / CS (engines_exact.cu); Plain is exact: no median
    const bool med = median && e->backend != ST_BACKEND_PLAIN;
    double* est = out;
    if (med) {
      if (int rc = e->est.ensure(batch * e->D * nf * sizeof(double), st)) return rc;
      est = static_cast<double*>(e->est.p);
    }
    if (int rc = exact_iuv(e, batch, a, b, static_cast<int>(free_mode), est, st)) return rc;
    return med ? launch_median(est, static_cast<int>(batch), static_cast<int>(e->D),
                               static_cast<int>(nf), out, st)
               : ST_OK;
  }
  if (use_direct(e, batch, free_mode)) {  // time-domain correlation (correlate.cu)
    if (median && e->D <= 16)
      return iuv_fused_ab(e, batch, a, b, free_mode, 1, out, nullptr, nullptr, st);
    if (int rc = corr_sync(e, st)) return rc;
    if (!median) return corr_estimate(e, batch, a, b, free_mode, nullptr, out, st);
    if (int rc = e->est.ensure(batch * e->D * nf * sizeof(double), st)) return rc;
    double* est = static_cast<double*>(e->est.p);
    if (int rc = corr_estimate(e, batch, a, b, free_mode, nullptr, est, st)) return rc;
    return launch_median(est, static_cast<int>(batch), static_cast<int>(e->D),
                         static_cast<int>(nf), out, st);
  }
  if (median) {  // small batches: cluster estimator with the median fused in
    const int rc = iuv_fused_ab(e, batch, a, b, free_mode, 1, out, nullptr, nullptr, st);
    if (rc != 1) return rc;
  }
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
  if (is_exact(e)) {
    const bool med = median && e->backend != ST_BACKEND_PLAIN;
    double* est = out;
    if (med) {
      if (int rc = e->est.ensure(batch * e->D * sizeof(double), st)) return rc;
      est = static_cast<double*>(e->est.p);
    }
    if (int rc = exact_uvw(e, batch, u, v, w, est, st)) return rc;
    return med ? launch_median(est, static_cast<int>(batch), static_cast<int>(e->D), 1, out, st)
               : ST_OK;
  }
  if (use_direct(e, batch, 2)) {  // <w, T(u, v, I)> in the time domain (correlate.cu)
    if (median && e->D <= 16) return iuv_fused_ab(e, batch, u, v, 2, 4, out, nullptr, nullptr, st, w);
    if (int rc = corr_sync(e, st)) return rc;
    if (!median) return corr_estimate(e, batch, u, v, 2, w, out, st);
    if (int rc = e->est.ensure(batch * e->D * sizeof(double), st)) return rc;
    double* est = static_cast<double*>(e->est.p);
    if (int rc = corr_estimate(e, batch, u, v, 2, w, est, st)) return rc;
    return launch_median(est, static_cast<int>(batch), static_cast<int>(e->D), 1, out, st);
  }
  if (median) {  // small batches: <w, T(u, v, I)> per family on the cluster estimator, median fused
    const int rc = iuv_fused_ab(e, batch, u, v, 2, 4, out, nullptr, nullptr, st, w);
    if (rc != 1) return rc;
    // beyond one CTA per SM (config 3's 15 restarts x 10 families): the first
    // nb1 vectors on the one-CTA kernel + median, the rest as clusters on the
    // side stream (median fused), as launch_iuv splits its batch
    DeviceInfo di;
    if (int rc2 = device_info(&di)) return rc2;
    const size_t nb1 = static_cast<size_t>(di.sm_count) / e->D;
    if (!e->plan.large_p1 && nb1 > 0 && batch > nb1) {
      const size_t nb2 = batch - nb1;
      if (int rc2 = e->scratch.ensure(nb1 * e->D * e->plan.P * sizeof(double2), st)) return rc2;
      if (int rc2 = e->est.ensure((nb1 + nb2) * e->D * sizeof(double), st)) return rc2;
      const size_t had = e->cnt.bytes;
      if (int rc2 = e->cnt.ensure(std::max<size_t>(nb2, 64) * sizeof(int), st)) return rc2;
      if (e->cnt.bytes != had) FCS_CUDA_TRY(cudaMemsetAsync(e->cnt.p, 0, e->cnt.bytes, st));
      double* est = static_cast<double*>(e->est.p);
      IuvTail t;
      t.mode = 4;
      t.cnt = static_cast<int*>(e->cnt.p);
      t.out = out + nb1;
      t.wvec = w + nb1 * e->dims[2];
      cudaStream_t st2 = nullptr;
      FCS_CUDA_TRY(fork_side(st, &st2));
      const EngArgs args = e->args();
      // one-CTA part first (the submission order that keeps the two parts
      // concurrent on any caller stream, as launch_iuv's split)
      int rco = launch_uvw_dot(e->plan, args, static_cast<int>(nb1), u, v, w,
                               static_cast<double2*>(e->scratch.p), est, st);
      int rcc = launch_iuv_cluster(e->plan, args, static_cast<int>(nb2), u + nb1 * e->dims[0],
                                   v + nb1 * e->dims[1], 0, 1, 2, est + nb1 * e->D, t, st2);
      // join before the median: a join directly followed by the next call's
      // fork measured a serialising stall (tools/experiments/iuv_split_probe.py)
      FCS_CUDA_TRY(join_side(st));
      if (rcc == 0 && !rco)
        rco = launch_median(est, static_cast<int>(nb1), static_cast<int>(e->D), 1, out, st);
      if (rcc == 0) return rco;
      if (rcc != 1) return rcc;
    }
  }
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
  if (is_exact(e)) return exact_deflate(e, weight, u, v, w, st);
  if (e->backend == ST_BACKEND_TS) {
    // TsEngine::deflate (cpd.cpp:115-122): TS -= ts_sketch(w u o v o w) =
    // ((CP-form FCS of u o v o w) mod J), then the spectra are rebuilt.
    const size_t qbytes = 2 * e->D * e->plan.P * sizeof(double2);
    if (int rc = e->scratch.ensure(qbytes + e->D * e->jt * sizeof(double), st)) return rc;
    auto* q = static_cast<double2*>(e->scratch.p);
    auto* c = reinterpret_cast<double*>(static_cast<char*>(e->scratch.p) + qbytes);
    CpArgs a{};
    a.order = 3;
    const EngArgs ea = e->args();
    for (int n = 0; n < 3; ++n) {
      a.dims[n] = ea.dims[n];
      a.tab_off[n] = ea.tab_off[n];
      a.hash_lens[n] = ea.hash_len;
    }
    a.fam_stride = ea.fam_stride;
    a.factors[0] = u;
    a.factors[1] = v;
    a.factors[2] = w;
    a.weights = e->one;
    a.r_begin = 0;
    a.r_count = 1;
    if (int rc = launch_cp(e->plan, a, static_cast<int>(e->D), e->packed, q, c,
                           static_cast<int>(e->jt), 0, st))
      return rc;
    if (int rc = launch_ts_extend(c, static_cast<int>(e->D), static_cast<int>(e->jt),
                                  static_cast<int>(e->hash_len), e->ext, -weight, 1, st))
      return rc;
    return launch_spec_from_real(e->plan, e->ext, e->jt, static_cast<int>(e->jt),
                                 static_cast<int>(e->D), e->spec, st);
  }
  if (int rc = e->scratch.ensure(e->D * e->plan.P * sizeof(double2), st)) return rc;
  e->tsk_stale = true;  // rebuilt from the deflated spectra on the next direct estimate
  return launch_deflate(e->plan, e->args(), weight, u, v, w, static_cast<double2*>(e->scratch.p),
                        e->spec, st);
}

int st_engine_set_path(st_engine* e, int path) {
  FCS_CHECK_ARG(e != nullptr, "st_engine_set_path: null engine");
  FCS_CHECK_ARG(path == ST_PATH_AUTO || path == ST_PATH_SPECTRAL || path == ST_PATH_DIRECT,
                "st_engine_set_path: unknown path");
  e->path = path;
  return ST_OK;
}

}  // extern "C"
