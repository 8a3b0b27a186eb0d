// Shared host-side pieces of the contraction engine (engine.cu) and the CPD
// drivers built on it (cpd.cu).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <numbers>

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
int launch_uvw_dot(const FftPlan&, const EngArgs&, int, const double*, const double*, const double*,
                   double2*, double*, cudaStream_t);
int launch_cs_columns(const double*, int, int, const uint32_t*, int, double*, cudaStream_t);
int launch_normalize_rows(double*, int, int, cudaStream_t);
int launch_median_normalize(const double*, int, int, int, double*, cudaStream_t);
int launch_refine_update(double*, const double*, int, int*, cudaStream_t);
int launch_family_tables(size_t, const size_t*, const size_t*, size_t, const uint64_t*,
                         uint32_t*, cudaStream_t);
// ext[d][k] (+)= scale * sum_{m = k mod J, m < jt} in[d][m]   (engine.cu)
int launch_ts_extend(const double* in, int D, int jt, int J, double* ext, double scale,
                     int accumulate, cudaStream_t st);

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Stream-ordered scratch that only grows. Every use calls ensure() with its
// stream; when the stream differs from the previous user's, the new stream
// first waits (event) for the previous stream's work, so neither the buffer's
// contents nor a cudaFreeAsync on growth can race a kernel still reading it.
struct Scratch {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t last = nullptr;
  bool used = false;
  int ensure(size_t need, cudaStream_t st) {
    if (used && last != st) {
      cudaEvent_t ev;
      bool ok = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess;
      if (ok) {
        ok = cudaEventRecord(ev, last) == cudaSuccess && cudaStreamWaitEvent(st, ev, 0) == cudaSuccess;
        cudaEventDestroy(ev);
      }
      if (!ok) {  // the previous stream is gone: order against the whole device
        cudaGetLastError();
        FCS_CUDA_TRY(cudaDeviceSynchronize());
      }
    }
    last = st;
    used = true;
    if (need <= bytes) return ST_OK;
    if (p) FCS_CUDA_TRY(cudaFreeAsync(p, st));
    p = nullptr;
    bytes = 0;
    FCS_CUDA_TRY(malloc_async(&p, need, st));
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
inline void contracted(size_t f, int* c1, int* c2) {
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
  // random_unit (cpd.cpp:199-204): dim gaussians, then divide by the norm.
  void unit(double* u, size_t dim) {
    for (size_t i = 0; i < dim; ++i) u[i] = gaussian();
    double sq = 0.0;
    for (size_t i = 0; i < dim; ++i) sq += u[i] * u[i];
    const double norm = std::sqrt(sq);
    if (norm > 0)
      for (size_t i = 0; i < dim; ++i) u[i] /= norm;
  }
};

}  // namespace fcs

struct st_engine;
namespace fcs {
// Plain / HCS / CS backends (engines_exact.cu)
int exact_create(st_engine* e, int dtype, const void* tensor, cudaStream_t st);
int exact_iuv(st_engine* e, size_t batch, const double* a, const double* b, int f, double* est,
              cudaStream_t st);
int exact_uvw(st_engine* e, size_t batch, const double* u, const double* v, const double* w,
              double* est, cudaStream_t st);
int exact_deflate(st_engine* e, double weight, const double* u, const double* v, const double* w,
                  cudaStream_t st);
}  // namespace fcs

// The engine: D families' packed hash tables and the cached half spectra of
// the sketch each estimate correlates against.
//  FCS backend: S_d = F(FCS_d(T)), length J~ = 3J - 2 (FcsEngine, cpd.cpp:61-94).
//  TS backend:  S_d = F(ext_d) with ext_d[k] = TS_d(T)[k mod J] for k < 3J - 2.
//    The reference correlates at length J (circular, TsEngine cpd.cpp:96-126
//    -> iuv_spectral/uvw_spectral with n = J, estimators.cpp:213-233); every
//    index it reads, (k + j1 + j2) mod J with k, j1, j2 < J, equals the linear
//    index k + j1 + j2 < 3J - 2 into the J-periodic extension, so the FCS
//    kernels at length J~ compute the same estimates with no new kernel.
struct st_engine {
  int device = 0;
  int backend = ST_BACKEND_FCS;
  size_t dims[3] = {0, 0, 0};
  size_t hash_len = 0;
  size_t D = 0;
  size_t jt = 0;        // correlation length (3J - 2 for both backends)
  size_t slen = 0;      // sketch length (J~ for FCS, J for TS)
  fcs::FftPlan plan{};
  uint32_t* packed = nullptr;  // D x sum(dims)
  double2* spec = nullptr;     // D x P
  double* ext = nullptr;       // TS: D x jt periodic extension (real)
  double* one = nullptr;       // TS: device 1.0 (rank-one CP weight)
  double* dense = nullptr;     // Plain: the tensor; HCS: D x J^3 sketches; CS: D x J sketches
  uint64_t* seeds = nullptr;   // CS: the D long pairs' seeds
  fcs::Scratch scratch, est, vec, vec2;
  fcs::Scratch cnt;  // per-vector arrival counters of the fused cluster tail (kept zero)
  fcs::Scratch est2;  // per-family estimates of the rtpm restart step
  // time-domain sketches for the direct estimator (correlate.cu): FCS owns a
  // D x jt copy (rebuilt from spec after a deflation), TS aliases ext
  double* tsk = nullptr;
  bool tsk_own = false;
  bool tsk_stale = false;
  int path = 0;        // ST_PATH_AUTO / ST_PATH_SPECTRAL / ST_PATH_DIRECT
  fcs::Scratch corr;   // direct path: Q (batch x D x (2J - 1))
  fcs::EngArgs args() const {
    fcs::EngArgs e{};
    size_t off = 0;
    for (int n = 0; n < 3; ++n) {
      e.dims[n] = static_cast<int>(dims[n]);
      e.tab_off[n] = static_cast<int>(off);
      off += dims[n];
    }
    e.fam_stride = static_cast<int>(off);
    e.D = static_cast<int>(D);
    e.hash_len = static_cast<int>(hash_len);
    e.packed = packed;
    e.spec = spec;
    return e;
  }
};

namespace fcs {
// The cluster estimator with its fused tail (IuvTail modes 1-3) over `batch`
// vectors a (= b) with free mode 0; returns 1 when the cluster path does not
// apply (the caller runs the separate kernels).
int engine_iuv_fused(st_engine* e, size_t batch, const double* a, size_t free_mode, int mode,
                     double* out, double* best, int* stopped, cudaStream_t st);
// Direct (time-domain) estimator, correlate.cu.
bool corr_feasible(const st_engine* e, size_t free_mode);
// With a tail (mode 1-4, IuvTail of fft.cuh) the median over the families
// (and the rtpm row normalisation / refinement update) is fused into the
// readout kernel; tail->cnt must hold `batch` zeroed counters.
int corr_estimate(st_engine* e, size_t batch, const double* a, const double* b, size_t free_mode,
                  const double* w, double* est, cudaStream_t st, const IuvTail* tail = nullptr);
// Whether iuv / uvw over `batch` vectors with this free mode takes the direct
// path (engine.cu: path override, feasibility, cost rule); rebuilds e->tsk
// from the spectra when a deflation left it stale.
bool use_direct(st_engine* e, size_t batch, size_t free_mode);
int default_path();
int corr_sync(st_engine* e, cudaStream_t st);
inline bool is_exact(const st_engine* e) {
  return e->backend == ST_BACKEND_PLAIN || e->backend == ST_BACKEND_HCS ||
         e->backend == ST_BACKEND_CS;
}
}  // namespace fcs
