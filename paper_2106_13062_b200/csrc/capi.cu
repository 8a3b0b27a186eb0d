// C-ABI layer (include/fcs_b200.h): host-side validation, workspace and
// dispatch to the sm_100a kernels. No CPU compute path exists: every compute
// entry launches device kernels or fails.
#include <cuda_runtime.h>

#include <cmath>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <numbers>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace fcs {

thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int device_info(DeviceInfo* out) {
  static std::mutex mu;
  static DeviceInfo cache[64];
  int dev = 0;
  FCS_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(ST_ECUDA, "device index out of range");
  std::lock_guard<std::mutex> lock(mu);
  if (cache[dev].device != dev) {
    cudaDeviceProp p;
    FCS_CUDA_TRY(cudaGetDeviceProperties(&p, dev));
    if (p.major < 10) return fail(ST_ECUDA, "fcs_b200 requires an sm_100 (Blackwell) device");
    cache[dev].device = dev;
    cache[dev].sm_count = p.multiProcessorCount;
    cache[dev].smem_optin = p.sharedMemPerBlockOptin;
    cache[dev].l2_bytes = p.l2CacheSize;
  }
  *out = cache[dev];
  return ST_OK;
}

cudaError_t malloc_async_raw(void** p, size_t bytes, cudaStream_t st) {
  static std::once_flag once[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::call_once(once[dev & 63], [dev]() {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  });
  return cudaMallocAsync(p, bytes, st);
}

namespace {
struct SideStream {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
std::mutex g_side_mu;
SideStream g_side[64];
cudaError_t side_of(SideStream** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  SideStream& s = g_side[dev & 63];
  if (s.side == nullptr) {
    if ((e = cudaStreamCreateWithFlags(&s.side, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming)) != cudaSuccess)
      return e;
  }
  *out = &s;
  return cudaSuccess;
}
}  // namespace

cudaError_t fork_side(cudaStream_t st, cudaStream_t* side) {
  std::lock_guard<std::mutex> lock(g_side_mu);
  SideStream* s = nullptr;
  cudaError_t e = side_of(&s);
  if (e == cudaSuccess) e = cudaEventRecord(s->fork, st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s->side, s->fork, 0);
  if (e == cudaSuccess) *side = s->side;
  return e;
}

cudaError_t join_side(cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g_side_mu);
  SideStream* s = nullptr;
  cudaError_t e = side_of(&s);
  if (e == cudaSuccess) e = cudaEventRecord(s->join, s->side);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, s->join, 0);
  return e;
}

// kernels (hash.cu, fcs_dense.cu)
int launch_hash_tabulate(uint64_t, size_t, size_t, uint32_t*, int8_t*, cudaStream_t);
int launch_family_tables(size_t, const size_t*, const size_t*, size_t, const uint64_t*,
                         uint32_t*, cudaStream_t);
int launch_pack_tables(size_t, const uint32_t*, const int8_t*, uint32_t*, cudaStream_t);
int launch_device_gaussian(int, uint64_t, size_t, void*, cudaStream_t);

// RAII device buffer for the host-buffer conveniences.
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  int alloc(size_t bytes) {
    if (bytes == 0) bytes = 1;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return fail(ST_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return ST_OK;
  }
};

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Grow-only device buffer.
struct GrowBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t need) {
    if (need <= bytes && p) return ST_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, need ? need : 1);
    if (e != cudaSuccess) return fail(ST_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    bytes = need;
    return ST_OK;
  }
};

// Per-device state of the host-buffer entry: a copy stream, a compute stream,
// double-buffered staging and cached tables / output / workspace.
struct HostCtx {
  std::mutex mu;
  cudaStream_t copy = nullptr, comp = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
  GrowBuf buf[2], tab, out, ws;
};

int host_ctx(HostCtx** out) {
  static std::mutex mu;
  static HostCtx* ctx[64] = {};
  int dev = 0;
  FCS_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(ST_ECUDA, "device index out of range");
  std::lock_guard<std::mutex> lock(mu);
  if (!ctx[dev]) {
    // The side stream of fork_side is created before these two: created
    // after them it measured slower concurrency (config 3's split step 41 ->
    // 54 us after one host-buffer call), created first it does not.
    {
      std::lock_guard<std::mutex> side_lock(g_side_mu);
      SideStream* side = nullptr;
      FCS_CUDA_TRY(side_of(&side));
    }
    auto* c = new HostCtx();
    FCS_CUDA_TRY(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    FCS_CUDA_TRY(cudaStreamCreateWithFlags(&c->comp, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      FCS_CUDA_TRY(cudaEventCreateWithFlags(&c->copied[b], cudaEventDisableTiming));
      FCS_CUDA_TRY(cudaEventCreateWithFlags(&c->done[b], cudaEventDisableTiming));
    }
    ctx[dev] = c;
  }
  *out = ctx[dev];
  return ST_OK;
}

}  // namespace fcs

using namespace fcs;

extern "C" {

const char* st_last_error(void) { return g_last_error.c_str(); }

int st_abi_version(void) { return 3; }

int st_device_query(int* sm_count, size_t* smem_optin, size_t* l2_bytes) {
  DeviceInfo di;
  if (int rc = device_info(&di)) return rc;
  if (sm_count) *sm_count = di.sm_count;
  if (smem_optin) *smem_optin = di.smem_optin;
  if (l2_bytes) *l2_bytes = di.l2_bytes;
  return ST_OK;
}

uint64_t st_family_seed(uint64_t base_seed, size_t d) {
  return splitmix_draw(base_seed + static_cast<uint64_t>(d), 1);
}

int st_hash_tabulate(uint64_t seed, size_t input_dim, size_t hash_len, uint32_t* bucket,
                     int8_t* sign, void* stream) {
  FCS_CHECK_ARG(input_dim > 0 && hash_len > 0, "HashPair: dimensions must be positive");
  FCS_CHECK_ARG(input_dim < (1ull << 32), "HashPair: input_dim too large");
  return launch_hash_tabulate(seed, input_dim, hash_len, bucket, sign, as_stream(stream));
}

int st_family_tables(size_t order, const size_t* dims, const size_t* hash_lens,
                     size_t sketch_count, const uint64_t* master_seeds, uint32_t* packed,
                     void* stream) {
  FCS_CHECK_ARG(order >= 1 && order <= ST_MAX_ORDER, "HashFamily: need one hash length per mode");
  FCS_CHECK_ARG(sketch_count >= 1,
                "EstimatorConfig: hash_len and sketch_count must be >= 1");
  uint64_t total = 0;
  for (size_t n = 0; n < order; ++n) {
    FCS_CHECK_ARG(dims[n] > 0 && hash_lens[n] > 0, "HashPair: dimensions must be positive");
    FCS_CHECK_ARG(hash_lens[n] < (1ull << 30), "HashPair: hash_len too large");
    total += dims[n];
  }
  FCS_CHECK_ARG(total < (1ull << 32), "HashFamily: tables too large");
  return launch_family_tables(order, dims, hash_lens, sketch_count, master_seeds, packed,
                              as_stream(stream));
}

int st_pack_tables(size_t total, const uint32_t* bucket, const int8_t* sign, uint32_t* packed,
                   void* stream) {
  return launch_pack_tables(total, bucket, sign, packed, as_stream(stream));
}

size_t st_fcs_dense_workspace(int dtype, size_t order, const size_t* dims, size_t last_count,
                              size_t sketch_count, const size_t* hash_lens) {
  return dense_workspace(dtype, order, dims, last_count, sketch_count, hash_lens);
}

int st_fcs_dense_report(int dtype, size_t order, const size_t* dims, size_t last_count,
                        size_t sketch_count, const size_t* hash_lens, const void* workspace,
                        size_t workspace_bytes, int* fx_exponent, size_t* fallback_ctas,
                        size_t* ctas) {
  return dense_fx_report(dtype, order, dims, last_count, sketch_count, hash_lens, workspace,
                         workspace_bytes, fx_exponent, fallback_ctas, ctas);
}

int st_fcs_dense(int dtype, const void* tensor, size_t order, const size_t* dims,
                 size_t last_begin, size_t last_count, size_t sketch_count,
                 const uint32_t* packed, const size_t* hash_lens, double* out, int accumulate,
                 void* workspace, size_t workspace_bytes, void* stream) {
  return launch_fcs_dense(dtype, tensor, order, dims, last_begin, last_count, sketch_count,
                          packed, hash_lens, out, accumulate, workspace, workspace_bytes,
                          as_stream(stream));
}

namespace {
// st_fcs_dense_host with the families given by master seeds (K0 on the
// device) or by explicit host packed tables (uploaded).
int fcs_dense_host_impl(int dtype, const void* host_tensor, size_t order, const size_t* dims,
                        size_t last_begin, size_t last_count, size_t sketch_count,
                        const uint64_t* master_seeds, const uint32_t* host_packed,
                        const size_t* hash_lens, double* host_out) {
  FCS_CHECK_ARG(dtype == ST_F32 || dtype == ST_F64, "st_fcs_dense_host: unknown dtype");
  FCS_CHECK_ARG(order >= 1 && order <= ST_MAX_ORDER, "fcs_sketch: unsupported tensor order");
  FCS_CHECK_ARG(sketch_count >= 1, "EstimatorConfig: hash_len and sketch_count must be >= 1");
  size_t per_slab = 1, sum_dims = 0, sum_j = 0;
  for (size_t n = 0; n < order; ++n) {
    FCS_CHECK_ARG(dims[n] > 0 && hash_lens[n] > 0, "HashPair: dimensions must be positive");
    if (n + 1 < order) per_slab *= dims[n];
    sum_dims += dims[n];
    sum_j += hash_lens[n];
  }
  FCS_CHECK_ARG(last_begin + last_count <= dims[order - 1], "fcs_sketch: slab out of range");
  const size_t jt = sum_j - order + 1;
  const size_t esz = dtype == ST_F32 ? 4 : 8;
  HostCtx* hc = nullptr;
  if (int rc = host_ctx(&hc)) return rc;
  std::lock_guard<std::mutex> lock(hc->mu);
  // chunking of the slab along the last mode (order 1: a single chunk)
  const size_t nchunks = order == 1 ? 1 : std::min<size_t>(8, std::max<size_t>(1, last_count));
  const size_t per_chunk = (last_count + nchunks - 1) / nchunks;
  const size_t chunk_elems = (order == 1 ? last_count : per_chunk * per_slab);
  size_t ws = st_fcs_dense_workspace(dtype, order, dims, std::max<size_t>(per_chunk, 1),
                                     sketch_count, hash_lens);
  if (int rc = hc->buf[0].ensure(chunk_elems * esz)) return rc;
  if (int rc = hc->buf[1].ensure(chunk_elems * esz)) return rc;
  if (int rc = hc->tab.ensure(sketch_count * sum_dims * sizeof(uint32_t))) return rc;
  if (int rc = hc->out.ensure(sketch_count * jt * sizeof(double))) return rc;
  if (int rc = hc->ws.ensure(ws)) return rc;
  double* dout = static_cast<double*>(hc->out.p);
  // On any error return below, drain both streams before returning: an H2D
  // copy may still be reading the caller's host buffer.
  struct DrainOnError {
    HostCtx* hc;
    bool armed = true;
    ~DrainOnError() {
      if (armed) {
        cudaStreamSynchronize(hc->copy);
        cudaStreamSynchronize(hc->comp);
      }
    }
  } drain{hc};
  if (master_seeds) {
    if (int rc = st_family_tables(order, dims, hash_lens, sketch_count, master_seeds,
                                  static_cast<uint32_t*>(hc->tab.p), hc->comp))
      return rc;
  } else {
    FCS_CUDA_TRY(cudaMemcpyAsync(hc->tab.p, host_packed,
                                 sketch_count * sum_dims * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, hc->comp));
  }
  if (last_count == 0)
    FCS_CUDA_TRY(cudaMemsetAsync(dout, 0, sketch_count * jt * sizeof(double), hc->comp));
  const char* src = static_cast<const char*>(host_tensor);
  for (size_t k = 0; k * per_chunk < last_count; ++k) {
    const size_t lo = k * per_chunk, cnt = std::min(per_chunk, last_count - lo);
    const int b = static_cast<int>(k & 1);
    const size_t bytes = (order == 1 ? cnt : cnt * per_slab) * esz;
    // the copy may overwrite buffer b only after the sketch that used it finished
    FCS_CUDA_TRY(cudaStreamWaitEvent(hc->copy, hc->done[b], 0));
    FCS_CUDA_TRY(cudaMemcpyAsync(hc->buf[b].p, src + (order == 1 ? lo : lo * per_slab) * esz,
                                 bytes, cudaMemcpyHostToDevice, hc->copy));
    FCS_CUDA_TRY(cudaEventRecord(hc->copied[b], hc->copy));
    FCS_CUDA_TRY(cudaStreamWaitEvent(hc->comp, hc->copied[b], 0));
    if (int rc = st_fcs_dense(dtype, hc->buf[b].p, order, dims, last_begin + lo, cnt, sketch_count,
                              static_cast<uint32_t*>(hc->tab.p), hash_lens, dout, k > 0 ? 1 : 0,
                              hc->ws.p, ws, hc->comp))
      return rc;
    FCS_CUDA_TRY(cudaEventRecord(hc->done[b], hc->comp));
  }
  FCS_CUDA_TRY(cudaMemcpyAsync(host_out, dout, sketch_count * jt * sizeof(double),
                               cudaMemcpyDeviceToHost, hc->comp));
  FCS_CUDA_TRY(cudaStreamSynchronize(hc->comp));
  drain.armed = false;
  return ST_OK;
}
}  // namespace

int st_fcs_dense_host(int dtype, const void* host_tensor, size_t order, const size_t* dims,
                      size_t last_begin, size_t last_count, size_t sketch_count,
                      const uint64_t* master_seeds, const size_t* hash_lens, double* host_out) {
  FCS_CHECK_ARG(master_seeds != nullptr, "st_fcs_dense_host: null seeds");
  return fcs_dense_host_impl(dtype, host_tensor, order, dims, last_begin, last_count,
                             sketch_count, master_seeds, nullptr, hash_lens, host_out);
}

int st_fcs_dense_host_tables(int dtype, const void* host_tensor, size_t order,
                             const size_t* dims, size_t last_begin, size_t last_count,
                             size_t sketch_count, const uint32_t* host_packed,
                             const size_t* hash_lens, double* host_out) {
  FCS_CHECK_ARG(host_packed != nullptr, "st_fcs_dense_host_tables: null tables");
  return fcs_dense_host_impl(dtype, host_tensor, order, dims, last_begin, last_count,
                             sketch_count, nullptr, host_packed, hash_lens, host_out);
}

int st_host_gaussian(uint64_t seed, size_t n, double* out, int threads) {
  // Pair p consumes draws 2p+1 (u1) and 2p+2 (u2) and yields (r cos, r sin):
  // exactly the serial next_gaussian sequence (rng.cpp:8-21), host libm.
  const size_t pairs = (n + 1) / 2;
  auto work = [&](size_t p0, size_t p1) {
    for (size_t p = p0; p < p1; ++p) {
      const uint64_t d1 = splitmix_draw(seed, 2 * p + 1);
      const uint64_t d2 = splitmix_draw(seed, 2 * p + 2);
      const double u1 = static_cast<double>((d1 >> 11) + 1) * 0x1.0p-53;
      const double u2 = static_cast<double>(d2 >> 11) * 0x1.0p-53;
      const double radius = std::sqrt(-2.0 * std::log(u1));
      const double angle = 2.0 * std::numbers::pi * u2;
      out[2 * p] = radius * std::cos(angle);
      if (2 * p + 1 < n) out[2 * p + 1] = radius * std::sin(angle);
    }
  };
  if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  if (pairs < (1u << 16) || threads == 1) {
    work(0, pairs);
    return ST_OK;
  }
  std::vector<std::thread> pool;
  const size_t per = (pairs + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const size_t p0 = std::min(pairs, t * per), p1 = std::min(pairs, p0 + per);
    pool.emplace_back(work, p0, p1);
  }
  for (auto& th : pool) th.join();
  return ST_OK;
}

int st_device_gaussian(int dtype, uint64_t seed, size_t n, void* out, void* stream) {
  FCS_CHECK_ARG(dtype == ST_F32 || dtype == ST_F64, "st_device_gaussian: unknown dtype");
  return launch_device_gaussian(dtype, seed, n, out, as_stream(stream));
}

}  // extern "C"
