// Shared device/host helpers for the FCS B200 library (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

#include "fcs_b200.h"

#if !defined(__CUDA_ARCH__) || __CUDA_ARCH__ >= 1000
#else
#error "fcs_b200 targets sm_100a only"
#endif

namespace fcs {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);

#define FCS_CUDA_TRY(expr)                                                        \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess)                                                        \
      return ::fcs::fail(ST_ECUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
  } while (0)

#define FCS_CHECK_ARG(cond, msg)                                                  \
  do {                                                                            \
    if (!(cond)) return ::fcs::fail(ST_EINVAL, msg);                              \
  } while (0)

// ------------------------------------------------------------- SplitMix64
// rng.hpp:16-21: the k-th draw (1-based) of SplitMix64(seed) is
// fmix64(seed + k * GAMMA); counter-based, so tables tabulate in parallel.
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

__host__ __device__ inline uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__host__ __device__ inline uint64_t splitmix_draw(uint64_t seed, uint64_t k) {
  return fmix64(seed + k * kGamma);
}

__host__ __device__ inline uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

// Packed per-index table entry: bucket in bits [0,31), sign in bit 31
// (1 = negative). Keeps one 4-byte load per index on the hot path.
__host__ __device__ inline uint32_t pack_entry(uint32_t bucket, int8_t sign) {
  return bucket | (sign < 0 ? 0x80000000u : 0u);
}

// Device properties cached per device (SM count, smem opt-in, L2 size).
struct DeviceInfo {
  int device = -1;
  int sm_count = 0;
  size_t smem_optin = 0;
  size_t l2_bytes = 0;
};
int device_info(DeviceInfo* out);

// Stream-ordered allocation from the device's default pool. The first call
// per device raises the pool's release threshold so freed blocks stay
// reserved across stream synchronisations (otherwise every call after a
// sync maps fresh memory: config 5's kron call 0.29 ms instead of 0.08 ms).
cudaError_t malloc_async_raw(void** p, size_t bytes, cudaStream_t st);
// Fork / join with a per-device non-blocking side stream inside one API call
// (independent launches that each fill only part of the device): fork_side
// orders the side stream after everything already on st and returns it;
// join_side orders st after everything enqueued on the side stream. The
// events are per device and reused (a wait binds to the latest record at
// enqueue time), so a call costs two record/wait pairs and no allocation.
cudaError_t fork_side(cudaStream_t st, cudaStream_t* side);
cudaError_t join_side(cudaStream_t st);
template <typename T>
inline cudaError_t malloc_async(T** p, size_t bytes, cudaStream_t st) {
  return malloc_async_raw(reinterpret_cast<void**>(p), bytes, st);
}

inline unsigned ceil_div(size_t a, size_t b) { return static_cast<unsigned>((a + b - 1) / b); }

// K1 launch (fcs_dense.cu). kind 0: FCS bucket sum, 1: HCS mixed radix.
// out_len != 0 overrides the per-family output length (kind 0 only): the
// row-batched sketches (codecs.cu) bake a row offset r * J~ into one mode's
// table entries and write rows x J~ values per family.
int dense_fx_report(int dtype, size_t order, const size_t* dims, size_t last_count, size_t D,
                    const size_t* hash_lens, const void* ws, size_t ws_bytes, int* S,
                    size_t* fallback, size_t* ctas);
size_t dense_workspace(int dtype, size_t order, const size_t* dims, size_t last_count, size_t D,
                       const size_t* hash_lens, int kind = 0, size_t out_len = 0);
int launch_fcs_dense(int dtype, const void* t, size_t order, const size_t* dims, size_t last_begin,
                     size_t last_count, size_t D, const uint32_t* packed, const size_t* hash_lens,
                     double* out, int accumulate, void* ws, size_t ws_bytes, cudaStream_t st,
                     size_t fam_stride = 0, int kind = 0, size_t out_len = 0);

}  // namespace fcs
