// K0: counter-based hash-table tabulation and synthetic data generation.
//
// HashPair (hashing.cpp:10-22) draws, for each index i in turn, the bucket
// from draw 2i+1 (Lemire mulhi reduction, rng.hpp:25-28) and the sign from the
// top bit of draw 2i+2. SplitMix64 is a counter generator (rng.hpp:16-21):
// draw k = fmix64(seed + k*GAMMA), so index i is computed independently by
// one thread, bit-exact with the serial stream.
#include "common.cuh"

namespace fcs {

__global__ void hash_tabulate_kernel(uint64_t seed, uint32_t n, uint64_t hash_len,
                                     uint32_t* __restrict__ bucket, int8_t* __restrict__ sign) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = 2ull * i;
  bucket[i] = static_cast<uint32_t>(mulhi64(splitmix_draw(seed, k + 1), hash_len));
  sign[i] = (splitmix_draw(seed, k + 2) >> 63) ? int8_t(-1) : int8_t(1);
}

// One family (all modes) into packed tables: mode n seeded master ^ n
// (hashing.cpp:50-53).
struct FamilyArgs {
  uint64_t master;
  int order;
  uint32_t offs[ST_MAX_ORDER + 1];
  uint64_t hash_len[ST_MAX_ORDER];
};

__global__ void family_tables_kernel(FamilyArgs a, uint32_t* __restrict__ packed) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.offs[a.order]) return;
  int n = 0;
  while (t >= a.offs[n + 1]) ++n;
  const uint64_t i = t - a.offs[n];
  const uint64_t seed = a.master ^ static_cast<uint64_t>(n);
  const uint32_t b = static_cast<uint32_t>(mulhi64(splitmix_draw(seed, 2 * i + 1), a.hash_len[n]));
  const bool neg = (splitmix_draw(seed, 2 * i + 2) >> 63) != 0;
  packed[t] = b | (neg ? 0x80000000u : 0u);
}

__global__ void pack_tables_kernel(uint64_t total, const uint32_t* __restrict__ bucket,
                                   const int8_t* __restrict__ sign, uint32_t* __restrict__ packed) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < total) packed[i] = pack_entry(bucket[i], sign[i]);
}

// Box-Muller on draws (2p+1, 2p+2) -> elements (2p, 2p+1): the same mapping
// as next_gaussian (rng.cpp:8-21), with CUDA libm.
template <typename T>
__global__ void device_gaussian_kernel(uint64_t seed, uint64_t n, T* __restrict__ out) {
  const uint64_t pairs = (n + 1) / 2;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < pairs;
       p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t d1 = splitmix_draw(seed, 2 * p + 1);
    const uint64_t d2 = splitmix_draw(seed, 2 * p + 2);
    const double u1 = static_cast<double>((d1 >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(d2 >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    double s, c;
    sincospi(2.0 * u2, &s, &c);
    out[2 * p] = static_cast<T>(r * c);
    if (2 * p + 1 < n) out[2 * p + 1] = static_cast<T>(r * s);
  }
}

int launch_hash_tabulate(uint64_t seed, size_t n, size_t hash_len, uint32_t* bucket,
                         int8_t* sign, cudaStream_t st) {
  if (n == 0) return ST_OK;
  hash_tabulate_kernel<<<ceil_div(n, 256), 256, 0, st>>>(seed, static_cast<uint32_t>(n),
                                                        hash_len, bucket, sign);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_family_tables(size_t order, const size_t* dims, const size_t* hash_lens, size_t D,
                         const uint64_t* seeds, uint32_t* packed, cudaStream_t st) {
  FamilyArgs a{};
  a.order = static_cast<int>(order);
  a.offs[0] = 0;
  for (size_t n = 0; n < order; ++n) {
    a.offs[n + 1] = a.offs[n] + static_cast<uint32_t>(dims[n]);
    a.hash_len[n] = hash_lens[n];
  }
  const uint32_t per = a.offs[order];
  for (size_t d = 0; d < D; ++d) {
    a.master = seeds[d];
    family_tables_kernel<<<ceil_div(per, 256), 256, 0, st>>>(a, packed + d * per);
  }
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_pack_tables(size_t total, const uint32_t* bucket, const int8_t* sign, uint32_t* packed,
                       cudaStream_t st) {
  if (total == 0) return ST_OK;
  pack_tables_kernel<<<ceil_div(total, 256), 256, 0, st>>>(total, bucket, sign, packed);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int launch_device_gaussian(int dtype, uint64_t seed, size_t n, void* out, cudaStream_t st) {
  if (n == 0) return ST_OK;
  DeviceInfo di;
  if (int rc = device_info(&di)) return rc;
  const unsigned blocks = static_cast<unsigned>(di.sm_count) * 8;
  if (dtype == ST_F32)
    device_gaussian_kernel<float><<<blocks, 256, 0, st>>>(seed, n, static_cast<float*>(out));
  else
    device_gaussian_kernel<double><<<blocks, 256, 0, st>>>(seed, n, static_cast<double*>(out));
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace fcs
