// Sparse-input FCS (north_star (1) "dense/sparse-tensor FCS"
// gives FCS of a tensor in O(nnz(T))). The reference has no sparse type: its
// dense path visits every entry and skips the zeros (for_each_nonzero,
// sketch.cpp:48-61), and each nonzero lands in the composed bucket of its
// multi-index (HashFamily::compose, hashing.cpp:83-98). Here the input is a
// COO list — values[k] at coords[k * order + n] — and the work is
// proportional to nnz: one thread per nonzero, the D families' tables staged
// in shared memory, and one native fp64 global reduction (RED.E.ADD.F64) per
// (nonzero, family) into the L2-resident D x J~ output. Duplicate
// coordinates add up (the sketch of the densified sum, by linearity);
// out-of-range coordinates are skipped and counted (the caller raises
// compose's "index out of range").
#include "dense_common.cuh"

namespace fcs {
namespace {

template <typename T>
__global__ void __launch_bounds__(256) fcs_coo_kernel(const T* __restrict__ values,
                                                      const uint32_t* __restrict__ coords,
                                                      uint64_t nnz, int order, int D,
                                                      CooArgs a, const uint32_t* __restrict__ packed,
                                                      double* __restrict__ out,
                                                      unsigned long long* __restrict__ invalid,
                                                      int smem_tables) {
  extern __shared__ uint32_t stab[];
  const uint32_t* tab = packed;
  if (smem_tables) {
    const uint32_t n = static_cast<uint32_t>(D) * a.fam_stride;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) stab[i] = __ldg(packed + i);
    __syncthreads();
    tab = stab;
  }
  unsigned long long bad = 0;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double v = static_cast<double>(values[k]);
    uint32_t idx[ST_MAX_ORDER];
    bool ok = true;
#pragma unroll
    for (int n = 0; n < ST_MAX_ORDER; ++n) {
      if (n < order) {
        idx[n] = __ldg(coords + k * order + n);
        ok = ok && idx[n] < a.dims[n];
      }
    }
    if (!ok) {
      ++bad;
      continue;
    }
    if (v == 0.0) continue;  // for_each_nonzero skips exact zeros
    for (int d = 0; d < D; ++d) {
      const uint32_t* t = tab + static_cast<uint64_t>(d) * a.fam_stride;
      uint32_t bucket = 0, sbit = 0;
#pragma unroll
      for (int n = 0; n < ST_MAX_ORDER; ++n) {
        if (n < order) {
          const uint32_t e = t[a.tab_off[n] + idx[n]];
          bucket += e & 0x7fffffffu;
          sbit ^= e & 0x80000000u;
        }
      }
      atomicAdd(out + static_cast<uint64_t>(d) * a.jt + bucket, sbit ? -v : v);
    }
  }
  if (invalid && bad) atomicAdd(invalid, bad);
}

}  // namespace

int launch_fcs_coo(int dtype, const void* values, const uint32_t* coords, size_t nnz, size_t order,
                   const size_t* dims, size_t D, const uint32_t* packed, const size_t* hash_lens,
                   double* out, int accumulate, unsigned long long* invalid, cudaStream_t st) {
  FCS_CHECK_ARG(dtype == ST_F32 || dtype == ST_F64, "st_fcs_coo: unknown dtype");
  FCS_CHECK_ARG(order >= 1 && order <= ST_MAX_ORDER, "fcs_sketch: unsupported tensor order");
  FCS_CHECK_ARG(D >= 1, "EstimatorConfig: hash_len and sketch_count must be >= 1");
  CooArgs a{};
  uint64_t sum_dims = 0, sum_j = 0;
  for (size_t n = 0; n < order; ++n) {
    FCS_CHECK_ARG(dims[n] > 0 && hash_lens[n] > 0, "HashPair: dimensions must be positive");
    FCS_CHECK_ARG(dims[n] < (1ull << 32), "fcs_sketch: dimension too large");
    a.dims[n] = static_cast<uint32_t>(dims[n]);
    a.tab_off[n] = static_cast<uint32_t>(sum_dims);
    sum_dims += dims[n];
    sum_j += hash_lens[n];
  }
  FCS_CHECK_ARG(sum_dims < (1ull << 32) && sum_j - order + 1 < (1ull << 31),
                "fcs_sketch: family too large");
  a.fam_stride = static_cast<uint32_t>(sum_dims);
  a.jt = static_cast<uint32_t>(sum_j - order + 1);
  const size_t out_elems = D * a.jt;
  if (!accumulate) FCS_CUDA_TRY(cudaMemsetAsync(out, 0, out_elems * sizeof(double), st));
  if (nnz == 0) return ST_OK;
  DeviceInfo di;
  if (int rc = device_info(&di)) return rc;
  const size_t tab_bytes = D * sum_dims * sizeof(uint32_t);
  const int smem_tables = tab_bytes <= 96 * 1024 ? 1 : 0;
  const size_t smem = smem_tables ? tab_bytes : 0;
  const unsigned grid = static_cast<unsigned>(
      std::min<uint64_t>((nnz + 255) / 256, static_cast<uint64_t>(di.sm_count) * 8));
  if (dtype == ST_F32) {
    if (smem > 48 * 1024)
      FCS_CUDA_TRY(cudaFuncSetAttribute(fcs_coo_kernel<float>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    fcs_coo_kernel<float><<<grid, 256, smem, st>>>(static_cast<const float*>(values), coords, nnz,
                                                   static_cast<int>(order), static_cast<int>(D),
                                                   a, packed, out, invalid, smem_tables);
  } else {
    if (smem > 48 * 1024)
      FCS_CUDA_TRY(cudaFuncSetAttribute(fcs_coo_kernel<double>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    fcs_coo_kernel<double><<<grid, 256, smem, st>>>(static_cast<const double*>(values), coords,
                                                    nnz, static_cast<int>(order),
                                                    static_cast<int>(D), a, packed, out, invalid,
                                                    smem_tables);
  }
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace fcs

using namespace fcs;

extern "C" int st_fcs_coo(int dtype, const void* values, const uint32_t* coords, size_t nnz,
                          size_t order, const size_t* dims, size_t sketch_count,
                          const uint32_t* packed, const size_t* hash_lens, double* out,
                          int accumulate, unsigned long long* invalid, void* stream) {
  return launch_fcs_coo(dtype, values, coords, nnz, order, dims, sketch_count, packed, hash_lens,
                        out, accumulate, invalid, static_cast<cudaStream_t>(stream));
}
