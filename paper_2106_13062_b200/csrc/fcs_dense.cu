// K1: dense fast count sketch — streaming scatter of vec(T) into
// bucket sum_n h_n(i_n) with sign prod_n s_n(i_n), D families per launch.
//
// Reference: fcs_sketch(const DenseTensor&, const HashFamily&),
// sketch.cpp:187-201, over the odometer walk for_each_nonzero,
// sketch.cpp:48-61 (zeros skipped). The reference sums serially in fp64;
// here each block privatises one family's sketch in shared memory, streams a
// contiguous range of mode-0 fibers (coalesced loads of the fastest mode),
// and the per-block partials are reduced in a fixed order in fp64
// (deterministic).
//
// Work decomposition: a "fiber" is one mode-0 column T[:, i_1, ..., i_{N-1}]
// (I_0 contiguous elements). Its offset c = sum_{n>=1} h_n(i_n) and sign
// sigma = prod_{n>=1} s_n(i_n) are warp-uniform, so the per-element work is
// one packed mode-0 table load, one add and one shared-memory accumulate.
#include <algorithm>

#include "common.cuh"

namespace fcs {

struct DenseArgs {
  int order;
  int D;
  uint32_t dims[ST_MAX_ORDER];
  uint32_t tab_off[ST_MAX_ORDER];  // start of mode n inside one family's tables
  uint32_t fam_stride;             // sum(dims): distance between families
  uint32_t jt;                     // composed length J~
  uint32_t last_begin;             // first i_{N-1} of this slab
  uint32_t i0_shift;               // mode-0 table shift (order-1 slabs only)
  uint64_t fibers;                 // mode-0 fibers in this slab
  uint64_t fibers_per_chunk;
};

// Offset and sign bit of fiber f (slab-local) for the family at `tab`.
__device__ __forceinline__ void fiber_offset(const DenseArgs& a, const uint32_t* __restrict__ tab,
                                             uint64_t f, uint32_t& c, uint32_t& sbit) {
  c = 0;
  sbit = 0;
  for (int n = 1; n < a.order; ++n) {
    uint64_t i;
    if (n < a.order - 1) {
      i = f % a.dims[n];
      f /= a.dims[n];
    } else {
      i = f + a.last_begin;
    }
    const uint32_t e = __ldg(tab + a.tab_off[n] + i);
    c += e & 0x7fffffffu;
    sbit ^= e & 0x80000000u;
  }
}

template <typename Tacc>
__device__ __forceinline__ Tacc signed_val(Tacc v, uint32_t sbit) {
  return sbit ? -v : v;
}

// Block-private shared-memory sketch of family d = blockIdx.x % D over the
// fiber chunk blockIdx.x / D; partial written to part[chunk][d][:].
template <typename Tin, typename Tacc>
__global__ void __launch_bounds__(1024) fcs_dense_smem_kernel(DenseArgs a,
                                                              const Tin* __restrict__ t,
                                                              const uint32_t* __restrict__ packed,
                                                              Tacc* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tacc* sk = reinterpret_cast<Tacc*>(smem_raw);
  const int d = blockIdx.x % a.D;
  const uint64_t chunk = blockIdx.x / a.D;
  const uint32_t* tab = packed + static_cast<uint64_t>(d) * a.fam_stride;
  const uint32_t* tab0 = tab + a.i0_shift;

  for (uint32_t b = threadIdx.x; b < a.jt; b += blockDim.x) sk[b] = Tacc(0);
  __syncthreads();

  const uint64_t f_begin = chunk * a.fibers_per_chunk;
  const uint64_t f_end = min(a.fibers, f_begin + a.fibers_per_chunk);
  const uint32_t i0n = a.dims[0];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;

  for (uint64_t f = f_begin + warp; f < f_end; f += nwarps) {
    uint32_t c, sbit;
    fiber_offset(a, tab, f, c, sbit);
    const Tin* fib = t + f * i0n;
    uint32_t i = lane;
    // 4 independent loads in flight per lane before the accumulates.
    for (; i + 96 < i0n; i += 128) {
      Tacc v[4];
      uint32_t e[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[k] = static_cast<Tacc>(__ldcs(fib + i + 32 * k));
        e[k] = __ldg(tab0 + i + 32 * k);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (v[k] != Tacc(0))
          atomicAdd(&sk[(e[k] & 0x7fffffffu) + c], signed_val(v[k], (e[k] ^ sbit) & 0x80000000u));
      }
    }
    for (; i < i0n; i += 32) {
      const Tacc v = static_cast<Tacc>(__ldcs(fib + i));
      const uint32_t e = __ldg(tab0 + i);
      if (v != Tacc(0))
        atomicAdd(&sk[(e & 0x7fffffffu) + c], signed_val(v, (e ^ sbit) & 0x80000000u));
    }
  }
  __syncthreads();
  Tacc* dst = part + (chunk * a.D + d) * static_cast<uint64_t>(a.jt);
  for (uint32_t b = threadIdx.x; b < a.jt; b += blockDim.x) dst[b] = sk[b];
}

// Fixed-order fp64 reduction of the chunk partials: out[d][b] (+)= sum_c part[c][d][b].
template <typename Tacc>
__global__ void reduce_partials_kernel(const Tacc* __restrict__ part, uint64_t nchunk,
                                       uint64_t per_chunk, double* __restrict__ out,
                                       int accumulate) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= per_chunk) return;
  double acc = accumulate ? out[i] : 0.0;
  for (uint64_t c = 0; c < nchunk; ++c) acc += static_cast<double>(part[c * per_chunk + i]);
  out[i] = acc;
}

// Fallback when one family's sketch does not fit in shared memory: fp64
// atomics straight into the (L2-resident) output. Correct for any J~.
template <typename Tin>
__global__ void fcs_dense_global_kernel(DenseArgs a, const Tin* __restrict__ t,
                                        const uint32_t* __restrict__ packed,
                                        double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t gwarp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t i0n = a.dims[0];
  for (uint64_t w = gwarp; w < a.fibers * a.D; w += nw) {
    const int d = static_cast<int>(w % a.D);
    const uint64_t f = w / a.D;
    const uint32_t* tab = packed + static_cast<uint64_t>(d) * a.fam_stride;
    uint32_t c, sbit;
    fiber_offset(a, tab, f, c, sbit);
    double* o = out + static_cast<uint64_t>(d) * a.jt;
    for (uint32_t i = lane; i < i0n; i += 32) {
      const double v = static_cast<double>(t[f * i0n + i]);
      const uint32_t e = __ldg(tab + a.i0_shift + i);
      if (v != 0.0) atomicAdd(&o[(e & 0x7fffffffu) + c], ((e ^ sbit) & 0x80000000u) ? -v : v);
    }
  }
}

namespace {

struct Plan {
  bool smem = false;
  size_t smem_bytes = 0;
  int threads = 0;
  uint64_t nchunk = 0;
  size_t ws = 0;
};

template <typename Tin, typename Tacc>
int make_plan(const DenseArgs& a, Plan* p) {
  DeviceInfo di;
  if (int rc = device_info(&di)) return rc;
  p->smem_bytes = static_cast<size_t>(a.jt) * sizeof(Tacc);
  if (p->smem_bytes > di.smem_optin) {
    p->smem = false;
    p->ws = 0;
    return ST_OK;
  }
  p->smem = true;
  auto kern = fcs_dense_smem_kernel<Tin, Tacc>;
  FCS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(p->smem_bytes)));
  // One 1024-thread block per SM when the sketch fills shared memory,
  // otherwise 512-thread blocks packed by occupancy.
  p->threads = p->smem_bytes > di.smem_optin / 2 ? 1024 : 512;
  int per_sm = 0;
  FCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, p->threads,
                                                             p->smem_bytes));
  per_sm = std::max(per_sm, 1);
  const uint64_t resident = static_cast<uint64_t>(per_sm) * di.sm_count;
  uint64_t nchunk = std::max<uint64_t>(1, resident / static_cast<uint64_t>(a.D));
  // Keep at least a few fibers per warp so table setup amortises.
  const uint64_t min_fibers = std::max<uint64_t>(1, static_cast<uint64_t>(p->threads / 32));
  nchunk = std::min<uint64_t>(nchunk, std::max<uint64_t>(1, a.fibers / min_fibers));
  p->nchunk = nchunk;
  p->ws = nchunk * a.D * static_cast<size_t>(a.jt) * sizeof(Tacc);
  return ST_OK;
}

int fill_args(size_t order, const size_t* dims, size_t last_begin, size_t last_count, size_t D,
              const size_t* hash_lens, DenseArgs* a) {
  FCS_CHECK_ARG(order >= 1 && order <= ST_MAX_ORDER, "fcs_sketch: unsupported tensor order");
  FCS_CHECK_ARG(D >= 1, "EstimatorConfig: hash_len and sketch_count must be >= 1");
  *a = DenseArgs{};
  a->order = static_cast<int>(order);
  a->D = static_cast<int>(D);
  uint64_t sum_dims = 0, sum_j = 0;
  for (size_t n = 0; n < order; ++n) {
    FCS_CHECK_ARG(dims[n] > 0 && hash_lens[n] > 0, "HashPair: dimensions must be positive");
    FCS_CHECK_ARG(dims[n] < (1u << 31) && hash_lens[n] < (1u << 30),
                  "fcs_sketch: dimension too large");
    a->dims[n] = static_cast<uint32_t>(dims[n]);
    a->tab_off[n] = static_cast<uint32_t>(sum_dims);
    sum_dims += dims[n];
    sum_j += hash_lens[n];
  }
  FCS_CHECK_ARG(sum_dims < (1ull << 32) && sum_j - order + 1 < (1ull << 31),
                "fcs_sketch: family too large");
  FCS_CHECK_ARG(last_begin + last_count <= dims[order - 1], "fcs_sketch: slab out of range");
  a->fam_stride = static_cast<uint32_t>(sum_dims);
  a->jt = static_cast<uint32_t>(sum_j - order + 1);
  a->last_begin = static_cast<uint32_t>(last_begin);
  uint64_t fibers = last_count;
  for (size_t n = 1; n + 1 < order; ++n) fibers *= dims[n];
  if (order == 1) fibers = last_count ? 1 : 0;  // a vector is one fiber
  a->fibers = fibers;
  if (order == 1) {
    a->dims[0] = static_cast<uint32_t>(last_count);
    a->i0_shift = static_cast<uint32_t>(last_begin);
    a->last_begin = 0;
  }
  return ST_OK;
}

template <typename Tin, typename Tacc>
int run_dense(DenseArgs a, const Tin* t, const uint32_t* packed, double* out, int accumulate,
              void* ws, size_t ws_bytes, cudaStream_t st) {
  const size_t out_elems = static_cast<size_t>(a.D) * a.jt;
  if (a.fibers == 0) {
    if (!accumulate) FCS_CUDA_TRY(cudaMemsetAsync(out, 0, out_elems * sizeof(double), st));
    return ST_OK;
  }
  Plan p;
  if (int rc = make_plan<Tin, Tacc>(a, &p)) return rc;
  if (!p.smem) {
    if (!accumulate) FCS_CUDA_TRY(cudaMemsetAsync(out, 0, out_elems * sizeof(double), st));
    DeviceInfo di;
    if (int rc = device_info(&di)) return rc;
    fcs_dense_global_kernel<Tin><<<di.sm_count * 4, 512, 0, st>>>(a, t, packed, out);
    FCS_CUDA_TRY(cudaGetLastError());
    return ST_OK;
  }
  FCS_CHECK_ARG(ws != nullptr && ws_bytes >= p.ws, "st_fcs_dense: workspace too small");
  a.fibers_per_chunk = (a.fibers + p.nchunk - 1) / p.nchunk;
  const uint64_t nchunk = (a.fibers + a.fibers_per_chunk - 1) / a.fibers_per_chunk;
  Tacc* part = static_cast<Tacc*>(ws);
  fcs_dense_smem_kernel<Tin, Tacc>
      <<<static_cast<unsigned>(nchunk * a.D), p.threads, p.smem_bytes, st>>>(a, t, packed, part);
  FCS_CUDA_TRY(cudaGetLastError());
  reduce_partials_kernel<Tacc><<<ceil_div(out_elems, 256), 256, 0, st>>>(part, nchunk, out_elems,
                                                                         out, accumulate);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace

size_t dense_workspace(int dtype, size_t order, const size_t* dims, size_t last_count, size_t D,
                       const size_t* hash_lens) {
  DenseArgs a;
  if (fill_args(order, dims, 0, last_count, D, hash_lens, &a) != ST_OK) return 0;
  Plan p;
  const int rc = dtype == ST_F32 ? make_plan<float, float>(a, &p) : make_plan<double, double>(a, &p);
  return rc == ST_OK ? p.ws : 0;
}

int launch_fcs_dense(int dtype, const void* t, size_t order, const size_t* dims, size_t last_begin,
                     size_t last_count, size_t D, const uint32_t* packed, const size_t* hash_lens,
                     double* out, int accumulate, void* ws, size_t ws_bytes, cudaStream_t st,
                     size_t fam_stride) {
  DenseArgs a;
  if (int rc = fill_args(order, dims, last_begin, last_count, D, hash_lens, &a)) return rc;
  if (fam_stride) a.fam_stride = static_cast<uint32_t>(fam_stride);
  if (dtype == ST_F32)
    return run_dense<float, float>(a, static_cast<const float*>(t), packed, out, accumulate, ws,
                                   ws_bytes, st);
  if (dtype == ST_F64)
    return run_dense<double, double>(a, static_cast<const double*>(t), packed, out, accumulate, ws,
                                     ws_bytes, st);
  return fail(ST_EINVAL, "st_fcs_dense: unknown dtype");
}

}  // namespace fcs
