// Tensor sketch (TS) and higher-order count sketch (HCS) entry points, the
// adjacent rows of the FCS API.
//
//  * TS dense (sketch.cpp:135-149) buckets by (sum_n h_n) mod J: it is the
//    J-periodic fold of the FCS of the same tensor, so it reuses K1 and adds
//    a fold. TS of a CP tensor (sketch.cpp:151-155) is the circular
//    convolution at length J of the factor count sketches = the fold of their
//    linear convolution, i.e. of the CP-form FCS (K2-K5).
//  * HCS dense (sketch.cpp:157-173) is K1 with mixed-radix bucket
//    sum_n h_n * prod_{m<n} J_m into a J_0 x ... x J_{N-1} tensor
//    (DenseArgs::mult). HCS of a CP tensor (sketch.cpp:175-185) is
//    densify(CpTensor(w, {CS_n(U^(n))})): count sketch of every factor column,
//    then a weighted sum of outer products.
#include <algorithm>

#include "common.cuh"

namespace fcs {


namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// out[d][b] (+)= sum_{q >= 0, b + qJ < jt} in[d][b + qJ]
__global__ void fold_kernel(const double* __restrict__ in, int D, uint32_t jt, uint32_t J,
                            double* __restrict__ out, int accumulate) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<uint64_t>(D) * J) return;
  const uint64_t d = i / J;
  const uint32_t b = static_cast<uint32_t>(i - d * J);
  double acc = accumulate ? out[i] : 0.0;
  for (uint32_t k = b; k < jt; k += J) acc += in[d * jt + k];
  out[i] = acc;
}

// Per (family d, mode n) count sketch of the R factor columns:
// cs[d][n] is J_n x R column-major at offset cs_off[n] within family d's block.
struct HcsCpArgs {
  int order;
  int rank;
  int dims[ST_MAX_ORDER];
  int J[ST_MAX_ORDER];
  int tab_off[ST_MAX_ORDER];
  int cs_off[ST_MAX_ORDER];
  int fam_stride;
  int cs_stride;  // doubles per family block
  const double* factors[ST_MAX_ORDER];
  const double* weights;
  uint64_t out_len;  // prod J_n
};

__global__ void hcs_cs_kernel(HcsCpArgs a, const uint32_t* __restrict__ packed, double* cs) {
  const int d = blockIdx.y;
  const uint32_t* tab = packed + static_cast<size_t>(d) * a.fam_stride;
  double* blk = cs + static_cast<size_t>(d) * a.cs_stride;
  for (int n = 0; n < a.order; ++n) {
    const size_t cnt = static_cast<size_t>(a.dims[n]) * a.rank;
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < cnt;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
      const int i = static_cast<int>(k % a.dims[n]);
      const int r = static_cast<int>(k / a.dims[n]);
      const double v = a.factors[n][k];  // I_n x R column-major
      if (v == 0.0) continue;            // cs_sketch_columns skips zeros (sketch.cpp:128)
      const uint32_t e = __ldg(tab + a.tab_off[n] + i);
      atomicAdd(blk + a.cs_off[n] + static_cast<size_t>(r) * a.J[n] + (e & 0x7fffffffu),
                (e >> 31) ? -v : v);
    }
  }
}

// out[d][j] (+)= sum_{r: w_r != 0} w_r prod_n cs_n[d][j_n, r] (densify, tensor.cpp:86-115)
__global__ void hcs_outer_kernel(HcsCpArgs a, const double* __restrict__ cs, int D,
                                 double* __restrict__ out, int accumulate) {
  const uint64_t total = static_cast<uint64_t>(D) * a.out_len;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t d = i / a.out_len;
    uint64_t rem = i - d * a.out_len;
    int jn[ST_MAX_ORDER];
    for (int n = 0; n < a.order; ++n) {
      jn[n] = static_cast<int>(rem % a.J[n]);
      rem /= a.J[n];
    }
    const double* blk = cs + d * a.cs_stride;
    double acc = 0.0;
    for (int r = 0; r < a.rank; ++r) {
      const double w = a.weights[r];
      if (w == 0.0) continue;
      double p = w;
      for (int n = 0; n < a.order; ++n) p *= blk[a.cs_off[n] + static_cast<size_t>(r) * a.J[n] + jn[n]];
      acc += p;
    }
    out[i] = accumulate ? out[i] + acc : acc;
  }
}

int check_equal_lens(size_t order, const size_t* hash_lens) {
  for (size_t n = 1; n < order; ++n)
    FCS_CHECK_ARG(hash_lens[n] == hash_lens[0], "ts_sketch: all hash lengths must be equal");
  return ST_OK;
}

size_t composed(size_t order, const size_t* hash_lens) {
  size_t s = 0;
  for (size_t n = 0; n < order; ++n) s += hash_lens[n];
  return s - order + 1;
}

}  // namespace

// out[d][b] = sum_q in[d][b + qJ] (TS = FCS mod J), for codecs.cu.
int st_ts_fold(const double* in, int D, uint32_t jt, uint32_t J, double* out, cudaStream_t st) {
  fold_kernel<<<ceil_div(static_cast<size_t>(D) * J, 256), 256, 0, st>>>(in, D, jt, J, out, 0);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace fcs

using namespace fcs;

extern "C" {

size_t st_ts_dense_workspace(int dtype, size_t order, const size_t* dims, size_t last_count,
                             size_t sketch_count, const size_t* hash_lens) {
  return align_up(dense_workspace(dtype, order, dims, last_count, sketch_count, hash_lens, 0)) +
         sketch_count * composed(order, hash_lens) * sizeof(double);
}

int st_ts_dense(int dtype, const void* tensor, size_t order, const size_t* dims, size_t last_begin,
                size_t last_count, size_t sketch_count, const uint32_t* packed,
                const size_t* hash_lens, double* out, int accumulate, void* workspace,
                size_t workspace_bytes, void* stream) {
  FCS_CHECK_ARG(order >= 1 && order <= ST_MAX_ORDER, "ts_sketch: unsupported tensor order");
  if (int rc = check_equal_lens(order, hash_lens)) return rc;
  const size_t need = st_ts_dense_workspace(dtype, order, dims, last_count, sketch_count, hash_lens);
  FCS_CHECK_ARG(workspace && workspace_bytes >= need, "st_ts_dense: workspace too small");
  const size_t dws = dense_workspace(dtype, order, dims, last_count, sketch_count, hash_lens, 0);
  double* fcs = reinterpret_cast<double*>(static_cast<char*>(workspace) + align_up(dws));
  cudaStream_t st = as_stream(stream);
  if (int rc = launch_fcs_dense(dtype, tensor, order, dims, last_begin, last_count, sketch_count,
                                packed, hash_lens, fcs, 0, workspace, dws, st))
    return rc;
  const size_t jt = composed(order, hash_lens), J = hash_lens[0];
  fold_kernel<<<ceil_div(sketch_count * J, 256), 256, 0, st>>>(
      fcs, static_cast<int>(sketch_count), static_cast<uint32_t>(jt), static_cast<uint32_t>(J), out,
      accumulate);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

size_t st_fcs_cp_workspace(size_t, const size_t*, size_t, size_t, const size_t*);
int st_fcs_cp(const double*, size_t, size_t, const size_t*, const double* const*, size_t, size_t,
              size_t, const uint32_t*, const size_t*, double*, int, void*, size_t, void*);

size_t st_ts_cp_workspace(size_t order, const size_t* dims, size_t rank, size_t sketch_count,
                          const size_t* hash_lens) {
  const size_t cw = st_fcs_cp_workspace(order, dims, rank, sketch_count, hash_lens);
  if (cw == 0) return 0;
  return align_up(cw) + sketch_count * composed(order, hash_lens) * sizeof(double);
}

int st_ts_cp(const double* weights, size_t rank, size_t order, const size_t* dims,
             const double* const* factors, size_t r_begin, size_t r_count, size_t sketch_count,
             const uint32_t* packed, const size_t* hash_lens, double* out, int accumulate,
             void* workspace, size_t workspace_bytes, void* stream) {
  FCS_CHECK_ARG(order >= 1 && order <= ST_MAX_ORDER, "ts_sketch: unsupported tensor order");
  if (int rc = check_equal_lens(order, hash_lens)) return rc;
  const size_t cw = st_fcs_cp_workspace(order, dims, rank, sketch_count, hash_lens);
  FCS_CHECK_ARG(cw > 0, "ts_sketch: composed length exceeds the shared-memory FFT");
  const size_t need = align_up(cw) + sketch_count * composed(order, hash_lens) * sizeof(double);
  FCS_CHECK_ARG(workspace && workspace_bytes >= need, "st_ts_cp: workspace too small");
  double* fcs = reinterpret_cast<double*>(static_cast<char*>(workspace) + align_up(cw));
  if (int rc = st_fcs_cp(weights, rank, order, dims, factors, r_begin, r_count, sketch_count,
                         packed, hash_lens, fcs, 0, workspace, cw, stream))
    return rc;
  const size_t jt = composed(order, hash_lens), J = hash_lens[0];
  fold_kernel<<<ceil_div(sketch_count * J, 256), 256, 0, as_stream(stream)>>>(
      fcs, static_cast<int>(sketch_count), static_cast<uint32_t>(jt), static_cast<uint32_t>(J), out,
      accumulate);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

size_t st_hcs_dense_workspace(int dtype, size_t order, const size_t* dims, size_t last_count,
                              size_t sketch_count, const size_t* hash_lens) {
  return dense_workspace(dtype, order, dims, last_count, sketch_count, hash_lens, 1);
}

int st_hcs_dense(int dtype, const void* tensor, size_t order, const size_t* dims,
                 size_t last_begin, size_t last_count, size_t sketch_count, const uint32_t* packed,
                 const size_t* hash_lens, double* out, int accumulate, void* workspace,
                 size_t workspace_bytes, void* stream) {
  return launch_fcs_dense(dtype, tensor, order, dims, last_begin, last_count, sketch_count, packed,
                          hash_lens, out, accumulate, workspace, workspace_bytes,
                          as_stream(stream), 0, 1);
}

size_t st_hcs_cp_workspace(size_t order, const size_t* dims, size_t rank, size_t sketch_count,
                           const size_t* hash_lens) {
  (void)dims;
  size_t sj = 0;
  for (size_t n = 0; n < order; ++n) sj += hash_lens[n];
  return std::max<size_t>(1, sketch_count * sj * std::max<size_t>(rank, 1) * sizeof(double));
}

int st_hcs_cp(const double* weights, size_t rank, size_t order, const size_t* dims,
              const double* const* factors, size_t sketch_count, const uint32_t* packed,
              const size_t* hash_lens, double* out, int accumulate, void* workspace,
              size_t workspace_bytes, void* stream) {
  FCS_CHECK_ARG(order >= 1 && order <= ST_MAX_ORDER, "CpTensor: no factors");
  FCS_CHECK_ARG(sketch_count >= 1, "EstimatorConfig: hash_len and sketch_count must be >= 1");
  HcsCpArgs a{};
  a.order = static_cast<int>(order);
  a.rank = static_cast<int>(rank);
  a.weights = weights;
  size_t off = 0, csoff = 0;
  uint64_t prod = 1;
  for (size_t n = 0; n < order; ++n) {
    FCS_CHECK_ARG(dims[n] > 0 && hash_lens[n] > 0, "HashPair: dimensions must be positive");
    a.dims[n] = static_cast<int>(dims[n]);
    a.J[n] = static_cast<int>(hash_lens[n]);
    a.tab_off[n] = static_cast<int>(off);
    a.cs_off[n] = static_cast<int>(csoff);
    a.factors[n] = factors[n];
    off += dims[n];
    csoff += hash_lens[n] * rank;
    prod *= hash_lens[n];
  }
  FCS_CHECK_ARG(prod < (1ull << 40), "hcs_sketch: sketch tensor too large");
  a.fam_stride = static_cast<int>(off);
  a.cs_stride = static_cast<int>(csoff);
  a.out_len = prod;
  const size_t need = st_hcs_cp_workspace(order, dims, rank, sketch_count, hash_lens);
  FCS_CHECK_ARG(workspace && workspace_bytes >= need, "st_hcs_cp: workspace too small");
  cudaStream_t st = as_stream(stream);
  double* cs = static_cast<double*>(workspace);
  FCS_CUDA_TRY(cudaMemsetAsync(cs, 0, sketch_count * csoff * sizeof(double), st));
  if (rank > 0) {
    hcs_cs_kernel<<<dim3(64, static_cast<unsigned>(sketch_count)), 256, 0, st>>>(a, packed, cs);
    FCS_CUDA_TRY(cudaGetLastError());
  }
  const uint64_t total = sketch_count * prod;
  hcs_outer_kernel<<<static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 148 * 16)), 256,
                     0, st>>>(a, cs, static_cast<int>(sketch_count), out, accumulate);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // extern "C"
