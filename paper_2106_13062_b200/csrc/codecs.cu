// Sketch-domain codecs and estimates around the FCS path (SURVEY.md §8(f)
// ranks 3-4; the reference specifies them in SPEC.md:371-435 and PAPER.md
// §4.2-4.3 but does not implement them, so the spec is the contract):
//  * st_estimate_inner       — estimate_inner / inner_once (estimators.cpp:193-207),
//                              inner_once_ts (estimators.cpp:235-239),
//  * st_regression_forward   — Y = median_d FCS_d(X rows) FCS_d(W rows)^T + b
//                              (Eq. 20),
//  * st_fcs_contraction      — FCS(A (x)_{3,1} B) = sum_l FCS(A(:,:,l)) * FCS(B(l,:,:))
//                              (§4.3.2); L = 1 is compress_kron,
//  * st_sketch_decompress    — median_d s(i) FCS_d[sum_n h_n(i_n)],
//  * st_kron_decompress_all  — the full (I1 I3) x (I2 I4) reconstruction.
//
// Row-batched sketches: a batch of R tensors that share one family is one K1
// launch over an order-(N+1) tensor whose batch mode's table holds r * len
// (sign +): each row's composed buckets land in its own len-slot segment.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "engine.cuh"

namespace fcs {

int st_ts_fold(const double* in, int D, uint32_t jt, uint32_t J, double* out, cudaStream_t st);

namespace {

struct Dims4 {
  uint32_t d[4];
};

// out[d] = [base tables of the hashed modes | r * row_len for the batch mode]
// (batch_first: the batch mode is mode 0, else the last mode).
__global__ void batch_tables_kernel(const uint32_t* __restrict__ base, uint32_t base_stride,
                                    uint32_t base_len, int D, uint32_t rows, uint32_t row_len,
                                    int batch_first, uint32_t* __restrict__ out) {
  const uint32_t stride = base_len + rows;
  const size_t n = static_cast<size_t>(D) * stride;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t d = i / stride;
    const uint32_t k = static_cast<uint32_t>(i - d * stride);
    uint32_t v;
    if (batch_first)
      v = k < rows ? k * row_len : __ldg(base + d * base_stride + (k - rows));
    else
      v = k < base_len ? __ldg(base + d * base_stride + k) : (k - base_len) * row_len;
    out[i] = v;
  }
}

// est[d] = <a_d, b_d> in a fixed order (one CTA per family).
__global__ void dots_kernel(const double* __restrict__ a, const double* __restrict__ b, int len,
                            double* __restrict__ est) {
  __shared__ double red[32];
  const size_t off = static_cast<size_t>(blockIdx.x) * len;
  double acc = 0.0;
  for (int k = threadIdx.x; k < len; k += blockDim.x) acc += a[off + k] * b[off + k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) est[blockIdx.x] = t;
  }
}

// est[b][d][c] = <SX_d[b], SW_d[c]> over the J~ sketch coordinates: a 16 x 16
// output tile per CTA, 32-wide k panels staged in shared memory.
constexpr int kTile = 16, kPanel = 32;
__global__ void sketch_gemm_kernel(const double* __restrict__ SX, const double* __restrict__ SW,
                                   int B, int Cn, int D, int len, double* __restrict__ est) {
  __shared__ double xs[kTile][kPanel + 1];
  __shared__ double ws[kTile][kPanel + 1];
  const int d = blockIdx.z;
  const int b0 = blockIdx.y * kTile, c0 = blockIdx.x * kTile;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 16 x 16
  const double* X = SX + static_cast<size_t>(d) * B * len;
  const double* W = SW + static_cast<size_t>(d) * Cn * len;
  double acc = 0.0;
  for (int k0 = 0; k0 < len; k0 += kPanel) {
    for (int q = ty * kTile + tx; q < kTile * kPanel; q += kTile * kTile) {
      const int r = q / kPanel, k = q % kPanel;
      xs[r][k] = (b0 + r < B && k0 + k < len) ? X[static_cast<size_t>(b0 + r) * len + k0 + k] : 0.0;
      ws[r][k] = (c0 + r < Cn && k0 + k < len) ? W[static_cast<size_t>(c0 + r) * len + k0 + k] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < kPanel; ++k) acc += xs[ty][k] * ws[tx][k];
    __syncthreads();
  }
  const int b = b0 + ty, c = c0 + tx;
  if (b < B && c < Cn) est[(static_cast<size_t>(b) * D + d) * Cn + c] = acc;
}

__global__ void add_bias_kernel(double* __restrict__ y, const double* __restrict__ bias, int B,
                                int Cn) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < B * Cn) y[i] += bias[i % Cn];
}

// acc[d][s] = sum_l FA[d][l][s] * FB[d][l][s] (packed half spectra, fixed order).
__global__ void pair_product_sum_kernel(const double2* __restrict__ FA,
                                        const double2* __restrict__ FB, int L, int P,
                                        double2* __restrict__ acc) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int d = blockIdx.y;
  if (s >= P) return;
  double2 a = make_double2(0.0, 0.0);
  const size_t base = static_cast<size_t>(d) * L * P + s;
  for (int l = 0; l < L; ++l) {
    const size_t o = base + static_cast<size_t>(l) * P;
    a = cadd(a, hmul(FA[o], FB[o], s == 0));
  }
  acc[static_cast<size_t>(d) * P + s] = a;
}

// out[q] = median_d prod_n s_n(i_n) * sk_d[(sum_n h_n(i_n)) mod len]; the
// multi-index of query q comes from idx (count x order) or, for the Kronecker
// reconstruction (idx == nullptr), from the column-major (I1 I3) x (I2 I4)
// position: row = I3 i1 + i3, col = I4 i2 + i4.
__global__ void decompress_kernel(const double* __restrict__ sk, int D, uint32_t len,
                                  const uint32_t* __restrict__ packed, uint32_t fam_stride,
                                  int order, Dims4 dims, size_t count,
                                  const uint32_t* __restrict__ idx, double* __restrict__ out) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < count;
       q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    uint32_t ii[ST_MAX_ORDER];
    if (idx) {
      for (int n = 0; n < order; ++n) ii[n] = idx[q * order + n];
    } else {
      const uint64_t rows = static_cast<uint64_t>(dims.d[0]) * dims.d[2];
      const uint64_t row = q % rows, col = q / rows;
      ii[0] = static_cast<uint32_t>(row / dims.d[2]);
      ii[2] = static_cast<uint32_t>(row % dims.d[2]);
      ii[1] = static_cast<uint32_t>(col / dims.d[3]);
      ii[3] = static_cast<uint32_t>(col % dims.d[3]);
    }
    double v[64];
    for (int d = 0; d < D; ++d) {
      const uint32_t* tab = packed + static_cast<size_t>(d) * fam_stride;
      uint64_t h = 0;
      uint32_t sbit = 0, off = 0;
      for (int n = 0; n < order; ++n) {
        const uint32_t e = __ldg(tab + off + ii[n]);
        h += e & 0x7fffffffu;
        sbit ^= e & 0x80000000u;
        off += dims.d[n];
      }
      const double z = __ldg(sk + static_cast<size_t>(d) * len + h % len);
      const double x = sbit ? -z : z;
      int k = d;  // insertion into the sorted prefix (median_reduce, estimators.cpp:117-138)
      while (k > 0 && v[k - 1] > x) {
        v[k] = v[k - 1];
        --k;
      }
      v[k] = x;
    }
    out[q] = (D & 1) ? v[D / 2] : 0.5 * (v[D / 2 - 1] + v[D / 2]);
  }
}

struct DevMem {
  std::vector<void*> ptrs;
  cudaStream_t st;
  explicit DevMem(cudaStream_t s) : st(s) {}
  ~DevMem() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
  template <typename T>
  int alloc(T** p, size_t n) {
    *p = nullptr;
    void* q = nullptr;
    FCS_CUDA_TRY(malloc_async(&q, std::max<size_t>(1, n * sizeof(T)), st));
    ptrs.push_back(q);
    *p = static_cast<T*>(q);
    return ST_OK;
  }
};

int batch_tables(const uint32_t* base, size_t base_stride, size_t base_len, size_t D, size_t rows,
                 size_t row_len, bool batch_first, uint32_t* out, cudaStream_t st) {
  const size_t n = D * (base_len + rows);
  batch_tables_kernel<<<std::min<unsigned>(ceil_div(n, 256), 4096), 256, 0, st>>>(
      base, static_cast<uint32_t>(base_stride), static_cast<uint32_t>(base_len),
      static_cast<int>(D), static_cast<uint32_t>(rows), static_cast<uint32_t>(row_len),
      batch_first ? 1 : 0, out);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

// K1 over `rows` order-N tensors sharing each family: out[d][r][0..row_len).
int rows_sketch(int dtype, const void* x, size_t order, const size_t* dims, size_t rows,
                size_t row_len, size_t D, const uint32_t* base, size_t base_stride,
                size_t base_off, DevMem& mem, double* out, cudaStream_t st) {
  size_t sum_dims = 0;
  for (size_t n = 0; n < order; ++n) sum_dims += dims[n];
  uint32_t* tabs;
  if (int rc = mem.alloc(&tabs, D * (sum_dims + rows))) return rc;
  if (int rc = batch_tables(base + base_off, base_stride, sum_dims, D, rows, row_len, false,
                            tabs, st))
    return rc;
  size_t bd[ST_MAX_ORDER + 1], bl[ST_MAX_ORDER + 1];
  for (size_t n = 0; n < order; ++n) {
    bd[n] = dims[n];
    bl[n] = 1;  // only the output length matters (out_len below)
  }
  bd[order] = rows;
  bl[order] = 1;
  const size_t out_len = rows * row_len;
  const size_t wsb = dense_workspace(dtype, order + 1, bd, rows, D, bl, 0, out_len);
  char* ws;
  if (int rc = mem.alloc(&ws, wsb)) return rc;
  return launch_fcs_dense(dtype, x, order + 1, bd, 0, rows, D, tabs, bl, out, 0, ws, wsb, st, 0, 0,
                          out_len);
}

std::vector<uint64_t> family_seeds(uint64_t seed, size_t D) {
  std::vector<uint64_t> s(D);
  for (size_t d = 0; d < D; ++d) s[d] = splitmix_draw(seed + static_cast<uint64_t>(d), 1);
  return s;  // families_for (estimators.cpp:104-115)
}

}  // namespace
}  // namespace fcs

using namespace fcs;

extern "C" {

int st_estimate_inner(int kind, int dtype, const void* a, const void* b, size_t order,
                      const size_t* dims, size_t hash_len, size_t sketch_count, uint64_t seed,
                      double* estimates, double* out, void* stream) {
  FCS_CHECK_ARG(kind == ST_SKETCH_FCS || kind == ST_SKETCH_TS, "estimate_inner: unknown sketch");
  FCS_CHECK_ARG(dtype == ST_F32 || dtype == ST_F64, "estimate_inner: unknown dtype");
  FCS_CHECK_ARG(order >= 1 && order <= ST_MAX_ORDER, "fcs_sketch: unsupported tensor order");
  FCS_CHECK_ARG(hash_len > 0 && sketch_count > 0,
                "EstimatorConfig: hash_len and sketch_count must be >= 1");
  FCS_CHECK_ARG(sketch_count >= 1, "median_reduce: empty input");
  size_t sum_dims = 0;
  for (size_t n = 0; n < order; ++n) {
    FCS_CHECK_ARG(dims[n] > 0, "HashPair: dimensions must be positive");
    sum_dims += dims[n];
  }
  cudaStream_t st = as_stream(stream);
  DevMem mem(st);
  const size_t D = sketch_count;
  std::vector<size_t> hl(order, hash_len);
  const size_t jt = order * hash_len - order + 1;
  const size_t len = kind == ST_SKETCH_TS ? hash_len : jt;
  uint32_t* packed;
  double *sa, *sb, *est, *med;
  if (int rc = mem.alloc(&packed, D * sum_dims)) return rc;
  if (int rc = mem.alloc(&sa, 2 * D * jt)) return rc;
  if (int rc = mem.alloc(&est, D + 1)) return rc;
  sb = sa + D * jt;
  med = est + D;
  const std::vector<uint64_t> seeds = family_seeds(seed, D);
  if (int rc = launch_family_tables(order, dims, hl.data(), D, seeds.data(), packed, st)) return rc;
  const size_t wsb = dense_workspace(dtype, order, dims, dims[order - 1], D, hl.data());
  char* ws;
  if (int rc = mem.alloc(&ws, wsb)) return rc;
  for (int side = 0; side < 2; ++side) {
    double* o = side ? sb : sa;
    if (int rc = launch_fcs_dense(dtype, side ? b : a, order, dims, 0, dims[order - 1], D, packed,
                                  hl.data(), o, 0, ws, wsb, st))
      return rc;
    if (kind == ST_SKETCH_TS) {  // ts_sketch = FCS mod J (ts_hcs.cu), compacted in place
      double* f;
      if (int rc = mem.alloc(&f, D * hash_len)) return rc;
      if (int rc = st_ts_fold(o, static_cast<int>(D), static_cast<uint32_t>(jt),
                              static_cast<uint32_t>(hash_len), f, st))
        return rc;
      FCS_CUDA_TRY(cudaMemcpyAsync(o, f, D * hash_len * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
  }
  dots_kernel<<<static_cast<unsigned>(D), 256, 0, st>>>(sa, sb, static_cast<int>(len), est);
  FCS_CUDA_TRY(cudaGetLastError());
  if (int rc = launch_median(est, 1, static_cast<int>(D), 1, med, st)) return rc;
  if (estimates)
    FCS_CUDA_TRY(cudaMemcpyAsync(estimates, est, D * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (out) {
    FCS_CUDA_TRY(cudaMemcpyAsync(out, med, sizeof(double), cudaMemcpyDeviceToHost, st));
    FCS_CUDA_TRY(cudaStreamSynchronize(st));
  }
  return ST_OK;
}

int st_sketch_dots(size_t count, size_t len, const double* a, const double* b, double* out,
                   void* stream) {
  if (count == 0) return ST_OK;
  FCS_CHECK_ARG(len < (1ull << 31), "st_sketch_dots: sketch too long");
  dots_kernel<<<static_cast<unsigned>(count), 256, 0, as_stream(stream)>>>(
      a, b, static_cast<int>(len), out);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int st_regression_forward(int dtype, const void* x, size_t batch, const void* w, size_t classes,
                          const double* bias, size_t order, const size_t* dims, size_t hash_len,
                          size_t sketch_count, uint64_t seed, double* y, void* stream) {
  FCS_CHECK_ARG(dtype == ST_F32 || dtype == ST_F64, "sketched_regression_forward: unknown dtype");
  FCS_CHECK_ARG(order >= 1 && order < ST_MAX_ORDER, "fcs_sketch: unsupported tensor order");
  FCS_CHECK_ARG(hash_len > 0 && sketch_count > 0,
                "EstimatorConfig: hash_len and sketch_count must be >= 1");
  FCS_CHECK_ARG(sketch_count >= 1, "median_reduce: empty input");
  if (batch == 0 || classes == 0) return ST_OK;
  size_t sum_dims = 0;
  for (size_t n = 0; n < order; ++n) {
    FCS_CHECK_ARG(dims[n] > 0, "HashPair: dimensions must be positive");
    sum_dims += dims[n];
  }
  cudaStream_t st = as_stream(stream);
  DevMem mem(st);
  const size_t D = sketch_count;
  const size_t jt = order * hash_len - order + 1;
  std::vector<size_t> hl(order, hash_len);
  uint32_t* packed;
  double *sx, *sw, *est;
  if (int rc = mem.alloc(&packed, D * sum_dims)) return rc;
  if (int rc = mem.alloc(&sx, D * batch * jt)) return rc;
  if (int rc = mem.alloc(&sw, D * classes * jt)) return rc;
  if (int rc = mem.alloc(&est, batch * D * classes)) return rc;
  const std::vector<uint64_t> seeds = family_seeds(seed, D);
  if (int rc = launch_family_tables(order, dims, hl.data(), D, seeds.data(), packed, st)) return rc;
  if (int rc = rows_sketch(dtype, x, order, dims, batch, jt, D, packed, sum_dims, 0, mem, sx, st))
    return rc;
  if (int rc = rows_sketch(dtype, w, order, dims, classes, jt, D, packed, sum_dims, 0, mem, sw, st))
    return rc;
  const dim3 grid(ceil_div(classes, kTile), ceil_div(batch, kTile), static_cast<unsigned>(D));
  sketch_gemm_kernel<<<grid, dim3(kTile, kTile), 0, st>>>(sx, sw, static_cast<int>(batch),
                                                          static_cast<int>(classes),
                                                          static_cast<int>(D),
                                                          static_cast<int>(jt), est);
  FCS_CUDA_TRY(cudaGetLastError());
  if (int rc = launch_median(est, static_cast<int>(batch), static_cast<int>(D),
                             static_cast<int>(classes), y, st))
    return rc;
  if (bias) {
    add_bias_kernel<<<ceil_div(batch * classes, 256), 256, 0, st>>>(y, bias, static_cast<int>(batch),
                                                                    static_cast<int>(classes));
    FCS_CUDA_TRY(cudaGetLastError());
  }
  return ST_OK;
}

int st_fcs_contraction(int dtype, const void* a, const size_t* dims_a, const void* b,
                       const size_t* dims_b, size_t sketch_count, const uint32_t* packed,
                       const size_t* hash_lens, double* out, void* stream) {
  FCS_CHECK_ARG(dtype == ST_F32 || dtype == ST_F64, "compress_contraction: unknown dtype");
  FCS_CHECK_ARG(dims_a[2] == dims_b[0], "compress_contraction: contracted dimensions differ");
  FCS_CHECK_ARG(sketch_count >= 1, "EstimatorConfig: hash_len and sketch_count must be >= 1");
  for (int n = 0; n < 3; ++n)
    FCS_CHECK_ARG(dims_a[n] > 0 && dims_b[n] > 0, "DenseTensor: zero dimension");
  for (int n = 0; n < 4; ++n) FCS_CHECK_ARG(hash_lens[n] > 0, "HashPair: dimensions must be positive");
  cudaStream_t st = as_stream(stream);
  DevMem mem(st);
  const size_t D = sketch_count, L = dims_a[2];
  const size_t I1 = dims_a[0], I2 = dims_a[1], I3 = dims_b[1], I4 = dims_b[2];
  const size_t stride = I1 + I2 + I3 + I4;
  const size_t la = hash_lens[0] + hash_lens[1] - 1, lb = hash_lens[2] + hash_lens[3] - 1;
  const size_t lo = la + lb - 1;  // 4J - 3 for equal hash lengths
  FftPlan pl;
  if (int rc = get_fft_plan(lo, &pl)) return rc;
  uint32_t *ta, *tb;
  double *sa, *sb;
  double2 *fa, *fb, *acc;
  if (int rc = mem.alloc(&ta, D * (I1 + I2 + L))) return rc;
  if (int rc = mem.alloc(&tb, D * (L + I3 + I4))) return rc;
  if (int rc = mem.alloc(&sa, D * L * la)) return rc;
  if (int rc = mem.alloc(&sb, D * L * lb)) return rc;
  if (int rc = mem.alloc(&fa, 2 * D * L * pl.P + D * pl.P)) return rc;
  fb = fa + D * L * pl.P;
  acc = fb + D * L * pl.P;
  // A(:,:,l) under pairs 0,1 -> row l of sa; B(l,:,:) under pairs 2,3 -> row l of sb
  if (int rc = batch_tables(packed, stride, I1 + I2, D, L, la, false, ta, st)) return rc;
  if (int rc = batch_tables(packed + I1 + I2, stride, I3 + I4, D, L, lb, true, tb, st)) return rc;
  const size_t one[3] = {1, 1, 1};
  const size_t da[3] = {I1, I2, L}, db[3] = {L, I3, I4};
  const size_t wsa = dense_workspace(dtype, 3, da, L, D, one, 0, L * la);
  const size_t wsb = dense_workspace(dtype, 3, db, I4, D, one, 0, L * lb);
  char* ws;
  if (int rc = mem.alloc(&ws, std::max(wsa, wsb))) return rc;
  if (int rc = launch_fcs_dense(dtype, a, 3, da, 0, L, D, ta, one, sa, 0, ws, wsa, st, 0, 0, L * la))
    return rc;
  if (int rc = launch_fcs_dense(dtype, b, 3, db, 0, I4, D, tb, one, sb, 0, ws, wsb, st, 0, 0, L * lb))
    return rc;
  // sum_l F(sa_l) F(sb_l), one inverse per family (§4.3.2)
  if (int rc = launch_spec_from_real(pl, sa, la, static_cast<int>(la), static_cast<int>(D * L), fa, st))
    return rc;
  if (int rc = launch_spec_from_real(pl, sb, lb, static_cast<int>(lb), static_cast<int>(D * L), fb, st))
    return rc;
  pair_product_sum_kernel<<<dim3(ceil_div(pl.P, 256), static_cast<unsigned>(D)), 256, 0, st>>>(
      fa, fb, static_cast<int>(L), pl.P, acc);
  FCS_CUDA_TRY(cudaGetLastError());
  return launch_real_from_spec(pl, acc, static_cast<int>(D), out, lo, static_cast<int>(lo), 0, st);
}

int st_sketch_decompress(const double* sketch, size_t sketch_count, size_t len,
                         const uint32_t* packed, size_t order, const size_t* dims, size_t count,
                         const uint32_t* idx, double* out, void* stream) {
  FCS_CHECK_ARG(order >= 1 && order <= 4, "decompress: order 1..4 supported");
  FCS_CHECK_ARG(sketch_count >= 1 && sketch_count <= 64, "median_reduce: 1..64 sketches");
  FCS_CHECK_ARG(len > 0, "decompress: empty sketch");
  if (count == 0) return ST_OK;
  FCS_CHECK_ARG(idx != nullptr, "decompress: null index array");
  Dims4 d4{};
  size_t stride = 0;
  for (size_t n = 0; n < order; ++n) {
    d4.d[n] = static_cast<uint32_t>(dims[n]);
    stride += dims[n];
  }
  cudaStream_t st = as_stream(stream);
  decompress_kernel<<<std::min<unsigned>(ceil_div(count, 256), 8192), 256, 0, st>>>(
      sketch, static_cast<int>(sketch_count), static_cast<uint32_t>(len), packed,
      static_cast<uint32_t>(stride), static_cast<int>(order), d4, count, idx, out);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int st_kron_decompress_all(const double* sketch, size_t sketch_count, size_t len,
                           const uint32_t* packed, const size_t* dims4, double* out, void* stream) {
  FCS_CHECK_ARG(sketch_count >= 1 && sketch_count <= 64, "median_reduce: 1..64 sketches");
  FCS_CHECK_ARG(len > 0, "decompress: empty sketch");
  Dims4 d4{};
  size_t stride = 0;
  for (int n = 0; n < 4; ++n) {
    FCS_CHECK_ARG(dims4[n] > 0, "DenseTensor: zero dimension");
    d4.d[n] = static_cast<uint32_t>(dims4[n]);
    stride += dims4[n];
  }
  const size_t count = dims4[0] * dims4[1] * dims4[2] * dims4[3];
  cudaStream_t st = as_stream(stream);
  decompress_kernel<<<std::min<unsigned>(ceil_div(count, 256), 8192), 256, 0, st>>>(
      sketch, static_cast<int>(sketch_count), static_cast<uint32_t>(len), packed,
      static_cast<uint32_t>(stride), 4, d4, count, nullptr, out);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // extern "C"
