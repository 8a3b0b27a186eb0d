// CP decomposition drivers on the contraction engine (cpd.cpp:234-392):
//  * st_rtpm / st_rtpm_backend — symmetric robust tensor power method,
//  * st_rtpm_asym — the alternating rank-1 variant for general order-3 tensors,
//  * st_als — alternating least squares with engine MTTKRP columns and exact
//    Gram solves,
//  * st_residual_norm — || T - densify(cp) ||_F / || T ||_F on the device.
// Restarts (rtpm, rtpm_asym) and MTTKRP columns (als) are batched into one
// engine call each; the control flow, the initial-vector stream and the argmax
// rule follow the reference so that the same estimates yield the same result.
#include <math_constants.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "engine.cuh"

namespace fcs {
namespace {

__device__ double cta_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < static_cast<int>(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  __syncthreads();
  return t;  // valid in thread 0
}

constexpr int kResThreads = 256;

// Per CTA: sum over its mode-0 fibers of (cp - t)^2 and t^2. A fiber (j, k)
// stages c_r = w_r A1[j,r] A2[k,r] in shared memory; thread i forms
// sum_r A0[i,r] c_r (column-major factors: coalesced over i).
template <typename T>
__global__ void __launch_bounds__(kResThreads)
    residual_kernel(const T* __restrict__ t, int I0, int I1, int I2, const double* __restrict__ w,
                    int R, const double* __restrict__ A0, const double* __restrict__ A1,
                    const double* __restrict__ A2, double* __restrict__ part) {
  extern __shared__ double c[];
  __shared__ double red[32];
  const size_t fibers = static_cast<size_t>(I1) * I2;
  double num = 0.0, den = 0.0;
  for (size_t f = blockIdx.x; f < fibers; f += gridDim.x) {
    const int j = static_cast<int>(f % I1), k = static_cast<int>(f / I1);
    __syncthreads();
    for (int r = threadIdx.x; r < R; r += blockDim.x)
      c[r] = w[r] * A1[j + static_cast<size_t>(r) * I1] * A2[k + static_cast<size_t>(r) * I2];
    __syncthreads();
    const T* fib = t + f * I0;
    for (int i = threadIdx.x; i < I0; i += blockDim.x) {
      double v = 0.0;
      for (int r = 0; r < R; ++r) v += A0[i + static_cast<size_t>(r) * I0] * c[r];
      const double x = static_cast<double>(fib[i]);
      num += (v - x) * (v - x);
      den += x * x;
    }
  }
  const double sn = cta_sum(num, red);
  const double sd = cta_sum(den, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = sn;
    part[2 * blockIdx.x + 1] = sd;
  }
}

// Fixed-order sum of the per-CTA partials (deterministic for a fixed grid).
__global__ void residual_final_kernel(const double* __restrict__ part, int n, double* out) {
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
  a = cta_sum(a, red);
  b = cta_sum(b, red);
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = b;
  }
}

// densify (tensor.cpp:86-115): out[l] = sum_r w_r prod_n U_n[i_n(l), r] for an
// order-N CP tensor (factors I_n x R column-major), flat column-major l.
struct DensifyArgs {
  int order, rank;
  int dims[ST_MAX_ORDER];
  const double* factors[ST_MAX_ORDER];
  const double* weights;
};
__global__ void densify_kernel(DensifyArgs a, size_t total, double* __restrict__ out) {
  for (size_t l = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; l < total;
       l += static_cast<size_t>(gridDim.x) * blockDim.x) {
    int idx[ST_MAX_ORDER];
    size_t rem = l;
    for (int n = 0; n < a.order; ++n) {
      idx[n] = static_cast<int>(rem % a.dims[n]);
      rem /= a.dims[n];
    }
    double s = 0.0;
    for (int r = 0; r < a.rank; ++r) {
      double p = a.weights[r];
      for (int n = 0; n < a.order; ++n) p *= a.factors[n][idx[n] + static_cast<size_t>(r) * a.dims[n]];
      s += p;
    }
    out[l] = s;
  }
}

// psnr partials (cpd.cpp:394-403): per CTA max |ref| and sum (ref - est)^2.
template <typename T>
__global__ void psnr_kernel(const T* __restrict__ ref, const T* __restrict__ est, size_t n,
                            double* __restrict__ part) {
  __shared__ double red[32];
  double mx = 0.0, se = 0.0;
  for (size_t l = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; l < n;
       l += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const double r = static_cast<double>(ref[l]), d = r - static_cast<double>(est[l]);
    mx = fmax(mx, fabs(r));
    se += d * d;
  }
  se = cta_sum(se, red);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __shared__ double mred[32];
  if ((threadIdx.x & 31) == 0) mred[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (unsigned w = 0; w < (blockDim.x >> 5); ++w) m = fmax(m, mred[w]);
    part[2 * blockIdx.x] = m;
    part[2 * blockIdx.x + 1] = se;
  }
}

__global__ void negate_kernel(double* v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = -v[i];
}

// residual_norm (cpd.cpp:385-392) from device factors; sums returned on host.
int residual_sums(int dtype, const void* t, const size_t* dims, const double* w, size_t R,
                  const double* A0, const double* A1, const double* A2, double* part, int nblk,
                  double* sums_dev, double* sums_host, cudaStream_t st) {
  const size_t smem = std::max<size_t>(1, R) * sizeof(double);
  const int I0 = static_cast<int>(dims[0]), I1 = static_cast<int>(dims[1]),
            I2 = static_cast<int>(dims[2]);
  if (dtype == ST_F32) {
    FCS_CUDA_TRY(cudaFuncSetAttribute(residual_kernel<float>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    residual_kernel<float><<<nblk, kResThreads, smem, st>>>(static_cast<const float*>(t), I0, I1,
                                                            I2, w, static_cast<int>(R), A0, A1, A2,
                                                            part);
  } else {
    FCS_CUDA_TRY(cudaFuncSetAttribute(residual_kernel<double>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    residual_kernel<double><<<nblk, kResThreads, smem, st>>>(static_cast<const double*>(t), I0, I1,
                                                             I2, w, static_cast<int>(R), A0, A1,
                                                             A2, part);
  }
  FCS_CUDA_TRY(cudaGetLastError());
  residual_final_kernel<<<1, 256, 0, st>>>(part, nblk, sums_dev);
  FCS_CUDA_TRY(cudaGetLastError());
  FCS_CUDA_TRY(cudaMemcpyAsync(sums_host, sums_dev, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  FCS_CUDA_TRY(cudaStreamSynchronize(st));
  return ST_OK;
}

double residual_from_sums(const double* s) {
  const double num = std::sqrt(s[0]), denom = std::sqrt(s[1]);
  if (denom == 0.0) return num == 0.0 ? 0.0 : std::numeric_limits<double>::infinity();
  return num / denom;
}

int residual_blocks() {
  DeviceInfo di;
  if (device_info(&di) != ST_OK) return 148 * 8;
  return di.sm_count * 8;
}

// ---------------------------------------------------------------- host LA
// Minimum-norm least-squares solve of G X = B (G: n x n, B: n x m, both
// column-major), as Eigen's completeOrthogonalDecomposition().solve used by
// als (cpd.cpp:369-370): Householder QR with column pivoting, numerical rank
// = #{i : |r_ii| > eps * n * max_k |r_kk|}, then the minimum-norm solution
// of the rank-r trapezoidal system through a QR of its transpose.
void householder(std::vector<double>& a, int lda, int rows, int col, int row0, std::vector<double>& v,
                 double* beta) {
  const int len = rows - row0;
  v.assign(len, 0.0);
  double sigma = 0.0;
  for (int i = 1; i < len; ++i) sigma += a[(row0 + i) + col * lda] * a[(row0 + i) + col * lda];
  const double x0 = a[row0 + col * lda];
  v[0] = 1.0;
  for (int i = 1; i < len; ++i) v[i] = a[(row0 + i) + col * lda];
  if (sigma == 0.0) {
    *beta = 0.0;
    return;
  }
  const double mu = std::sqrt(x0 * x0 + sigma);
  const double v0 = x0 <= 0 ? x0 - mu : -sigma / (x0 + mu);
  *beta = 2.0 * v0 * v0 / (sigma + v0 * v0);
  for (int i = 1; i < len; ++i) v[i] /= v0;
}

void min_norm_solve(int n, const std::vector<double>& G, int m, const std::vector<double>& B,
                    std::vector<double>& X) {
  std::vector<double> a = G, b = B;
  std::vector<int> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  std::vector<double> norms(n);
  for (int c = 0; c < n; ++c) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i + c * n] * a[i + c * n];
    norms[c] = s;
  }
  std::vector<double> v;
  for (int k = 0; k < n; ++k) {  // pivoted QR: A P = Q R, b <- Q^T b
    int best = k;
    for (int c = k + 1; c < n; ++c)
      if (norms[c] > norms[best]) best = c;
    if (best != k) {
      for (int i = 0; i < n; ++i) std::swap(a[i + k * n], a[i + best * n]);
      std::swap(norms[k], norms[best]);
      std::swap(perm[k], perm[best]);
    }
    double beta;
    householder(a, n, n, k, k, v, &beta);
    // apply to columns k..n-1 of a and to b
    for (int c = k; c < n; ++c) {
      double s = 0.0;
      for (int i = 0; i < n - k; ++i) s += v[i] * a[(k + i) + c * n];
      s *= beta;
      for (int i = 0; i < n - k; ++i) a[(k + i) + c * n] -= s * v[i];
    }
    for (int c = 0; c < m; ++c) {
      double s = 0.0;
      for (int i = 0; i < n - k; ++i) s += v[i] * b[(k + i) + c * n];
      s *= beta;
      for (int i = 0; i < n - k; ++i) b[(k + i) + c * n] -= s * v[i];
    }
    for (int c = k + 1; c < n; ++c) {  // downdate the remaining column norms
      double s = 0.0;
      for (int i = k + 1; i < n; ++i) s += a[i + c * n] * a[i + c * n];
      norms[c] = s;
    }
  }
  double maxpivot = 0.0;
  for (int i = 0; i < n; ++i) maxpivot = std::max(maxpivot, std::fabs(a[i + i * n]));
  const double thr = std::numeric_limits<double>::epsilon() * n * maxpivot;
  int r = 0;
  for (int i = 0; i < n; ++i) r += std::fabs(a[i + i * n]) > thr;
  X.assign(static_cast<size_t>(n) * m, 0.0);
  if (r == 0) return;
  // y (in the pivoted basis) = min-norm solution of [R11 R12] y = c, c = (Q^T b)[0:r]:
  // M^T = Q2 R2 (n x r), y = Q2 R2^{-T} c.
  std::vector<double> mt(static_cast<size_t>(n) * r);  // M^T, n x r
  for (int i = 0; i < r; ++i)
    for (int c = i; c < n; ++c) mt[c + i * n] = a[i + c * n];
  std::vector<std::vector<double>> vs(r);
  std::vector<double> betas(r);
  for (int k = 0; k < r; ++k) {
    householder(mt, n, n, k, k, vs[k], &betas[k]);
    for (int c = k; c < r; ++c) {
      double s = 0.0;
      for (int i = 0; i < n - k; ++i) s += vs[k][i] * mt[(k + i) + c * n];
      s *= betas[k];
      for (int i = 0; i < n - k; ++i) mt[(k + i) + c * n] -= s * vs[k][i];
    }
  }
  std::vector<double> z(n);
  for (int col = 0; col < m; ++col) {
    // solve R2^T z1 = c (forward substitution), z = [z1; 0]
    std::fill(z.begin(), z.end(), 0.0);
    for (int i = 0; i < r; ++i) {
      double s = b[i + col * n];
      for (int k = 0; k < i; ++k) s -= mt[k + i * n] * z[k];
      z[i] = s / mt[i + i * n];
    }
    for (int k = r - 1; k >= 0; --k) {  // y = Q2 z
      double s = 0.0;
      for (int i = 0; i < n - k; ++i) s += vs[k][i] * z[k + i];
      s *= betas[k];
      for (int i = 0; i < n - k; ++i) z[k + i] -= s * vs[k][i];
    }
    for (int i = 0; i < n; ++i) X[perm[i] + static_cast<size_t>(col) * n] = z[i];
  }
}

struct EngineGuard {
  st_engine* e = nullptr;
  ~EngineGuard() { st_engine_destroy(e); }
};

// rtpm (cpd.cpp:234-277) on an engine.
// Device-side steps of rtpm between the engine calls, so a whole run needs
// one host synchronisation (the reference's control flow, cpd.cpp:234-277):
// the restart argmax with strict > (first wins, NaN never wins) copying the
// winner to best, and the component's bookkeeping.
__global__ void rtpm_argmax_kernel(const double* __restrict__ vals, int L,
                                   const double* __restrict__ U, int dim,
                                   double* __restrict__ best, int* __restrict__ bad) {
  __shared__ int arg;
  if (threadIdx.x == 0) {
    double bv = -CUDART_INF;
    int a = -1;
    for (int l = 0; l < L; ++l)
      if (vals[l] > bv) {
        bv = vals[l];
        a = l;
      }
    if (a < 0) *bad = 1;  // no finite candidate: reported after the run
    arg = a < 0 ? 0 : a;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < dim; i += blockDim.x) best[i] = U[static_cast<size_t>(arg) * dim + i];
}

// weight = the refined contraction value: weights[r], factor column r, and
// the weighted vector the deflation subtracts (weight u o u o u =
// u o u o (weight u): linear in the last factor).
__global__ void rtpm_component_kernel(const double* __restrict__ val,
                                      const double* __restrict__ best, int dim,
                                      double* __restrict__ weight_out,
                                      double* __restrict__ factor_out,
                                      double* __restrict__ wbest) {
  const double w = *val;
  if (threadIdx.x == 0) *weight_out = w;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) {
    factor_out[i] = best[i];
    wbest[i] = w * best[i];
  }
}

int rtpm_on(st_engine* e, size_t dim, size_t rank, size_t L, size_t num_iters, uint64_t seed,
            double* weights, double* factor, cudaStream_t st) {
  // device: the R x L initial vectors, two L x dim iterate buffers, best /
  // next / weighted best, values, R weights, R x dim factors, flags
  const size_t need = (rank * L + 2 * L + 3) * dim * sizeof(double) +
                      (L + 1 + rank) * sizeof(double) + rank * dim * sizeof(double) + 16;
  if (int rc = e->vec.ensure(need, st)) return rc;
  double* U0 = static_cast<double*>(e->vec.p);
  double* Ubuf = U0 + rank * L * dim;
  double* Ybuf = Ubuf + L * dim;
  double* best = Ybuf + L * dim;
  double* next = best + dim;
  double* wbest = next + dim;
  double* vals = wbest + dim;
  double* wdev = vals + L + 1;
  double* fdev = wdev + rank;
  int* flags = reinterpret_cast<int*>(fdev + rank * dim);  // [0] stopped, [1] no finite candidate
  // every component's initial vectors up front, in the reference's draw order
  std::vector<double> hU(rank * L * dim);
  HostRng rng(splitmix_draw(seed ^ 0x7274706dULL, 1));  // init_rng (cpd.cpp:245)
  for (size_t i = 0; i < rank * L; ++i) rng.unit(hU.data() + i * dim, dim);
  FCS_CUDA_TRY(cudaMemcpyAsync(U0, hU.data(), hU.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  FCS_CUDA_TRY(cudaMemsetAsync(flags, 0, 2 * sizeof(int), st));
  const int tpb = 256;
  for (size_t r = 0; r < rank; ++r) {
    double* U = Ubuf;
    double* Y = Ybuf;
    FCS_CUDA_TRY(cudaMemcpyAsync(U, U0 + r * L * dim, L * dim * sizeof(double),
                                 cudaMemcpyDeviceToDevice, st));
    // L restarts advance in lockstep; a row whose norm underflows stays zero,
    // exactly like the reference's early break (iuu(0) = 0).
    for (size_t it = 0; it < num_iters; ++it) {
      // small batches: one cluster kernel with the median and the row
      // normalisation fused in; else estimator, median and normalisation kernels
      const int rc = engine_iuv_fused(e, L, U, 0, 2, Y, nullptr, nullptr, st);
      if (rc == 1) {
        if (is_exact(e)) {
          if (int rc2 = st_engine_iuv(e, L, U, U, 0, Y, 1, st)) return rc2;
          if (int rc2 = launch_normalize_rows(Y, static_cast<int>(L), static_cast<int>(dim), st))
            return rc2;
        } else {  // per-family estimates, then one median + normalisation kernel
          if (int rc2 = e->est2.ensure(L * e->D * dim * sizeof(double), st)) return rc2;
          double* est = static_cast<double*>(e->est2.p);
          if (int rc2 = st_engine_iuv(e, L, U, U, 0, est, 0, st)) return rc2;
          if (int rc2 = launch_median_normalize(est, static_cast<int>(L), static_cast<int>(e->D),
                                                static_cast<int>(dim), Y, st))
            return rc2;
        }
      } else if (rc) {
        return rc;
      }
      std::swap(U, Y);
    }
    if (int rc = st_engine_uvw(e, L, U, U, U, vals, 1, st)) return rc;
    rtpm_argmax_kernel<<<1, tpb, 0, st>>>(vals, static_cast<int>(L), U, static_cast<int>(dim), best,
                                          flags + 1);
    FCS_CUDA_TRY(cudaGetLastError());
    FCS_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(int), st));
    for (size_t it = 0; it < num_iters; ++it) {  // refinement (cpd.cpp:266-270)
      const int rc = engine_iuv_fused(e, 1, best, 0, 3, next, best, flags, st);
      if (rc == 1) {
        if (int rc2 = st_engine_iuv(e, 1, best, best, 0, next, 1, st)) return rc2;
        if (int rc2 = launch_refine_update(best, next, static_cast<int>(dim), flags, st))
          return rc2;
      } else if (rc) {
        return rc;
      }
    }
    if (int rc = st_engine_uvw(e, 1, best, best, best, vals, 1, st)) return rc;
    rtpm_component_kernel<<<1, tpb, 0, st>>>(vals, best, static_cast<int>(dim), wdev + r,
                                             fdev + r * dim, wbest);
    FCS_CUDA_TRY(cudaGetLastError());
    if (int rc = st_engine_deflate(e, 1.0, best, best, wbest, st)) return rc;
  }
  int bad = 0;
  FCS_CUDA_TRY(cudaMemcpyAsync(weights, wdev, rank * sizeof(double), cudaMemcpyDeviceToHost, st));
  FCS_CUDA_TRY(cudaMemcpyAsync(factor, fdev, rank * dim * sizeof(double), cudaMemcpyDeviceToHost, st));
  FCS_CUDA_TRY(cudaMemcpyAsync(&bad, flags + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  FCS_CUDA_TRY(cudaStreamSynchronize(st));
  if (bad) return fail(ST_ENUMERIC, "rtpm: no candidate with a finite contraction value");
  return ST_OK;
}

}  // namespace
}  // namespace fcs

using namespace fcs;

extern "C" {

int st_rtpm_backend(int backend, int dtype, const void* tensor, size_t dim, size_t rank,
                    size_t num_inits, size_t num_iters, size_t hash_len, size_t sketch_count,
                    uint64_t seed, double* weights, double* factor, void* stream) {
  FCS_CHECK_ARG(dim > 0, "DenseTensor: zero dimension");
  FCS_CHECK_ARG(rank > 0 && num_inits > 0 && num_iters > 0,
                "rtpm: rank, inits, and iterations must be >= 1");
  cudaStream_t st = as_stream(stream);
  const size_t dims[3] = {dim, dim, dim};
  EngineGuard g;
  if (int rc = st_engine_create_backend(&g.e, backend, dtype, tensor, dims, hash_len, sketch_count,
                                        seed, st))
    return rc;
  return rtpm_on(g.e, dim, rank, num_inits, num_iters, seed, weights, factor, st);
}

int st_rtpm(int dtype, const void* tensor, size_t dim, size_t rank, size_t num_inits,
            size_t num_iters, size_t hash_len, size_t sketch_count, uint64_t seed,
            double* weights, double* factor, void* stream) {
  return st_rtpm_backend(ST_BACKEND_FCS, dtype, tensor, dim, rank, num_inits, num_iters, hash_len,
                         sketch_count, seed, weights, factor, stream);
}

int st_rtpm_asym(int backend, int dtype, const void* tensor, const size_t* dims, size_t rank,
                 size_t num_inits, size_t num_iters, size_t hash_len, size_t sketch_count,
                 uint64_t seed, double* weights, double* factors, void* stream) {
  FCS_CHECK_ARG(rank > 0 && num_inits > 0 && num_iters > 0,
                "rtpm_asym: rank, inits, and iterations must be >= 1");
  for (int n = 0; n < 3; ++n) FCS_CHECK_ARG(dims[n] > 0, "DenseTensor: zero dimension");
  cudaStream_t st = as_stream(stream);
  EngineGuard g;
  if (int rc = st_engine_create_backend(&g.e, backend, dtype, tensor, dims, hash_len, sketch_count,
                                        seed, st))
    return rc;
  st_engine* e = g.e;
  const size_t L = num_inits;
  const size_t I[3] = {dims[0], dims[1], dims[2]};
  const size_t sum_i = I[0] + I[1] + I[2];
  if (int rc = e->vec.ensure((L * sum_i + sum_i + L + 1) * sizeof(double), st)) return rc;
  double* U[3];
  U[0] = static_cast<double*>(e->vec.p);
  U[1] = U[0] + L * I[0];
  U[2] = U[1] + L * I[1];
  double* B[3];
  B[0] = U[2] + L * I[2];
  B[1] = B[0] + I[0];
  B[2] = B[1] + I[1];
  double* vals = B[2] + I[2];
  std::vector<double> hU[3] = {std::vector<double>(L * I[0]), std::vector<double>(L * I[1]),
                               std::vector<double>(L * I[2])};
  std::vector<double> hvals(L), hb;
  HostRng rng(splitmix_draw(seed ^ 0x72743161ULL, 1));  // init_rng (cpd.cpp:285)
  size_t off[3] = {0, I[0] * rank, (I[0] + I[1]) * rank};
  // one alternating sweep over the three modes on `rows` vectors (cpd.cpp:298-305)
  auto sweep = [&](double* const* V, size_t rows) -> int {
    for (int m = 0; m < 3; ++m) {
      int c1, c2;
      contracted(m, &c1, &c2);
      if (int rc = st_engine_iuv(e, rows, V[c1], V[c2], m, V[m], 1, st)) return rc;
      if (int rc = launch_normalize_rows(V[m], static_cast<int>(rows), static_cast<int>(I[m]), st))
        return rc;
    }
    return ST_OK;
  };
  for (size_t r = 0; r < rank; ++r) {
    for (size_t l = 0; l < L; ++l)
      for (int n = 0; n < 3; ++n) rng.unit(hU[n].data() + l * I[n], I[n]);
    for (int n = 0; n < 3; ++n)
      FCS_CUDA_TRY(cudaMemcpyAsync(U[n], hU[n].data(), L * I[n] * sizeof(double),
                                   cudaMemcpyHostToDevice, st));
    // Note: the in-place update reads V[c1], V[c2] and writes V[m], m distinct.
    for (size_t it = 0; it < num_iters; ++it)
      if (int rc = sweep(U, L)) return rc;
    if (int rc = st_engine_uvw(e, L, U[0], U[1], U[2], vals, 1, st)) return rc;
    FCS_CUDA_TRY(cudaMemcpyAsync(hvals.data(), vals, L * sizeof(double), cudaMemcpyDeviceToHost, st));
    FCS_CUDA_TRY(cudaStreamSynchronize(st));
    double best_value = -std::numeric_limits<double>::infinity();
    long arg = -1;
    for (size_t l = 0; l < L; ++l) {
      const double v = std::fabs(hvals[l]);
      if (v > best_value) {  // strict >, first wins (cpd.cpp:307-311)
        best_value = v;
        arg = static_cast<long>(l);
      }
    }
    if (arg < 0) return fail(ST_ENUMERIC, "rtpm_asym: no candidate with a finite contraction value");
    for (int n = 0; n < 3; ++n)
      FCS_CUDA_TRY(cudaMemcpyAsync(B[n], U[n] + arg * I[n], I[n] * sizeof(double),
                                   cudaMemcpyDeviceToDevice, st));
    for (size_t it = 0; it < num_iters; ++it)  // refinement (cpd.cpp:313-320)
      if (int rc = sweep(B, 1)) return rc;
    if (int rc = st_engine_uvw(e, 1, B[0], B[1], B[2], vals, 1, st)) return rc;
    double weight = 0.0;
    FCS_CUDA_TRY(cudaMemcpyAsync(&weight, vals, sizeof(double), cudaMemcpyDeviceToHost, st));
    FCS_CUDA_TRY(cudaStreamSynchronize(st));
    if (weight < 0) {  // absorb the sign into the first factor (cpd.cpp:322-325)
      negate_kernel<<<ceil_div(I[0], 256), 256, 0, st>>>(B[0], static_cast<int>(I[0]));
      FCS_CUDA_TRY(cudaGetLastError());
      weight = -weight;
    }
    weights[r] = weight;
    for (int n = 0; n < 3; ++n)
      FCS_CUDA_TRY(cudaMemcpyAsync(factors + off[n] + r * I[n], B[n], I[n] * sizeof(double),
                                   cudaMemcpyDeviceToHost, st));
    if (int rc = st_engine_deflate(e, weight, B[0], B[1], B[2], st)) return rc;
  }
  FCS_CUDA_TRY(cudaStreamSynchronize(st));
  return ST_OK;
}

int st_densify(size_t order, const size_t* dims, size_t rank, const double* weights,
               const double* const* factors, double* out, void* stream) {
  FCS_CHECK_ARG(order >= 1 && order <= ST_MAX_ORDER, "CpTensor: no factors");
  DensifyArgs a{};
  a.order = static_cast<int>(order);
  a.rank = static_cast<int>(rank);
  a.weights = weights;
  size_t total = 1;
  for (size_t n = 0; n < order; ++n) {
    FCS_CHECK_ARG(dims[n] > 0, "DenseTensor: zero dimension");
    a.dims[n] = static_cast<int>(dims[n]);
    a.factors[n] = factors[n];
    total *= dims[n];
  }
  const unsigned grid = static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 16384));
  densify_kernel<<<grid, 256, 0, as_stream(stream)>>>(a, total, out);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int st_psnr(int dtype, const void* reference, const void* estimate, size_t n, double* out,
            void* stream) {
  FCS_CHECK_ARG(dtype == ST_F32 || dtype == ST_F64, "psnr: unknown dtype");
  FCS_CHECK_ARG(n > 0 && out != nullptr, "psnr: empty tensors");
  cudaStream_t st = as_stream(stream);
  const int nblk = residual_blocks();
  double* part = nullptr;
  FCS_CUDA_TRY(malloc_async(reinterpret_cast<void**>(&part), 2 * nblk * sizeof(double), st));
  if (dtype == ST_F64)
    psnr_kernel<double><<<nblk, 256, 0, st>>>(static_cast<const double*>(reference),
                                              static_cast<const double*>(estimate), n, part);
  else
    psnr_kernel<float><<<nblk, 256, 0, st>>>(static_cast<const float*>(reference),
                                             static_cast<const float*>(estimate), n, part);
  std::vector<double> h(2 * nblk);
  const cudaError_t le = cudaGetLastError();
  const cudaError_t ce =
      cudaMemcpyAsync(h.data(), part, 2 * nblk * sizeof(double), cudaMemcpyDeviceToHost, st);
  const cudaError_t se = cudaStreamSynchronize(st);
  cudaFreeAsync(part, st);
  FCS_CUDA_TRY(le);
  FCS_CUDA_TRY(ce);
  FCS_CUDA_TRY(se);
  double peak = 0.0, sse = 0.0;
  for (int b = 0; b < nblk; ++b) {
    peak = std::max(peak, h[2 * b]);
    sse += h[2 * b + 1];
  }
  const double mse = sse / static_cast<double>(n);
  *out = mse == 0.0 ? 99.0 : std::min(10.0 * std::log10(peak * peak / mse), 99.0);
  return ST_OK;
}

int st_residual_norm(int dtype, const void* tensor, const size_t* dims, const double* weights,
                     size_t rank, const double* factors, double* out, void* stream) {
  FCS_CHECK_ARG(dtype == ST_F32 || dtype == ST_F64, "st_residual_norm: unknown dtype");
  for (int n = 0; n < 3; ++n) FCS_CHECK_ARG(dims[n] > 0, "DenseTensor: zero dimension");
  FCS_CHECK_ARG(out != nullptr, "st_residual_norm: null output");
  cudaStream_t st = as_stream(stream);
  const int nblk = residual_blocks();
  double* part = nullptr;
  FCS_CUDA_TRY(malloc_async(reinterpret_cast<void**>(&part), (2 * nblk + 2) * sizeof(double), st));
  double sums[2];
  const double* A0 = factors;
  const double* A1 = A0 + dims[0] * rank;
  const double* A2 = A1 + dims[1] * rank;
  const int rc = residual_sums(dtype, tensor, dims, weights, rank, A0, A1, A2, part, nblk,
                               part + 2 * nblk, sums, st);
  cudaFreeAsync(part, st);
  if (rc) return rc;
  *out = residual_from_sums(sums);
  return ST_OK;
}

int st_als(int backend, int dtype, const void* tensor, const size_t* dims, size_t rank,
           size_t max_iters, double tol, size_t hash_len, size_t sketch_count, uint64_t seed,
           double* weights, double* factors, size_t* sweeps, void* stream) {
  FCS_CHECK_ARG(rank > 0 && max_iters > 0, "als: rank and iterations must be >= 1");
  for (int n = 0; n < 3; ++n) FCS_CHECK_ARG(dims[n] > 0, "DenseTensor: zero dimension");
  cudaStream_t st = as_stream(stream);
  EngineGuard g;
  if (int rc = st_engine_create_backend(&g.e, backend, dtype, tensor, dims, hash_len, sketch_count,
                                        seed, st))
    return rc;
  st_engine* e = g.e;
  const size_t R = rank;
  const size_t I[3] = {dims[0], dims[1], dims[2]};
  const size_t sum_i = I[0] + I[1] + I[2];
  const size_t imax = std::max({I[0], I[1], I[2]});
  const int nblk = residual_blocks();
  // device: factors (packed like the output), mttkrp (imax x R), weights, residual partials
  if (int rc = e->vec.ensure((sum_i * R + imax * R + R + 2 * nblk + 2) * sizeof(double), st))
    return rc;
  double* dF[3];
  dF[0] = static_cast<double*>(e->vec.p);
  dF[1] = dF[0] + I[0] * R;
  dF[2] = dF[1] + I[1] * R;
  double* dM = dF[2] + I[2] * R;
  double* dW = dM + imax * R;
  double* part = dW + R;
  std::vector<double> F[3] = {std::vector<double>(I[0] * R), std::vector<double>(I[1] * R),
                              std::vector<double>(I[2] * R)};
  HostRng rng(splitmix_draw(seed ^ 0x616c73ULL, 1));  // init_rng (cpd.cpp:346)
  for (int n = 0; n < 3; ++n)
    for (size_t r = 0; r < R; ++r) rng.unit(F[n].data() + r * I[n], I[n]);
  std::vector<double> w(R, 1.0), M(imax * R), gram(R * R), X;
  for (int n = 0; n < 3; ++n)
    FCS_CUDA_TRY(cudaMemcpyAsync(dF[n], F[n].data(), I[n] * R * sizeof(double),
                                 cudaMemcpyHostToDevice, st));
  double prev = std::numeric_limits<double>::infinity();
  size_t done = 0;
  for (size_t sweep = 0; sweep < max_iters; ++sweep) {
    for (int mode = 0; mode < 3; ++mode) {
      int o1, o2;
      contracted(mode, &o1, &o2);
      const size_t im = I[mode];
      // MTTKRP columns: R engine contractions in one batch (cpd.cpp:363-366);
      // row r of the batch output is column r of the I_mode x R matrix.
      if (int rc = st_engine_iuv(e, R, dF[o1], dF[o2], mode, dM, 1, st)) return rc;
      FCS_CUDA_TRY(cudaMemcpyAsync(M.data(), dM, im * R * sizeof(double), cudaMemcpyDeviceToHost, st));
      // gram = (F_o1^T F_o1) .* (F_o2^T F_o2) (cpd.cpp:367-368), exact on the host
      for (size_t a = 0; a < R; ++a)
        for (size_t b = 0; b < R; ++b) {
          double s1 = 0.0, s2 = 0.0;
          const double* x1 = F[o1].data();
          const double* x2 = F[o2].data();
          for (size_t i = 0; i < I[o1]; ++i) s1 += x1[i + a * I[o1]] * x1[i + b * I[o1]];
          for (size_t i = 0; i < I[o2]; ++i) s2 += x2[i + a * I[o2]] * x2[i + b * I[o2]];
          gram[a + b * R] = s1 * s2;
        }
      FCS_CUDA_TRY(cudaStreamSynchronize(st));
      // F_mode = (gram^+ M^T)^T (cpd.cpp:369-370)
      std::vector<double> Mt(R * im);
      for (size_t i = 0; i < im; ++i)
        for (size_t r = 0; r < R; ++r) Mt[r + i * R] = M[i + r * im];
      min_norm_solve(static_cast<int>(R), gram, static_cast<int>(im), Mt, X);
      for (size_t i = 0; i < im; ++i)
        for (size_t r = 0; r < R; ++r) F[mode][i + r * im] = X[r + i * R];
      for (size_t r = 0; r < R; ++r) {  // cpd.cpp:371-375
        double s = 0.0;
        for (size_t i = 0; i < im; ++i) s += F[mode][i + r * im] * F[mode][i + r * im];
        const double norm = std::sqrt(s);
        w[r] = norm;
        if (norm > 1e-150)
          for (size_t i = 0; i < im; ++i) F[mode][i + r * im] /= norm;
      }
      FCS_CUDA_TRY(cudaMemcpyAsync(dF[mode], F[mode].data(), im * R * sizeof(double),
                                   cudaMemcpyHostToDevice, st));
    }
    FCS_CUDA_TRY(cudaMemcpyAsync(dW, w.data(), R * sizeof(double), cudaMemcpyHostToDevice, st));
    double sums[2];
    if (int rc = residual_sums(dtype, tensor, dims, dW, R, dF[0], dF[1], dF[2], part, nblk,
                               part + 2 * nblk, sums, st))
      return rc;
    const double residual = residual_from_sums(sums);
    done = sweep + 1;
    if (std::fabs(prev - residual) < tol) break;  // cpd.cpp:378-380
    prev = residual;
  }
  for (size_t r = 0; r < R; ++r) weights[r] = w[r];
  size_t off = 0;
  for (int n = 0; n < 3; ++n) {
    std::copy(F[n].begin(), F[n].end(), factors + off);
    off += I[n] * R;
  }
  if (sweeps) *sweeps = done;
  FCS_CUDA_TRY(cudaStreamSynchronize(st));
  return ST_OK;
}

}  // extern "C"
