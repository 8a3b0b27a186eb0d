// Spectral paths for composed lengths beyond one CTA's shared memory
// (J~ > kMaxFftM): the same half-spectrum algebra as spectral.cu on a
// two-level ("four-step") transform in global memory.
//
// The packed complex sequence z[n] = x[2n] + i x[2n+1] (P = P1 P2 points,
// n = n1 P2 + n2) is transformed as
//   Y[k1][n2] = w_P^{n2 k1} sum_{n1} z[n1 P2 + n2] w_P1^{n1 k1}   (column pass, P1-point)
//   Z[k1 + P1 k2] = sum_{n2} Y[k1][n2] w_P2^{n2 k2}                 (row pass, P2-point)
// with each P1- / P2-point transform done by the shared-memory DIF of
// fft.cuh in its digit-reversed slot order. Z[k] lands at position
// pos(k) = f2p_a[k mod P1] * P2 + f2p_b[k / P1]; pos(0) = 0. The r2c pair
// pass then maps (Z[k], Z[P-k]) to the Hermitian half spectrum exactly as
// fft.cuh's post / pre pair maps do, so every pointwise kernel (products, conjugates,
// Parseval sums with the two real bins in slot 0) is layout-agnostic and the
// inverse runs the passes backwards (DIT rows, conjugate twiddle, DIT columns).
//
// Reference semantics are those of spectral.cu (fft.cpp:42-84 with padding
// to any M >= J~, estimators.cpp:38-90 for the estimators).
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "fft.cuh"

namespace fcs {

namespace {

__device__ __forceinline__ double2 root_p(int64_t e, int64_t P) {
  // exp(-2 pi i e / P), e reduced exactly first
  double s, c;
  sincospi(-2.0 * static_cast<double>(e % P) / static_cast<double>(P), &s, &c);
  return make_double2(c, s);
}

__device__ __forceinline__ size_t lpos(const LargeFft& L, int64_t k) {
  const int64_t k1 = k % L.P1, k2 = k / L.P1;
  return static_cast<size_t>(L.a.f2p[k1]) * L.P2 + L.b.f2p[k2];
}

// Column pass: one CTA per (column n2, item). Zero-padded real input rows.
__global__ void __launch_bounds__(kFftThreads) lf_cols_fwd(LargeFft L, const double* __restrict__ x,
                                                           size_t ldx, int64_t len,
                                                           double2* __restrict__ Y) {
  extern __shared__ __align__(16) double2 lsm[];
  double2* tw = lsm;
  double2* buf = lsm + table_slots(L.a);
  load_twiddles(tw, L.a);
  const int n2 = blockIdx.x;
  const size_t item = blockIdx.y;
  const double* xi = x + item * ldx;
  for (int n1 = threadIdx.x; n1 < L.P1; n1 += blockDim.x) {
    const int64_t t = 2 * (static_cast<int64_t>(n1) * L.P2 + n2);
    buf[swz(n1)] = make_double2(t < len ? xi[t] : 0.0, t + 1 < len ? xi[t + 1] : 0.0);
  }
  __syncthreads();
  fft_forward(buf, L.a, tw);
  const int* f2p = smem_f2p(tw, L.a);
  double2* y = Y + item * static_cast<size_t>(L.P);
  for (int k1 = threadIdx.x; k1 < L.P1; k1 += blockDim.x) {
    const int s1 = f2p[k1];
    y[static_cast<size_t>(s1) * L.P2 + n2] =
        cmul(buf[swz(s1)], root_p(static_cast<int64_t>(n2) * k1, L.P));
  }
}

// Row pass (in place): one CTA per (row slot s1, item).
__global__ void __launch_bounds__(kFftThreads) lf_rows_fwd(LargeFft L, double2* __restrict__ Z) {
  extern __shared__ __align__(16) double2 lsm[];
  double2* tw = lsm;
  double2* buf = lsm + table_slots(L.b);
  load_twiddles(tw, L.b);
  double2* row = Z + blockIdx.y * static_cast<size_t>(L.P) + static_cast<size_t>(blockIdx.x) * L.P2;
  for (int n2 = threadIdx.x; n2 < L.P2; n2 += blockDim.x) buf[swz(n2)] = row[n2];
  __syncthreads();
  fft_forward(buf, L.b, tw);
  for (int s2 = threadIdx.x; s2 < L.P2; s2 += blockDim.x) row[s2] = buf[swz(s2)];
}

// r2c / c2r pair pass over (k, P-k) (fft.cuh post_pair / pre_pair), one thread per pair.
template <bool kPost>
__global__ void lf_pairs(LargeFft L, double2* __restrict__ Z, int items) {
  const int64_t half = L.P / 2;
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k > half) return;
  double2* z = Z + blockIdx.y * static_cast<size_t>(L.P);
  if (k == 0) {
    const double2 v = z[0];
    z[0] = kPost ? make_double2(v.x + v.y, v.x - v.y) : make_double2(0.5 * (v.x + v.y), 0.5 * (v.x - v.y));
    return;
  }
  const size_t pa = lpos(L, k), pb = lpos(L, L.P - k);
  double2 va = z[pa], vb = z[pb];
  const double2 w = root_p(k, L.M);
  if (kPost) post_pair(va, vb, w);
  else pre_pair(va, vb, w);
  z[pa] = va;
  if (pb != pa) z[pb] = vb;
  (void)items;
}

// Inverse row pass (in place): DIT over the row's slots, then the conjugate
// column twiddle w_P^{-n2 k1}.
__global__ void __launch_bounds__(kFftThreads) lf_rows_inv(LargeFft L, double2* __restrict__ Z) {
  extern __shared__ __align__(16) double2 lsm[];
  double2* tw = lsm;
  double2* buf = lsm + table_slots(L.b);
  load_twiddles(tw, L.b);
  const int s1 = blockIdx.x;
  const int k1 = L.p2f_a[s1];
  double2* row = Z + blockIdx.y * static_cast<size_t>(L.P) + static_cast<size_t>(s1) * L.P2;
  for (int s2 = threadIdx.x; s2 < L.P2; s2 += blockDim.x) buf[swz(s2)] = row[s2];
  __syncthreads();
  fft_inverse(buf, L.b, tw);
  for (int n2 = threadIdx.x; n2 < L.P2; n2 += blockDim.x)
    row[n2] = cmul(buf[swz(n2)], cconj(root_p(static_cast<int64_t>(n2) * k1, L.P)));
}

// Inverse column pass: DIT over the column's row slots -> natural n1; the
// real sequence x[2n], x[2n+1] (n = n1 P2 + n2) scaled by 1/P.
__global__ void __launch_bounds__(kFftThreads) lf_cols_inv(LargeFft L, const double2* __restrict__ Z,
                                                           double* __restrict__ out, size_t ldo,
                                                           int64_t out_len, int accumulate) {
  extern __shared__ __align__(16) double2 lsm[];
  double2* tw = lsm;
  double2* buf = lsm + table_slots(L.a);
  load_twiddles(tw, L.a);
  const int n2 = blockIdx.x;
  const size_t item = blockIdx.y;
  const double2* z = Z + item * static_cast<size_t>(L.P);
  for (int s1 = threadIdx.x; s1 < L.P1; s1 += blockDim.x)
    buf[swz(s1)] = z[static_cast<size_t>(s1) * L.P2 + n2];
  __syncthreads();
  fft_inverse(buf, L.a, tw);
  const double inv = 1.0 / L.P;
  double* o = out + item * ldo;
  for (int n1 = threadIdx.x; n1 < L.P1; n1 += blockDim.x) {
    const int64_t t = 2 * (static_cast<int64_t>(n1) * L.P2 + n2);
    const double2 v = buf[swz(n1)];
    if (t < out_len) o[t] = accumulate ? o[t] + v.x * inv : v.x * inv;
    if (t + 1 < out_len) o[t + 1] = accumulate ? o[t + 1] + v.y * inv : v.y * inv;
  }
}

// ------------------------------------------------------ pointwise kernels
// Count sketches of `rows` vectors (row r at U + r * ldu, I entries) under D
// families, into zeroed real rows out[(r * sr + d * sd) * J].
__global__ void lf_cs_rows(const double* __restrict__ U, size_t ldu, int I, int rows,
                           const uint32_t* __restrict__ packed, int fam_stride, int tab_off, int D,
                           int J, size_t sr, size_t sd, double* __restrict__ out) {
  const size_t n = static_cast<size_t>(rows) * I;
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = q / I;
    const int i = static_cast<int>(q - r * I);
    const double v = U[r * ldu + i];
    if (v == 0.0) continue;  // cs_sketch skips zeros (sketch.cpp:105-116)
    for (int d = 0; d < D; ++d) {
      const uint32_t e = __ldg(packed + static_cast<size_t>(d) * fam_stride + tab_off + i);
      atomicAdd(out + (r * sr + d * sd) * J + (e & 0x7fffffffu), (e >> 31) ? -v : v);
    }
  }
}

// a[item] = a[item] (*) b[item] (half-spectrum product), optional scale.
__global__ void lf_mul(double2* __restrict__ a, const double2* __restrict__ b, size_t n, int P) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<size_t>(gridDim.x) * blockDim.x)
    a[q] = hmul(a[q], b[q], q % P == 0);
}

// G[b][d] = S_d * conj(Fa Fb) (iuv_spectral's product, estimators.cpp:80-83).
__global__ void lf_iuv_combine(const double2* __restrict__ S, double2* __restrict__ Fa,
                               const double2* __restrict__ Fb, int D, int P, size_t n) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t item = q / P;
    const int s = static_cast<int>(q - item * P);
    const int d = static_cast<int>(item % D);
    const bool z = s == 0;
    Fa[q] = hmul(S[static_cast<size_t>(d) * P + s], hconj(hmul(Fa[q], Fb[q], z), z), z);
  }
}

// est[item] = s_f(i) z[item][h_f(i)] (iuv_spectral's readout, estimators.cpp:84-89).
__global__ void lf_gather(const double* __restrict__ z, size_t ldz, const uint32_t* __restrict__ packed,
                          int fam_stride, int tab_off, int D, int nf, size_t items,
                          double* __restrict__ est) {
  const size_t n = items * nf;
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t item = q / nf;
    const int i = static_cast<int>(q - item * nf);
    const int d = static_cast<int>(item % D);
    const uint32_t e = __ldg(packed + static_cast<size_t>(d) * fam_stride + tab_off + i);
    const double v = z[item * ldz + (e & 0x7fffffffu)];
    est[q] = (e >> 31) ? -v : v;
  }
}

// est[item] = (1/M) sum_s Re(S_d conj(Fu Fv Fw)) with the slot-0 pair of real
// bins counted once and every other slot twice (uvw_spectral + spectral_dot).
__global__ void lf_uvw_dot(const double2* __restrict__ S, const double2* __restrict__ Fu,
                           const double2* __restrict__ Fv, const double2* __restrict__ Fw, int D,
                           int P, int M, double* __restrict__ est) {
  __shared__ double red[32];
  const size_t item = blockIdx.x;
  const int d = static_cast<int>(item % D);
  const double2* s = S + static_cast<size_t>(d) * P;
  const size_t off = item * P;
  double acc = 0.0;
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    const bool z = q == 0;
    const double2 g = hmul(hmul(Fu[off + q], Fv[off + q], z), Fw[off + q], z);
    const double re = s[q].x * g.x + s[q].y * g.y;
    acc += z ? re : 2.0 * re;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) est[item] = t / M;
  }
}

// S_d -= weight * Fu Fv Fw (K9 by linearity).
__global__ void lf_deflate(double2* __restrict__ S, const double2* __restrict__ Fu,
                           const double2* __restrict__ Fv, const double2* __restrict__ Fw,
                           double weight, int P, size_t n) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const bool z = q % P == 0;
    S[q] = csub(S[q], cscale(hmul(hmul(Fu[q], Fv[q], z), Fw[q], z), weight));
  }
}

// acc[d] = sum_r w_r Q[d][r] (fixed order; zero weights skipped, sketch.cpp:75).
__global__ void lf_rank_sum(const double2* __restrict__ Q, const double* __restrict__ w,
                            int r_begin, int R, int P, int D, double2* __restrict__ acc) {
  const size_t n = static_cast<size_t>(D) * P;
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t d = q / P;
    const int s = static_cast<int>(q - d * P);
    double2 a = make_double2(0.0, 0.0);
    for (int r = 0; r < R; ++r) {
      const double wr = w[r_begin + r];
      if (wr == 0.0) continue;
      a = cadd(a, cscale(Q[(d * R + r) * static_cast<size_t>(P) + s], wr));
    }
    acc[q] = a;
  }
}

unsigned grid_for(size_t n) { return static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 16384)); }

size_t large_smem(const FftPlan& sub) {
  return static_cast<size_t>(sub.P + table_slots(sub)) * sizeof(double2);
}

template <typename K>
int set_smem(K kernel, size_t bytes) {
  FCS_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(bytes)));
  return ST_OK;
}

struct DevTmp {
  void* p = nullptr;
  cudaStream_t st;
  explicit DevTmp(cudaStream_t s) : st(s) {}
  ~DevTmp() {
    if (p) cudaFreeAsync(p, st);
  }
  int alloc(size_t bytes) {
    FCS_CUDA_TRY(malloc_async(&p, std::max<size_t>(bytes, 1), st));
    return ST_OK;
  }
};

}  // namespace

// -------------------------------------------------------------- transforms
int large_rfft(const FftPlan& pl, const double* x, size_t ldx, int64_t len, int items,
               double2* spec, cudaStream_t st) {
  if (items == 0) return ST_OK;
  LargeFft L;
  if (int rc = get_large_fft(pl, &L)) return rc;
  const size_t sa = large_smem(L.a), sb = large_smem(L.b);
  if (int rc = set_smem(lf_cols_fwd, sa)) return rc;
  if (int rc = set_smem(lf_rows_fwd, sb)) return rc;
  lf_cols_fwd<<<dim3(L.P2, items), kFftThreads, sa, st>>>(L, x, ldx, len, spec);
  FCS_CUDA_TRY(cudaGetLastError());
  lf_rows_fwd<<<dim3(L.P1, items), kFftThreads, sb, st>>>(L, spec);
  FCS_CUDA_TRY(cudaGetLastError());
  lf_pairs<true><<<dim3(ceil_div(L.P / 2 + 1, 256), items), 256, 0, st>>>(L, spec, items);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int large_irfft(const FftPlan& pl, double2* spec, int items, double* out, size_t ldo,
                int64_t out_len, int accumulate, cudaStream_t st) {
  if (items == 0) return ST_OK;
  LargeFft L;
  if (int rc = get_large_fft(pl, &L)) return rc;
  const size_t sa = large_smem(L.a), sb = large_smem(L.b);
  if (int rc = set_smem(lf_rows_inv, sb)) return rc;
  if (int rc = set_smem(lf_cols_inv, sa)) return rc;
  lf_pairs<false><<<dim3(ceil_div(L.P / 2 + 1, 256), items), 256, 0, st>>>(L, spec, items);
  FCS_CUDA_TRY(cudaGetLastError());
  lf_rows_inv<<<dim3(L.P1, items), kFftThreads, sb, st>>>(L, spec);
  FCS_CUDA_TRY(cudaGetLastError());
  lf_cols_inv<<<dim3(L.P2, items), kFftThreads, sa, st>>>(L, spec, out, ldo, out_len, accumulate);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

// ------------------------------------------------------------ operations
int large_real_from_spec(const FftPlan& pl, const double2* spec, int items, double* out,
                         size_t ldo, int out_len, int accumulate, cudaStream_t st) {
  DevTmp tmp(st);
  const size_t bytes = static_cast<size_t>(items) * pl.P * sizeof(double2);
  if (int rc = tmp.alloc(bytes)) return rc;
  FCS_CUDA_TRY(cudaMemcpyAsync(tmp.p, spec, bytes, cudaMemcpyDeviceToDevice, st));
  return large_irfft(pl, static_cast<double2*>(tmp.p), items, out, ldo, out_len, accumulate, st);
}

int large_conv(const FftPlan& pl, const double* a, int la, size_t lda, const double* b, int lb,
               size_t ldb, int items, double* out, size_t ldo, cudaStream_t st) {
  DevTmp tmp(st);
  const size_t n = static_cast<size_t>(items) * pl.P;
  if (int rc = tmp.alloc(2 * n * sizeof(double2))) return rc;
  auto* fa = static_cast<double2*>(tmp.p);
  double2* fb = fa + n;
  if (int rc = large_rfft(pl, a, lda, la, items, fa, st)) return rc;
  if (int rc = large_rfft(pl, b, ldb, lb, items, fb, st)) return rc;
  lf_mul<<<grid_for(n), 256, 0, st>>>(fa, fb, n, pl.P);
  FCS_CUDA_TRY(cudaGetLastError());
  return large_irfft(pl, fa, items, out, ldo, la + lb - 1, 0, st);
}

// Count sketches of `rows` vectors for mode tab_off under all D families,
// then their spectra: spec[(r * sr + d * sd)].
static int cs_spectra(const FftPlan& pl, const double* U, size_t ldu, int I, int rows,
                      const uint32_t* packed, int fam_stride, int tab_off, int D, int J, size_t sr,
                      size_t sd, double* real_tmp, double2* spec, cudaStream_t st) {
  const size_t items = static_cast<size_t>(rows) * D;
  FCS_CUDA_TRY(cudaMemsetAsync(real_tmp, 0, items * J * sizeof(double), st));
  lf_cs_rows<<<grid_for(static_cast<size_t>(rows) * I), 256, 0, st>>>(
      U, ldu, I, rows, packed, fam_stride, tab_off, D, J, sr, sd, real_tmp);
  FCS_CUDA_TRY(cudaGetLastError());
  return large_rfft(pl, real_tmp, J, J, static_cast<int>(items), spec, st);
}

int large_iuv(const FftPlan& pl, const EngArgs& e, int batch, const double* A, const double* B,
              int c1, int c2, int f, int J, double* est, cudaStream_t st) {
  const size_t items = static_cast<size_t>(batch) * e.D;
  const size_t n = items * pl.P;
  DevTmp tmp(st);
  if (int rc = tmp.alloc(2 * n * sizeof(double2) + items * J * sizeof(double))) return rc;
  auto* fa = static_cast<double2*>(tmp.p);
  double2* fb = fa + n;
  auto* real = reinterpret_cast<double*>(fb + n);
  // item = b * D + d (as the fused kernel)
  if (int rc = cs_spectra(pl, A, e.dims[c1], e.dims[c1], batch, e.packed, e.fam_stride,
                          e.tab_off[c1], e.D, J, e.D, 1, real, fa, st))
    return rc;
  if (int rc = cs_spectra(pl, B, e.dims[c2], e.dims[c2], batch, e.packed, e.fam_stride,
                          e.tab_off[c2], e.D, J, e.D, 1, real, fb, st))
    return rc;
  lf_iuv_combine<<<grid_for(n), 256, 0, st>>>(e.spec, fa, fb, e.D, pl.P, n);
  FCS_CUDA_TRY(cudaGetLastError());
  if (int rc = large_irfft(pl, fa, static_cast<int>(items), real, J, J, 0, st)) return rc;
  lf_gather<<<grid_for(items * e.dims[f]), 256, 0, st>>>(real, J, e.packed, e.fam_stride,
                                                         e.tab_off[f], e.D, e.dims[f], items, est);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int large_uvw(const FftPlan& pl, const EngArgs& e, int batch, const double* U, const double* V,
              const double* W, int J, double* est, cudaStream_t st) {
  const size_t items = static_cast<size_t>(batch) * e.D;
  const size_t n = items * pl.P;
  DevTmp tmp(st);
  if (int rc = tmp.alloc(3 * n * sizeof(double2) + items * J * sizeof(double))) return rc;
  auto* fu = static_cast<double2*>(tmp.p);
  double2* fv = fu + n;
  double2* fw = fv + n;
  auto* real = reinterpret_cast<double*>(fw + n);
  const double* vecs[3] = {U, V, W};
  double2* specs[3] = {fu, fv, fw};
  for (int m = 0; m < 3; ++m)
    if (int rc = cs_spectra(pl, vecs[m], e.dims[m], e.dims[m], batch, e.packed, e.fam_stride,
                            e.tab_off[m], e.D, J, e.D, 1, real, specs[m], st))
      return rc;
  lf_uvw_dot<<<static_cast<unsigned>(items), 256, 0, st>>>(e.spec, fu, fv, fw, e.D, pl.P, pl.M, est);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int large_deflate(const FftPlan& pl, const EngArgs& e, double weight, const double* U,
                  const double* V, const double* W, int J, double2* spec, cudaStream_t st) {
  const size_t n = static_cast<size_t>(e.D) * pl.P;
  DevTmp tmp(st);
  if (int rc = tmp.alloc(3 * n * sizeof(double2) + static_cast<size_t>(e.D) * J * sizeof(double)))
    return rc;
  auto* fu = static_cast<double2*>(tmp.p);
  double2* fv = fu + n;
  double2* fw = fv + n;
  auto* real = reinterpret_cast<double*>(fw + n);
  const double* vecs[3] = {U, V, W};
  double2* specs[3] = {fu, fv, fw};
  for (int m = 0; m < 3; ++m)
    if (int rc = cs_spectra(pl, vecs[m], e.dims[m], e.dims[m], 1, e.packed, e.fam_stride,
                            e.tab_off[m], e.D, J, e.D, 1, real, specs[m], st))
      return rc;
  lf_deflate<<<grid_for(n), 256, 0, st>>>(spec, fu, fv, fw, weight, pl.P, n);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

// CP-form FCS (K2-K5): per mode the count sketches of the factor columns
// under every family, their spectra multiplied across modes, weighted sum
// over ranks, one inverse per family.
int large_cp(const FftPlan& pl, const CpArgs& a, int D, const uint32_t* packed, const int* J,
             double* out, int jt, int accumulate, cudaStream_t st) {
  const int R = a.r_count;
  const size_t items = static_cast<size_t>(D) * std::max(R, 1);
  const size_t n = items * pl.P;
  int jmax = 1;
  for (int m = 0; m < a.order; ++m) jmax = std::max(jmax, J[m]);
  DevTmp tmp(st);
  if (int rc = tmp.alloc((2 * n + static_cast<size_t>(D) * pl.P) * sizeof(double2) +
                         items * jmax * sizeof(double)))
    return rc;
  auto* q = static_cast<double2*>(tmp.p);
  double2* f = q + n;
  double2* acc = f + n;
  auto* real = reinterpret_cast<double*>(acc + static_cast<size_t>(D) * pl.P);
  if (R > 0) {
    for (int m = 0; m < a.order; ++m) {
      // factor columns r_begin.. are rows of length I_m; item = d * R + r
      const double* cols = a.factors[m] + static_cast<size_t>(a.r_begin) * a.dims[m];
      if (int rc = cs_spectra(pl, cols, a.dims[m], a.dims[m], R, packed, a.fam_stride,
                              a.tab_off[m], D, J[m], 1, R, real, m == 0 ? q : f, st))
        return rc;
      if (m > 0) {
        lf_mul<<<grid_for(n), 256, 0, st>>>(q, f, n, pl.P);
        FCS_CUDA_TRY(cudaGetLastError());
      }
    }
  }
  if (R > 0) {
    lf_rank_sum<<<grid_for(static_cast<size_t>(D) * pl.P), 256, 0, st>>>(q, a.weights, a.r_begin, R,
                                                                        pl.P, D, acc);
    FCS_CUDA_TRY(cudaGetLastError());
  } else {
    FCS_CUDA_TRY(cudaMemsetAsync(acc, 0, static_cast<size_t>(D) * pl.P * sizeof(double2), st));
  }
  return large_irfft(pl, acc, D, out, jt, jt, accumulate, st);
}

// ------------------------------------------------------------------ plans
int get_large_fft(const FftPlan& pl, LargeFft* out) {
  int dev = 0;
  FCS_CUDA_TRY(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<std::pair<int, int>, LargeFft> cache;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({dev, pl.M});
    if (it != cache.end()) {
      *out = it->second;
      return ST_OK;
    }
  }
  LargeFft L{};
  L.M = pl.M;
  L.P = pl.P;
  L.P1 = pl.large_p1;
  L.P2 = pl.P / pl.large_p1;
  if (int rc = get_fft_plan(2 * static_cast<size_t>(L.P1), &L.a)) return rc;
  if (int rc = get_fft_plan(2 * static_cast<size_t>(L.P2), &L.b)) return rc;
  if (L.a.P != L.P1 || L.b.P != L.P2) return fail(ST_EINVAL, "fft: inconsistent two-level plan");
  std::vector<int> f2p(L.P1), p2f(L.P1);
  FCS_CUDA_TRY(cudaMemcpy(f2p.data(), L.a.f2p, L.P1 * sizeof(int), cudaMemcpyDeviceToHost));
  for (int k = 0; k < L.P1; ++k) p2f[f2p[k]] = k;
  int* dp2f = nullptr;
  FCS_CUDA_TRY(cudaMalloc(&dp2f, L.P1 * sizeof(int)));
  FCS_CUDA_TRY(cudaMemcpy(dp2f, p2f.data(), L.P1 * sizeof(int), cudaMemcpyHostToDevice));
  L.p2f_a = dp2f;
  std::lock_guard<std::mutex> lock(mu);
  cache[{dev, pl.M}] = L;
  *out = L;
  return ST_OK;
}



// ------------------------------------------- exact-length DFT (Bluestein)
// The reference's dft / idft_real (fft.cpp:42-73) transform at EXACTLY
// n = J~ points (FFTW, any n, e.g. 8998 = 2 * 11 * 409). The spectral paths
// above pad to a smooth M instead, which is exact for every value the
// estimators read; the public dft / idft_real / fft_convolve / precompute_z
// entries, whose callers see every bin, use the chirp-z identity
//   jk = (j^2 + k^2 - (k - j)^2) / 2:
//   X[k] = ch_k sum_j (x_j ch_j) conj(ch_{k-j}),  ch_m = exp(s pi i m^2 / n)
// (s = -1 forward, +1 inverse): one circular convolution at a smooth complex
// length P >= 2n - 1 done with the library's own FFTs (fft.cuh in shared
// memory up to P = 6144, the two-level transform above beyond), m^2 reduced
// modulo 2n in integers before sincospi.
namespace {

__device__ __forceinline__ double2 chirp(int64_t m, int64_t n, double sign) {
  const int64_t r = (m % (2 * n)) * (m % (2 * n)) % (2 * n);
  double s, c;
  sincospi(sign * static_cast<double>(r) / static_cast<double>(n), &s, &c);
  return make_double2(c, s);
}

// A[item][j] = x_j ch_j (j < min(len, n)), 0 up to P. Real (xr) or complex (xc) rows.
__global__ void bs_prep_a(const double* __restrict__ xr, const double2* __restrict__ xc,
                          size_t ldx, int64_t len, int64_t n, int64_t P, double sign,
                          double2* __restrict__ A) {
  const size_t item = blockIdx.y;
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < P;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    if (j < n && j < len) {
      const double2 x = xr ? make_double2(xr[item * ldx + j], 0.0) : xc[item * ldx + j];
      v = cmul(x, chirp(j, n, sign));
    }
    A[item * P + j] = v;
  }
}

// B[m] = conj(ch_m) for |m| < n on the circle of P points, 0 elsewhere.
__global__ void bs_prep_b(int64_t n, int64_t P, double sign, double2* __restrict__ B) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < P;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    if (j < n) v = cconj(chirp(j, n, sign));
    else if (P - j < n) v = cconj(chirp(P - j, n, sign));
    B[j] = v;
  }
}

// In-place complex FFT of `items` rows of P points in global memory with a
// one-CTA plan: forward leaves the digit-reversed slot order, inverse takes
// it and returns natural order (unnormalised).
template <bool kForward>
__global__ void __launch_bounds__(kFftThreads) bs_cfft(FftPlan pl, double2* __restrict__ data) {
  extern __shared__ __align__(16) double2 bsm[];
  double2* tw = bsm;
  double2* buf = bsm + table_slots(pl, false);
  load_twiddles(tw, pl, false);
  double2* row = data + blockIdx.x * static_cast<size_t>(pl.P);
  for (int i = threadIdx.x; i < pl.P; i += blockDim.x) buf[swz(i)] = row[i];
  __syncthreads();
  if (kForward) {
    fft_forward(buf, pl, tw);
  } else {
    fft_inverse(buf, pl, tw);
  }
  for (int i = threadIdx.x; i < pl.P; i += blockDim.x) row[i] = buf[swz(i)];
}

__global__ void bs_mul(double2* __restrict__ A, const double2* __restrict__ B, int64_t P,
                       size_t total) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<size_t>(gridDim.x) * blockDim.x)
    A[q] = cmul(A[q], B[q % P]);
}

// out[item][k] = scale * ch_k conv[k], k < n.
__global__ void bs_final(const double2* __restrict__ A, int64_t n, int64_t P, double sign,
                         double scale, double2* __restrict__ out) {
  const size_t item = blockIdx.y;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[item * n + k] = cscale(cmul(A[item * P + k], chirp(k, n, sign)), scale);
}

// Real part scaled by 1/n into out, and per-row sums of re^2 and im^2 (fixed
// order: thread strides, then a shared-memory tree) for the residue check.
__global__ void bs_real_part(const double2* __restrict__ X, int64_t n, double* __restrict__ out,
                             double* __restrict__ norms) {
  __shared__ double sr[256], si[256];
  const size_t item = blockIdx.x;
  const double inv = 1.0 / static_cast<double>(n);
  double r2 = 0.0, i2 = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    const double2 v = X[item * n + k];
    const double re = v.x * inv, im = v.y * inv;
    out[item * n + k] = re;
    r2 += re * re;
    i2 += im * im;
  }
  sr[threadIdx.x] = r2;
  si[threadIdx.x] = i2;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (static_cast<int>(threadIdx.x) < s) {
      sr[threadIdx.x] += sr[threadIdx.x + s];
      si[threadIdx.x] += si[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    norms[2 * item] = sr[0];
    norms[2 * item + 1] = si[0];
  }
}

// G = S conj(Fa) conj(Fb) over n bins (precompute_z, estimators.cpp:151-167).
__global__ void bs_z_combine(const double2* __restrict__ S, const double2* __restrict__ Fa,
                             const double2* __restrict__ Fb, int64_t n, double2* __restrict__ G) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    G[k] = cmul(S[k], cconj(cmul(Fa[k], Fb[k])));
}

// acc[k] *= next[k] (fft_convolve's product, fft.cpp:79-82).
__global__ void bs_cmul_inplace(double2* __restrict__ acc, const double2* __restrict__ next,
                                int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    acc[k] = cmul(acc[k], next[k]);
}

unsigned grid64(int64_t n) {
  return static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 4096));
}

}  // namespace

// X = exact n-point DFT (sign -1) or unnormalised inverse (sign +1) of
// `items` rows: real rows xr (ldx apart, len used, zero-padded / truncated
// to n) or complex rows xc (ldx apart). out: items x n complex.
int exact_dft(const double* xr, const double2* xc, size_t ldx, size_t len, size_t n, int items,
              double sign, double2* out, cudaStream_t st) {
  if (items == 0) return ST_OK;
  FftPlan pl;
  if (int rc = get_fft_plan(2 * (2 * n - 1), &pl)) return rc;
  const int64_t P = pl.P;
  DevTmp tmp(st);
  if (int rc = tmp.alloc((static_cast<size_t>(items) + 1) * P * sizeof(double2))) return rc;
  auto* A = static_cast<double2*>(tmp.p);
  double2* B = A + static_cast<size_t>(items) * P;
  bs_prep_a<<<dim3(grid64(P), items), 256, 0, st>>>(xr, xc, ldx, static_cast<int64_t>(len),
                                                      static_cast<int64_t>(n), P, sign, A);
  FCS_CUDA_TRY(cudaGetLastError());
  bs_prep_b<<<grid64(P), 256, 0, st>>>(static_cast<int64_t>(n), P, sign, B);
  FCS_CUDA_TRY(cudaGetLastError());
  double scale = 1.0;
  if (!pl.large_p1) {
    const size_t sm = fft_smem_bytes(pl, false);
    if (int rc = set_smem(bs_cfft<true>, sm)) return rc;
    if (int rc = set_smem(bs_cfft<false>, sm)) return rc;
    bs_cfft<true><<<items + 1, kFftThreads, sm, st>>>(pl, A);  // rows of A, then B
    FCS_CUDA_TRY(cudaGetLastError());
    bs_mul<<<grid64(static_cast<int64_t>(items) * P), 256, 0, st>>>(
        A, B, P, static_cast<size_t>(items) * P);
    FCS_CUDA_TRY(cudaGetLastError());
    bs_cfft<false><<<items, kFftThreads, sm, st>>>(pl, A);
    FCS_CUDA_TRY(cudaGetLastError());
    scale = 1.0 / static_cast<double>(P);
  } else {
    LargeFft L;
    if (int rc = get_large_fft(pl, &L)) return rc;
    const size_t sa = large_smem(L.a), sb = large_smem(L.b);
    if (int rc = set_smem(lf_cols_fwd, sa)) return rc;
    if (int rc = set_smem(lf_rows_fwd, sb)) return rc;
    if (int rc = set_smem(lf_rows_inv, sb)) return rc;
    if (int rc = set_smem(lf_cols_inv, sa)) return rc;
    // complex rows viewed as packed reals: lf_cols_fwd's z[m] = x[2m] + i x[2m+1]
    double* Ad = reinterpret_cast<double*>(A);
    lf_cols_fwd<<<dim3(L.P2, items + 1), kFftThreads, sa, st>>>(L, Ad, 2 * P, 2 * P, A);
    FCS_CUDA_TRY(cudaGetLastError());
    lf_rows_fwd<<<dim3(L.P1, items + 1), kFftThreads, sb, st>>>(L, A);
    FCS_CUDA_TRY(cudaGetLastError());
    bs_mul<<<grid64(static_cast<int64_t>(items) * P), 256, 0, st>>>(
        A, B, P, static_cast<size_t>(items) * P);
    FCS_CUDA_TRY(cudaGetLastError());
    lf_rows_inv<<<dim3(L.P1, items), kFftThreads, sb, st>>>(L, A);
    FCS_CUDA_TRY(cudaGetLastError());
    lf_cols_inv<<<dim3(L.P2, items), kFftThreads, sa, st>>>(L, A, Ad, 2 * P, 2 * P, 0);
    FCS_CUDA_TRY(cudaGetLastError());
  }
  bs_final<<<dim3(grid64(static_cast<int64_t>(n)), items), 256, 0, st>>>(
      A, static_cast<int64_t>(n), P, sign, scale, out);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

// idft_real of `items` rows of n bins: out = Re(IDFT) / n, and the residue
// check of fft.cpp:69-71 (synchronous when check != 0).
int exact_idft_real(const double2* spec, size_t n, int items, double* out, int check,
                    cudaStream_t st) {
  if (items == 0) return ST_OK;
  DevTmp tmp(st);
  if (int rc = tmp.alloc(static_cast<size_t>(items) * n * sizeof(double2) + 16 * items + 16))
    return rc;
  auto* X = static_cast<double2*>(tmp.p);
  auto* norms = reinterpret_cast<double*>(X + static_cast<size_t>(items) * n);
  if (int rc = exact_dft(nullptr, spec, n, n, n, items, +1.0, X, st)) return rc;
  bs_real_part<<<items, 256, 0, st>>>(X, static_cast<int64_t>(n), out, norms);
  FCS_CUDA_TRY(cudaGetLastError());
  if (check) {
    std::vector<double> h(2 * static_cast<size_t>(items));
    FCS_CUDA_TRY(cudaMemcpyAsync(h.data(), norms, h.size() * sizeof(double),
                                 cudaMemcpyDeviceToHost, st));
    FCS_CUDA_TRY(cudaStreamSynchronize(st));
    for (int i = 0; i < items; ++i)
      if (std::sqrt(h[2 * i + 1]) > 1e-9 * std::sqrt(h[2 * i]) + 1e-12)
        return fail(ST_ENUMERIC, "idft_real: inverse transform is not real");
  }
  return ST_OK;
}

// fft_convolve (fft.cpp:75-84): F^-1(prod_i F(x_i, n)) at exactly n points.
int exact_fft_convolve(const double* const* inputs, const size_t* lens, size_t k, size_t n,
                       double* out, cudaStream_t st) {
  DevTmp tmp(st);
  if (int rc = tmp.alloc(2 * n * sizeof(double2))) return rc;
  auto* acc = static_cast<double2*>(tmp.p);
  double2* nxt = acc + n;
  if (int rc = exact_dft(inputs[0], nullptr, 0, lens[0], n, 1, -1.0, acc, st)) return rc;
  for (size_t i = 1; i < k; ++i) {
    if (int rc = exact_dft(inputs[i], nullptr, 0, lens[i], n, 1, -1.0, nxt, st)) return rc;
    bs_cmul_inplace<<<grid64(static_cast<int64_t>(n)), 256, 0, st>>>(acc, nxt,
                                                                      static_cast<int64_t>(n));
    FCS_CUDA_TRY(cudaGetLastError());
  }
  return exact_idft_real(acc, n, 1, out, 1, st);
}

// precompute_z (estimators.cpp:151-167): z = idft_real(S conj(F cs_a) conj(F cs_b)) at n.
int exact_precompute_z(const double2* spectrum, size_t n, const double* csa, size_t ja,
                       const double* csb, size_t jb, double* z, cudaStream_t st) {
  DevTmp tmp(st);
  if (int rc = tmp.alloc(3 * n * sizeof(double2))) return rc;
  auto* fa = static_cast<double2*>(tmp.p);
  double2* fb = fa + n;
  double2* g = fb + n;
  if (int rc = exact_dft(csa, nullptr, 0, ja, n, 1, -1.0, fa, st)) return rc;
  if (int rc = exact_dft(csb, nullptr, 0, jb, n, 1, -1.0, fb, st)) return rc;
  bs_z_combine<<<grid64(static_cast<int64_t>(n)), 256, 0, st>>>(spectrum, fa, fb,
                                                                  static_cast<int64_t>(n), g);
  FCS_CUDA_TRY(cudaGetLastError());
  return exact_idft_real(g, n, 1, z, 1, st);
}

}  // namespace fcs
