// The remaining contraction-engine backends of make_contraction_engine
// (cpd.cpp:220-232): Plain (exact, cpd.cpp:36-59), HCS (cpd.cpp:128-158) and
// long-pair CS (cpd.cpp:160-197). All three reduce to the same batched
// order-3 contractions — contract3_free / contract3 (tensor.cpp:181-226) —
// over a "virtual" tensor per group g:
//   Plain: the fp64 tensor itself (one group);
//   HCS:   family d's J x J x J higher-order count sketch, contracted with the
//          count sketches of the vectors, then read out through the free
//          mode's pair (estimators.cpp:241-275);
//   CS:    X_d[l] = s_d(l) * sk_d[h_d(l)] with family d's long pair (h_d, s_d)
//          over all prod I_n flat indices, hashed on the fly from its seed
//          (estimators.cpp:277-350; the reference tabulates the same pair).
// Contractions batch items (vector pairs x groups) in chunks of kCB items per
// CTA, one CTA per last-mode slice, with fixed-order reductions.
#include <cuda_runtime.h>

#include <algorithm>

#include "engine.cuh"

namespace fcs {
namespace {

constexpr int kCB = 8;  // items per CTA chunk
constexpr int kThreads = 256;

struct DenseAcc {
  const double* X;
  size_t gstride;
  __device__ __forceinline__ double at(int g, size_t l) const { return X[g * gstride + l]; }
};

struct CsAcc {
  const double* sk;  // G x J
  const uint64_t* seeds;
  uint64_t J;
  __device__ __forceinline__ double at(int g, size_t l) const {
    const uint64_t s = seeds[g];
    const uint32_t h = static_cast<uint32_t>(mulhi64(splitmix_draw(s, 2 * l + 1), J));
    const double v = sk[g * J + h];
    return (splitmix_draw(s, 2 * l + 2) >> 63) ? -v : v;
  }
};

// Items (g, b), g < G groups, b < B vectors. Vector rows: kVecItem -> row
// g * B + b, kVecShared -> row b (same vectors for every group), kVecBG -> row
// b * G + g. Outputs are written in (b, g) order: row b * G + g.
enum { kVecItem = 0, kVecShared = 1, kVecBG = 2 };
struct Geo {
  int I[3];
  int G, B;
  int vec_mode;
  const double* A;  // contracted on the first contracted mode
  size_t lda;
  const double* V;  // contracted on the second contracted mode
  size_t ldv;
};

__device__ __forceinline__ size_t vec_row(const Geo& q, int g, int b) {
  return q.vec_mode == kVecShared ? static_cast<size_t>(b)
         : q.vec_mode == kVecBG   ? static_cast<size_t>(b) * q.G + g
                                  : static_cast<size_t>(g) * q.B + b;
}

__device__ __forceinline__ void chunk_of(const Geo& q, int c, int* g, int* b0, int* nb) {
  const int ncpg = (q.B + kCB - 1) / kCB;
  *g = c / ncpg;
  *b0 = (c % ncpg) * kCB;
  *nb = min(kCB, q.B - *b0);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// free mode 0 (contract3_free case 0): part[k][b*G+g][i0] = v_k * (slice_k a)_i0, 0 if v_k == 0
template <typename Acc>
__global__ void __launch_bounds__(kThreads) free0_kernel(Acc x, Geo q, double* __restrict__ part) {
  const int k = blockIdx.x;
  int g, b0, nb;
  chunk_of(q, blockIdx.y, &g, &b0, &nb);
  const size_t items = static_cast<size_t>(q.G) * q.B;
  const int I0 = q.I[0], I1 = q.I[1];
  const double* ar[kCB];
  double vk[kCB];
#pragma unroll
  for (int t = 0; t < kCB; ++t) {
    const int b = min(b0 + t, q.B - 1);
    ar[t] = q.A + vec_row(q, g, b) * q.lda;
    vk[t] = t < nb ? __ldg(q.V + vec_row(q, g, b) * q.ldv + k) : 0.0;
  }
  for (int i0 = threadIdx.x; i0 < I0; i0 += blockDim.x) {
    double acc[kCB];
#pragma unroll
    for (int t = 0; t < kCB; ++t) acc[t] = 0.0;
    const size_t base = static_cast<size_t>(k) * I1 * I0 + i0;
    for (int i1 = 0; i1 < I1; ++i1) {
      const double v = x.at(g, base + static_cast<size_t>(i1) * I0);
#pragma unroll
      for (int t = 0; t < kCB; ++t) acc[t] += v * __ldg(ar[t] + i1);
    }
#pragma unroll
    for (int t = 0; t < kCB; ++t)
      if (t < nb)
        part[(static_cast<size_t>(k) * items + static_cast<size_t>(b0 + t) * q.G + g) * I0 + i0] =
            vk[t] != 0.0 ? vk[t] * acc[t] : 0.0;
  }
}

// free mode 1 (case 1): part[k][b*G+g][i1] = v_k * (slice_k^T a)_i1
template <typename Acc>
__global__ void __launch_bounds__(kThreads) free1_kernel(Acc x, Geo q, double* __restrict__ part) {
  const int k = blockIdx.x;
  int g, b0, nb;
  chunk_of(q, blockIdx.y, &g, &b0, &nb);
  const size_t items = static_cast<size_t>(q.G) * q.B;
  const int I0 = q.I[0], I1 = q.I[1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* ar[kCB];
#pragma unroll
  for (int t = 0; t < kCB; ++t) ar[t] = q.A + vec_row(q, g, min(b0 + t, q.B - 1)) * q.lda;
  for (int i1 = warp; i1 < I1; i1 += nw) {
    double acc[kCB];
#pragma unroll
    for (int t = 0; t < kCB; ++t) acc[t] = 0.0;
    const size_t base = (static_cast<size_t>(k) * I1 + i1) * I0;
    for (int i0 = lane; i0 < I0; i0 += 32) {
      const double v = x.at(g, base + i0);
#pragma unroll
      for (int t = 0; t < kCB; ++t) acc[t] += v * __ldg(ar[t] + i0);
    }
#pragma unroll
    for (int t = 0; t < kCB; ++t) {
      const double s = warp_sum(acc[t]);
      if (lane == 0 && t < nb) {
        const double vk = __ldg(q.V + vec_row(q, g, b0 + t) * q.ldv + k);
        part[(static_cast<size_t>(k) * items + static_cast<size_t>(b0 + t) * q.G + g) * I1 + i1] =
            vk != 0.0 ? vk * s : 0.0;
      }
    }
  }
}

// free mode 2 (case 2): out[b*G+g][k] = a^T slice_k v
template <typename Acc>
__global__ void __launch_bounds__(kThreads) free2_kernel(Acc x, Geo q, double* __restrict__ out) {
  __shared__ double red[kThreads / 32][kCB];
  const int k = blockIdx.x;
  int g, b0, nb;
  chunk_of(q, blockIdx.y, &g, &b0, &nb);
  const int I0 = q.I[0], I1 = q.I[1], I2 = q.I[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* ar[kCB];
  const double* vr[kCB];
#pragma unroll
  for (int t = 0; t < kCB; ++t) {
    const size_t row = vec_row(q, g, min(b0 + t, q.B - 1));
    ar[t] = q.A + row * q.lda;
    vr[t] = q.V + row * q.ldv;
  }
  double tot[kCB];
#pragma unroll
  for (int t = 0; t < kCB; ++t) tot[t] = 0.0;
  for (int i1 = warp; i1 < I1; i1 += nw) {
    double acc[kCB];
#pragma unroll
    for (int t = 0; t < kCB; ++t) acc[t] = 0.0;
    const size_t base = (static_cast<size_t>(k) * I1 + i1) * I0;
    for (int i0 = lane; i0 < I0; i0 += 32) {
      const double v = x.at(g, base + i0);
#pragma unroll
      for (int t = 0; t < kCB; ++t) acc[t] += v * __ldg(ar[t] + i0);
    }
#pragma unroll
    for (int t = 0; t < kCB; ++t) tot[t] += warp_sum(acc[t]) * __ldg(vr[t] + i1);
  }
  if (lane == 0)
#pragma unroll
    for (int t = 0; t < kCB; ++t) red[warp][t] = tot[t];
  __syncthreads();
  if (static_cast<int>(threadIdx.x) < nb) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w][threadIdx.x];
    out[(static_cast<size_t>(b0 + threadIdx.x) * q.G + g) * I2 + k] = s;
  }
}

// out[r] = sum_k part[k][r] (fixed order)
__global__ void reduce_k_kernel(const double* __restrict__ part, int K, size_t per_k,
                                double* __restrict__ out) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < per_k;
       q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < K; ++k) s += part[static_cast<size_t>(k) * per_k + q];
    out[q] = s;
  }
}

// est[r] = sum_{k: w_k != 0} w_k m[r][k], w row r / w_div (contract3's loop, tensor.cpp:190-195)
__global__ void dot_w_kernel(const double* __restrict__ m, const double* __restrict__ W,
                             size_t ldw, int w_div, int I2, double* __restrict__ est) {
  __shared__ double red[32];
  const size_t r = blockIdx.x;
  const double* w = W + (r / w_div) * ldw;
  double s = 0.0;
  for (int k = threadIdx.x; k < I2; k += blockDim.x)
    if (w[k] != 0.0) s += w[k] * m[r * I2 + k];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) est[r] = t;
  }
}

// X_g[i0,i1,i2] -= weight * u_g[i0] v_g[i1] w_g[i2] (densify(rank_one), tensor.cpp:86-115)
__global__ void deflate_dense_kernel(double* __restrict__ X, size_t gstride, int G, int I0, int I1,
                                     const double* __restrict__ U, const double* __restrict__ V,
                                     const double* __restrict__ W, int I2, double weight) {
  const size_t n = static_cast<size_t>(G) * gstride;
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t g = q / gstride;
    size_t l = q - g * gstride;
    const int i0 = static_cast<int>(l % I0);
    l /= I0;
    const int i1 = static_cast<int>(l % I1);
    const int i2 = static_cast<int>(l / I1);
    X[q] -= weight * U[g * I0 + i0] * V[g * I1 + i1] * W[g * I2 + i2];
  }
}

// sk_g[h_g(l)] += scale * s_g(l) * value(l) over all flat indices l: cs_sketch of
// vec(T) (kRankOne false) or of densify(u o v o w) (true), zeros skipped
// (sketch.cpp:105-116). Shared-memory privatised when J fits.
template <bool kRankOne, typename Tin>
__global__ void cs_long_kernel(const Tin* __restrict__ t, const double* __restrict__ U,
                               const double* __restrict__ V, const double* __restrict__ W, int I0,
                               int I1, size_t total, const uint64_t* __restrict__ seeds, int G,
                               uint64_t J, double scale, double* __restrict__ sk, int use_smem) {
  extern __shared__ double acc[];
  for (int g = 0; g < G; ++g) {
    if (use_smem) {
      for (uint64_t b = threadIdx.x; b < J; b += blockDim.x) acc[b] = 0.0;
      __syncthreads();
    }
    const uint64_t s = seeds[g];
    for (size_t l = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; l < total;
         l += static_cast<size_t>(gridDim.x) * blockDim.x) {
      double v;
      if (kRankOne) {
        const size_t r = l / I0;
        v = U[l - r * I0] * V[r % I1] * W[r / I1];
      } else {
        v = static_cast<double>(t[l]);
      }
      if (v == 0.0) continue;
      const uint32_t h = static_cast<uint32_t>(mulhi64(splitmix_draw(s, 2 * l + 1), J));
      const double sv = ((splitmix_draw(s, 2 * l + 2) >> 63) ? -v : v) * scale;
      atomicAdd(use_smem ? acc + h : sk + g * J + h, sv);
    }
    if (use_smem) {
      __syncthreads();
      for (uint64_t b = threadIdx.x; b < J; b += blockDim.x)
        if (acc[b] != 0.0) atomicAdd(sk + g * J + b, acc[b]);
      __syncthreads();
    }
  }
}

// Count sketches of `rows` vectors (row r at U + r * ldu, I entries) under the
// D families' mode tables, into zeroed rows out[(r * D + d) * J].
__global__ void cs_rows_kernel(const double* __restrict__ U, size_t ldu, int I, int rows,
                               const uint32_t* __restrict__ packed, int fam_stride, int tab_off,
                               int D, int J, double* __restrict__ out) {
  const size_t n = static_cast<size_t>(rows) * I;
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = q / I;
    const int i = static_cast<int>(q - r * I);
    const double v = U[r * ldu + i];
    if (v == 0.0) continue;
    for (int d = 0; d < D; ++d) {
      const uint32_t e = __ldg(packed + static_cast<size_t>(d) * fam_stride + tab_off + i);
      atomicAdd(out + (r * D + d) * J + (e & 0x7fffffffu), (e >> 31) ? -v : v);
    }
  }
}

// est[r][i] = s_f(i) w[r][h_f(i)], r = b * D + d (the HCS readout, estimators.cpp:264-271)
__global__ void gather_kernel(const double* __restrict__ w, int J, const uint32_t* __restrict__ packed,
                              int fam_stride, int tab_off, int D, int nf, size_t rows,
                              double* __restrict__ est) {
  const size_t n = rows * nf;
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = q / nf;
    const int i = static_cast<int>(q - r * nf);
    const uint32_t e = __ldg(packed + (r % D) * fam_stride + tab_off + i);
    const double v = w[r * J + (e & 0x7fffffffu)];
    est[q] = (e >> 31) ? -v : v;
  }
}

__global__ void widen_kernel(const float* __restrict__ in, double* __restrict__ out, size_t n) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<size_t>(gridDim.x) * blockDim.x)
    out[q] = static_cast<double>(in[q]);
}

unsigned grid_for(size_t n) { return static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 8192)); }

// Batched contraction with the identity at free mode f; out rows b * G + g.
template <typename Acc>
int contract(const Acc& x, const Geo& q, int f, double* out, Scratch& scr, cudaStream_t st) {
  const size_t items = static_cast<size_t>(q.G) * q.B;
  if (items == 0) return ST_OK;
  const dim3 grid(q.I[2], q.G * ((q.B + kCB - 1) / kCB));
  if (f == 2) {
    free2_kernel<Acc><<<grid, kThreads, 0, st>>>(x, q, out);
    FCS_CUDA_TRY(cudaGetLastError());
    return ST_OK;
  }
  const size_t per_k = items * q.I[f];
  if (int rc = scr.ensure(static_cast<size_t>(q.I[2]) * per_k * sizeof(double), st)) return rc;
  auto* part = static_cast<double*>(scr.p);
  if (f == 0)
    free0_kernel<Acc><<<grid, kThreads, 0, st>>>(x, q, part);
  else
    free1_kernel<Acc><<<grid, kThreads, 0, st>>>(x, q, part);
  FCS_CUDA_TRY(cudaGetLastError());
  reduce_k_kernel<<<grid_for(per_k), 256, 0, st>>>(part, q.I[2], per_k, out);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

Geo make_geo(const int* I, int G, int B, int vec_mode, const double* A, size_t lda,
             const double* V, size_t ldv) {
  Geo q{};
  for (int n = 0; n < 3; ++n) q.I[n] = I[n];
  q.G = G;
  q.B = B;
  q.vec_mode = vec_mode;
  q.A = A;
  q.lda = lda;
  q.V = V;
  q.ldv = ldv;
  return q;
}

// HCS: count sketches of batch rows of `vecs` (length dims[m]) under every
// family's mode-m pair, rows (b * D + d) of length J.
int hcs_cs(st_engine* e, const double* vecs, size_t batch, int m, double* out, cudaStream_t st) {
  const size_t J = e->hash_len, D = e->D;
  FCS_CUDA_TRY(cudaMemsetAsync(out, 0, batch * D * J * sizeof(double), st));
  const EngArgs ea = e->args();
  cs_rows_kernel<<<grid_for(batch * e->dims[m]), 256, 0, st>>>(
      vecs, e->dims[m], static_cast<int>(e->dims[m]), static_cast<int>(batch), e->packed,
      ea.fam_stride, ea.tab_off[m], static_cast<int>(D), static_cast<int>(J), out);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace

// ------------------------------------------------------------ engine hooks
int exact_create(st_engine* e, int dtype, const void* tensor, cudaStream_t st) {
  const size_t n = e->dims[0] * e->dims[1] * e->dims[2];
  const int D = static_cast<int>(e->D);
  if (e->backend == ST_BACKEND_PLAIN) {  // PlainEngine holds the tensor (cpd.cpp:38)
    e->slen = 0;
    FCS_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&e->dense), n * sizeof(double)));
    if (dtype == ST_F64) {
      FCS_CUDA_TRY(cudaMemcpyAsync(e->dense, tensor, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    } else {
      widen_kernel<<<grid_for(n), 256, 0, st>>>(static_cast<const float*>(tensor), e->dense, n);
      FCS_CUDA_TRY(cudaGetLastError());
    }
    return ST_OK;
  }
  if (e->backend == ST_BACKEND_HCS) {  // precompute_hcs per family (estimators.cpp:241-243)
    const size_t J = e->hash_len;
    FCS_CHECK_ARG(J * J * J < (1ull << 31), "hcs_sketch: sketch tensor too large");
    e->slen = J * J * J;
    FCS_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&e->dense), D * e->slen * sizeof(double)));
    const size_t hl[3] = {J, J, J};
    const size_t wsb = dense_workspace(dtype, 3, e->dims, e->dims[2], D, hl, 1);
    void* ws = nullptr;
    FCS_CUDA_TRY(malloc_async(&ws, std::max<size_t>(wsb, 1), st));
    const int rc = launch_fcs_dense(dtype, tensor, 3, e->dims, 0, e->dims[2], D, e->packed, hl,
                                    e->dense, 0, ws, wsb, st, 0, 1);
    cudaFreeAsync(ws, st);
    return rc;
  }
  FCS_CHECK_ARG(e->backend == ST_BACKEND_CS, "make_contraction_engine: unknown backend");
  // D long pairs HashPair(prod I, J, family_seed(seed, d)) (cpd.cpp:162-166)
  const uint64_t J = e->hash_len;
  e->slen = J;
  FCS_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&e->dense), D * J * sizeof(double)));
  FCS_CUDA_TRY(cudaMemsetAsync(e->dense, 0, D * J * sizeof(double), st));
  DeviceInfo di;
  if (int rc = device_info(&di)) return rc;
  const size_t smem = J * sizeof(double);
  const int use_smem = smem <= 48 * 1024;
  const unsigned grid = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, di.sm_count * 8));
  const int I0 = static_cast<int>(e->dims[0]), I1 = static_cast<int>(e->dims[1]);
  if (dtype == ST_F64)
    cs_long_kernel<false, double><<<grid, 256, use_smem ? smem : 0, st>>>(
        static_cast<const double*>(tensor), nullptr, nullptr, nullptr, I0, I1, n, e->seeds, D, J,
        1.0, e->dense, use_smem);
  else
    cs_long_kernel<false, float><<<grid, 256, use_smem ? smem : 0, st>>>(
        static_cast<const float*>(tensor), nullptr, nullptr, nullptr, I0, I1, n, e->seeds, D, J,
        1.0, e->dense, use_smem);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

// est: batch x D x I_f for HCS / CS, batch x I_f for Plain (D = 1 output).
int exact_iuv(st_engine* e, size_t batch, const double* a, const double* b, int f, double* est,
              cudaStream_t st) {
  int c1, c2;
  contracted(f, &c1, &c2);
  const int I[3] = {static_cast<int>(e->dims[0]), static_cast<int>(e->dims[1]),
                    static_cast<int>(e->dims[2])};
  const int B = static_cast<int>(batch), D = static_cast<int>(e->D);
  if (e->backend == ST_BACKEND_PLAIN)
    return contract(DenseAcc{e->dense, 0}, make_geo(I, 1, B, kVecItem, a, I[c1], b, I[c2]), f, est,
                    e->scratch, st);
  if (e->backend == ST_BACKEND_CS)
    return contract(CsAcc{e->dense, e->seeds, e->hash_len},
                    make_geo(I, D, B, kVecShared, a, I[c1], b, I[c2]), f, est, e->scratch, st);
  // HCS: contract3_free(sketch_d, CS(a), CS(b), f) -> J-vector, then s_f(i) w[h_f(i)]
  const int J = static_cast<int>(e->hash_len);
  const size_t rows = batch * D;
  if (int rc = e->vec2.ensure(3 * rows * J * sizeof(double), st)) return rc;
  auto* csa = static_cast<double*>(e->vec2.p);
  double* csb = csa + rows * J;
  double* w = csb + rows * J;
  if (int rc = hcs_cs(e, a, batch, c1, csa, st)) return rc;
  if (int rc = hcs_cs(e, b, batch, c2, csb, st)) return rc;
  const int JJ[3] = {J, J, J};
  if (int rc = contract(DenseAcc{e->dense, e->slen}, make_geo(JJ, D, B, kVecBG, csa, J, csb, J), f,
                        w, e->scratch, st))
    return rc;
  const EngArgs ea = e->args();
  gather_kernel<<<grid_for(rows * I[f]), 256, 0, st>>>(w, J, e->packed, ea.fam_stride, ea.tab_off[f],
                                                       D, I[f], rows, est);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

// est: batch x D (batch for Plain).
int exact_uvw(st_engine* e, size_t batch, const double* u, const double* v, const double* w,
              double* est, cudaStream_t st) {
  const int I[3] = {static_cast<int>(e->dims[0]), static_cast<int>(e->dims[1]),
                    static_cast<int>(e->dims[2])};
  const int B = static_cast<int>(batch), D = static_cast<int>(e->D);
  if (e->backend == ST_BACKEND_PLAIN || e->backend == ST_BACKEND_CS) {
    const int G = e->backend == ST_BACKEND_PLAIN ? 1 : D;
    if (int rc = e->vec2.ensure(batch * G * I[2] * sizeof(double), st)) return rc;
    auto* m = static_cast<double*>(e->vec2.p);
    int rc;
    if (e->backend == ST_BACKEND_PLAIN)
      rc = contract(DenseAcc{e->dense, 0}, make_geo(I, 1, B, kVecItem, u, I[0], v, I[1]), 2, m,
                    e->scratch, st);
    else
      rc = contract(CsAcc{e->dense, e->seeds, e->hash_len},
                    make_geo(I, D, B, kVecShared, u, I[0], v, I[1]), 2, m, e->scratch, st);
    if (rc) return rc;
    dot_w_kernel<<<static_cast<unsigned>(batch * G), 256, 0, st>>>(m, w, I[2], G, I[2], est);
    FCS_CUDA_TRY(cudaGetLastError());
    return ST_OK;
  }
  // HCS: contract3(sketch_d, CS(u), CS(v), CS(w)) (estimators.cpp:245-255)
  const int J = static_cast<int>(e->hash_len);
  const size_t rows = batch * D;
  if (int rc = e->vec2.ensure(4 * rows * J * sizeof(double), st)) return rc;
  auto* cu = static_cast<double*>(e->vec2.p);
  double* cv = cu + rows * J;
  double* cw = cv + rows * J;
  double* m = cw + rows * J;
  if (int rc = hcs_cs(e, u, batch, 0, cu, st)) return rc;
  if (int rc = hcs_cs(e, v, batch, 1, cv, st)) return rc;
  if (int rc = hcs_cs(e, w, batch, 2, cw, st)) return rc;
  const int JJ[3] = {J, J, J};
  if (int rc = contract(DenseAcc{e->dense, e->slen}, make_geo(JJ, D, B, kVecBG, cu, J, cv, J), 2,
                        m, e->scratch, st))
    return rc;
  dot_w_kernel<<<static_cast<unsigned>(rows), 256, 0, st>>>(m, cw, J, 1, J, est);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int exact_deflate(st_engine* e, double weight, const double* u, const double* v, const double* w,
                  cudaStream_t st) {
  const int I0 = static_cast<int>(e->dims[0]), I1 = static_cast<int>(e->dims[1]),
            I2 = static_cast<int>(e->dims[2]);
  if (e->backend == ST_BACKEND_PLAIN) {  // tensor_ -= densify(rank_one) (cpd.cpp:52-55)
    const size_t n = static_cast<size_t>(I0) * I1 * I2;
    deflate_dense_kernel<<<grid_for(n), 256, 0, st>>>(e->dense, n, 1, I0, I1, u, v, w, I2, weight);
    FCS_CUDA_TRY(cudaGetLastError());
    return ST_OK;
  }
  if (e->backend == ST_BACKEND_CS) {  // sketch -= cs_sketch(densify(rank_one)) (cpd.cpp:182-189)
    const size_t n = static_cast<size_t>(I0) * I1 * I2;
    DeviceInfo di;
    if (int rc = device_info(&di)) return rc;
    const size_t smem = e->hash_len * sizeof(double);
    const int use_smem = smem <= 48 * 1024;
    const unsigned grid = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, di.sm_count * 8));
    cs_long_kernel<true, double><<<grid, 256, use_smem ? smem : 0, st>>>(
        nullptr, u, v, w, I0, I1, n, e->seeds, static_cast<int>(e->D), e->hash_len, -weight,
        e->dense, use_smem);
    FCS_CUDA_TRY(cudaGetLastError());
    return ST_OK;
  }
  // HCS: sketch -= hcs_sketch(rank_one) = weight * CS(u) o CS(v) o CS(w) (cpd.cpp:148-153)
  const int J = static_cast<int>(e->hash_len), D = static_cast<int>(e->D);
  if (int rc = e->vec2.ensure(3 * static_cast<size_t>(D) * J * sizeof(double), st)) return rc;
  auto* cu = static_cast<double*>(e->vec2.p);
  double* cv = cu + static_cast<size_t>(D) * J;
  double* cw = cv + static_cast<size_t>(D) * J;
  if (int rc = hcs_cs(e, u, 1, 0, cu, st)) return rc;
  if (int rc = hcs_cs(e, v, 1, 1, cv, st)) return rc;
  if (int rc = hcs_cs(e, w, 1, 2, cw, st)) return rc;
  deflate_dense_kernel<<<grid_for(static_cast<size_t>(D) * e->slen), 256, 0, st>>>(
      e->dense, e->slen, D, J, J, cu, cv, cw, J, weight);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace fcs
