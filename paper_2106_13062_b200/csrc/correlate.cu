// Time-domain evaluation of the sketched contraction (the "direct" estimator
// path of the FCS / TS engines).
//
// The reference estimates T(I,a,b) for family d as (estimators.cpp:66-90)
//   z = idft_real(S_d . conj(F cs_a) . conj(F cs_b)),  est[i] = s_f(i) z[h_f(i)],
// with S_d = F(FCS_d(T)) at n = J~ = 3J - 2. In the time domain z is the
// circular cross-correlation z[m] = sum_j sk[(m + j) mod n] (cs_a * cs_b)[j]
// of the sketch with the linear convolution of the two count sketches; for
// the m the readout needs (m = h_f(i) < J) and the convolution's support
// (j <= 2J - 2) the index m + j <= 3J - 3 < n never wraps, so
//   est[i] = s_f(i) sum_{i1} a'(i1) Q[h_f(i) + h_c1(i1)],
//   Q[k]   = sum_{i2} b'(i2) sk[k + h_c2(i2)],   k < 2J - 1,
// with a'(i1) = s_c1(i1) a[i1] and b'(i2) = s_c2(i2) b[i2] (cs_sketch,
// sketch.cpp:105-116, kept as nonzero lists: a collision is two terms of the
// same sum). T(u,v,w) is <w, T(u,v,I)> (spectral_dot, estimators.cpp:38-64,
// by linearity). Same estimate, no transform: the inputs are sparse (at most
// I_n nonzeros of J per mode) and only I_f outputs are read, so where I is
// small against J the (2J - 1) x I_c2 product per item is cheaper than the
// length-n transforms, which run latency-bound at one item per SM. engine.cu
// picks the path per call by a cost rule fitted to measured A/B runs
// (profiles/corr_sweep_r02.txt; config 3 stays on the transforms);
// st_engine_set_path overrides it.
//
// Q, per family, is a product of a Hankel matrix of the sketch with the
// batch's B' (rows = the contracted mode's indices, split into bucket ranges
// so each CTA's sketch window is KT + J / ranks):
// corr_q_mma_kernel (batches of 2+): the fp64 tensor cores, mma.sync
//   m8n8k4.f64 (DMMA) — A(m, kk) = sk[k + m + h(row kk)] gathered from the
//   shared-memory window, B(kk, n) = B'(row kk, v); 8 or 16 vectors per CTA.
// corr_q_kernel (one vector, or ST_CORR_DFMA): DFMA, each thread KR k's x VB
//   vectors in registers, rows software-pipelined; for one vector a
//   matrix-vector product bound by shared-memory loads.
// corr_z_kernel: the readout, one item (vector, family) per CTA or its outputs
//   split over G CTAs within one wave: the range partials of Q_{v,d} summed
//   in a fixed order into shared memory, est[i] = s_f(i) sum_{i1} a'(i1)
//   Q[h_f(i) + h_c1(i1)] (row order), outputs dealt to lanes round-robin over
//   their bucket class mod 16 (fewer bank conflicts in the gathers); for
//   T(u,v,w) the block sum sum_i w[i] est[i]; the median over the families
//   (and the rtpm normalisation / refinement update) fused by the vector's
//   last CTA (tail.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>

#include "engine.cuh"
#include "tail.cuh"

namespace fcs {
namespace {

constexpr int kQChunk = 128;  // B' rows staged per pass
constexpr int kZThreads = 256;
constexpr int kMaxSplit = 4;

// Q partial of bucket range ks: the rows i2 whose bucket h(i2) lies in
// [hlo, hhi) = [ks*J/ksplit, (ks+1)*J/ksplit) (ascending i2), so the CTA's
// sketch window is KT + (hhi - hlo) - 1 instead of KT + J - 1:
// Qp[ks][v][d][k] = sum_{i2 : h(i2) in range} sk[k + h(i2)] B'(i2, v).
template <int TH, int VB, int KR>
__global__ void __launch_bounds__(TH)
corr_q_kernel(const double* __restrict__ sk, int jt, const uint32_t* __restrict__ packed,
              int fam_stride, int tab_c2, int n2, const double* __restrict__ b, int batch, int D,
              int K, int ktiles, int ksplit, int J, double* __restrict__ Qp) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int KT = TH * KR;
  int blk = blockIdx.x;
  const int kt = blk % ktiles;
  blk /= ktiles;
  const int d = blk % D;
  blk /= D;
  const int ks = blk % ksplit;
  const int v0 = (blk / ksplit) * VB;
  const int hlo = static_cast<int>(static_cast<long>(ks) * J / ksplit);
  const int hhi = static_cast<int>(static_cast<long>(ks + 1) * J / ksplit);
  const int win = KT + (hhi - hlo) - 1;
  double* sS = reinterpret_cast<double*>(smem);
  double* sB = sS + ((win + 1) & ~1);  // 16-byte aligned rows of VB
  int* sH = reinterpret_cast<int*>(sB + kQChunk * VB);
  int* sC = sH + kQChunk;  // signed (i2 + 1) of each staged row
  __shared__ int s_cnt;
  const int k0 = kt * KT;
  const double* S = sk + static_cast<size_t>(d) * jt + hlo;
  // the sketch window sk[k0 + hlo ...] by asynchronous 8-byte copies, all in
  // flight at once (a load-then-store loop serialises one L2 round trip each)
  for (int i = threadIdx.x; i < win; i += TH) {
    const int g = k0 + i;
    if (g + hlo < jt) {
      const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(sS + i));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(S + g));
    } else {
      sS[i] = 0.0;
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  const uint32_t* tab = packed + static_cast<size_t>(d) * fam_stride + tab_c2;
  double acc[KR][VB];
#pragma unroll
  for (int r = 0; r < KR; ++r)
#pragma unroll
    for (int v = 0; v < VB; ++v) acc[r][v] = 0.0;
  const int lane = threadIdx.x & 31;
  __shared__ int s_scan;
  int scan = 0;
  while (scan < n2) {
    __syncthreads();  // previous chunk consumed
    if (threadIdx.x < 32) {  // warp 0: the next <= kQChunk rows in range, ascending i2
      int cnt = 0;
      for (; scan < n2 && cnt + 32 <= kQChunk; scan += 32) {
        const int c = scan + lane;
        const uint32_t e = c < n2 ? __ldg(tab + c) : 0u;
        const int h = static_cast<int>(e & 0x7fffffffu);
        const bool in = c < n2 && h >= hlo && h < hhi;
        const unsigned m = __ballot_sync(0xffffffffu, in);
        if (in) {
          const int pos = cnt + __popc(m & ((1u << lane) - 1));
          sC[pos] = (e & 0x80000000u) ? -(c + 1) : (c + 1);
          sH[pos] = h - hlo;
        }
        cnt += __popc(m);
      }
      if (lane == 0) {
        s_cnt = cnt;
        s_scan = scan;
      }
    }
    __syncthreads();
    scan = s_scan;
    const int cn = s_cnt;
    if (cn == 0) continue;
    for (int i = threadIdx.x; i < cn * VB; i += TH) {  // raw b rows, all copies in flight
      const int r = i / VB, v = i - r * VB;
      if (v0 + v < batch) {
        const int cs = sC[r];
        const int c = (cs < 0 ? -cs : cs) - 1;
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(sB + i));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst),
                     "l"(b + static_cast<size_t>(v0 + v) * n2 + c));
      } else {
        sB[i] = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    for (int i = threadIdx.x; i < cn * VB; i += TH)  // B' = s_c2(i2) b
      if (sC[i / VB] < 0) sB[i] = -sB[i];
    __syncthreads();
    // software-pipelined rows: the next row's sketch values and B' are loaded
    // while the current row's KR x VB multiply-adds issue
    const double* sp = sS + threadIdx.x;
    double sv[KR], bv[VB];
    {
      const int h0 = sH[0];
#pragma unroll
      for (int r = 0; r < KR; ++r) sv[r] = sp[h0 + r * TH];
#pragma unroll
      for (int v = 0; v < VB; ++v) bv[v] = sB[v];
    }
    for (int c = 0; c < cn; ++c) {
      const int cn1 = min(c + 1, cn - 1);
      const int h1 = sH[cn1];
      double sn[KR], bn[VB];
#pragma unroll
      for (int r = 0; r < KR; ++r) sn[r] = sp[h1 + r * TH];
#pragma unroll
      for (int v = 0; v < VB; ++v) bn[v] = sB[cn1 * VB + v];
#pragma unroll
      for (int v = 0; v < VB; ++v)
#pragma unroll
        for (int r = 0; r < KR; ++r) acc[r][v] = fma(sv[r], bv[v], acc[r][v]);
#pragma unroll
      for (int r = 0; r < KR; ++r) sv[r] = sn[r];
#pragma unroll
      for (int v = 0; v < VB; ++v) bv[v] = bn[v];
    }
  }
  double* out = Qp + static_cast<size_t>(ks) * batch * D * K;
#pragma unroll
  for (int r = 0; r < KR; ++r) {
    const int k = k0 + threadIdx.x + r * TH;
    if (k >= K) continue;
#pragma unroll
    for (int v = 0; v < VB; ++v)
      if (v0 + v < batch) out[(static_cast<size_t>(v0 + v) * D + d) * K + k] = acc[r][v];
  }
}

// The same Q partial on the fp64 tensor cores (DMMA, mma.sync m8n8k4.f64):
// per warp MT x NT tiles of 8 k x 8 vectors, the k dimension of the MMA
// running over 4 staged rows: A(m, kk) = sk[k + m + h(row kk)] (a Hankel
// tile gathered from the sketch window), B(kk, n) = B'(row kk, v0 + n).
// One m8n8k4 is 256 multiply-adds for two fragment loads per lane, so the
// shared-memory pipe is far from binding and the tensor pipe reaches its
// rate from 8 warps per SM (tools/microbench/dmma_peak.cu: 36.6 TFLOP/s at
// 8 warps, while DFMA needs 2 issuing warps per SMSP for 32.5).
template <int NT, int MT>
__global__ void __launch_bounds__(128)
corr_q_mma_kernel(const double* __restrict__ sk, int jt, const uint32_t* __restrict__ packed,
                  int fam_stride, int tab_c2, int n2, const double* __restrict__ b, int batch,
                  int D, int K, int ktiles, int ksplit, int J, double* __restrict__ Qp) {
  constexpr int TH = 128, VB = 8 * NT, KT = 4 * 8 * MT;
  extern __shared__ __align__(16) unsigned char smem[];
  int blk = blockIdx.x;
  const int kt = blk % ktiles;
  blk /= ktiles;
  const int d = blk % D;
  blk /= D;
  const int ks = blk % ksplit;
  const int v0 = (blk / ksplit) * VB;
  const int hlo = static_cast<int>(static_cast<long>(ks) * J / ksplit);
  const int hhi = static_cast<int>(static_cast<long>(ks + 1) * J / ksplit);
  const int win = KT + (hhi - hlo) - 1;
  double* sS = reinterpret_cast<double*>(smem);
  double* sB = sS + ((win + 1) & ~1);
  int* sH = reinterpret_cast<int*>(sB + kQChunk * VB);
  int* sC = sH + kQChunk;
  __shared__ int s_cnt, s_scan;
  const int k0 = kt * KT;
  const double* S = sk + static_cast<size_t>(d) * jt + hlo;
  for (int i = threadIdx.x; i < win; i += TH) {
    const int g = k0 + i;
    if (g + hlo < jt) {
      const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(sS + i));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(S + g));
    } else {
      sS[i] = 0.0;
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  const uint32_t* tab = packed + static_cast<size_t>(d) * fam_stride + tab_c2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gm = lane >> 2, tg = lane & 3;  // fragment row / column group
  double acc[MT][NT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  int scan = 0;
  while (scan < n2) {
    __syncthreads();
    if (threadIdx.x < 32) {
      int cnt = 0;
      for (; scan < n2 && cnt + 32 <= kQChunk; scan += 32) {
        const int c = scan + lane;
        const uint32_t e = c < n2 ? __ldg(tab + c) : 0u;
        const int h = static_cast<int>(e & 0x7fffffffu);
        const bool in = c < n2 && h >= hlo && h < hhi;
        const unsigned m = __ballot_sync(0xffffffffu, in);
        if (in) {
          const int pos = cnt + __popc(m & ((1u << lane) - 1));
          sC[pos] = (e & 0x80000000u) ? -(c + 1) : (c + 1);
          sH[pos] = h - hlo;
        }
        cnt += __popc(m);
      }
      if (lane == 0) {
        s_cnt = cnt;
        s_scan = scan;
      }
    }
    __syncthreads();
    scan = s_scan;
    const int cn = s_cnt;
    if (cn == 0) continue;
    const int cn4 = (cn + 3) & ~3;  // rows padded to the MMA depth with B' = 0
    for (int i = threadIdx.x; i < cn4 * VB; i += TH) {
      const int r = i / VB, v = i - r * VB;
      if (r < cn && v0 + v < batch) {
        const int cs = sC[r];
        const int c = (cs < 0 ? -cs : cs) - 1;
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(sB + i));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst),
                     "l"(b + static_cast<size_t>(v0 + v) * n2 + c));
      } else {
        sB[i] = 0.0;
        if (v == 0 && r >= cn) sH[r] = 0;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    for (int i = threadIdx.x; i < cn * VB; i += TH)  // B' = s_c2(i2) b
      if (sC[i / VB] < 0) sB[i] = -sB[i];
    __syncthreads();
    const double* sa = sS + warp * 8 * MT + gm;
    for (int r4 = 0; r4 < cn4; r4 += 4) {
      const int h = sH[r4 + tg];
      double bf[NT];
#pragma unroll
      for (int n = 0; n < NT; ++n) bf[n] = sB[(r4 + tg) * VB + n * 8 + gm];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const double af = sa[m * 8 + h];
#pragma unroll
        for (int n = 0; n < NT; ++n)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(acc[m][n][0]), "+d"(acc[m][n][1])
              : "d"(af), "d"(bf[n]));
      }
    }
  }
  double* out = Qp + static_cast<size_t>(ks) * batch * D * K;
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    const int k = k0 + warp * 8 * MT + m * 8 + gm;
    if (k >= K) continue;
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int v = v0 + n * 8 + 2 * tg + j;
        if (v < batch) out[(static_cast<size_t>(v) * D + d) * K + k] = acc[m][n][j];
      }
  }
}

// One CTA per (vector, family): Q = sum of the ksplit partials (fixed order)
// in shared memory; thread (i, p) sums the i1 in part p of n1 for output i
// (4 independent accumulators), parts added in order.
// MODE 0: est[(v*D + d)*nf + i]; MODE 1: est[v*D + d] = sum_i w[v][i] est_i.
template <int MODE>
__global__ void __launch_bounds__(kZThreads)
corr_z_kernel(const double* __restrict__ Qp, int ksplit, size_t qstride, int K,
              const uint32_t* __restrict__ packed, int fam_stride, int tab_c1, int n1, int tab_f,
              int nf, const double* __restrict__ a, int D, const double* __restrict__ w, int G,
              double* __restrict__ est, IuvTail tail) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* sQ = reinterpret_cast<double*>(smem);
  double2* sAH = reinterpret_cast<double2*>(sQ + ((K + 1) & ~1));  // {a', bucket}
  double* sPart = reinterpret_cast<double*>(sAH + n1);               // [P][W]
  __shared__ double red[kZThreads / 32 + 1];
  const int item = blockIdx.x / G, g = blockIdx.x - item * G;  // G CTAs split the outputs
  const int v = item / D, d = item - v * D;
  const int nfg = (nf + G - 1) / G;
  const int ib = min(nf, g * nfg), ie = min(nf, ib + nfg);
  // Q = sum of the partials, eight rows of every partial in flight per thread
  const double* q0 = Qp + static_cast<size_t>(item) * K;
  for (int i = threadIdx.x; i < K; i += 8 * kZThreads) {
    double x[8][kMaxSplit];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int p = 0; p < kMaxSplit; ++p) {
        const int ii = i + j * kZThreads;
        x[j][p] = (p < ksplit && ii < K) ? q0[p * qstride + ii] : 0.0;
      }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double y = x[j][0];
#pragma unroll
      for (int p = 1; p < kMaxSplit; ++p)
        if (p < ksplit) y += x[j][p];
      if (i + j * kZThreads < K) sQ[i + j * kZThreads] = y;
    }
  }
  const uint32_t* tab1 = packed + static_cast<size_t>(d) * fam_stride + tab_c1;
  const uint32_t* tabf = packed + static_cast<size_t>(d) * fam_stride + tab_f;
  const double* av = a + static_cast<size_t>(v) * n1;
  for (int c = threadIdx.x; c < n1; c += kZThreads) {
    const uint32_t e = __ldg(tab1 + c);
    const double x = av[c];
    sAH[c] = make_double2((e & 0x80000000u) ? -x : x,
                          __hiloint2double(0, static_cast<int>(e & 0x7fffffffu)));
  }
  // Lane order of the outputs: the gather of output i at row c reads
  // sQ[h_f(i) + h_c1(c)], whose 8-byte bank is (h_f(i) + h_c1(c)) mod 16 — the
  // row shifts every lane's bank alike, so outputs dealt round-robin over the
  // 16 classes h_f(i) mod 16 keep each warp's 32 gathers at ~2 lanes per bank
  // (random outputs: ~4.5 wavefronts per gather). Any order gives the same
  // sums (each output is summed by one thread in row order).
  __shared__ int cls_cnt[16];
  const int ne = ie - ib;
  int* sRank = reinterpret_cast<int*>(sPart + kZThreads);  // (class << 16 | rank) per output
  int* sOrd = sRank + ne;                                   // position -> output
  if (threadIdx.x < 16) cls_cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < ne; k += kZThreads) {
    const int cls = static_cast<int>(__ldg(tabf + ib + k) & 15u);
    sRank[k] = (cls << 16) | atomicAdd(&cls_cnt[cls], 1);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < ne; k += kZThreads) {
    const int cls = sRank[k] >> 16, j = sRank[k] & 0xffff;
    int pos = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int n = cls_cnt[q];
      pos += min(j, n) + (q < cls && n > j ? 1 : 0);
    }
    sOrd[pos] = ib + k;
  }
  __syncthreads();
  const int W = max(1, min(ie - ib, kZThreads));
  const int P = kZThreads / W;
  const int iw = threadIdx.x % W, p = threadIdx.x / W;
  const int per = (n1 + P - 1) / P;
  const int cb = min(n1, p * per), ce = min(n1, cb + per);
  double part_w = 0.0;
  for (int i0 = ib; i0 < ie; i0 += W) {
    const int i = i0 + iw < ie ? sOrd[i0 + iw - ib] : ie;
    if (p < P && i < ie) {
      double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
      const double* q = sQ + (__ldg(tabf + i) & 0x7fffffffu);
      int c = cb;
      for (; c + 4 <= ce; c += 4) {
        const double2 e0 = sAH[c], e1 = sAH[c + 1], e2 = sAH[c + 2], e3 = sAH[c + 3];
        acc0 = fma(e0.x, q[__double2loint(e0.y)], acc0);
        acc1 = fma(e1.x, q[__double2loint(e1.y)], acc1);
        acc2 = fma(e2.x, q[__double2loint(e2.y)], acc2);
        acc3 = fma(e3.x, q[__double2loint(e3.y)], acc3);
      }
      for (; c < ce; ++c) {
        const double2 e0 = sAH[c];
        acc0 = fma(e0.x, q[__double2loint(e0.y)], acc0);
      }
      sPart[p * W + iw] = (acc0 + acc1) + (acc2 + acc3);
    }
    __syncthreads();
    if (p == 0 && i < ie) {
      double x = sPart[iw];
      for (int r = 1; r < P; ++r) x += sPart[r * W + iw];
      if (__ldg(tabf + i) & 0x80000000u) x = -x;
      if (MODE == 0)
        est[static_cast<size_t>(item) * nf + i] = x;
      else
        part_w += w[static_cast<size_t>(v) * nf + i] * x;
    }
    __syncthreads();
  }
  if (MODE == 1) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part_w += __shfl_xor_sync(0xffffffffu, part_w, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part_w;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s2 = 0.0;
      for (int k = 0; k < kZThreads / 32; ++k) s2 += red[k];
      est[item] = s2;
    }
  }
  if (tail.mode != 0)  // the last of vector v's D x G CTAs: median (+ normalise / refine)
    estimator_tail<kZThreads>(tail, est, v, D, MODE == 1 ? 1 : nf, D * G, red);
}

std::mutex g_mu;
std::map<std::pair<const void*, int>, size_t> g_smem;

template <typename Kern>
int ensure_smem(Kern kernel, size_t bytes) {
  int dev = 0;
  FCS_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  size_t& cur = g_smem[{reinterpret_cast<const void*>(kernel), dev}];
  if (bytes > cur) {
    FCS_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(bytes)));
    cur = bytes;
  }
  return ST_OK;
}

constexpr int kQKr = 4;
constexpr int kQMaxThreads = 128;

size_t q_smem(int J, int VB, int TH, int ks = 1) {
  const int win = TH * kQKr + (J + ks - 1) / ks;
  return static_cast<size_t>((win + 1) & ~1) * sizeof(double) +
         static_cast<size_t>(kQChunk) * VB * sizeof(double) + 2 * kQChunk * sizeof(int);
}
size_t z_smem(int K, int n1, int nf) {
  return static_cast<size_t>((K + 1) & ~1) * sizeof(double) + n1 * sizeof(double2) +
         kZThreads * sizeof(double) +  // sPart: P x W <= kZThreads
         2 * static_cast<size_t>(nf) * sizeof(int);  // output ranks and lane order
}

template <int TH, int VB>
int launch_q_vb(const double* sk, int jt, const uint32_t* packed, int fam_stride, int tab_c2,
                int n2, const double* b, int batch, int D, int K, int J, int ks, double* Qp,
                cudaStream_t st) {
  constexpr int KT = TH * kQKr;
  const int ktiles = (K + KT - 1) / KT;
  const int vblocks = (batch + VB - 1) / VB;
  const size_t sm = q_smem(J, VB, TH, ks);
  auto kern = corr_q_kernel<TH, VB, kQKr>;
  if (int rc = ensure_smem(kern, sm)) return rc;
  kern<<<static_cast<unsigned>(ktiles) * D * vblocks * ks, TH, sm, st>>>(
      sk, jt, packed, fam_stride, tab_c2, n2, b, batch, D, K, ktiles, ks, J, Qp);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

constexpr int kMmaMt = 8;

template <int NT>
int launch_q_mma(const double* sk, int jt, const uint32_t* packed, int fam_stride, int tab_c2,
                 int n2, const double* b, int batch, int D, int K, int J, int ks, double* Qp,
                 cudaStream_t st) {
  constexpr int KT = 4 * 8 * kMmaMt;
  const int ktiles = (K + KT - 1) / KT;
  const int vblocks = (batch + 8 * NT - 1) / (8 * NT);
  const int win = KT + (J + ks - 1) / ks;
  const size_t sm = static_cast<size_t>((win + 1) & ~1) * sizeof(double) +
                    static_cast<size_t>(kQChunk) * 8 * NT * sizeof(double) +
                    2 * kQChunk * sizeof(int);
  auto kern = corr_q_mma_kernel<NT, kMmaMt>;
  if (int rc = ensure_smem(kern, sm)) return rc;
  kern<<<static_cast<unsigned>(ktiles) * D * vblocks * ks, 128, sm, st>>>(
      sk, jt, packed, fam_stride, tab_c2, n2, b, batch, D, K, ktiles, ks, J, Qp);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

// Bucket-range splits: enough CTAs for ~12 resident warps per SM, each range
// at least 32 buckets wide, at most kMaxSplit ranges (the Z kernel reads
// every split's partial row).
int q_split(int ctas, int warps_per_cta, int J, int sms) {
  int ks = 1;
  while (ks < kMaxSplit && ctas * warps_per_cta * ks < 12 * sms && J / (2 * ks) >= 32) ks *= 2;
  return ks;
}

}  // namespace

// Largest hash length the direct path takes (Q_{v,d} of 2J - 1 doubles and
// the sketch window in one CTA's shared memory).
bool corr_feasible(const st_engine* e, size_t free_mode) {
  DeviceInfo di;
  if (device_info(&di)) return false;
  int c1, c2;
  contracted(free_mode, &c1, &c2);
  const int J = static_cast<int>(e->hash_len);
  const int K = 2 * J - 1;
  if (e->dims[c1] > 4096 || e->dims[free_mode] > (1u << 20)) return false;
  return z_smem(K, static_cast<int>(e->dims[c1]), static_cast<int>(e->dims[free_mode])) <=
             di.smem_optin &&
         q_smem(J, 16, 64) <= di.smem_optin && q_smem(J, 4, kQMaxThreads) <= di.smem_optin;
}

// est = per-family estimates (batch x D x nf), or with w != nullptr the
// per-family T(a, b, w) (batch x D); needs e->tsk current.
int corr_estimate(st_engine* e, size_t batch, const double* a, const double* b, size_t free_mode,
                  const double* w, double* est, cudaStream_t st, const IuvTail* tail) {
  int c1, c2;
  contracted(free_mode, &c1, &c2);
  DeviceInfo di;
  if (int rc = device_info(&di)) return rc;
  const EngArgs g = e->args();
  const int J = static_cast<int>(e->hash_len);
  const int K = 2 * J - 1;
  const int D = static_cast<int>(e->D);
  const int nb = static_cast<int>(batch);
  const double* sk = e->tsk;
  const int jt = static_cast<int>(e->jt);
  const int n2 = g.dims[c2];
  // vector-block width and CTA size: wide blocks (FMA-bound) use 64 threads
  // so the launch still has warps on every SM
  // batches of 2+: the tensor-core kernel (vector blocks of 8 or 16); a single
  // vector: the DFMA kernel (a matrix-vector product, shared-memory bound)
  const bool mma = nb >= 2 && !std::getenv("ST_CORR_DFMA");
  const int VB = mma ? (nb > 8 ? 16 : 8) : (nb >= 12 ? 16 : nb >= 6 ? 8 : nb >= 3 ? 4 : nb == 2 ? 2 : 1);
  const int TH = mma ? 128 : VB >= 8 ? 64 : kQMaxThreads;
  const int KT = mma ? 4 * 8 * kMmaMt : TH * kQKr;
  const int ctas = ((K + KT - 1) / KT) * D * ((nb + VB - 1) / VB);
  const int ks = q_split(ctas, TH / 32, J, di.sm_count);
  const size_t qstride = batch * e->D * K;
  if (int rc = e->corr.ensure(ks * qstride * sizeof(double), st)) return rc;
  auto* Qp = static_cast<double*>(e->corr.p);
  const int tab = g.tab_off[c2];
  int rc;
  if (mma) {
    rc = VB == 16 ? launch_q_mma<2>(sk, jt, g.packed, g.fam_stride, tab, n2, b, nb, D, K, J, ks, Qp, st)
                  : launch_q_mma<1>(sk, jt, g.packed, g.fam_stride, tab, n2, b, nb, D, K, J, ks, Qp, st);
  } else {
    switch (VB) {
      case 16: rc = launch_q_vb<64, 16>(sk, jt, g.packed, g.fam_stride, tab, n2, b, nb, D, K, J, ks, Qp, st); break;
      case 8: rc = launch_q_vb<64, 8>(sk, jt, g.packed, g.fam_stride, tab, n2, b, nb, D, K, J, ks, Qp, st); break;
      case 4: rc = launch_q_vb<kQMaxThreads, 4>(sk, jt, g.packed, g.fam_stride, tab, n2, b, nb, D, K, J, ks, Qp, st); break;
      case 2: rc = launch_q_vb<kQMaxThreads, 2>(sk, jt, g.packed, g.fam_stride, tab, n2, b, nb, D, K, J, ks, Qp, st); break;
      default: rc = launch_q_vb<kQMaxThreads, 1>(sk, jt, g.packed, g.fam_stride, tab, n2, b, nb, D, K, J, ks, Qp, st); break;
    }
  }
  if (rc) return rc;
  const int n1 = g.dims[c1], nf = g.dims[free_mode];
  const size_t sm = z_smem(K, n1, nf);
  const int items = nb * D;
  // few items (the rtpm refinement): split each item's outputs over G CTAs,
  // as many as keep the launch within ONE wave of resident CTAs (a launch a
  // few CTAs past a wave doubles its span: config 3's 150 items x 2 groups =
  // 300 CTAs on 296 slots measured 19 us, one group 150 CTAs ...)
  int occ = 1;
  {
    static std::mutex mu;
    static std::map<std::pair<int, size_t>, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_pair(di.device * 2 + (w ? 1 : 0), sm);
    auto it = cache.find(key);
    if (it == cache.end()) {
      int n = 0;
      if (w) {
        if (int rc2 = ensure_smem(corr_z_kernel<1>, sm)) return rc2;
        FCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, corr_z_kernel<1>, kZThreads, sm));
      } else {
        if (int rc2 = ensure_smem(corr_z_kernel<0>, sm)) return rc2;
        FCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, corr_z_kernel<0>, kZThreads, sm));
      }
      it = cache.emplace(key, std::max(n, 1)).first;
    }
    occ = it->second;
  }
  const int slots = occ * di.sm_count;
  const int G = w ? 1 : std::max(1, std::min(slots / std::max(items, 1), (nf + 31) / 32));
  IuvTail tl;
  if (tail) tl = *tail;
  const unsigned grid = static_cast<unsigned>(items) * G;
  if (w) {
    if (int rc2 = ensure_smem(corr_z_kernel<1>, sm)) return rc2;
    corr_z_kernel<1><<<grid, kZThreads, sm, st>>>(Qp, ks, qstride, K, g.packed, g.fam_stride,
                                                 g.tab_off[c1], n1, g.tab_off[free_mode], nf, a,
                                                 D, w, G, est, tl);
  } else {
    if (int rc2 = ensure_smem(corr_z_kernel<0>, sm)) return rc2;
    corr_z_kernel<0><<<grid, kZThreads, sm, st>>>(Qp, ks, qstride, K, g.packed, g.fam_stride,
                                                 g.tab_off[c1], n1, g.tab_off[free_mode], nf, a,
                                                 D, nullptr, G, est, tl);
  }
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace fcs
