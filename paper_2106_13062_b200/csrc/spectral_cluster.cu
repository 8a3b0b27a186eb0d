// K6 over a thread-block cluster: the sketched contraction T(I, a, b) of one
// (vector, family) item spread over 8 CTAs that exchange their transposes
// through distributed shared memory (iuv_spectral, estimators.cpp:66-90).
//
// The one-CTA kernel (spectral.cu, iuv1_kernel) runs one item per CTA at 8
// warps: each P = 4608-point pass is fp64-issue and latency bound, and a
// batch of 10-150 items leaves most SMs idle (config 3: 12.6 % warps active,
// the batch-1 refinement step on 10 SMs). Here an item is a cluster of 8 CTAs
// and the length-M transforms are four-step transforms whose transposes go
// over DSMEM:
//
//   forward, complex M = 64 * N2 points of w = cs_a + i cs_b (n = n1 + 64 n2):
//     F1  CTA r: columns n1 in [8r, 8r+8): N2-point DFTs over n2 (two radix
//         passes), twiddle w_M^{n1 k2}, store to the owner of k2 (remote);
//     F3  CTA r: its k2 rows (mirror-closed: k2 and N2 - k2 together):
//         64-point DFTs over n1 -> X[k2 + N2 k1];
//   product: A = (X[k] + conj X[-k]) / 2, B = (X[k] - conj X[-k]) / 2i
//         (both real sketches from one complex transform; -k stays in the
//         CTA), G = S_d conj(A B), then the c2r pre map over (k, k + M/2)
//         (same row) -> U[k], k < P = M/2;
//   inverse, P = 32 * N2 points (k = k2 + N2 k1):
//     I1  per k2 row: 32-point inverse DFT over k1, twiddle w_P^{-m1 k2},
//         store to the owner of m1 (CTA r: m1 in [4r, 4r+4));
//     I3  per m1: N2-point inverse DFT over k2 -> u[m1 + 32 m2] =
//         P (z[2m] + i z[2m+1]);
//   gather est[i] = s_f(i) z[h_f(i)] by the CTA that holds z[h_f(i)].
//
// The cached spectrum S_d is read in frequency order through the plan's
// frequency -> slot table. Same arithmetic as the one-CTA path up to fp64
// round-off (different factorisation of the same transform length).
//
// Users of the same distributed transform (ClFft): the estimator with its
// fused tails (IuvTail: median over the D families by the last cluster to
// finish, the rtpm row normalisation / refinement update, and T(u,v,w) as
// <w, T(u,v,I)> per family), the row-pair linear convolution (config 5) and
// the per-family inverse of a half spectrum (the CP sketch's last step).
// M = 64 N2 with N2 in {32, 48, 64, 96, 128, 144, 192}.
#include <cooperative_groups.h>
#include <cstdlib>

#include "fft.cuh"
#include "median.cuh"

namespace fcs {

namespace cg = cooperative_groups;

namespace {

constexpr int kClC = 8;          // CTAs per item
constexpr int kN1 = 64;          // forward: M = 64 N2

template <int RA, int RB>
struct ClGeom {
  static constexpr int N2 = RA * RB;
  static constexpr int M = kN1 * N2;
  static constexpr int P = M / 2;
  static constexpr int Q = N2 / (2 * kClC);  // mirror classes of k2 per CTA
  static constexpr int ROWS = 2 * Q;         // k2 rows per CTA
  static constexpr int COLS = kN1 / kClC;    // n1 columns per CTA
  static constexpr int M1 = 32 / kClC;       // inverse m1 per CTA
  static_assert(N2 % (2 * kClC) == 0, "N2 must be a multiple of 16");
  // U rows (ROWS x 32) and the I3 rows (M1 x N2) share the F1 column buffer
  static_assert(ROWS * 32 + M1 * N2 <= COLS * N2, "column buffer too small");
  static constexpr int kTw = (1 << kTwLoBits) + (M >> kTwLoBits);
  static constexpr size_t smem_bytes() {
    return static_cast<size_t>(kTw + COLS * N2 + ROWS * kN1) * sizeof(double2);
  }
};

// Slot swizzle of the DSMEM-exchanged buffers: bits 0-2 (16-byte slot in a
// 128-byte wavefront) XOR bits 3-5 and 4-6, so the stride-1, -4, -8 and -16
// slot patterns of the passes fall on distinct bank groups.
__device__ __forceinline__ int sw(int s) { return s ^ (((s >> 3) ^ (s >> 4)) & 7); }
__device__ __forceinline__ int pick3(const int* v, int i) { return i == 0 ? v[0] : i == 1 ? v[1] : v[2]; }

// k2 -> (owning CTA, local row); row -> k2. Class c = min(k2, N2 - k2) except
// that k2 = N2/2 joins class 0 (with k2 = 0) as its second member.
template <int N2, int Q>
__device__ __forceinline__ void k2_owner(int k2, int& owner, int& row) {
  const int h = N2 / 2;
  const int cls = k2 == h ? 0 : min(k2, N2 - k2);
  const int member = (k2 == 0 || k2 < h) ? 0 : 1;
  owner = cls / Q;
  row = 2 * (cls % Q) + member;
}
template <int N2, int Q>
__device__ __forceinline__ int row_k2(int r, int row) {
  const int cls = r * Q + (row >> 1);
  if ((row & 1) == 0) return cls;
  return cls == 0 ? N2 / 2 : N2 - cls;
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// The distributed transform shared by the cluster kernels. Buffers (slot
// indices swizzled by sw): colbuf [COLS][N2] F1 columns, later U rows
// [ROWS][32] and the I3 rows [M1][N2] behind them; rowbuf [ROWS][64] F3 rows.
template <int RA, int RB, int kThreads>
struct ClFft {
  using Gm = ClGeom<RA, RB>;
  static constexpr int N2 = Gm::N2, M = Gm::M, P = Gm::P, Q = Gm::Q, ROWS = Gm::ROWS,
                       COLS = Gm::COLS, M1 = Gm::M1;
  static constexpr int hi = 1 << kTwLoBits;
  const double2* tw;
  double2* colbuf;
  double2* rowbuf;
  double2* ubuf;
  double2* ibuf;
  int r, t0;

  __device__ ClFft(unsigned char* smem, int rank)
      : tw(reinterpret_cast<double2*>(smem)), r(rank), t0(threadIdx.x) {
    colbuf = reinterpret_cast<double2*>(smem) + Gm::kTw;
    rowbuf = colbuf + COLS * N2;
    ubuf = colbuf;
    ibuf = colbuf + ROWS * 32;  // F1 columns are dead after the first cluster barrier
  }

  // F1 pass A: DFT_RB over b of x[a + RA b], twiddle w_N2^{a kb}
  __device__ void f1a() const {
    for (int u = t0; u < COLS * RA; u += kThreads) {
      const int j = u / RA, a = u % RA;
      const int c = j * N2 + a;
      double2 x[RB];
#pragma unroll
      for (int q = 0; q < RB; ++q) x[q] = colbuf[sw(c + RA * q)];
      RegDft<RB>::run(x, -1.0);
#pragma unroll
      for (int kb = 1; kb < RB; ++kb)
        if (a) x[kb] = cmul(x[kb], twiddle(tw, hi, static_cast<uint32_t>((kN1 * a * kb) % M)));
#pragma unroll
      for (int q = 0; q < RB; ++q) colbuf[sw(c + RA * q)] = x[q];
    }
  }
  // F1 pass B: DFT_RA over a -> t[kb + RB ka]; twiddle w_M^{n1 k2}; to the owner of k2;
  // then the cluster barrier and F3 (64-point DFTs over n1, 8 x 8, in place:
  // slot ka + 8 kb <- X[k2 + N2 (kb + 8 ka)])
  __device__ void f1b_f3(cg::cluster_group& cl) const {
    for (int u = t0; u < COLS * RB; u += kThreads) {
      const int j = u / RB, kb = u % RB;
      const int n1 = COLS * r + j;
      const int c = j * N2 + RA * kb;
      double2 y[RA];
#pragma unroll
      for (int q = 0; q < RA; ++q) y[q] = colbuf[sw(c + q)];
      RegDft<RA>::run(y, -1.0);
#pragma unroll
      for (int ka = 0; ka < RA; ++ka) {
        const int k2 = kb + RB * ka;
        const double2 v =
            (n1 * k2) ? cmul(y[ka], twiddle(tw, hi, static_cast<uint32_t>(n1 * k2))) : y[ka];
        int owner, row;
        k2_owner<N2, Q>(k2, owner, row);
        double2* dst = cl.map_shared_rank(rowbuf, owner);
        dst[sw(row * kN1 + n1)] = v;
      }
    }
    cl.sync();
    for (int u = t0; u < ROWS * 8; u += kThreads) {
      const int row = u >> 3, a = u & 7;
      const int c = row * kN1 + a;
      double2 x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = rowbuf[sw(c + 8 * q)];
      RegDft<8>::run(x, -1.0);
#pragma unroll
      for (int kb = 1; kb < 8; ++kb)
        if (a) x[kb] = cmul(x[kb], twiddle(tw, hi, static_cast<uint32_t>(N2 * a * kb)));
#pragma unroll
      for (int q = 0; q < 8; ++q) rowbuf[sw(c + 8 * q)] = x[q];
    }
    __syncthreads();
    for (int u = t0; u < ROWS * 8; u += kThreads) {
      const int row = u >> 3, kb = u & 7;
      const int c = row * kN1 + 8 * kb;
      double2 y[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) y[q] = rowbuf[sw(c + q)];
      RegDft<8>::run(y, -1.0);
#pragma unroll
      for (int q = 0; q < 8; ++q) rowbuf[sw(c + q)] = y[q];
    }
    __syncthreads();
  }
  // Spectra of both real inputs at k = k2 + N2 kk (w = a + i b): A = (X[k] + conj X[-k]) / 2,
  // B = (X[k] - conj X[-k]) / 2i; -k stays in this CTA.
  __device__ void spectra(int row, int k2, int kk, double2& a2, double2& b2) const {
    const int mrow = (k2 == 0 || k2 == N2 / 2) ? row : (row ^ 1);
    const int km = k2 == 0 ? ((kN1 - kk) & (kN1 - 1)) : (kN1 - 1 - kk);
    const double2 X = rowbuf[sw(row * kN1 + (kk >> 3) + 8 * (kk & 7))];
    const double2 Xm = rowbuf[sw(mrow * kN1 + (km >> 3) + 8 * (km & 7))];
    a2 = make_double2(0.5 * (X.x + Xm.x), 0.5 * (X.y - Xm.y));
    b2 = make_double2(0.5 * (X.y + Xm.y), -0.5 * (X.x - Xm.x));
  }
  // The c2r pre map of G at k and k + P (k = k2 + N2 k1, k1 < 32) into U.
  __device__ void put_u(int row, int k2, int k1, double2 g0, double2 g1) const {
    const int k = k2 + N2 * k1;
    const double2 ev = make_double2(0.5 * (g0.x + g1.x), 0.5 * (g0.y + g1.y));
    double2 ov = make_double2(0.5 * (g0.x - g1.x), 0.5 * (g0.y - g1.y));
    if (k) ov = cmul(ov, cconj(twiddle(tw, hi, static_cast<uint32_t>(k))));
    ubuf[sw(row * 32 + k1)] = make_double2(ev.x - ov.y, ev.y + ov.x);
  }
  // I1 (32-point inverse DFTs over k1 = a + 4 b), twiddle w_P^{-m1 k2}, to the
  // owner of m1; the cluster barrier; I3 (N2-point inverse DFTs over k2):
  // ibuf slot ma + RA mb of local row m1 % M1 <- P u[m1 + 32 (mb + RB ma)].
  __device__ void inverse(cg::cluster_group& cl) const {
    for (int u = t0; u < ROWS * 4; u += kThreads) {
      const int row = u >> 2, a = u & 3;
      const int c = row * 32 + a;
      double2 x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = ubuf[sw(c + 4 * q)];
      RegDft<8>::run(x, +1.0);
#pragma unroll
      for (int mb = 1; mb < 8; ++mb)
        if (a)
          x[mb] = cmul(x[mb], cconj(twiddle(tw, hi, static_cast<uint32_t>((M / 32) * a * mb))));
#pragma unroll
      for (int q = 0; q < 8; ++q) ubuf[sw(c + 4 * q)] = x[q];
    }
    __syncthreads();
    for (int u = t0; u < ROWS * 8; u += kThreads) {
      const int row = u >> 3, mb = u & 7;
      const int k2 = row_k2<N2, Q>(r, row);
      const int c = row * 32 + 4 * mb;
      double2 y[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) y[q] = ubuf[sw(c + q)];
      RegDft<4>::run(y, +1.0);
#pragma unroll
      for (int ma = 0; ma < 4; ++ma) {
        const int m1 = mb + 8 * ma;
        const int e2 = (2 * m1 * k2) % M;  // w_P^{m1 k2} = w_M^{2 m1 k2}
        const double2 v =
            e2 ? cmul(y[ma], cconj(twiddle(tw, hi, static_cast<uint32_t>(e2)))) : y[ma];
        double2* dst = cl.map_shared_rank(ibuf, m1 / M1);
        dst[sw((m1 % M1) * N2 + k2)] = v;
      }
    }
    cl.sync();
    for (int u = t0; u < M1 * RA; u += kThreads) {
      const int ml = u / RA, a = u % RA;
      const int c = ml * N2 + a;
      double2 x[RB];
#pragma unroll
      for (int q = 0; q < RB; ++q) x[q] = ibuf[sw(c + RA * q)];
      RegDft<RB>::run(x, +1.0);
#pragma unroll
      for (int mb = 1; mb < RB; ++mb)
        if (a)
          x[mb] = cmul(x[mb], cconj(twiddle(tw, hi, static_cast<uint32_t>((kN1 * a * mb) % M))));
#pragma unroll
      for (int q = 0; q < RB; ++q) ibuf[sw(c + RA * q)] = x[q];
    }
    __syncthreads();
    for (int u = t0; u < M1 * RB; u += kThreads) {
      const int ml = u / RB, mb = u % RB;
      const int c = ml * N2 + RA * mb;
      double2 y[RA];
#pragma unroll
      for (int q = 0; q < RA; ++q) y[q] = ibuf[sw(c + q)];
      RegDft<RA>::run(y, +1.0);
#pragma unroll
      for (int q = 0; q < RA; ++q) ibuf[sw(c + q)] = y[q];
    }
    __syncthreads();
  }
  // z[h] (times P) if this CTA holds it: u[h / 2], component h % 2
  __device__ bool owns(int h) const { return ((h >> 1) & 31) / M1 == r; }
  __device__ double zval(int h) const {
    const int m = h >> 1;
    const int m1 = m & 31, m2 = m >> 5;
    const double2 v = ibuf[sw((m1 % M1) * N2 + (m2 / RB) + RA * (m2 % RB))];
    return (h & 1) ? v.y : v.x;
  }
  // twiddle table: loads issued into registers (stored by store_tw)
  static constexpr int kTwPer = (Gm::kTw + kThreads - 1) / kThreads;
  __device__ void load_tw(const FftPlan& pl, double2 (&twr)[kTwPer]) const {
#pragma unroll
    for (int q = 0; q < kTwPer; ++q) {
      const int i = t0 + q * kThreads;
      if (i < Gm::kTw) twr[q] = __ldg(pl.tw + i);
    }
  }
  __device__ void store_tw(const double2 (&twr)[kTwPer]) const {
#pragma unroll
    for (int q = 0; q < kTwPer; ++q) {
      const int i = t0 + q * kThreads;
      if (i < Gm::kTw) const_cast<double2*>(tw)[i] = twr[q];
    }
  }
};

// For batches that fit one wave of clusters: the spectrum values are fetched
// at the start and held in registers through the forward passes. (A
// throughput form for larger batches — fetched before the product, 96
// registers, 5 CTAs/SM — measured 47.8 us at config 3's 150 items against
// 46.7 us for the one-CTA kernel, so larger batches stay there.)
template <int RA, int RB, int kClThreads>
__global__ void __cluster_dims__(kClC, 1, 1) __launch_bounds__(kClThreads, 3)
    iuv_cluster_kernel(FftPlan pl, EngArgs e, const double* __restrict__ A,
                       const double* __restrict__ B, int c1, int c2, int f,
                       double* __restrict__ est, IuvTail tail) {
  using F = ClFft<RA, RB, kClThreads>;
  constexpr int N2 = F::N2, M = F::M, P = F::P, Q = F::Q, ROWS = F::ROWS, COLS = F::COLS;
  constexpr int kGU = (ROWS * 32 + kClThreads - 1) / kClThreads;  // product units per thread
  constexpr int kGather = 2;                                       // gather entries per thread
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cg::cluster_group cl = cg::this_cluster();
  const F fx(smem_raw, static_cast<int>(cl.block_rank()));
  const int r = fx.r, t0 = fx.t0;
  const int item = blockIdx.x / kClC;
  const int bvec = item / e.D, d = item % e.D;
  // every CTA of the cluster has started before anyone writes remote memory
  cluster_arrive();
  const uint32_t* tab = e.packed + static_cast<size_t>(d) * e.fam_stride;
  const int na = pick3(e.dims, c1), nb = pick3(e.dims, c2), nf = pick3(e.dims, f);
  const uint32_t* ta = tab + pick3(e.tab_off, c1);
  const uint32_t* tb = tab + pick3(e.tab_off, c2);
  const uint32_t* tf = tab + pick3(e.tab_off, f);
  const double* av = A + static_cast<size_t>(bvec) * na;
  const double* bv = B + static_cast<size_t>(bvec) * nb;
  // Early loads, all in flight together: twiddles, the count-sketch inputs,
  // the gather table entries and the slots of this thread's spectrum values.
  double2 twr[F::kTwPer];  // stored after the scatter, so both load streams overlap
  fx.load_tw(pl, twr);
  constexpr int kSc = 4;  // scatter inputs per thread per round
  for (int i = t0; i < COLS * N2; i += kClThreads) fx.colbuf[i] = make_double2(0.0, 0.0);
  uint32_t gt[kGather];
#pragma unroll
  for (int g = 0; g < kGather; ++g) {
    const int i = t0 + g * kClThreads;
    gt[g] = i < nf ? __ldg(tf + i) : 0u;
  }
  const double2* sp = e.spec + static_cast<size_t>(d) * P;
  int sslot[kGU][2];
#pragma unroll
  for (int g = 0; g < kGU; ++g) {
    const int u = t0 + g * kClThreads;
    const int row = u >> 5, k1 = u & 31;
    const int k2 = row_k2<N2, Q>(r, row < ROWS ? row : 0);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = k2 + N2 * (k1 + 32 * h);
      const int kh = k <= P ? k : M - k;  // half-spectrum frequency
      // the real bins (kh = 0, P) sit in slot f2p[0]
      sslot[g][h] = u < ROWS * 32 ? __ldg(pl.f2p + (kh == P ? 0 : kh)) : 0;
    }
  }
  __syncthreads();
  for (int i0 = t0; i0 < na + nb; i0 += kSc * kClThreads) {
    double v[kSc];
    uint32_t t[kSc];
#pragma unroll
    for (int q = 0; q < kSc; ++q) {
      const int i = i0 + q * kClThreads;
      v[q] = 0.0;
      t[q] = 0u;
      if (i < na) {
        v[q] = av[i];
        t[q] = __ldg(ta + i);
      } else if (i < na + nb) {
        v[q] = bv[i - na];
        t[q] = __ldg(tb + i - na);
      }
    }
#pragma unroll
    for (int q = 0; q < kSc; ++q) {
      const int i = i0 + q * kClThreads;
      const uint32_t h = t[q] & 0x7fffffffu;
      const int n1 = static_cast<int>(h & 63u);
      if (v[q] == 0.0 || n1 / COLS != r) continue;
      double2& s = fx.colbuf[sw((n1 % COLS) * N2 + static_cast<int>(h >> 6))];
      atomicAdd(i < na ? &s.x : &s.y, (t[q] >> 31) ? -v[q] : v[q]);
    }
  }
  fx.store_tw(twr);
  __syncthreads();
  fx.f1a();
  // spectrum values for the product phase, in flight through the forward passes
  // (raw slot values: the real-bin / conjugate selection happens at the use,
  // so no instruction waits on these loads before the forward passes)
  double2 sv[kGU][2];
#pragma unroll
  for (int g = 0; g < kGU; ++g) {
#pragma unroll
    for (int h = 0; h < 2; ++h) sv[g][h] = __ldg(sp + sslot[g][h]);
  }
  __syncthreads();
  cluster_wait();
  fx.f1b_f3(cl);
  // G = S_d conj(A B) and the c2r pre map
#pragma unroll
  for (int g = 0; g < kGU; ++g) {
    const int u = t0 + g * kClThreads;
    if (u >= ROWS * 32) break;
    const int row = u >> 5, k1 = u & 31;
    const int k2 = row_k2<N2, Q>(r, row);
    double2 gg[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double2 a2, b2;
      fx.spectra(row, k2, k1 + 32 * h, a2, b2);
      const int k = k2 + N2 * (k1 + 32 * h);
      const int kh = k <= P ? k : M - k;
      double2 sx = sv[g][h];
      if (kh == 0) sx = make_double2(sx.x, 0.0);
      else if (kh == P) sx = make_double2(sx.y, 0.0);
      else if (k > P) sx = cconj(sx);
      gg[h] = cmul(sx, cconj(cmul(a2, b2)));
    }
    fx.put_u(row, k2, k1, gg[0], gg[1]);
  }
  __syncthreads();
  fx.inverse(cl);
  // gather: z[h] = u[h / 2] component h % 2, scaled 1 / P. Tail mode 4
  // (T(u, v, w)): instead of the estimates, their dot product with w — the
  // family's T(u, v, w) by linearity — summed over the CTAs in a fixed order.
  const bool dotw = tail.mode == 4;
  double* o = est + static_cast<size_t>(item) * nf;
  const double* wv = dotw ? tail.wvec + static_cast<size_t>(bvec) * nf : nullptr;
  const double inv = 1.0 / P;
  double dacc = 0.0;
#pragma unroll
  for (int g = 0; g < kGather; ++g) {
    const int i = t0 + g * kClThreads;
    if (i >= nf) break;
    const uint32_t t = gt[g];
    const int h = static_cast<int>(t & 0x7fffffffu);
    if (!fx.owns(h)) continue;
    const double z = fx.zval(h) * inv;
    if (dotw) dacc += wv[i] * ((t >> 31) ? -z : z);
    else o[i] = (t >> 31) ? -z : z;
  }
  for (int i = t0 + kGather * kClThreads; i < nf; i += kClThreads) {  // nf > 256
    const uint32_t t = __ldg(tf + i);
    const int h = static_cast<int>(t & 0x7fffffffu);
    if (!fx.owns(h)) continue;
    const double z = fx.zval(h) * inv;
    if (dotw) dacc += wv[i] * ((t >> 31) ? -z : z);
    else o[i] = (t >> 31) ? -z : z;
  }
  if (dotw) {  // est[item] = sum over the CTAs (rank order) of the block sums
    __shared__ double wred[kClThreads / 32];
    __shared__ double wpart[kClC];
#pragma unroll
    for (int q = 16; q > 0; q >>= 1) dacc += __shfl_xor_sync(0xffffffffu, dacc, q);
    if ((t0 & 31) == 0) wred[t0 >> 5] = dacc;
    __syncthreads();
    if (t0 == 0) {
      double sblk = 0.0;
#pragma unroll
      for (int q = 0; q < kClThreads / 32; ++q) sblk += wred[q];
      *cl.map_shared_rank(&wpart[r], 0) = sblk;
    }
    cl.sync();
    if (r == 0 && t0 == 0) {
      double sum = 0.0;
#pragma unroll
      for (int q = 0; q < kClC; ++q) sum += wpart[q];
      est[item] = sum;
    }
  }
  if (tail.mode != 0) {
    // The last of the D clusters of vector bvec (per-vector arrival counter)
    // takes the median over the families with all 8 CTAs, then (modes 2, 3)
    // the row norm from per-CTA partials exchanged over DSMEM.
    __shared__ int last;
    __shared__ double part[kClC];
    __shared__ double red[kClThreads / 32];
    __threadfence();
    cl.sync();
    if (r == 0 && t0 == 0) {
      const int old = atomicAdd(tail.cnt + bvec, 1);
      const int is_last = old == e.D - 1;
      if (is_last) tail.cnt[bvec] = 0;  // every cluster of bvec has arrived: ready for the next launch
      for (int q = 0; q < kClC; ++q) *cl.map_shared_rank(&last, q) = is_last;
    }
    cl.sync();
    if (!last) return;
    __threadfence();
    if (tail.mode == 3 && *reinterpret_cast<volatile int*>(tail.stopped)) return;
    const int nt = dotw ? 1 : nf;  // values per family: one contraction value, or the row
    const double* col0 = est + static_cast<size_t>(bvec) * e.D * nt;
    double* ob = tail.out + static_cast<size_t>(bvec) * nt;
    double acc = 0.0;
    for (int i = r * kClThreads + t0; i < nt; i += kClC * kClThreads) {
      const double m = median_col(col0 + i, e.D, nt, [](const double* p) { return __ldcg(p); });
      ob[i] = m;
      acc += m * m;
    }
    if (tail.mode == 1 || tail.mode == 4) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((t0 & 31) == 0) red[t0 >> 5] = acc;
    __syncthreads();
    if (t0 < kClC) {  // this CTA's partial to every CTA of the cluster (slot r)
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kClThreads / 32; ++w) s += red[w];
      *cl.map_shared_rank(&part[r], t0) = s;
    }
    cl.sync();
    double tot = 0.0;
#pragma unroll
    for (int q = 0; q < kClC; ++q) tot += part[q];
    const double nv = sqrt(tot);
    if (tail.mode == 2) {
      for (int i = r * kClThreads + t0; i < nf; i += kClC * kClThreads)
        ob[i] = nv < 1e-150 ? 0.0 : ob[i] / nv;
    } else {
      if (nv < 1e-150) {
        if (r == 0 && t0 == 0) *tail.stopped = 1;
        return;
      }
      for (int i = r * kClThreads + t0; i < nf; i += kClC * kClThreads) tail.best[i] = ob[i] / nv;
    }
  }
}

// Linear convolution of row pairs (fft_convolve of two sequences,
// fft.cpp:75-84; config 5's Kronecker composition): one cluster per item,
// w = a + i b transformed once, G = A B, out[t] = z[t] for t < la + lb - 1.
template <int RA, int RB, int kClThreads>
__global__ void __cluster_dims__(kClC, 1, 1) __launch_bounds__(kClThreads, 3)
    conv_cluster_kernel(FftPlan pl, const double* __restrict__ a, int la, size_t lda,
                        const double* __restrict__ b, int lb, size_t ldb,
                        double* __restrict__ out, size_t ldo) {
  using F = ClFft<RA, RB, kClThreads>;
  constexpr int N2 = F::N2, P = F::P, ROWS = F::ROWS, COLS = F::COLS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cg::cluster_group cl = cg::this_cluster();
  const F fx(smem_raw, static_cast<int>(cl.block_rank()));
  const int r = fx.r, t0 = fx.t0;
  const int item = blockIdx.x / kClC;
  cluster_arrive();
  double2 twr[F::kTwPer];
  fx.load_tw(pl, twr);
  const double* ar = a + static_cast<size_t>(item) * lda;
  const double* br = b + static_cast<size_t>(item) * ldb;
  // this CTA's columns n1 = 8 r + j: w[n1 + 64 n2] for every n2 (zero past the rows)
  for (int i = t0; i < COLS * N2; i += kClThreads) {
    const int j = i / N2, n2 = i % N2;
    const int n = COLS * r + j + kN1 * n2;
    fx.colbuf[sw(i)] = make_double2(n < la ? __ldg(ar + n) : 0.0, n < lb ? __ldg(br + n) : 0.0);
  }
  fx.store_tw(twr);
  __syncthreads();
  fx.f1a();
  __syncthreads();
  cluster_wait();
  fx.f1b_f3(cl);
  for (int u = t0; u < ROWS * 32; u += kClThreads) {
    const int row = u >> 5, k1 = u & 31;
    const int k2 = row_k2<N2, F::Q>(r, row);
    double2 gg[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double2 a2, b2;
      fx.spectra(row, k2, k1 + 32 * h, a2, b2);
      gg[h] = cmul(a2, b2);
    }
    fx.put_u(row, k2, k1, gg[0], gg[1]);
  }
  __syncthreads();
  fx.inverse(cl);
  // out[t] = z[t] / P for the t this CTA holds: t = 2m + c, m1 = m % 32 in [4r, 4r + 4)
  const int lo = la + lb - 1;
  double* o = out + static_cast<size_t>(item) * ldo;
  const double inv = 1.0 / P;
  for (int i = t0; i < F::M1 * N2 * 2; i += kClThreads) {
    const int ml = i / (2 * N2), rest = i % (2 * N2);
    const int m2 = rest >> 1, c = rest & 1;
    const int t = 2 * (F::M1 * r + ml + 32 * m2) + c;
    if (t < lo) o[t] = fx.zval(t) * inv;
  }
}

// K5 over a cluster: the inverse of the summed CP spectrum of family d
// (cp_sum_kernel: the one-CTA plan's half spectrum in slot order, read in
// frequency order through the frequency -> slot table), out[d][t] (+)= z[t]
// for t < jt. D clusters instead of D CTAs.
template <int RA, int RB, int kClThreads>
__global__ void __cluster_dims__(kClC, 1, 1) __launch_bounds__(kClThreads, 3)
    spec_inverse_cluster_kernel(FftPlan pl, const double2* __restrict__ acc,
                                double* __restrict__ out, int jt, int accumulate) {
  using F = ClFft<RA, RB, kClThreads>;
  constexpr int N2 = F::N2, M = F::M, P = F::P, ROWS = F::ROWS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cg::cluster_group cl = cg::this_cluster();
  const F fx(smem_raw, static_cast<int>(cl.block_rank()));
  const int r = fx.r, t0 = fx.t0;
  const int d = blockIdx.x / kClC;
  cluster_arrive();
  double2 twr[F::kTwPer];
  fx.load_tw(pl, twr);
  const double2* sp = acc + static_cast<size_t>(d) * P;
  // the full spectrum G[k] from the half spectrum (slot f2p[0] holds X0, XP)
  auto G = [&](int k) {
    const int kh = k <= P ? k : M - k;
    if (kh == 0) return make_double2(__ldg(&sp[__ldg(pl.f2p)].x), 0.0);
    if (kh == P) return make_double2(__ldg(&sp[__ldg(pl.f2p)].y), 0.0);
    const double2 v = __ldg(sp + __ldg(pl.f2p + kh));
    return k > P ? cconj(v) : v;
  };
  fx.store_tw(twr);
  __syncthreads();
  for (int u = t0; u < ROWS * 32; u += kClThreads) {
    const int row = u >> 5, k1 = u & 31;
    const int k2 = row_k2<N2, F::Q>(r, row);
    fx.put_u(row, k2, k1, G(k2 + N2 * k1), G(k2 + N2 * (k1 + 32)));
  }
  __syncthreads();
  cluster_wait();
  fx.inverse(cl);
  double* o = out + static_cast<size_t>(d) * jt;
  const double inv = 1.0 / P;
  for (int i = t0; i < F::M1 * N2 * 2; i += kClThreads) {
    const int ml = i / (2 * N2), rest = i % (2 * N2);
    const int m2 = rest >> 1, c = rest & 1;
    const int t = 2 * (F::M1 * r + ml + 32 * m2) + c;
    if (t < jt) {
      const double v = fx.zval(t) * inv;
      o[t] = accumulate ? o[t] + v : v;
    }
  }
}

// K9 over a cluster: deflation S_d -= weight F(cs_u) F(cs_v) F(cs_w) of
// family d (deflate_kernel; cpd.cpp:79-87 in the frequency domain): w1 =
// cs_u + i cs_v transformed once (both spectra by the Hermitian split), their
// product kept per k in shared memory, then cs_w transformed; each CTA updates
// the half-spectrum slots of its k (k <= M/2; slot f2p[0] holds X0, X_{M/2}).
template <int RA, int RB, int kClThreads>
__global__ void __cluster_dims__(kClC, 1, 1) __launch_bounds__(kClThreads, 3)
    deflate_cluster_kernel(FftPlan pl, EngArgs e, double weight, const double* __restrict__ U,
                           const double* __restrict__ V, const double* __restrict__ W,
                           double2* __restrict__ spec) {
  using F = ClFft<RA, RB, kClThreads>;
  constexpr int N2 = F::N2, P = F::P, Q = F::Q, ROWS = F::ROWS, COLS = F::COLS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cg::cluster_group cl = cg::this_cluster();
  const F fx(smem_raw, static_cast<int>(cl.block_rank()));
  double2* abbuf = fx.rowbuf + ROWS * kN1;  // A B per k of this CTA's rows
  const int r = fx.r, t0 = fx.t0;
  const int d = blockIdx.x / kClC;
  cluster_arrive();
  double2 twr[F::kTwPer];
  fx.load_tw(pl, twr);
  const uint32_t* tab = e.packed + static_cast<size_t>(d) * e.fam_stride;
  // count sketch into this CTA's columns: first (real) and optional second (imag) vector
  auto scatter = [&](const double* x0, int n0, const uint32_t* t0p, const double* x1, int n1,
                     const uint32_t* t1p) {
    for (int i = t0; i < COLS * N2; i += kClThreads) fx.colbuf[i] = make_double2(0.0, 0.0);
    __syncthreads();
    for (int i = t0; i < n0 + n1; i += kClThreads) {
      const bool first = i < n0;
      const double v = first ? x0[i] : x1[i - n0];
      if (v == 0.0) continue;
      const uint32_t t = __ldg(first ? t0p + i : t1p + (i - n0));
      const uint32_t h = t & 0x7fffffffu;
      const int n1c = static_cast<int>(h & 63u);
      if (n1c / COLS != r) continue;
      double2& sl = fx.colbuf[sw((n1c % COLS) * N2 + static_cast<int>(h >> 6))];
      atomicAdd(first ? &sl.x : &sl.y, (t >> 31) ? -v : v);
    }
  };
  scatter(U, e.dims[0], tab + e.tab_off[0], V, e.dims[1], tab + e.tab_off[1]);
  fx.store_tw(twr);
  __syncthreads();
  fx.f1a();
  __syncthreads();
  cluster_wait();
  fx.f1b_f3(cl);
  for (int u = t0; u < ROWS * kN1; u += kClThreads) {
    const int row = u >> 6, kk = u & 63;
    const int k2 = row_k2<N2, Q>(r, row);
    double2 a2, b2;
    fx.spectra(row, k2, kk, a2, b2);
    abbuf[row * kN1 + kk] = cmul(a2, b2);
  }
  __syncthreads();
  cluster_arrive();  // every CTA has read its rows before the second transform writes them
  scatter(W, e.dims[2], tab + e.tab_off[2], nullptr, 0, nullptr);
  __syncthreads();
  fx.f1a();
  __syncthreads();
  cluster_wait();
  fx.f1b_f3(cl);
  double2* S = spec + static_cast<size_t>(d) * P;
  for (int u = t0; u < ROWS * kN1; u += kClThreads) {
    const int row = u >> 6, kk = u & 63;
    const int k2 = row_k2<N2, Q>(r, row);
    const int k = k2 + N2 * kk;
    if (k > P) continue;
    const double2 c = fx.rowbuf[sw(row * kN1 + (kk >> 3) + 8 * (kk & 7))];
    const double2 g = cmul(abbuf[row * kN1 + kk], c);
    if (k == 0) {
      S[__ldg(pl.f2p)].x -= weight * g.x;
    } else if (k == P) {
      S[__ldg(pl.f2p)].y -= weight * g.x;
    } else {
      double2& sv = S[__ldg(pl.f2p + k)];
      sv = make_double2(sv.x - weight * g.x, sv.y - weight * g.y);
    }
  }
}

template <int RA, int RB, typename K>
int cluster_prep(K k, int* max_clusters_out) {
  using Gm = ClGeom<RA, RB>;
  const size_t smem = Gm::smem_bytes();
  // once per device and kernel: the shared-memory opt-in and the number of
  // clusters that fit the device at once
  static int max_clusters_dev[64];
  static bool init_dev[64];
  int dev = 0;
  FCS_CUDA_TRY(cudaGetDevice(&dev));
  if (!init_dev[dev & 63]) {
    FCS_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kClC);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    int n = 0;
    FCS_CUDA_TRY(cudaOccupancyMaxActiveClusters(&n, k, &cfg));
    max_clusters_dev[dev & 63] = n;
    init_dev[dev & 63] = true;
  }
  *max_clusters_out = max_clusters_dev[dev & 63];
  return ST_OK;
}

template <int RA, int RB>
int launch_cl(const FftPlan& pl, const EngArgs& e, int batch, const double* A, const double* B,
              int c1, int c2, int f, double* est, const IuvTail& tail, cudaStream_t st) {
  auto k = iuv_cluster_kernel<RA, RB, 128>;
  int max_clusters = 0;
  if (int rc = cluster_prep<RA, RB>(k, &max_clusters)) return rc;
  // one wave only: beyond it the one-CTA kernel's throughput wins
  if (static_cast<long>(batch) * e.D > max_clusters) return 1;
  const unsigned grid = static_cast<unsigned>(batch) * e.D * kClC;
  k<<<grid, 128, ClGeom<RA, RB>::smem_bytes(), st>>>(pl, e, A, B, c1, c2, f, est, tail);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

template <int RA, int RB>
int launch_conv_cl(const FftPlan& pl, const double* a, int la, size_t lda, const double* b, int lb,
                   size_t ldb, int items, double* out, size_t ldo, cudaStream_t st) {
  auto k = conv_cluster_kernel<RA, RB, 128>;
  int max_clusters = 0;
  if (int rc = cluster_prep<RA, RB>(k, &max_clusters)) return rc;
  if (items > max_clusters) return 1;
  k<<<static_cast<unsigned>(items) * kClC, 128, ClGeom<RA, RB>::smem_bytes(), st>>>(
      pl, a, la, lda, b, lb, ldb, out, ldo);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

template <int RA, int RB>
int launch_inv_cl(const FftPlan& pl, const double2* acc, int D, double* out, int jt, int accumulate,
                  cudaStream_t st) {
  auto k = spec_inverse_cluster_kernel<RA, RB, 128>;
  int max_clusters = 0;
  if (int rc = cluster_prep<RA, RB>(k, &max_clusters)) return rc;
  if (D > max_clusters) return 1;
  k<<<static_cast<unsigned>(D) * kClC, 128, ClGeom<RA, RB>::smem_bytes(), st>>>(pl, acc, out, jt,
                                                                               accumulate);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

template <int RA, int RB>
int launch_defl_cl(const FftPlan& pl, const EngArgs& e, double weight, const double* U,
                   const double* V, const double* W, double2* spec, cudaStream_t st) {
  auto k = deflate_cluster_kernel<RA, RB, 128>;
  const size_t smem = ClGeom<RA, RB>::smem_bytes() +
                      static_cast<size_t>(ClGeom<RA, RB>::ROWS) * kN1 * sizeof(double2);
  static bool attr[64];
  int dev = 0;
  FCS_CUDA_TRY(cudaGetDevice(&dev));
  if (!attr[dev & 63]) {
    FCS_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    attr[dev & 63] = true;
  }
  k<<<static_cast<unsigned>(e.D) * kClC, 128, smem, st>>>(pl, e, weight, U, V, W, spec);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace

int launch_deflate_cluster(const FftPlan& pl, const EngArgs& e, double weight, const double* U,
                           const double* V, const double* W, double2* spec, cudaStream_t st) {
  static const bool off = std::getenv("ST_IUV_CLUSTER_OFF") != nullptr;  // A/B probe
  if (off || pl.large_p1 || e.D <= 0 || e.D > 32) return 1;
  switch (pl.M) {
    case 12288: return launch_defl_cl<16, 12>(pl, e, weight, U, V, W, spec, st);
    case 9216: return launch_defl_cl<16, 9>(pl, e, weight, U, V, W, spec, st);
    case 8192: return launch_defl_cl<16, 8>(pl, e, weight, U, V, W, spec, st);
    case 6144: return launch_defl_cl<16, 6>(pl, e, weight, U, V, W, spec, st);
    case 4096: return launch_defl_cl<16, 4>(pl, e, weight, U, V, W, spec, st);
    case 3072: return launch_defl_cl<16, 3>(pl, e, weight, U, V, W, spec, st);
    case 2048: return launch_defl_cl<16, 2>(pl, e, weight, U, V, W, spec, st);
    default: return 1;
  }
}

int launch_spec_inverse_cluster(const FftPlan& pl, const double2* acc, int D, double* out, int jt,
                                int accumulate, cudaStream_t st) {
  static const bool off = std::getenv("ST_IUV_CLUSTER_OFF") != nullptr;  // A/B probe
  if (off || pl.large_p1 || D <= 0) return 1;
  switch (pl.M) {
    case 12288: return launch_inv_cl<16, 12>(pl, acc, D, out, jt, accumulate, st);
    case 9216: return launch_inv_cl<16, 9>(pl, acc, D, out, jt, accumulate, st);
    case 8192: return launch_inv_cl<16, 8>(pl, acc, D, out, jt, accumulate, st);
    case 6144: return launch_inv_cl<16, 6>(pl, acc, D, out, jt, accumulate, st);
    case 4096: return launch_inv_cl<16, 4>(pl, acc, D, out, jt, accumulate, st);
    case 3072: return launch_inv_cl<16, 3>(pl, acc, D, out, jt, accumulate, st);
    case 2048: return launch_inv_cl<16, 2>(pl, acc, D, out, jt, accumulate, st);
    default: return 1;
  }
}

int launch_iuv_cluster(const FftPlan& pl, const EngArgs& e, int batch, const double* A,
                       const double* B, int c1, int c2, int f, double* est, const IuvTail& tail,
                       cudaStream_t st) {
  static const bool off = std::getenv("ST_IUV_CLUSTER_OFF") != nullptr;  // A/B probe
  if (off || pl.large_p1 || batch <= 0) return 1;
  switch (pl.M) {
    case 9216: return launch_cl<16, 9>(pl, e, batch, A, B, c1, c2, f, est, tail, st);
    case 8192: return launch_cl<16, 8>(pl, e, batch, A, B, c1, c2, f, est, tail, st);
    // small transforms too (batch-1 step with the median, D = 10, 100-long
    // vectors: M = 3072 20.5 -> 13.8 us, M = 2048 18.5 -> 12.3 us)
    case 12288: return launch_cl<16, 12>(pl, e, batch, A, B, c1, c2, f, est, tail, st);
    case 6144: return launch_cl<16, 6>(pl, e, batch, A, B, c1, c2, f, est, tail, st);
    case 4096: return launch_cl<16, 4>(pl, e, batch, A, B, c1, c2, f, est, tail, st);
    case 3072: return launch_cl<16, 3>(pl, e, batch, A, B, c1, c2, f, est, tail, st);
    case 2048: return launch_cl<16, 2>(pl, e, batch, A, B, c1, c2, f, est, tail, st);
    default: return 1;
  }
}

int launch_conv_cluster(const FftPlan& pl, const double* a, int la, size_t lda, const double* b,
                        int lb, size_t ldb, int items, double* out, size_t ldo, cudaStream_t st) {
  static const bool off = std::getenv("ST_IUV_CLUSTER_OFF") != nullptr;  // A/B probe
  if (off || pl.large_p1 || items <= 0) return 1;
  switch (pl.M) {
    case 9216: return launch_conv_cl<16, 9>(pl, a, la, lda, b, lb, ldb, items, out, ldo, st);
    case 8192: return launch_conv_cl<16, 8>(pl, a, la, lda, b, lb, ldb, items, out, ldo, st);
    case 12288: return launch_conv_cl<16, 12>(pl, a, la, lda, b, lb, ldb, items, out, ldo, st);
    case 6144: return launch_conv_cl<16, 6>(pl, a, la, lda, b, lb, ldb, items, out, ldo, st);
    case 4096: return launch_conv_cl<16, 4>(pl, a, la, lda, b, lb, ldb, items, out, ldo, st);
    case 3072: return launch_conv_cl<16, 3>(pl, a, la, lda, b, lb, ldb, items, out, ldo, st);
    case 2048: return launch_conv_cl<16, 2>(pl, a, la, lda, b, lb, ldb, items, out, ldo, st);
    default: return 1;
  }
}

}  // namespace fcs
