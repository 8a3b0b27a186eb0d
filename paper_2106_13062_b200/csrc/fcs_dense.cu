// K1: dense fast count sketch — streaming scatter of vec(T) into
// bucket sum_n h_n(i_n) with sign prod_n s_n(i_n), D families per launch.
//
// Reference: fcs_sketch(const DenseTensor&, const HashFamily&),
// sketch.cpp:187-201, over the odometer walk for_each_nonzero,
// sketch.cpp:48-61 (zeros skipped; adding +/-0 is equivalent). The reference
// sums serially in fp64; here each CTA privatises ONE family's full sketch in
// shared memory and streams a contiguous chunk of mode-0 fibers (a "fiber" is
// the I_0 contiguous elements T[:, i_1, ..., i_{N-1}], whose offset
// c = sum_{n>=1} h_n(i_n) and sign are warp-uniform). Grid index d is the
// fastest-varying, so the D CTAs that read the same chunk run together and
// share it through L2. Per-CTA partials are reduced in a fixed order in fp64.
//
// float32 fast path (fcs_dense_fx_kernel): shared-memory float atomics are
// compare-and-swap loops on sm_100a, integer atomics are native
// (ATOMS.ADD). The fp32 path therefore accumulates in int32 fixed point with
// a scale 2^S chosen from a sampled bound on the partial sums; every
// accumulate returns the old word, so overflow (and non-finite input) is
// detected exactly, and a CTA that overflowed redoes its chunk with float
// atomics. Rounding error per element <= 2^-(S+1) (K1). The
// sample statistics are reduced in a fixed order, so S — and the whole fixed-
// point result — is the same on every run. For D >= 2 the fiber's 128-byte
// lines are regrouped per load step to spread each ATOMS over more banks
// (fx_group_kernel, searched once per table set and cached on the device).
#include <algorithm>
#include <climits>
#include <vector>
#include <map>
#include <mutex>
#include <cstdlib>
#include <cmath>

#include "dense_common.cuh"

namespace fcs {
// Streaming 16-byte load that does not allocate in L1: the tensor is read
// once per CTA, and L1 shares its SRAM and data pipe with the shared-memory
// sketch and its atomics (config 4: 2.47 -> 2.33 ms vs __ldg, 2.50 ms __ldcs).
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

// Sampled statistics of the input and the fixed-point exponent derived from them.
struct FxStats {
  double maxabs;     // max |x| over the kept sample
  int S;             // fixed-point fractional bits
  double sum;
  double sumsq;
  double count;
};
// Per-fiber partial of the sample (fx_sample_warps), reduced in a fixed order
// by fx_scale_device: no contended atomics, and the chosen scale (hence the
// fixed-point rounding) is the same on every run.
struct FxPart {
  double mx;
  double s, s2, cnt;
};
// Fixed-point format limits: int32 words (fp32 input) and int64 words as two
// int32 halves (fp64 input). elem: largest |x * 2^S| the magic-number rounding
// keeps exact (the range check catches anything beyond); part: the largest
// designed partial (the wrap guard trips at twice it); max_s: largest S whose
// 2^S is finite in the input type.
struct FxLimits {
  double elem, part;
  int max_s;
};
// What a fixed-point kernel needs to derive S itself (fx_scale_device).
struct FxScaleArgs {
  const FxPart* parts;
  int nparts;
  double n_center;  // expected elements per busiest bucket per CTA
  FxStats* stats;   // written by CTA 0
};
constexpr FxLimits kFx32{4194304.0 /* 2^22 */, 1073741824.0 /* 2^30 */, 120};
constexpr FxLimits kFx64{2251799813685248.0 /* 2^51 */, 2305843009213693952.0 /* 2^61 */, 1000};
// A CTA whose largest |partial| stays below 2^kFxSmallBits (and is not zero)
// saw data far smaller than the sample predicted: its fixed-point rounding
// would be coarse relative to its own values, so it redoes its chunk with
// float atomics, like an overflowing CTA (the c4 N(0,1) partials peak near 2^28).
constexpr int kFxSmallBits = 16;
constexpr int kFxMaxSample = 2048;   // sampled fibers = sample CTAs = partials

// ------------------------------------------------------------------ kernels
// Generic block-private kernel (any shape, fp32 or fp64): one family per CTA,
// fibers strided over warps, shared-memory atomicAdd.
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
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (uint64_t f = f_begin + warp; f < f_end; f += nwarps) {
    uint32_t c, sbit;
    fiber_offset(a, tab, f, c, sbit);
    const Tin* fib = t + f * i0n;
    uint32_t i = lane;
    for (; i + 96 < i0n; i += 128) {  // 4 independent loads in flight per lane
      Tacc v[4];
      uint32_t e[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[k] = static_cast<Tacc>(__ldcs(fib + i + 32 * k));
        e[k] = __ldg(tab0 + i + 32 * k);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (v[k] != Tacc(0))
          atomicAdd(&sk[(e[k] & 0x7fffffffu) + c], signed_val(v[k], (e[k] ^ sbit) & 0x80000000u));
    }
    for (; i < i0n; i += 32) {
      const Tacc v = static_cast<Tacc>(__ldcs(fib + i));
      const uint32_t e = __ldg(tab0 + i);
      if (v != Tacc(0)) atomicAdd(&sk[(e & 0x7fffffffu) + c], signed_val(v, (e ^ sbit) & 0x80000000u));
    }
  }
  __syncthreads();
  Tacc* dst = part + (chunk * a.D + d) * static_cast<uint64_t>(a.jt);
  for (uint32_t b = threadIdx.x; b < a.jt; b += blockDim.x) dst[b] = sk[b];
}

// Fixed-point exponent: the largest S with a comfortable margin between the
// expected largest per-CTA bucket partial and 2^31 (bias * N + 8 sigma sqrt(N)
// + max, N = the expected count of elements a CTA adds to its busiest bucket).
// The statistics are ROBUST to outliers: a sampled fiber whose max |x| lies
// more than 4 standard deviations above the mean of log max|x| over the
// sampled fibers is left out, so one huge element (which its CTA handles by
// the exact range check + float fallback) cannot coarsen the scale for the
// whole tensor. Every reduction runs in a fixed order, so S is the same on
// every run.
// Fixed-order block reduction of K values at once: xor tree inside each warp,
// then warp 0 reduces the per-warp values (identity-padded to 32 lanes) with
// the same tree; every thread gets the results. op(i, x, y) combines value i.
template <int K, typename Op>
__device__ __forceinline__ void block_reduce(double (&v)[K], double (*red)[K], Op op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < K; ++i) v[i] = op(i, v[i], __shfl_xor_sync(0xffffffffu, v[i], o));
  __syncthreads();  // red is reused across calls
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int i = 0; i < K; ++i) red[threadIdx.x >> 5][i] = v[i];
  __syncthreads();
  if (threadIdx.x < 32) {
    double w[K];
#pragma unroll
    for (int i = 0; i < K; ++i) w[i] = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x][i] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < K; ++i) w[i] = op(i, w[i], __shfl_xor_sync(0xffffffffu, w[i], o));
    if (threadIdx.x == 0)
#pragma unroll
      for (int i = 0; i < K; ++i) red[32][i] = w[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = red[32][i];
}

// Computed redundantly (and identically) by every CTA of a fixed-point
// kernel from the sample partials before it scatters; CTA 0 also stores the
// statistics for the reduction and st_fcs_dense_report. All threads of the
// CTA must call it (it synchronises); blockDim.x == 512 (each thread holds
// up to kFxMaxSample / 512 partials in registers: one load round).
__device__ int fx_scale_device(const FxPart* __restrict__ parts, int nparts, double n_center,
                               FxLimits lim, FxStats* st) {
  constexpr int kPer = kFxMaxSample / 512;
  __shared__ double red[33][4];
  FxPart mine[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int q = threadIdx.x + j * blockDim.x;
    mine[j] = q < nparts ? parts[q] : FxPart{0.0, 0.0, 0.0, 0.0};
  }
  // mean and spread of log2 max|x| over the fibers with a nonzero max
  double lv[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const double m = mine[j].mx;
    if (m > 0.0 && m <= 1.7976931348623157e308) {
      const double lg = log2(m);
      lv[0] += lg;
      lv[1] += lg * lg;
      lv[2] += 1.0;
    }
  }
  block_reduce<3>(lv, reinterpret_cast<double(*)[3]>(red),
                  [](int, double x, double y) { return x + y; });
  const double ln = lv[2];
  const double lmean = ln > 0.0 ? lv[0] / ln : 0.0;
  const double lsd = ln > 0.0 ? sqrt(fmax(lv[1] / ln - lmean * lmean, 0.0)) : 0.0;
  const double cut = exp2(lmean + 4.0 * lsd + 1.0);  // + 1: never cut a tight (sd ~ 0) sample
  // fixed-order reduction of the kept sample partials: max, sum, sum of squares, count
  double sv[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    if (ln >= 16.0 && mine[j].mx > cut) continue;  // small samples keep everything
    sv[0] = fmax(sv[0], mine[j].mx);
    sv[1] += mine[j].s;
    sv[2] += mine[j].s2;
    sv[3] += mine[j].cnt;
  }
  block_reduce<4>(sv, red, [](int i, double x, double y) { return i == 0 ? fmax(x, y) : x + y; });
  const double pm = sv[0], ps = sv[1], ps2 = sv[2], pc = sv[3];
  __shared__ int s_out;
  if (threadIdx.x == 0) {
    const double n = fmax(pc, 1.0);
    const double mean = ps / n;
    const double rms = sqrt(fmax(ps2 / n, 0.0));
    const double mx = pm;
    const double bound = fabs(mean) * n_center + 8.0 * rms * sqrt(n_center) + 2.0 * mx;
    // An all-zero sample gives the top exponent: any element of the tensor
    // above 2^-(max_s) * elem then trips the exact range check and its CTA
    // redoes the chunk with float atomics, so a sample that missed the data
    // costs time, never accuracy. Small-magnitude data gets a large S.
    int S = lim.max_s;
    if (bound > 0.0) S = static_cast<int>(floor(log2(lim.part / bound)));
    // single elements must stay inside the exact-rounding range with a 1.5x
    // margin over the sampled maximum (an element beyond it is caught exactly
    // and its CTA falls back; N(0,1): sample max ~5, tensor max ~6.1)
    if (mx > 0.0) S = min(S, static_cast<int>(floor(log2(lim.elem / (1.5 * mx)))));
    S = max(-lim.max_s, min(lim.max_s, S));
    s_out = S;
    if (st != nullptr) {
      st->maxabs = pm;
      st->sum = ps;
      st->sumsq = ps2;
      st->count = pc;
      st->S = S;
    }
  }
  __syncthreads();
  return s_out;
}

// One CTA: the scale of a call from its sample partials (fx_scale_device),
// stored for the scatter, the reduction and st_fcs_dense_report.
__global__ void __launch_bounds__(512) fx_scale_kernel(FxScaleArgs sc, FxLimits lim) {
  fx_scale_device(sc.parts, sc.nparts, sc.n_center, lim, sc.stats);
}

// Bank-aware load order for the fx kernel. A warp's fiber is 4*NV 128-byte
// lines; load step j brings 4 whole lines (coalesced) and issues 4 ATOMS
// instructions, instruction k taking element k of every lane's float4. The
// ATOMS bank of element i is (h0(i) + c) mod 32 with c common to the whole
// fiber, so the bank conflicts of an instruction depend on h0 alone, and the
// cost of a grouping is sum over steps and k of the largest bank count.
// groups[d][j][q] = line of slot q (lanes 8q..8q+7) at step j — any
// permutation of the lines is correct (the grouping only moves wavefronts).
//
// One CTA per family: (1) a fingerprint of the family's mode-0 table looks up
// a device-side cache of earlier groupings (a hit is checked to be a
// permutation before use, so a stale or torn entry can cost speed, never
// correctness); on a miss (2) greedy construction — per step, seed with the
// worst remaining line, then add the line that minimises the group cost —
// then (3) up to kFxSearchIters rounds of parallel swap search (scaled with
// the tensor size so the one-off search stays a few % of one sketch): each warp prices
// one pseudo-random swap of two lines between two steps (lane = bank), the
// best swap is applied if it does not raise the cost (plateau moves allowed).
// Config-4 tables: greedy ~2.9, searched ~2.7 wavefronts per ATOMS
// (random order ~3.6).
constexpr int kFxSearchIters = 256;  // search rounds for a 2^30-element tensor (scaled down below)
constexpr int kFxCacheSlots = 64;
struct FxGroupEntry {
  unsigned long long fp;
  uint8_t g[32];
};

__device__ __forceinline__ unsigned long long fx_mix(unsigned long long x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void __launch_bounds__(1024) fx_group_kernel(const uint32_t* __restrict__ packed,
                                                        uint32_t fam_stride, uint32_t i0_shift,
                                                        int nsteps, int iters,
                                                        uint8_t* __restrict__ groups,
                                                        FxGroupEntry* __restrict__ cache) {
  __shared__ uint8_t lh[32][4][32];  // [line][k][bank] element counts
  __shared__ int h[4][32];           // current group's counts (greedy)
  __shared__ int H[8][4][32];        // per-step bank counts (search)
  __shared__ int cost[32];           // greedy: per-line price; search: per-step cost
  __shared__ int cand[32][6];        // search: delta, j1, q1, j2, q2, c1 | c2 << 16
  __shared__ uint8_t g[8][4];
  __shared__ unsigned long long fp_part[32];
  __shared__ uint32_t used;
  __shared__ int hit;
  const int d = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t* tab = packed + static_cast<uint64_t>(d) * fam_stride + i0_shift;
  const int nlines = 4 * nsteps;
  // (1) fingerprint of the line residues (bucket mod 32 is all the grouping
  // depends on) and the step count; cache lookup
  uint32_t bank = 0;
  unsigned long long f = 0;
  if (w < nlines) {
    bank = __ldg(tab + 32 * w + lane) & 31u;  // element t = lane of line w
    f = fx_mix((static_cast<unsigned long long>(32 * w + lane) << 8) | bank);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) f ^= __shfl_xor_sync(0xffffffffu, f, o);
  if (lane == 0) fp_part[w] = f;
  if (threadIdx.x == 0) {
    used = 0;
    hit = 0;
  }
  __syncthreads();
  const unsigned long long fp = [&] {
    unsigned long long x = fx_mix(static_cast<unsigned long long>(nsteps) + 0x9e3779b97f4a7c15ull);
    for (int i = 0; i < 32; ++i) x ^= fp_part[i];
    return x | 1ull;  // never 0 (empty slot)
  }();
  FxGroupEntry* slot = cache ? cache + (fp % kFxCacheSlots) : nullptr;
  if (slot != nullptr && threadIdx.x < 32) {
    const bool same = *reinterpret_cast<volatile unsigned long long*>(&slot->fp) == fp;
    const uint32_t line = lane < nlines ? reinterpret_cast<volatile uint8_t*>(slot->g)[lane] : 0u;
    const uint32_t mask = __reduce_or_sync(0xffffffffu, lane < nlines ? 1u << (line & 31u) : 0u);
    const bool perm = same && mask == (nlines == 32 ? 0xffffffffu : (1u << nlines) - 1u) &&
                      __all_sync(0xffffffffu, lane >= nlines || line < static_cast<uint32_t>(nlines));
    if (perm) {
      if (lane < nlines) groups[static_cast<size_t>(d) * nlines + lane] = static_cast<uint8_t>(line);
      if (lane == 0) hit = 1;
    }
  }
  __syncthreads();
  if (hit) return;
  // (2) greedy
  if (w < nlines) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int cnt = 0;  // elements t = k (mod 4) of line w that land in bank `lane`
#pragma unroll
      for (int t = k; t < 32; t += 4) cnt += (__shfl_sync(0xffffffffu, bank, t) == static_cast<uint32_t>(lane));
      lh[w][k][lane] = static_cast<uint8_t>(cnt);
    }
  }
  for (int j = 0; j < nsteps; ++j) {
    if (threadIdx.x < 128) h[threadIdx.x >> 5][lane] = 0;
    __syncthreads();
    for (int pick = 0; pick < 4; ++pick) {
      if (w < nlines) {
        int c = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          int v = h[k][lane] + lh[w][k][lane];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
          c += v;
        }
        if (lane == 0) cost[w] = c;
      }
      __syncthreads();
      if (w == 0) {
        // warp argmin over key = (signed cost, line): ties go to the lowest line
        const bool ok = lane < nlines && !(used >> lane & 1u);
        int key = ok ? ((pick == 0 ? 4096 - cost[lane] : cost[lane]) << 5) | lane : 0x7fffffff;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
        const int b = key & 31;
#pragma unroll
        for (int k = 0; k < 4; ++k) h[k][lane] += lh[b][k][lane];  // warp 0 owns h
        if (lane == 0) {
          used |= 1u << b;
          g[j][pick] = static_cast<uint8_t>(b);
        }
      }
      __syncthreads();
    }
  }
  // (3) parallel swap search
  for (int i = threadIdx.x; i < nsteps * 128; i += blockDim.x) {
    const int j = i >> 7, k = (i >> 5) & 3, b = i & 31;
    H[j][k][b] = lh[g[j][0]][k][b] + lh[g[j][1]][k][b] + lh[g[j][2]][k][b] + lh[g[j][3]][k][b];
  }
  __syncthreads();
  if (w < nsteps) {
    int c = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int v = H[w][k][lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
      c += v;
    }
    if (lane == 0) cost[w] = c;
  }
  __syncthreads();
  for (int it = 0; it < (nsteps >= 2 ? iters : 0); ++it) {
    {
      // 32-bit draws; nsteps is a power of two (2, 4 or 8)
      const uint32_t r = static_cast<uint32_t>(
          fx_mix((static_cast<unsigned long long>(d) << 40) ^ (static_cast<unsigned long long>(it) << 8) ^
                 static_cast<unsigned long long>(w)));
      const int j1 = static_cast<int>(r & static_cast<uint32_t>(nsteps - 1));
      const int j2 = (j1 + 1 + static_cast<int>((r >> 8) % static_cast<uint32_t>(nsteps - 1))) &
                     (nsteps - 1);
      const int q1 = static_cast<int>((r >> 20) & 3), q2 = static_cast<int>((r >> 24) & 3);
      const int a = g[j1][q1], b = g[j2][q2];
      int c1 = 0, c2 = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        int v1 = H[j1][k][lane] - lh[a][k][lane] + lh[b][k][lane];
        int v2 = H[j2][k][lane] - lh[b][k][lane] + lh[a][k][lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          v1 = max(v1, __shfl_xor_sync(0xffffffffu, v1, o));
          v2 = max(v2, __shfl_xor_sync(0xffffffffu, v2, o));
        }
        c1 += v1;
        c2 += v2;
      }
      if (lane == 0) {
        cand[w][0] = c1 + c2 - cost[j1] - cost[j2];
        cand[w][1] = j1;
        cand[w][2] = q1;
        cand[w][3] = j2;
        cand[w][4] = q2;
        cand[w][5] = c1 | (c2 << 16);
      }
    }
    __syncthreads();
    // best candidate (ties: lowest warp), applied if it does not raise the cost
    int key = ((cand[lane][0] + 1024) << 5) | lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
    const int bw = key & 31;
    if (cand[bw][0] <= 0) {
      const int j1 = cand[bw][1], q1 = cand[bw][2], j2 = cand[bw][3], q2 = cand[bw][4];
      const int a = g[j1][q1], b = g[j2][q2];
      if (threadIdx.x < 128) {
        const int k = threadIdx.x >> 5;
        H[j1][k][lane] += lh[b][k][lane] - lh[a][k][lane];
        H[j2][k][lane] += lh[a][k][lane] - lh[b][k][lane];
      }
      __syncthreads();  // every thread has read g / cand before the swap below
      if (threadIdx.x == 0) {
        g[j1][q1] = static_cast<uint8_t>(b);
        g[j2][q2] = static_cast<uint8_t>(a);
        cost[j1] = cand[bw][5] & 0xffff;
        cost[j2] = cand[bw][5] >> 16;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x < nlines) {
    const uint8_t line = g[threadIdx.x >> 2][threadIdx.x & 3];
    groups[static_cast<size_t>(d) * nlines + threadIdx.x] = line;
    if (slot != nullptr) slot->g[threadIdx.x] = line;
  }
  if (slot != nullptr) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) slot->fp = fp;  // published after the lines
  }
}

__device__ __forceinline__ void fiber_offset_fast(const DenseArgs& a, const uint32_t* tab,
                                                  uint64_t f, uint32_t& c, uint32_t& sbit) {
  if (a.order == 3 && a.fibers < 0xffffffffull) {
    const uint32_t ff = static_cast<uint32_t>(f);
    const uint32_t i2r = __umulhi(ff, a.inv_d1);  // ff / dims[1] (exact: ff < 2^32 / dims[1])
    const uint32_t q2 = ff - i2r * a.dims[1] >= a.dims[1] ? i2r + 1 : i2r;
    const uint32_t i1 = ff - q2 * a.dims[1], i2 = q2 + a.last_begin;
    const uint32_t e1 = __ldg(tab + a.tab_off[1] + i1), e2 = __ldg(tab + a.tab_off[2] + i2);
    c = (e1 & 0x7fffffffu) * a.mult[1] + (e2 & 0x7fffffffu) * a.mult[2];
    sbit = (e1 ^ e2) & 0x80000000u;
  } else {
    fiber_offset(a, tab, f, c, sbit);
  }
}

// float32 fast path (I_0 % 4 == 0, 16-byte aligned fibers, I_0 <= 128 * NV):
// warp per fiber, lane-owned mode-0 indices with their table entries in
// registers, NV 128-bit loads per lane with the next fiber prefetched,
// int32 fixed-point shared-memory accumulation with exact overflow detection.
__device__ void fx_float_redo(const DenseArgs& a, const float* __restrict__ t,
                              const uint32_t* __restrict__ tab, float scale, uint64_t chunk,
                              bool skip_diverted, float* skf, uint32_t r_lo = 0,
                              uint32_t r_cnt = 0xffffffffu);

// kRedo = false: the scatter; kRedo = true: the same loop over the chunks the
// scatter flagged (flag 2: an element out of the fixed-point range), each
// out-of-range element diverted to an fp64 reduction into `divert` (D x J~,
// added by reduce_fx_kernel) so the chunk stays in fixed point; a chunk that
// wraps (or was flagged for wrap / tiny partials, flag 4) is redone with fp32
// shared atomics (fx_float_redo), skipping what was diverted.
template <int NV, int SPLIT, int THREADS, bool kFull, bool kGroup = false, bool kRedo = false>
__global__ void __launch_bounds__(THREADS, 1) fcs_dense_fx_kernel(DenseArgs a,
                                                              const float* __restrict__ t,
                                                              const uint32_t* __restrict__ packed,
                                                              const FxStats* __restrict__ st,
                                                              int32_t* __restrict__ part,
                                                              int* __restrict__ flags,
                                                              const uint8_t* __restrict__ groups,
                                                              double* __restrict__ divert) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int32_t* sk = reinterpret_cast<int32_t*>(smem_raw);
  const int d = blockIdx.x % a.D;
  const uint64_t chunk = blockIdx.x / a.D;
  const uint32_t* tab = packed + static_cast<uint64_t>(d) * a.fam_stride;
  int in_flag = 0;
  if constexpr (kRedo) {
    in_flag = flags[chunk * a.D + d];
    if (!(in_flag & 2)) return;
    if (in_flag & 4) {  // wrap or tiny partials: the fixed point cannot help
      fx_float_redo(a, t, tab, ldexpf(1.0f, st->S), chunk, false,
                    reinterpret_cast<float*>(smem_raw));
      int32_t* dst = part + (chunk * a.D + d) * static_cast<uint64_t>(a.jt);
      for (uint32_t b = threadIdx.x; b < a.jt; b += blockDim.x) dst[b] = sk[b];
      if (threadIdx.x == 0) flags[chunk * a.D + d] = 1;
      return;
    }
  }
  double* dv = kRedo ? divert + static_cast<uint64_t>(d) * a.jt : nullptr;
  const float scale = ldexpf(1.0f, st->S);
  for (uint32_t b = threadIdx.x; b < a.jt; b += blockDim.x) sk[b] = 0;

  // SPLIT warps share a fiber: warp w takes part w % SPLIT (32*NV vectors) of
  // fiber group w / SPLIT.
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int warp = wid / SPLIT, nwarps = (blockDim.x >> 5) / SPLIT;
  const uint32_t vbase = static_cast<uint32_t>(wid % SPLIT) * 32u * NV;
  const uint32_t i0n = a.dims[0];
  const uint32_t nvec = i0n / 4;
  // Vector this lane loads at step j: lane + 32 j, or with the bank-aware
  // grouping (kFull only) 8 * line + (lane & 7), line = groups[d][j][lane / 8];
  // the indices are kept packed four per register (vmap).
  constexpr bool kMapped = kGroup && kFull && SPLIT == 1;  // vector map in vmap
  const bool grouped = kMapped && groups != nullptr;
  uint32_t vmap[(NV + 3) / 4];
#pragma unroll
  for (int w = 0; w < (NV + 3) / 4; ++w) vmap[w] = 0;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const uint32_t v = grouped ? 8u * groups[(static_cast<size_t>(d) * NV + j) * 4 + (lane >> 3)] +
                                     (lane & 7u)
                               : static_cast<uint32_t>(lane + 32 * j);
    vmap[j / 4] |= (v & 0xffu) << (8 * (j % 4));
  }
  uint32_t e0[NV][4];  // packed mode-0 entries (bucket | sign << 31)
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const uint32_t v = kMapped ? ((vmap[j / 4] >> (8 * (j % 4))) & 0xffu)
                               : vbase + lane + 32 * j;
#pragma unroll
    for (int k = 0; k < 4; ++k) e0[j][k] = v < nvec ? __ldg(tab + a.i0_shift + v * 4 + k) : 0u;
  }
  __syncthreads();

  const uint64_t f_begin = chunk * a.fibers_per_chunk;
  const uint64_t f_end = min(a.fibers, f_begin + a.fibers_per_chunk);
  float4 cur[NV], nxt[NV];
  auto load = [&](uint64_t fib, float4* dst) {
    const float4* src = reinterpret_cast<const float4*>(t + fib * i0n);
    if constexpr (kMapped) {
#pragma unroll
      for (int j = 0; j < NV; ++j) dst[j] = ld_stream(src + ((vmap[j / 4] >> (8 * (j % 4))) & 0xffu));
    } else {
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (vbase + lane + 32 * j < nvec) dst[j] = ld_stream(src + vbase + lane + 32 * j);
    }
  };
  uint64_t f = f_begin + warp;
  if (f < f_end) load(f, cur);
  const uint32_t sk_base = static_cast<uint32_t>(__cvta_generic_to_shared(sk));
  uint32_t ovf_acc = 0;  // bit 31: some partial reached |old| >= 2^30 (wrap guard)
  uint32_t rng_acc = 0;  // bits >= 23: a converted element was out of range / non-finite
  // One fiber: the fiber sign goes into the scale; the byte address of bucket
  // h0 + c is base + 4c + (entry << 2), the shift discarding the entry's sign bit.
  auto scatter = [&](const float4* vals, uint64_t fib) {
    uint32_t c, sbit;
    fiber_offset_fast(a, tab, fib, c, sbit);
    const float scale_f = sbit ? -scale : scale;
    uint32_t base_c = sk_base + 4u * c;
    // opaque to the optimiser: keeps the per-element address a single
    // LEA(entry, base_c) instead of (c + entry) * 4 + a rematerialised window base
    asm volatile("" : "+r"(base_c));
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      if (kFull || vbase + lane + 32 * j < nvec) {  // kFull: every lane owns whole vectors
        const float* x = reinterpret_cast<const float*>(&vals[j]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t e = e0[j][k];
          // x ^ (e & sign): one LOP3 per use (volatile: a hoisted e & sign
          // would double the 4*NV live table registers and spill)
          uint32_t xsb;
          asm volatile("lop3.b32 %0, %1, %2, 0x80000000, 0x78;"
                       : "=r"(xsb)
                       : "r"(__float_as_uint(x[k])), "r"(e));
          const float xs = __uint_as_float(xsb);
          // round-to-nearest int via the 1.5 * 2^23 magic number: for |y| < 2^22
          // the sum's bits are 0x4B400000 + round(y), exponent 0x96; any other
          // exponent (out of range, Inf, NaN) leaves bits >= 23 in bits ^ 0x4B000000
          const uint32_t bits = __float_as_uint(fmaf(xs, scale_f, 12582912.0f));
          int32_t q;
          if constexpr (kRedo) {
            q = static_cast<int32_t>(bits - 0x4B400000u);
            if ((bits ^ 0x4B000000u) >> 23) {  // exact fp64 reduction instead
              atomicAdd(dv + (e & 0x7fffffffu) + c,
                        static_cast<double>(scale_f < 0.f ? -xs : xs));
              q = 0;
            }
          } else {
            rng_acc |= bits ^ 0x4B000000u;
            q = static_cast<int32_t>(bits - 0x4B400000u);
          }
          int32_t old;
          asm volatile("atom.shared.add.s32 %0, [%1], %2;"
                       : "=r"(old)
                       : "r"(base_c + (e << 2)), "r"(q));
          // guard band: |q| < 2^22, so a partial can only wrap after passing
          // through |old| >= 2^30, which sets bit 31 of old + 2^30
          ovf_acc |= static_cast<uint32_t>(old) + 0x40000000u;
        }
      }
    }
  };
  // Ping-pong between the two register buffers (no copies).
  for (; f < f_end; f += 2 * nwarps) {
    if (f + nwarps < f_end) load(f + nwarps, nxt);
    scatter(cur, f);
    if (f + nwarps >= f_end) break;
    if (f + 2 * nwarps < f_end) load(f + 2 * nwarps, cur);
    scatter(nxt, f + nwarps);
  }
  if constexpr (kRedo) {
    const bool wrapped = __syncthreads_or(static_cast<int>(ovf_acc >> 31));
    if (wrapped)
      fx_float_redo(a, t, tab, scale, chunk, true, reinterpret_cast<float*>(smem_raw));
    int32_t* dst = part + (chunk * a.D + d) * static_cast<uint64_t>(a.jt);
    for (uint32_t b = threadIdx.x; b < a.jt; b += blockDim.x) dst[b] = sk[b];
    if (threadIdx.x == 0) flags[chunk * a.D + d] = wrapped ? 1 : 8;  // 8: fixed point, redone
    return;
  }
  // A CTA that saw an out-of-range or non-finite element (range), a partial
  // reaching 2^30 (wrap), or only nonzero-but-tiny partials (precision guard,
  // kFxSmallBits) leaves its chunk to the kRedo instantiation: flag 2 (+4 when
  // the fixed point cannot help: wrap or tiny partials).
  const bool wrapped = __syncthreads_or(static_cast<int>(ovf_acc >> 31));
  const bool ranged = __syncthreads_or(static_cast<int>((rng_acc >> 23) != 0));
  bool tiny = false;
  if (!wrapped && !ranged) {  // precision guard: all partials nonzero-but-tiny
    int nz = 0, big = 0;
    for (uint32_t b = threadIdx.x; b < a.jt; b += blockDim.x) {
      const int32_t v = sk[b];
      const uint32_t m = static_cast<uint32_t>(v < 0 ? -v : v);
      nz |= m != 0u;
      big |= (m >> kFxSmallBits) != 0u;
    }
    const bool any_big = __syncthreads_or(big);
    tiny = __syncthreads_or(nz) && !any_big;
  }
  // (an out-of-range element also adds a garbage word, which can fake a wrap:
  // with `ranged` the redo decides about wrapping itself)
  if (threadIdx.x == 0)
    flags[chunk * a.D + d] =
        (wrapped || ranged || tiny) ? (2 | ((!ranged && (wrapped || tiny)) ? 4 : 0)) : 0;
  if (wrapped || ranged || tiny) return;
  int32_t* dst = part + (chunk * a.D + d) * static_cast<uint64_t>(a.jt);
  for (uint32_t b = threadIdx.x; b < a.jt; b += blockDim.x) dst[b] = sk[b];
}

// fp32 shared-atomic redo of one chunk into skf (the CTA's sketch memory);
// skip_diverted: leave out the elements the fixed-point redo diverted (out of
// range at this scale) — they are already in `divert`.
// r_lo / r_cnt: only buckets [r_lo, r_lo + r_cnt) (a bucket-range CTA; skf
// holds that range); the defaults take every bucket.
__device__ void fx_float_redo(const DenseArgs& a, const float* __restrict__ t,
                              const uint32_t* __restrict__ tab, float scale, uint64_t chunk,
                              bool skip_diverted, float* skf, uint32_t r_lo, uint32_t r_cnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint64_t f_begin = chunk * a.fibers_per_chunk;
  const uint64_t f_end = min(a.fibers, f_begin + a.fibers_per_chunk);
  const uint32_t i0n = a.dims[0];
  r_cnt = min(r_cnt, a.jt);
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < r_cnt; b += blockDim.x) skf[b] = 0.f;
  __syncthreads();
  for (uint64_t g = f_begin + warp; g < f_end; g += nwarps) {
    uint32_t c, sbit;
    fiber_offset(a, tab, g, c, sbit);
    const float scale_f = sbit ? -scale : scale;
    for (uint32_t i = lane; i < i0n; i += 32) {
      const float x = __ldcs(t + g * i0n + i);
      const uint32_t e = __ldg(tab + a.i0_shift + i);
      if (skip_diverted) {
        const float xs = __uint_as_float(__float_as_uint(x) ^ (e & 0x80000000u));
        if ((__float_as_uint(fmaf(xs, scale_f, 12582912.0f)) ^ 0x4B000000u) >> 23) continue;
      }
      const uint32_t lb = (e & 0x7fffffffu) + c - r_lo;
      if (lb < r_cnt)
        atomicAdd(&skf[lb], __uint_as_float(__float_as_uint(x) ^ ((e ^ sbit) & 0x80000000u)));
    }
  }
  __syncthreads();
}

// float64 fixed-point path (any order >= 2, I_0 <= 1024): shared-memory
// fp64 atomics are CAS loops on sm_100a (measured 1.2 random updates/clk/SM
// vs 9.8 for int32 ATOMS.ADD, profiles/fp64_peak.json), so each bucket holds
// a 64-bit fixed-point partial as two int32 words (lo: unsigned, hi: signed;
// separate arrays so both words of one instruction spread over 32 banks).
// An element becomes q = round(x 2^S) by the fp64 magic number 1.5 * 2^52
// (exact for |x 2^S| < 2^51); lo += q_lo returns the old word, whose carry
// goes with q_hi into hi — every carry is exact because each add's carry is
// a function of its own returned old value, whatever order adds arrive in.
// The element range (exponent of the magic sum) and a guard band on hi
// (|partial| reaching 2^61) are checked exactly; a CTA that trips either
// redoes its chunk with fp64 CAS atomics. Partials are summed exactly in
// 128-bit integers in the reduction, then scaled by 2^-S once.
// Lane-owned mode-0 indices i_0 = lane + 32 k (k < NV) with their table
// entries in registers; each lane keeps NV loads in flight per fiber.
constexpr double kMagic64 = 6755399441055744.0;  // 1.5 * 2^52 (bits 0x4338000000000000)

__device__ __forceinline__ double ld_stream64(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
// fp32 input to the 64-bit fixed point (fp32 tensors the int32 kernel does not
// take: I_0 % 4 != 0); widened exactly.
__device__ __forceinline__ double ld_stream64(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return static_cast<double>(v);
}

// Warp-level sample statistics of fiber k * fibers / nsample into parts[k]
// (per-fiber order fixed).
template <typename Tin>
__device__ void fx_sample_warps(const DenseArgs& a, const Tin* __restrict__ t, uint64_t nsample,
                                FxPart* __restrict__ parts) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  const uint32_t i0n = a.dims[0];
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
       k < nsample; k += nw) {
    const uint64_t f = (k * a.fibers) / nsample;
    double mx = 0.0, s = 0.0, s2 = 0.0, cnt = 0.0;
    for (uint32_t i = lane; i < i0n; i += 32) {
      const double x = static_cast<double>(t[f * i0n + i]);
      mx = fmax(mx, fabs(x));
      s += x;
      s2 += x * x;
      cnt += 1.0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      s += __shfl_xor_sync(0xffffffffu, s, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if (lane == 0) parts[k] = FxPart{mx, s, s2, cnt};
  }
}

template <typename Tin>
__global__ void __launch_bounds__(256) fx_sample_warps_kernel(DenseArgs a, const Tin* __restrict__ t,
                                                              uint64_t nsample,
                                                              FxPart* __restrict__ parts,
                                                              double* __restrict__ zero = nullptr,
                                                              uint64_t nzero = 0) {
  fx_sample_warps<Tin>(a, t, nsample, parts);
  // the fp64 diversion buffer of the fp32 path, cleared here instead of by a memset
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nzero;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    zero[i] = 0.0;
}

// Sampled fibers: an eighth of the tensor's fibers, at least 256, at most 2048.
inline uint64_t fx_nsample(uint64_t fibers) {
  return std::min<uint64_t>(fibers, std::min<uint64_t>(kFxMaxSample,
                                                       std::max<uint64_t>(256, fibers / 8)));
}

__device__ __forceinline__ double i128_to_double(__int128 acc);

template <typename Tin, int NV, bool kFull, bool kRange>
__global__ void __launch_bounds__(512) fcs_dense_fx64_kernel(DenseArgs a,
                                                             const Tin* __restrict__ t,
                                                             const uint32_t* __restrict__ packed,
                                                             const FxStats* __restrict__ st,
                                                             uint32_t* __restrict__ part,
                                                             int* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* lo = reinterpret_cast<uint32_t*>(smem_raw);
  const int d = blockIdx.x % a.D;
  // kRange: this CTA holds buckets [r_lo, r_lo + r_cnt) of its family (plus
  // 32 dummy buckets: an element of another range adds 0 to bucket `lane`
  // past the range, so no predicate and no bank conflict)
  const uint32_t rp = kRange ? (blockIdx.x / a.D) % a.rparts : 0u;
  const uint64_t chunk = kRange ? blockIdx.x / (a.D * a.rparts) : blockIdx.x / a.D;
  const uint32_t span = kRange ? a.rspan : a.jt;
  const uint32_t r_lo = rp * span;
  const uint32_t r_cnt = kRange ? min(span, a.jt - r_lo) : a.jt;
  const uint32_t words = kRange ? span + 32u : a.jt;  // per word array
  const uint64_t prow = kRange ? (chunk * a.D + d) * a.rparts + rp : chunk * a.D + d;
  const uint32_t* tab = packed + static_cast<uint64_t>(d) * a.fam_stride;
  const double scale = ldexp(1.0, st->S);
  for (uint32_t b = threadIdx.x; b < 2 * words; b += blockDim.x) lo[b] = 0u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t i0n = a.dims[0];
  // I_0 > 1024: warp w takes segment w % 2^lseg of the fibers (entries
  // s0 .. s0 + slen of every fiber), 16 / 2^lseg fibers at a time
  const uint32_t s0 = (static_cast<uint32_t>(warp) & ((1u << a.lseg) - 1u)) * a.seg_len;
  const uint32_t slen = min(a.seg_len, i0n - s0);
  const int fstride = nwarps >> a.lseg;
  // mode-0 buckets two per register (bucket < jt <= 29056 < 2^16) and signs
  // as a bit mask (bit k: entry i_0 = s0 + lane + 32 k). Entries past the
  // segment load no data (x = 0 adds q = 0) and point at bucket `lane`:
  // distinct banks, so the padding lanes cost no conflicts and need no predicate.
  uint32_t bk[(NV + 1) / 2];
  uint32_t smask = 0;
#pragma unroll
  for (int k = 0; k < (NV + 1) / 2; ++k) bk[k] = 0u;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const uint32_t i = lane + 32u * k;
    const uint32_t e = i < slen ? __ldg(tab + a.i0_shift + s0 + i) : static_cast<uint32_t>(lane);
    bk[k / 2] |= (e & 0xffffu) << (16 * (k % 2));
    smask |= (e >> 31) << k;
  }
  __syncthreads();
  const uint64_t f_begin = chunk * a.fibers_per_chunk;
  const uint64_t f_end = min(a.fibers, f_begin + a.fibers_per_chunk);
  const uint32_t lo_base = static_cast<uint32_t>(__cvta_generic_to_shared(lo));
  const uint32_t hi_off = 4u * words;
  uint32_t rng_acc = 0, ovf_acc = 0;
  // A fiber is NB batches of LB entries per lane; the next batch's loads (of
  // this fiber or the next) are in flight while the current batch is
  // scattered (two register buffers, ping-pong, batch index compile-time).
  constexpr int LB = NV < 16 ? NV : 16;
  constexpr int NB = NV / LB;
  constexpr int G = LB < 4 ? LB : 4;
  auto load = [&]<int KB>(uint64_t f, double* x) {
    const Tin* fib = t + f * i0n + s0;
#pragma unroll
    for (int k = 0; k < LB; ++k)
      x[k] = (kFull || lane + 32u * (KB + k) < slen) ? ld_stream64(fib + lane + 32 * (KB + k)) : 0.0;
  };
  uint32_t base_c = 0, fmask = 0;
  auto scatter = [&]<int KB>(uint64_t f, const double* x) {
    if (KB == 0) {
      uint32_t c, sbit;
      fiber_offset_fast(a, tab, f, c, sbit);
      base_c = kRange ? c - r_lo : lo_base + 4u * c;  // kRange: range-relative offset
      fmask = smask ^ (sbit ? 0xffffffffu : 0u);  // bit k: final sign of entry k
    }
#pragma unroll
    for (int kg = 0; kg < LB; kg += G) {
      uint32_t qh[G], ql[G], ad[G], old[G];
#pragma unroll
      for (int k = 0; k < G; ++k) {
        constexpr int dummy = 0;
        (void)dummy;
        const int kk = KB + kg + k;
        const uint32_t e = (kk % 2) ? (bk[kk / 2] >> 16) : (bk[kk / 2] & 0xffffu);
        bool in_range = true;
        if constexpr (kRange) {
          const uint32_t lb = base_c + e;
          in_range = lb < r_cnt;
          ad[k] = lo_base + 4u * (in_range ? lb : span + static_cast<uint32_t>(lane));
        } else {
          ad[k] = base_c + (e << 2);
        }
        // sign: bit kk of fmask onto the top bit of x
        const uint64_t xb = static_cast<uint64_t>(__double_as_longlong(x[kg + k])) ^
                            (static_cast<uint64_t>((fmask << (31 - kk)) & 0x80000000u) << 32);
        const uint64_t bits = static_cast<uint64_t>(
            __double_as_longlong(fma(__longlong_as_double(xb), scale, kMagic64)));
        const uint32_t bh = static_cast<uint32_t>(bits >> 32);
        // exponent of the magic sum must stay 52 (0x433): else out of range / non-finite
        rng_acc |= bh ^ 0x43300000u;
        ql[k] = in_range ? static_cast<uint32_t>(bits) : 0u;  // the magic's low word is 0
        qh[k] = in_range ? bh - 0x43380000u : 0u;
      }
      // the low-word adds first (their returned values give the carries), then the high words
#pragma unroll
      for (int k = 0; k < G; ++k)
        asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old[k]) : "r"(ad[k]), "r"(ql[k]));
#pragma unroll
      for (int k = 0; k < G; ++k) {
        uint32_t hv, oh;
        // carry out of old + q_lo into q_hi
        asm("{ .reg .u32 tmp; add.cc.u32 tmp, %1, %2; addc.u32 %0, %3, 0; }"
            : "=r"(hv) : "r"(old[k]), "r"(ql[k]), "r"(qh[k]));
        asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(oh) : "r"(ad[k] + hi_off), "r"(hv));
        // guard band: |partial| >= 2^61 sets bit 31 of hi + 2^29 (one add moves hi < 2^20)
        ovf_acc |= oh + 0x20000000u;
      }
    }
  };
  double cur[LB], nxt[LB];
  uint64_t f = f_begin + (warp >> a.lseg);
  if (f < f_end) load.template operator()<0>(f, cur);
  if constexpr (NB == 1) {
    for (; f < f_end; f += 2 * fstride) {
      if (f + fstride < f_end) load.template operator()<0>(f + fstride, nxt);
      scatter.template operator()<0>(f, cur);
      if (f + fstride >= f_end) break;
      if (f + 2 * fstride < f_end) load.template operator()<0>(f + 2 * fstride, cur);
      scatter.template operator()<0>(f + fstride, nxt);
    }
  } else {
    static_assert(NB == 2, "NV = 32: two batches of 16");
    for (; f < f_end; f += fstride) {
      load.template operator()<LB>(f, nxt);
      scatter.template operator()<0>(f, cur);
      if (f + fstride < f_end) load.template operator()<0>(f + fstride, cur);
      scatter.template operator()<LB>(f, nxt);
    }
  }
  const int ovf = (ovf_acc >> 31) | ((rng_acc >> 20) != 0);
  const bool overflowed = __syncthreads_or(ovf);
  if (overflowed) {  // exact fallback for this CTA: fp64 atomics over the same chunk
    double* skd = reinterpret_cast<double*>(smem_raw);
    for (uint32_t b = threadIdx.x; b < r_cnt; b += blockDim.x) skd[b] = 0.0;
    __syncthreads();
    for (uint64_t g = f_begin + warp; g < f_end; g += nwarps) {
      uint32_t c, sbit;
      fiber_offset(a, tab, g, c, sbit);
      for (uint32_t i = lane; i < i0n; i += 32) {
        const double x = static_cast<double>(__ldcs(t + g * i0n + i));
        const uint32_t e = __ldg(tab + a.i0_shift + i);
        const uint32_t lb = (e & 0x7fffffffu) + c - r_lo;
        if (x != 0.0 && lb < r_cnt) atomicAdd(&skd[lb], ((e ^ sbit) & 0x80000000u) ? -x : x);
      }
    }
    __syncthreads();
  }
  // partial layout per (chunk, d[, range]): span lo words then span hi words
  // (or span doubles when flagged); kRange = false: span = J~
  uint32_t* dst = part + prow * 2ull * span;
  if (overflowed) {
    for (uint32_t b = threadIdx.x; b < 2 * r_cnt; b += blockDim.x) dst[b] = lo[b];
  } else {
    for (uint32_t b = threadIdx.x; b < r_cnt; b += blockDim.x) {
      dst[b] = lo[b];
      dst[span + b] = lo[words + b];
    }
  }
  if (threadIdx.x == 0) flags[prow] = overflowed ? 1 : 0;
}

// float32 fixed point with scalar loads (fp32 tensors off the float4 path:
// I_0 % 4 != 0 or a tensor not 16-byte aligned, I_0 <= 1024): the int32
// fixed point of fcs_dense_fx_kernel (same scale, range check, wrap guard and
// partial format) on the fx64 kernel's lane layout — i_0 = lane + 32 k,
// k < NV, buckets packed two per register, signs as a bit mask, padding lanes
// of a partial fiber adding 0 to bucket `lane`, batches of LB loads in flight.
// A flagged chunk (range, wrap or tiny partials) is redone with fp32 shared
// atomics. One LDG.32 per element moves the same 128-byte lines as the float4
// loads, so the LSU wavefronts per element are unchanged.
// kRange: J~ beyond shared memory — this CTA holds buckets [r_lo, r_lo +
// r_cnt) of its family (+ 32 dummy buckets), as fcs_dense_fx64_kernel.
template <int NV, bool kFull, bool kRange>
__global__ void __launch_bounds__(512) fcs_dense_fx32s_kernel(DenseArgs a,
                                                              const float* __restrict__ t,
                                                              const uint32_t* __restrict__ packed,
                                                              const FxStats* __restrict__ st,
                                                              int32_t* __restrict__ part,
                                                              int* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int32_t* sk = reinterpret_cast<int32_t*>(smem_raw);
  const int d = blockIdx.x % a.D;
  const uint32_t rp = kRange ? (blockIdx.x / a.D) % a.rparts : 0u;
  const uint64_t chunk = kRange ? blockIdx.x / (a.D * a.rparts) : blockIdx.x / a.D;
  const uint32_t span = kRange ? a.rspan : a.jt;
  const uint32_t r_lo = rp * span;
  const uint32_t r_cnt = kRange ? min(span, a.jt - r_lo) : a.jt;
  const uint64_t prow = kRange ? (chunk * a.D + d) * a.rparts + rp : chunk * a.D + d;
  const uint32_t* tab = packed + static_cast<uint64_t>(d) * a.fam_stride;
  const float scale = ldexpf(1.0f, st->S);
  for (uint32_t b = threadIdx.x; b < (kRange ? span + 32u : a.jt); b += blockDim.x) sk[b] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t i0n = a.dims[0];
  // I_0 > 1024: segments of the fibers per warp, as fcs_dense_fx64_kernel
  const uint32_t s0 = (static_cast<uint32_t>(warp) & ((1u << a.lseg) - 1u)) * a.seg_len;
  const uint32_t slen = min(a.seg_len, i0n - s0);
  const int fstride = nwarps >> a.lseg;
  uint32_t bk[(NV + 1) / 2];
  uint32_t smask = 0;
#pragma unroll
  for (int k = 0; k < (NV + 1) / 2; ++k) bk[k] = 0u;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const uint32_t i = lane + 32u * k;
    const uint32_t e = i < slen ? __ldg(tab + a.i0_shift + s0 + i) : static_cast<uint32_t>(lane);
    bk[k / 2] |= (e & 0xffffu) << (16 * (k % 2));
    smask |= (e >> 31) << k;
  }
  __syncthreads();
  const uint64_t f_begin = chunk * a.fibers_per_chunk;
  const uint64_t f_end = min(a.fibers, f_begin + a.fibers_per_chunk);
  const uint32_t sk_base = static_cast<uint32_t>(__cvta_generic_to_shared(sk));
  uint32_t rng_acc = 0, ovf_acc = 0;
  constexpr int LB = NV < 16 ? NV : 16;
  constexpr int NB = NV / LB;
  auto load = [&]<int KB>(uint64_t f, float* x) {
    const float* fib = t + f * i0n + s0;
#pragma unroll
    for (int k = 0; k < LB; ++k) {
      const uint32_t i = lane + 32u * (KB + k);
      if (kFull || i < slen) {
        asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(x[k]) : "l"(fib + i));
      } else {
        x[k] = 0.f;
      }
    }
  };
  uint32_t base_c = 0;
  float scale_f = scale;
  auto scatter = [&]<int KB>(uint64_t f, const float* x) {
    if (KB == 0) {
      uint32_t c, sbit;
      fiber_offset_fast(a, tab, f, c, sbit);
      base_c = kRange ? c - r_lo : sk_base + 4u * c;  // kRange: range-relative offset
      scale_f = sbit ? -scale : scale;
    }
#pragma unroll
    for (int k = 0; k < LB; ++k) {
      const int kk = KB + k;
      const uint32_t e = (kk % 2) ? (bk[kk / 2] >> 16) : (bk[kk / 2] & 0xffffu);
      const float xs = __uint_as_float(__float_as_uint(x[k]) ^
                                       ((smask >> kk) << 31));
      const uint32_t bits = __float_as_uint(fmaf(xs, scale_f, 12582912.0f));
      rng_acc |= bits ^ 0x4B000000u;
      int32_t q = static_cast<int32_t>(bits - 0x4B400000u);
      uint32_t addr;
      if constexpr (kRange) {  // another range's element adds 0 to dummy bucket `lane`
        const uint32_t lb = base_c + e;
        const bool in = lb < r_cnt;
        addr = sk_base + 4u * (in ? lb : span + static_cast<uint32_t>(lane));
        q = in ? q : 0;
      } else {
        addr = base_c + (e << 2);
      }
      int32_t old;
      asm volatile("atom.shared.add.s32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(q));
      ovf_acc |= static_cast<uint32_t>(old) + 0x40000000u;
    }
  };
  float cur[LB], nxt[LB];
  uint64_t f = f_begin + (warp >> a.lseg);
  if (f < f_end) load.template operator()<0>(f, cur);
  if constexpr (NB == 1) {
    for (; f < f_end; f += 2 * fstride) {
      if (f + fstride < f_end) load.template operator()<0>(f + fstride, nxt);
      scatter.template operator()<0>(f, cur);
      if (f + fstride >= f_end) break;
      if (f + 2 * fstride < f_end) load.template operator()<0>(f + 2 * fstride, cur);
      scatter.template operator()<0>(f + fstride, nxt);
    }
  } else {
    static_assert(NB == 2, "NV <= 32: at most two batches of 16");
    for (; f < f_end; f += fstride) {
      load.template operator()<LB>(f, nxt);
      scatter.template operator()<0>(f, cur);
      if (f + fstride < f_end) load.template operator()<0>(f + fstride, cur);
      scatter.template operator()<LB>(f, nxt);
    }
  }
  const bool bad = __syncthreads_or(static_cast<int>((ovf_acc >> 31) | ((rng_acc >> 23) != 0)));
  bool tiny = false;
  if (!bad) {  // precision guard (kFxSmallBits), as in fcs_dense_fx_kernel
    int nz = 0, big = 0;
    for (uint32_t b = threadIdx.x; b < r_cnt; b += blockDim.x) {
      const int32_t v = sk[b];
      const uint32_t m = static_cast<uint32_t>(v < 0 ? -v : v);
      nz |= m != 0u;
      big |= (m >> kFxSmallBits) != 0u;
    }
    const bool any_big = __syncthreads_or(big);
    tiny = __syncthreads_or(nz) && !any_big;
  }
  if (bad || tiny)
    fx_float_redo(a, t, tab, scale, chunk, false, reinterpret_cast<float*>(smem_raw), r_lo, r_cnt);
  // partial row per (chunk, d[, range]) of span words (kRange = false: span = J~)
  int32_t* dst = part + prow * static_cast<uint64_t>(span);
  for (uint32_t b = threadIdx.x; b < r_cnt; b += blockDim.x) dst[b] = sk[b];
  if (threadIdx.x == 0) flags[prow] = (bad || tiny) ? 1 : 0;
}

// out[d][b] (+)= 2^-S * (exact 128-bit sum of the fixed-point partials) + the
// fp64 partials of CTAs that fell back, both in a fixed order. 32 outputs x 32
// chunk lanes per CTA (like reduce_partials_kernel): lane y sums chunks
// y, y + 32, ..., then the 32 lane sums are combined in lane order.
__device__ __forceinline__ double i128_to_double(__int128 acc) {
  const int64_t top = static_cast<int64_t>(acc >> 64);
  if (top == 0 || top == -1) {
    const int64_t low = static_cast<int64_t>(acc);
    if (static_cast<__int128>(low) == acc) return static_cast<double>(low);
    return static_cast<double>(static_cast<int64_t>(acc >> 11)) * 2048.0;
  }
  return static_cast<double>(top) * 18446744073709551616.0 +
         static_cast<double>(static_cast<uint64_t>(acc));
}

__global__ void reduce_fx64_kernel(const uint32_t* __restrict__ part, const int* __restrict__ flags,
                                   uint64_t nchunk, int D, uint32_t jt, uint32_t rparts,
                                   uint32_t span, const FxStats* __restrict__ st,
                                   double* __restrict__ out, int accumulate) {
  __shared__ __int128 ired[32][33];
  __shared__ double dred[32][33];
  const uint64_t per = static_cast<uint64_t>(D) * jt;
  const uint64_t i = blockIdx.x * 32ull + threadIdx.x;
  __int128 acc = 0;
  double dacc = 0.0;
  if (i < per) {
    const int d = static_cast<int>(i / jt);
    const uint32_t bb = static_cast<uint32_t>(i - static_cast<uint64_t>(d) * jt);
    const uint32_t rp = bb / span, b = bb - rp * span;  // range part, bucket within it
    for (uint64_t c = threadIdx.y; c < nchunk; c += 32) {
      const uint64_t prow = (c * D + d) * rparts + rp;
      const uint32_t* row = part + prow * 2ull * span;
      if (flags[prow]) {
        dacc += reinterpret_cast<const double*>(row)[b];
      } else {
        acc += static_cast<int64_t>((static_cast<uint64_t>(row[span + b]) << 32) | row[b]);
      }
    }
  }
  ired[threadIdx.y][threadIdx.x] = acc;
  dred[threadIdx.y][threadIdx.x] = dacc;
  __syncthreads();
  if (threadIdx.y == 0 && i < per) {
    for (int y = 1; y < 32; ++y) {
      acc += ired[y][threadIdx.x];
      dacc += dred[y][threadIdx.x];
    }
    double r = ldexp(i128_to_double(acc), -st->S) + dacc;
    if (accumulate) r += out[i];
    out[i] = r;
  }
}

// Fixed-order fp64 reduction of the chunk partials: out[d][b] (+)= sum_c part[c][d][b].
// 32 outputs x 32 chunk lanes per CTA: lane y sums chunks y, y + 32, ...
// (coalesced over the 32 outputs), then the 32 lane sums are added in lane
// order — a fixed order, with 32x the memory-level parallelism of one thread
// per output (small tensors have few outputs and many chunks).
template <typename Tacc>
__global__ void reduce_partials_kernel(const Tacc* __restrict__ part, uint64_t nchunk,
                                       uint64_t per_chunk, double* __restrict__ out,
                                       int accumulate) {
  __shared__ double red[32][33];
  const uint64_t i = blockIdx.x * 32ull + threadIdx.x;
  double acc = 0.0;
  if (i < per_chunk)
    for (uint64_t c = threadIdx.y; c < nchunk; c += 32)
      acc += static_cast<double>(part[c * per_chunk + i]);
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && i < per_chunk) {
    double s = accumulate ? out[i] : 0.0;
    for (int y = 0; y < 32; ++y) s += red[y][threadIdx.x];
    out[i] = s;
  }
}

// Same for fixed-point partials (flag 0: int32 * 2^-S, flag 1: float bits).
// rparts > 1: per-(chunk, family, range) partial rows of span words (the
// bucket-range split of fcs_dense_fx32s_kernel); rparts = 1, span = J~ is the
// plain (chunk, family) layout.
__global__ void reduce_fx_kernel(const int32_t* __restrict__ part, const int* __restrict__ flags,
                                 uint64_t nchunk, int D, uint32_t jt,
                                 const FxStats* __restrict__ st, const double* __restrict__ divert,
                                 double* __restrict__ out, int accumulate, uint32_t rparts = 1,
                                 uint32_t span = 0) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t per0 = static_cast<uint64_t>(D) * jt;
  if (i >= per0) return;
  const int d0 = static_cast<int>(i / jt);
  if (rparts > 1) {  // ranged layout: one partial row per (chunk, family, range)
    const uint32_t b = static_cast<uint32_t>(i - static_cast<uint64_t>(d0) * jt);
    const uint32_t rp = b / span, lb = b - rp * span;
    const double inv = ldexp(1.0, -st->S);
    double acc = accumulate ? out[i] : 0.0;
    for (uint64_t c = 0; c < nchunk; ++c) {
      const uint64_t prow = (c * D + d0) * rparts + rp;
      const int32_t w = __ldcs(part + prow * span + lb);
      acc += __ldg(flags + prow) == 1 ? static_cast<double>(__int_as_float(w))
                                      : static_cast<double>(w) * inv;
    }
    out[i] = acc + divert[i];
    return;
  }
  const uint64_t per = per0;
  const int d = d0;
  const double inv = ldexp(1.0, -st->S);
  double acc = accumulate ? out[i] : 0.0;
  auto term = [&](int32_t w, int fl) {
    return fl == 1 ? static_cast<double>(__int_as_float(w)) : static_cast<double>(w) * inv;
  };
  uint64_t c = 0;
  constexpr int kU = 8;  // partials in flight, summed in chunk order (config 4: 37 chunks;
                         // 12.3 -> 11.3 us vs 4; a 32 x 8 chunk-lane layout: 28 us)
  for (; c + kU <= nchunk; c += kU) {
    int32_t w[kU];
    int fl[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      w[u] = __ldcs(part + (c + u) * per + i);
      fl[u] = __ldg(flags + (c + u) * D + d);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) acc += term(w[u], fl[u]);
  }
  for (; c < nchunk; ++c) acc += term(part[c * per + i], flags[c * D + d]);
  out[i] = acc + divert[i];
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

// -------------------------------------------------------------- planning
namespace {

// Per-device cache of fx line groupings (fx_group_kernel), zeroed once.
int fx_group_cache(FxGroupEntry** out) {
  static std::mutex mu;
  static std::map<int, FxGroupEntry*> per_dev;
  int dev = 0;
  FCS_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto it = per_dev.find(dev);
  if (it == per_dev.end()) {
    FxGroupEntry* p = nullptr;
    FCS_CUDA_TRY(cudaMalloc(&p, kFxCacheSlots * sizeof(FxGroupEntry)));
    FCS_CUDA_TRY(cudaMemset(p, 0, kFxCacheSlots * sizeof(FxGroupEntry)));
    it = per_dev.emplace(dev, p).first;
  }
  *out = it->second;
  return ST_OK;
}

enum class Path { Global, Smem, Fx, Fx32S, Fx64 };

struct Plan {
  Path path = Path::Global;
  uint32_t rparts = 1;  // fx64: bucket ranges per family (J~ beyond shared memory)
  uint32_t rspan = 0;
  bool group = false;  // fx: bank-aware load order
  size_t smem_bytes = 0;
  int threads = 0;
  int nv = 0;
  uint64_t nchunk = 0;
  size_t part_bytes = 0;
  size_t ws = 0;
};

// fx kernel variant for this shape (0: not applicable): 1..3 = one warp per
// fiber with 1/2/4/8 vectors per lane (512 threads). (Splitting a fiber over
// two warps at 1024 threads measured slower on B200: 3.5 vs 2.9 ms at config 4,
// the 64-register cap spills.)
int fx_nv(const DenseArgs& a) {
  if (a.dims[0] % 4 != 0) return 0;
  const uint32_t per_lane = (a.dims[0] / 4 + 31) / 32;
  if (per_lane == 0 || per_lane > 8) return 0;
  const int v = per_lane <= 1 ? 1 : per_lane <= 2 ? 2 : per_lane <= 4 ? 3 : 4;
  // 5..8: the same kernels without the per-vector guard when I_0 = 128 NV
  return a.dims[0] == (128u << (v - 1)) ? v + 4 : v;
}

using FxKernel = void (*)(DenseArgs, const float*, const uint32_t*, const FxStats*, int32_t*, int*,
                          const uint8_t*, double*);
template <bool kRedo>
FxKernel fx_kernel_t(int v, bool group) {
  if (group) {  // full-vector kernels with the bank-aware load order
    switch (v) {
      case 6: return fcs_dense_fx_kernel<2, 1, 512, true, true, kRedo>;
      case 7: return fcs_dense_fx_kernel<4, 1, 512, true, true, kRedo>;
      case 8: return fcs_dense_fx_kernel<8, 1, 512, true, true, kRedo>;
      default: break;
    }
  }
  switch (v) {
    case 1: return fcs_dense_fx_kernel<1, 1, 512, false, false, kRedo>;
    case 2: return fcs_dense_fx_kernel<2, 1, 512, false, false, kRedo>;
    case 3: return fcs_dense_fx_kernel<4, 1, 512, false, false, kRedo>;
    case 4: return fcs_dense_fx_kernel<8, 1, 512, false, false, kRedo>;
    case 5: return fcs_dense_fx_kernel<1, 1, 512, true, false, kRedo>;
    case 6: return fcs_dense_fx_kernel<2, 1, 512, true, false, kRedo>;
    case 7: return fcs_dense_fx_kernel<4, 1, 512, true, false, kRedo>;
    default: return fcs_dense_fx_kernel<8, 1, 512, true, false, kRedo>;
  }
}
FxKernel fx_kernel(int v, bool group, bool redo = false) {
  return redo ? fx_kernel_t<true>(v, group) : fx_kernel_t<false>(v, group);
}
inline int fx_threads(int) { return 512; }

// fx64 variant: NV = the smallest power of two with 32 NV >= I_0.
int fx64_nv(uint32_t i0) {
  int nv = 1;
  while (32u * nv < i0) nv <<= 1;
  return nv;
}

// Lane-owned fixed-point kernels (fx64, fx32s) take I_0 <= 16384: 2^lseg
// segments (one warp each, 16 warps per CTA) of seg_len <= 1024 entries, a
// multiple of 32 (the last segment shorter); NV from seg_len.
constexpr uint32_t kFxSegMaxI0 = 16384;
inline void fx_segments(uint32_t i0, uint32_t* seg_len, uint32_t* lseg) {
  uint32_t l = 0;
  while (((i0 + (1u << l) - 1) >> l) > 1024u) ++l;
  *lseg = l;
  *seg_len = (((i0 + (1u << l) - 1) >> l) + 31u) / 32u * 32u;
}
inline int fx_seg_nv(uint32_t i0) {
  uint32_t len, l;
  fx_segments(i0, &len, &l);
  return fx64_nv(len);
}
// every segment holds exactly 32 NV entries (no per-entry guard)
inline bool fx_seg_full(uint32_t i0) {
  uint32_t len, l;
  fx_segments(i0, &len, &l);
  return i0 == (32u * fx64_nv(len)) << l;
}
using Fx32sKernel = void (*)(DenseArgs, const float*, const uint32_t*, const FxStats*, int32_t*,
                             int*);
// fx32s variant: NV = the smallest power of two with 32 NV >= the segment length.
template <bool kRange>
Fx32sKernel fx32s_kernel_r(int nv, bool full) {
  switch (nv) {
    case 1: return full ? fcs_dense_fx32s_kernel<1, true, kRange> : fcs_dense_fx32s_kernel<1, false, kRange>;
    case 2: return full ? fcs_dense_fx32s_kernel<2, true, kRange> : fcs_dense_fx32s_kernel<2, false, kRange>;
    case 4: return full ? fcs_dense_fx32s_kernel<4, true, kRange> : fcs_dense_fx32s_kernel<4, false, kRange>;
    case 8: return full ? fcs_dense_fx32s_kernel<8, true, kRange> : fcs_dense_fx32s_kernel<8, false, kRange>;
    case 16:
      return full ? fcs_dense_fx32s_kernel<16, true, kRange>
                  : fcs_dense_fx32s_kernel<16, false, kRange>;
    default:
      return full ? fcs_dense_fx32s_kernel<32, true, kRange>
                  : fcs_dense_fx32s_kernel<32, false, kRange>;
  }
}
// range = true: the bucket-range split for J~ beyond shared memory
Fx32sKernel fx32s_kernel(int nv, bool full, bool range = false) {
  return range ? fx32s_kernel_r<true>(nv, full) : fx32s_kernel_r<false>(nv, full);
}

template <typename Tin>
using Fx64Kernel = void (*)(DenseArgs, const Tin*, const uint32_t*, const FxStats*, uint32_t*,
                            int*);
template <typename Tin, bool kRange>
Fx64Kernel<Tin> fx64_kernel_r(int nv, bool full) {
  switch (nv) {
    case 1: return full ? fcs_dense_fx64_kernel<Tin, 1, true, kRange> : fcs_dense_fx64_kernel<Tin, 1, false, kRange>;
    case 2: return full ? fcs_dense_fx64_kernel<Tin, 2, true, kRange> : fcs_dense_fx64_kernel<Tin, 2, false, kRange>;
    case 4: return full ? fcs_dense_fx64_kernel<Tin, 4, true, kRange> : fcs_dense_fx64_kernel<Tin, 4, false, kRange>;
    case 8: return full ? fcs_dense_fx64_kernel<Tin, 8, true, kRange> : fcs_dense_fx64_kernel<Tin, 8, false, kRange>;
    case 16:
      return full ? fcs_dense_fx64_kernel<Tin, 16, true, kRange>
                  : fcs_dense_fx64_kernel<Tin, 16, false, kRange>;
    default:
      return full ? fcs_dense_fx64_kernel<Tin, 32, true, kRange>
                  : fcs_dense_fx64_kernel<Tin, 32, false, kRange>;
  }
}
// range = true: the bucket-range split for J~ beyond shared memory
template <typename Tin>
Fx64Kernel<Tin> fx64_kernel(int nv, bool full, bool range = false) {
  return range ? fx64_kernel_r<Tin, true>(nv, full) : fx64_kernel_r<Tin, false>(nv, full);
}

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// The workspace depends only on the shape (never on the pointer), so
// st_fcs_dense_workspace never under-reports; an unaligned fp32 tensor simply
// takes the generic kernel with the same partition.
template <typename Tin, typename Tacc>
int make_plan_uncached(const DenseArgs& a, Plan* p);

// Opt a kernel in to the largest dynamic shared memory it can ever use (its
// static shared memory subtracted), so cached plans of any size launch.
template <typename K>
cudaError_t set_max_dynamic_smem(K k, const DeviceInfo& di) {
  cudaFuncAttributes at{};
  cudaError_t e = cudaFuncGetAttributes(&at, k);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(di.smem_optin - at.sharedSizeBytes));
}

// Plans depend only on the device, the dtype and the launch geometry; the
// cache keeps per-call host work (function attributes, occupancy queries)
// off the small-tensor path.
template <typename Tin, typename Tacc>
int make_plan(const DenseArgs& a, Plan* p) {
  static std::mutex mu;
  static std::map<std::vector<uint64_t>, Plan> cache;
  int dev = 0;
  FCS_CUDA_TRY(cudaGetDevice(&dev));
  std::vector<uint64_t> key = {static_cast<uint64_t>(dev), sizeof(Tin), sizeof(Tacc),
                               static_cast<uint64_t>(a.order), static_cast<uint64_t>(a.D), a.jt,
                               a.fibers};
  for (int n = 0; n < a.order; ++n) {
    key.push_back(a.dims[n]);
    key.push_back(a.mult[n]);
  }
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *p = it->second;
      return ST_OK;
    }
  }
  if (int rc = make_plan_uncached<Tin, Tacc>(a, p)) return rc;
  std::lock_guard<std::mutex> lock(mu);
  if (cache.size() > 4096) cache.clear();
  cache[key] = *p;
  return ST_OK;
}

template <typename Tin, typename Tacc>
int make_plan_uncached(const DenseArgs& a, Plan* p) {
  DeviceInfo di;
  if (int rc = device_info(&di)) return rc;
  p->smem_bytes = static_cast<size_t>(a.jt) * sizeof(Tacc);
  static const bool no_fx64_env = std::getenv("ST_FX64_OFF") != nullptr;  // A/B probe
  // lane-owned fixed-point kernels (64-bit for fp64 input, int32 for fp32 input
  // with scalar loads): their mode-0 buckets are packed in 16 bits
  const bool lane_fx_shape = a.order >= 2 && a.dims[0] <= kFxSegMaxI0 && a.j0 < 65536u &&
                             static_cast<double>(a.fibers) * a.dims[0] * a.D >= 8.0e6;
  const bool fx64_shape = sizeof(Tin) == 8 && lane_fx_shape && !no_fx64_env;
  const bool fx32_shape = sizeof(Tin) == 4 && lane_fx_shape;
  int per_sm = 0;
  if ((fx64_shape || fx32_shape) ? p->smem_bytes + 4096 > di.smem_optin
                                 : p->smem_bytes > di.smem_optin) {
    // fp64 with J~ beyond shared memory: the 64-bit fixed point over R bucket
    // ranges (one CTA per chunk, family and range; each element read R times
    // through L2) instead of fp64 global atomics (1024 x 1024 x 512,
    // J~ = 49,150, D = 1: 4.45 ms with global atomics)
    const size_t avail = di.smem_optin - 4096;  // static shared memory + the 32 dummy buckets
    const size_t wb = sizeof(Tin) == 8 ? 8 : 4;   // bytes per bucket
    const uint32_t R = static_cast<uint32_t>((static_cast<size_t>(a.jt) * wb + avail - 1) / avail);
    if (!(fx64_shape || fx32_shape) || R > 8) {
      p->path = Path::Global;
      p->ws = 0;
      return ST_OK;
    }
    p->rparts = R;
    p->rspan = (a.jt + R - 1) / R;
    p->nv = fx_seg_nv(a.dims[0]);
    p->threads = 512;
    p->smem_bytes = (static_cast<size_t>(p->rspan) + 32) * wb;
    if constexpr (sizeof(Tin) == 8) {
      p->path = Path::Fx64;
      auto k = fx64_kernel<Tin>(p->nv, fx_seg_full(a.dims[0]), true);
      FCS_CUDA_TRY(set_max_dynamic_smem(k, di));
      FCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, p->threads,
                                                                 p->smem_bytes));
    } else {  // fp32 (1024^3, J = 32768, D = 4: 23.8 ms with fp64 global atomics)
      p->path = Path::Fx32S;
      auto k = fx32s_kernel(p->nv, fx_seg_full(a.dims[0]), true);
      FCS_CUDA_TRY(set_max_dynamic_smem(k, di));
      FCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, p->threads,
                                                                 p->smem_bytes));
    }
  }
  if (p->rparts == 1) {
    p->nv = sizeof(Tin) == 4 ? fx_nv(a) : 0;
    // the fixed-point kernels also hold fx_scale_device's static scratch
    auto fits = [&](auto k) {
      cudaFuncAttributes at{};
      return cudaFuncGetAttributes(&at, k) == cudaSuccess &&
             p->smem_bytes + at.sharedSizeBytes <= di.smem_optin;
    };
    if (p->nv && !fits(fx_kernel(p->nv, false))) p->nv = 0;
    static const bool no_fx64 = std::getenv("ST_FX64_OFF") != nullptr;  // A/B probe
    // Below ~8M element-updates the call is launch/latency-bound and the CAS
    // kernel's two launches beat the fixed point's three (c1 100^3 D=1: 27.6 vs
    // 33.8 us; c5 operands: 37 vs 42 us); above it the fixed point wins (c3
    // build 200^3 D=10: 200 vs 292 us; 1024^3 J=8192 D=1: 1.44 vs 3.43 ms).
    const bool fx64_pays = static_cast<double>(a.fibers) * a.dims[0] * a.D >= 8.0e6;
    // fp32 shapes the float4 kernel does not take (I_0 % 4 != 0), I_0 <= 1024:
    // the same int32 fixed point with scalar loads
    const bool fx32s_ok = sizeof(Tin) == 4 && a.order >= 2 && a.dims[0] <= kFxSegMaxI0 &&
                          fits(fx32s_kernel(fx_seg_nv(a.dims[0]), false));
    if (sizeof(Tin) == 4 && !p->nv && fx32s_ok && fx64_pays) {
      p->path = Path::Fx32S;
      p->nv = fx_seg_nv(a.dims[0]);
      p->threads = 512;
      auto k = fx32s_kernel(p->nv, fx_seg_full(a.dims[0]));
      FCS_CUDA_TRY(set_max_dynamic_smem(k, di));
      FCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, p->threads,
                                                                 p->smem_bytes));
    } else if (sizeof(Tin) == 8 && a.order >= 2 && a.dims[0] <= kFxSegMaxI0 && !no_fx64 &&
               fx64_pays && fits(fx64_kernel<Tin>(fx_seg_nv(a.dims[0]), false))) {
      // fp64: 64-bit fixed point, 8 bytes per bucket
      p->path = Path::Fx64;
      p->nv = fx_seg_nv(a.dims[0]);
      p->threads = 512;
      const bool full = fx_seg_full(a.dims[0]);
      auto k = fx64_kernel<Tin>(p->nv, full);
      FCS_CUDA_TRY(set_max_dynamic_smem(k, di));
      FCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, p->threads,
                                                                 p->smem_bytes));
    } else if (p->nv) {
      p->path = Path::Fx;
      p->threads = fx_threads(p->nv);
      // the bank-aware order pays off when atomics bind: with the searched
      // groups, config-4 geometry D = 2: 1.333 -> 1.155 ms, D = 4: -4 %; with one
      // family the kernel is load-bound (D = 1: 0.722 vs 0.725 ms) and keeps
      // the immediate-offset loads.
      // ST_FX_NOGROUP=1 keeps the identity order (A/B probe).
      static const bool no_group = std::getenv("ST_FX_NOGROUP") != nullptr;
      p->group = p->nv >= 6 && a.D >= 2 && !no_group;
      auto k = fx_kernel(p->nv, p->group);
      FCS_CUDA_TRY(set_max_dynamic_smem(k, di));
      FCS_CUDA_TRY(set_max_dynamic_smem(fx_kernel(p->nv, p->group, true), di));
      if (fx32s_ok)  // an unaligned tensor on this plan takes the scalar-load kernel
        FCS_CUDA_TRY(set_max_dynamic_smem(
            fx32s_kernel(fx_seg_nv(a.dims[0]), fx_seg_full(a.dims[0])), di));
      FCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, p->threads,
                                                                 p->smem_bytes));
    } else {
      p->path = Path::Smem;
      auto k = fcs_dense_smem_kernel<Tin, Tacc>;
      FCS_CUDA_TRY(set_max_dynamic_smem(k, di));
      p->threads = p->smem_bytes > di.smem_optin / 2 ? 1024 : 512;
      FCS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, p->threads,
                                                                 p->smem_bytes));
    }
  }  // rparts == 1
  per_sm = std::max(per_sm, 1);
  const uint64_t resident = static_cast<uint64_t>(per_sm) * di.sm_count;
  uint64_t nchunk = std::max<uint64_t>(1, resident / (static_cast<uint64_t>(a.D) * p->rparts));
  // fixed point: at least ~4 fibers per warp of a 512-thread CTA (per-CTA
  // fixed costs — zeroing, writing the partial — dominate smaller shares);
  // the atomic kernel keeps 16 fibers per chunk (c1: 333 chunks, 22 us)
  const bool fixed = p->path == Path::Fx || p->path == Path::Fx32S || p->path == Path::Fx64;
  nchunk = std::min<uint64_t>(nchunk, std::max<uint64_t>(1, a.fibers / (fixed ? 64 : 16)));
  // Small tensors: each chunk writes (and the reduction re-reads) a D x J~
  // partial, so keep the partials to at most the tensor's bytes (config 1:
  // 592 -> 333 chunks; config 4 is unaffected).
  const uint64_t elems = a.fibers * a.dims[0];
  const uint64_t part_per_chunk = static_cast<uint64_t>(a.D) * a.jt * sizeof(Tacc);
  // ... but never below one CTA per SM (config 5's 512^2 operands, D = 8: 8 -> 19 chunks,
  // 103 -> 78 us per kron call)
  const uint64_t by_bytes = std::max<uint64_t>(1, elems * sizeof(Tin) / part_per_chunk);
  const uint64_t one_wave = (static_cast<uint64_t>(di.sm_count) + a.D - 1) / a.D;
  nchunk = std::min<uint64_t>(nchunk, std::max(by_bytes, one_wave));
  p->nchunk = nchunk;
  p->part_bytes = p->rparts > 1
                      ? nchunk * a.D * p->rparts * static_cast<size_t>(p->rspan) *
                            (p->path == Path::Fx64 ? 8 : 4)
                      : nchunk * a.D * static_cast<size_t>(a.jt) *
                            (p->path == Path::Fx64 ? 8 : sizeof(Tacc));  // Fx32S: int32 like Fx
  p->ws = align_up(p->part_bytes) + align_up(nchunk * a.D * p->rparts * sizeof(int)) +
          align_up(sizeof(FxStats)) + align_up(static_cast<size_t>(a.D) * 32) +
          align_up(kFxMaxSample * sizeof(FxPart)) +
          align_up(static_cast<size_t>(a.D) * a.jt * sizeof(double));  // fp32: divert
  return ST_OK;
}

// kind 0: FCS (bucket sum), kind 1: HCS (mixed-radix bucket, sketch.cpp:157-173).
int fill_args(size_t order, const size_t* dims, size_t last_begin, size_t last_count, size_t D,
              const size_t* hash_lens, DenseArgs* a, int kind = 0, size_t out_len = 0) {
  FCS_CHECK_ARG(order >= 1 && order <= ST_MAX_ORDER, "fcs_sketch: unsupported tensor order");
  FCS_CHECK_ARG(D >= 1, "EstimatorConfig: hash_len and sketch_count must be >= 1");
  *a = DenseArgs{};
  a->order = static_cast<int>(order);
  a->D = static_cast<int>(D);
  uint64_t sum_dims = 0, sum_j = 0, prod_j = 1;
  for (size_t n = 0; n < order; ++n) {
    FCS_CHECK_ARG(dims[n] > 0 && hash_lens[n] > 0, "HashPair: dimensions must be positive");
    FCS_CHECK_ARG(dims[n] < (1u << 31) && hash_lens[n] < (1u << 30),
                  "fcs_sketch: dimension too large");
    a->dims[n] = static_cast<uint32_t>(dims[n]);
    a->tab_off[n] = static_cast<uint32_t>(sum_dims);
    a->mult[n] = kind == 1 ? static_cast<uint32_t>(prod_j) : 1u;
    sum_dims += dims[n];
    sum_j += hash_lens[n];
    prod_j *= hash_lens[n];
    FCS_CHECK_ARG(kind == 0 || prod_j < (1ull << 31), "hcs_sketch: sketch tensor too large");
  }
  FCS_CHECK_ARG(sum_dims < (1ull << 32) && sum_j - order + 1 < (1ull << 31),
                "fcs_sketch: family too large");
  FCS_CHECK_ARG(last_begin + last_count <= dims[order - 1], "fcs_sketch: slab out of range");
  a->fam_stride = static_cast<uint32_t>(sum_dims);
  a->j0 = static_cast<uint32_t>(hash_lens[0]);
  a->jt = static_cast<uint32_t>(kind == 1 ? prod_j : sum_j - order + 1);
  if (out_len) {
    FCS_CHECK_ARG(kind == 0 && out_len < (1ull << 31), "fcs_sketch: batched output too large");
    a->jt = static_cast<uint32_t>(out_len);
  }
  if (order >= 2)
    a->inv_d1 = dims[1] > 1 ? static_cast<uint32_t>((1ull << 32) / dims[1]) : 0xffffffffu;
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
  if (p.path == Path::Global) {
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
  const bool aligned = (reinterpret_cast<uintptr_t>(t) & 15u) == 0;
  fx_segments(a.dims[0], &a.seg_len, &a.lseg);
  if (p.path == Path::Fx32S || (p.path == Path::Fx && !aligned && a.order >= 2 &&
                                 a.dims[0] <= 1024)) {
    char* base = static_cast<char*>(ws);
    auto* part = reinterpret_cast<int32_t*>(base);
    auto* flags = reinterpret_cast<int*>(base + align_up(p.part_bytes));
    auto* stats = reinterpret_cast<FxStats*>(base + align_up(p.part_bytes) +
                                             align_up(p.nchunk * a.D * p.rparts * sizeof(int)));
    auto* parts = reinterpret_cast<FxPart*>(base + align_up(p.part_bytes) +
                                            align_up(p.nchunk * a.D * p.rparts * sizeof(int)) +
                                            align_up(sizeof(FxStats)) +
                                            align_up(static_cast<size_t>(a.D) * 32));
    auto* divert = reinterpret_cast<double*>(
        base + align_up(p.part_bytes) + align_up(p.nchunk * a.D * p.rparts * sizeof(int)) +
        align_up(sizeof(FxStats)) + align_up(static_cast<size_t>(a.D) * 32) +
        align_up(kFxMaxSample * sizeof(FxPart)));
    const uint64_t nsample = fx_nsample(a.fibers);
    const double per_cta = static_cast<double>(a.fibers_per_chunk) * a.dims[0];
    const FxScaleArgs sc{parts, static_cast<int>(nsample), 3.0 * per_cta / a.jt + 16.0, stats};
    const float* tf = reinterpret_cast<const float*>(t);
    fx_sample_warps_kernel<float><<<ceil_div(nsample, 8), 256, 0, st>>>(a, tf, nsample, parts);
    FCS_CUDA_TRY(cudaGetLastError());
    fx_scale_kernel<<<1, 512, 0, st>>>(sc, kFx32);
    FCS_CUDA_TRY(cudaGetLastError());
    FCS_CUDA_TRY(cudaMemsetAsync(divert, 0, out_elems * sizeof(double), st));
    const int nv = fx_seg_nv(a.dims[0]);
    a.rparts = p.rparts;
    a.rspan = p.rparts > 1 ? p.rspan : a.jt;
    fx32s_kernel(nv, fx_seg_full(a.dims[0]), p.rparts > 1)<<<
        static_cast<unsigned>(nchunk * a.D * p.rparts), 512, p.smem_bytes, st>>>(a, tf, packed,
                                                                                stats, part, flags);
    FCS_CUDA_TRY(cudaGetLastError());
    reduce_fx_kernel<<<ceil_div(out_elems, 256), 256, 0, st>>>(part, flags, nchunk, a.D, a.jt,
                                                               stats, divert, out, accumulate,
                                                               a.rparts, a.rspan);
    FCS_CUDA_TRY(cudaGetLastError());
    return ST_OK;
  }
  if (p.path == Path::Fx && aligned) {
    char* base = static_cast<char*>(ws);
    auto* part = reinterpret_cast<int32_t*>(base);
    auto* flags = reinterpret_cast<int*>(base + align_up(p.part_bytes));
    auto* stats = reinterpret_cast<FxStats*>(base + align_up(p.part_bytes) +
                                             align_up(p.nchunk * a.D * p.rparts * sizeof(int)));
    auto* parts = reinterpret_cast<FxPart*>(base + align_up(p.part_bytes) +
                                            align_up(p.nchunk * a.D * p.rparts * sizeof(int)) +
                                            align_up(sizeof(FxStats)) +
                                            align_up(static_cast<size_t>(a.D) * 32));
    const uint64_t nsample = fx_nsample(a.fibers);
    const int nparts = static_cast<int>(nsample);  // one fiber per sample CTA
    auto* divert = reinterpret_cast<double*>(
        base + align_up(p.part_bytes) + align_up(p.nchunk * a.D * p.rparts * sizeof(int)) +
        align_up(sizeof(FxStats)) + align_up(static_cast<size_t>(a.D) * 32) +
        align_up(kFxMaxSample * sizeof(FxPart)));
    // (programmatic dependent launch of the chain measured no gain: 2.29-2.36 vs
    // 2.28-2.32 ms at config 4, tools/experiments/k1_pdl.txt)
    fx_sample_warps_kernel<float><<<ceil_div(nsample, 8), 256, 0, st>>>(
        a, reinterpret_cast<const float*>(t), nsample, parts, divert, out_elems);
    FCS_CUDA_TRY(cudaGetLastError());
    const double per_cta = static_cast<double>(a.fibers_per_chunk) * a.dims[0];
    const FxScaleArgs sc{parts, nparts, 3.0 * per_cta / a.jt + 16.0, stats};
    fx_scale_kernel<<<1, 512, 0, st>>>(sc, kFx32);
    FCS_CUDA_TRY(cudaGetLastError());
    // bank-aware load order for the full-vector kernels (I_0 = 128 NV, NV >= 2)
    uint8_t* groups = nullptr;
    const int nv_full = p.nv >= 6 ? 1 << (p.nv - 5) : 0;
    if (p.group) {
      groups = reinterpret_cast<uint8_t*>(base + align_up(p.part_bytes) +
                                          align_up(p.nchunk * a.D * p.rparts * sizeof(int)) +
                                          align_up(sizeof(FxStats)));
      FxGroupEntry* cache = nullptr;
      if (int rc = fx_group_cache(&cache)) return rc;
      const uint64_t elems = a.fibers * a.dims[0];
      const int iters = static_cast<int>(std::min<uint64_t>(kFxSearchIters, elems >> 22));
      fx_group_kernel<<<a.D, 1024, 0, st>>>(packed, a.fam_stride, a.i0_shift, nv_full, iters,
                                            groups, cache);
      FCS_CUDA_TRY(cudaGetLastError());
    }
    const float* tf = reinterpret_cast<const float*>(t);
    fx_kernel(p.nv, p.group)<<<static_cast<unsigned>(nchunk * a.D), p.threads, p.smem_bytes, st>>>(
        a, tf, packed, stats, part, flags, groups, divert);
    FCS_CUDA_TRY(cudaGetLastError());
    // redo of the flagged chunks (unflagged CTAs exit at once)
    fx_kernel(p.nv, p.group, true)<<<static_cast<unsigned>(nchunk * a.D), p.threads, p.smem_bytes,
                                     st>>>(a, tf, packed, stats, part, flags, groups, divert);
    FCS_CUDA_TRY(cudaGetLastError());
    reduce_fx_kernel<<<ceil_div(out_elems, 256), 256, 0, st>>>(part, flags, nchunk, a.D, a.jt,
                                                               stats, divert, out, accumulate);
    FCS_CUDA_TRY(cudaGetLastError());
    return ST_OK;
  }
  if (p.path == Path::Fx64) {
    char* base = static_cast<char*>(ws);
    auto* part = reinterpret_cast<uint32_t*>(base);
    auto* flags = reinterpret_cast<int*>(base + align_up(p.part_bytes));
    auto* stats = reinterpret_cast<FxStats*>(base + align_up(p.part_bytes) +
                                             align_up(p.nchunk * a.D * p.rparts * sizeof(int)));
    auto* parts = reinterpret_cast<FxPart*>(base + align_up(p.part_bytes) +
                                            align_up(p.nchunk * a.D * p.rparts * sizeof(int)) +
                                            align_up(sizeof(FxStats)) +
                                            align_up(static_cast<size_t>(a.D) * 32));
    const uint64_t nsample = fx_nsample(a.fibers);
    const int nparts = static_cast<int>(nsample);
    const double per_cta = static_cast<double>(a.fibers_per_chunk) * a.dims[0];
    const FxScaleArgs sc{parts, nparts, 3.0 * per_cta / a.jt + 16.0, stats};
    const bool full = fx_seg_full(a.dims[0]);
    fx_sample_warps_kernel<Tin><<<ceil_div(nsample, 8), 256, 0, st>>>(a, t, nsample, parts);
    FCS_CUDA_TRY(cudaGetLastError());
    fx_scale_kernel<<<1, 512, 0, st>>>(sc, kFx64);
    FCS_CUDA_TRY(cudaGetLastError());
    a.rparts = p.rparts;
    a.rspan = p.rparts > 1 ? p.rspan : a.jt;
    fx64_kernel<Tin>(p.nv, full, p.rparts > 1)<<<static_cast<unsigned>(nchunk * a.D * p.rparts),
                                                 p.threads, p.smem_bytes, st>>>(a, t, packed,
                                                                                stats, part, flags);
    FCS_CUDA_TRY(cudaGetLastError());
    reduce_fx64_kernel<<<ceil_div(out_elems, 32), dim3(32, 32), 0, st>>>(
        part, flags, nchunk, a.D, a.jt, a.rparts, a.rspan, stats, out, accumulate);
    FCS_CUDA_TRY(cudaGetLastError());
    return ST_OK;
  }
  int threads = p.threads;
  if (p.path == Path::Fx) {  // unaligned fp32 tensor: generic kernel, same partition
    DeviceInfo di;
    if (int rc = device_info(&di)) return rc;
    FCS_CUDA_TRY(set_max_dynamic_smem(fcs_dense_smem_kernel<Tin, Tacc>, di));
    threads = 1024;
  }
  Tacc* part = static_cast<Tacc*>(ws);
  fcs_dense_smem_kernel<Tin, Tacc>
      <<<static_cast<unsigned>(nchunk * a.D), threads, p.smem_bytes, st>>>(a, t, packed, part);
  FCS_CUDA_TRY(cudaGetLastError());
  reduce_partials_kernel<Tacc><<<ceil_div(out_elems, 32), dim3(32, 32), 0, st>>>(
      part, nchunk, out_elems, out, accumulate);
  FCS_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace

// Diagnostics of the last fp32 fixed-point call that used `ws` (synchronous):
// the exponent S, how many (chunk, family) CTAs fell back to float atomics,
// and how many there were. *S = INT_MIN and counts 0 when the call did not
// take the fixed-point kernel.
int dense_fx_report(int dtype, size_t order, const size_t* dims, size_t last_count, size_t D,
                    const size_t* hash_lens, const void* ws, size_t ws_bytes, int* S,
                    size_t* fallback, size_t* ctas) {
  DenseArgs a;
  if (int rc = fill_args(order, dims, 0, last_count, D, hash_lens, &a)) return rc;
  *S = INT32_MIN;
  *fallback = *ctas = 0;
  Plan p;
  if (int rc = dtype == ST_F32 ? make_plan<float, float>(a, &p) : make_plan<double, double>(a, &p))
    return rc;
  if ((p.path != Path::Fx && p.path != Path::Fx32S && p.path != Path::Fx64) || a.fibers == 0)
    return ST_OK;
  FCS_CHECK_ARG(ws != nullptr && ws_bytes >= p.ws, "st_fcs_dense_report: workspace too small");
  a.fibers_per_chunk = (a.fibers + p.nchunk - 1) / p.nchunk;
  const uint64_t nchunk = (a.fibers + a.fibers_per_chunk - 1) / a.fibers_per_chunk;
  const char* base = static_cast<const char*>(ws);
  std::vector<int> flags(nchunk * a.D * p.rparts);
  FCS_CUDA_TRY(cudaMemcpy(flags.data(), base + align_up(p.part_bytes), flags.size() * sizeof(int),
                          cudaMemcpyDeviceToHost));
  FxStats stats;
  FCS_CUDA_TRY(cudaMemcpy(&stats, base + align_up(p.part_bytes) + align_up(p.nchunk * a.D * p.rparts * sizeof(int)),
                          sizeof(FxStats), cudaMemcpyDeviceToHost));
  *S = stats.S;
  *ctas = flags.size();
  for (int f : flags) *fallback += f != 0;
  return ST_OK;
}

size_t dense_workspace(int dtype, size_t order, const size_t* dims, size_t last_count, size_t D,
                       const size_t* hash_lens, int kind, size_t out_len) {
  DenseArgs a;
  if (fill_args(order, dims, 0, last_count, D, hash_lens, &a, kind, out_len) != ST_OK) return 0;
  Plan p;
  const int rc = dtype == ST_F32 ? make_plan<float, float>(a, &p) : make_plan<double, double>(a, &p);
  return rc == ST_OK ? p.ws : 0;
}

int launch_fcs_dense(int dtype, const void* t, size_t order, const size_t* dims, size_t last_begin,
                     size_t last_count, size_t D, const uint32_t* packed, const size_t* hash_lens,
                     double* out, int accumulate, void* ws, size_t ws_bytes, cudaStream_t st,
                     size_t fam_stride, int kind, size_t out_len) {
  DenseArgs a;
  if (int rc = fill_args(order, dims, last_begin, last_count, D, hash_lens, &a, kind, out_len))
    return rc;
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
