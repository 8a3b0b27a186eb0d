// Microbenchmarks that ground the K1 design:
// shared-memory update throughput by primitive and address pattern, and the
// streaming read rate for 1x vs 4x (per-family) re-reads of a 4 GiB tensor.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_bench smem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kWords = 49152;   // 192 KB smem array (c4 sketch size)
constexpr int kIters = 4096;

__device__ __forceinline__ uint32_t lcg(uint32_t& s) { s = s * 1664525u + 1013904223u; return s; }

// mode: 0 plain RMW random, 1 atomicAdd f32 random, 2 atomicAdd i32 random,
// 3 plain RMW conflict-free, 4 atomicAdd i32 conflict-free, 5 atomicAdd f32 conflict-free,
// 6 LDS only random, 7 red.shared.add.u32 random (no return)
template <int MODE>
__global__ void __launch_bounds__(1024, 1) smem_kernel(float* out, unsigned long long* cycles) {
  extern __shared__ float sm[];
  for (int i = threadIdx.x; i < kWords; i += blockDim.x) sm[i] = 0.f;
  __syncthreads();
  uint32_t s = 12345u + threadIdx.x * 7919u + blockIdx.x * 104729u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float acc = 0.f;
  unsigned long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < kIters; ++it) {
    uint32_t r = lcg(s);
    uint32_t addr;
    if (MODE == 3 || MODE == 4 || MODE == 5) {
      // warp-uniform random base row, lanes on distinct banks; warps on disjoint rows
      uint32_t row = (__shfl_sync(0xffffffffu, r, 0) % (kWords / 32 / 32)) * 32 + warp;
      addr = row * 32 + lane;
    } else {
      addr = r % kWords;
    }
    if (MODE == 0 || MODE == 3) {
      sm[addr] += 1.0f;
    } else if (MODE == 1 || MODE == 5) {
      atomicAdd(&sm[addr], 1.0f);
    } else if (MODE == 2 || MODE == 4) {
      atomicAdd(reinterpret_cast<int*>(sm) + addr, static_cast<int>(r >> 29) + 1);
    } else if (MODE == 6) {
      acc += sm[addr];
    } else if (MODE == 7) {
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(static_cast<uint32_t>(
                       __cvta_generic_to_shared(reinterpret_cast<int*>(sm) + addr))), "r"((r >> 29) + 1));
    }
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) out[0] = acc;
  if (threadIdx.x < 32) out[blockIdx.x * 32 + threadIdx.x] = sm[threadIdx.x];
}

// Streaming read of a float tensor: grid of G CTAs, CTA b reads chunk (b / rep)
// of G/rep chunks, so the whole tensor is read `rep` times (rep CTAs per chunk).
__global__ void __launch_bounds__(1024, 1) stream_kernel(const float4* __restrict__ t, size_t n4,
                                                         int rep, float* out) {
  const int chunks = gridDim.x / rep;
  const int chunk = blockIdx.x / rep;
  const size_t per = (n4 + chunks - 1) / chunks;
  const size_t b = chunk * per, e = min(n4, b + per);
  float acc = 0.f;
  for (size_t i = b + threadIdx.x; i < e; i += blockDim.x) {
    float4 v = __ldcs(t + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

template <int MODE>
int run_smem(const char* name, float* out, unsigned long long* cyc, int sms) {
  auto k = smem_kernel<MODE>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 4));
  k<<<sms, 1024, kWords * 4>>>(out, cyc);
  CK(cudaDeviceSynchronize());
  unsigned long long h[256];
  CK(cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  printf("smem %-34s %7.2f updates/clk/SM\n", name, 1024.0 * kIters / avg);
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float* out;
  unsigned long long* cyc;
  CK(cudaMalloc(&out, 1 << 20));
  CK(cudaMalloc(&cyc, 256 * 8));
  run_smem<6>("LDS only, random", out, cyc, sms);
  run_smem<0>("plain RMW, random", out, cyc, sms);
  run_smem<3>("plain RMW, conflict-free", out, cyc, sms);
  run_smem<1>("atomicAdd f32, random", out, cyc, sms);
  run_smem<5>("atomicAdd f32, conflict-free", out, cyc, sms);
  run_smem<2>("atomicAdd i32, random", out, cyc, sms);
  run_smem<4>("atomicAdd i32, conflict-free", out, cyc, sms);
  run_smem<7>("red.shared.add.u32, random", out, cyc, sms);

  const size_t n = size_t(1) << 30;
  float4* t;
  CK(cudaMalloc(&t, n * 4));
  CK(cudaMemset(t, 0, n * 4));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep : {1, 2, 4}) {
    for (int w = 0; w < 2; ++w) stream_kernel<<<sms / 4 * 4, 1024>>>(t, n / 4, rep, out);
    cudaEventRecord(a);
    for (int w = 0; w < 5; ++w) stream_kernel<<<sms / 4 * 4, 1024>>>(t, n / 4, rep, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("stream 4 GiB read x%d (CTA-replicated): %.3f ms  -> %.0f GB/s unique, %.0f GB/s L2->SM\n",
           rep, ms, n * 4 / (ms * 1e-3) / 1e9, rep * n * 4 / (ms * 1e-3) / 1e9);
  }
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("sms %d clock %d kHz\n", sms, clk);
  return 0;
}
