// Design probe for K1 on the config-4 geometry (1024^3 fp32, J~=49150, D=4,
// one family per CTA, 148 CTAs): time of the scatter with different shared-
// memory update primitives, all else equal (vector loads, mode-0 table in
// registers, fiber-per-warp streaming, 16 warps/SM).
//   mode 0: atomicAdd f32 (CAS loop)   mode 1: red.shared.add.s32 fixed point
//   mode 2: plain RMW (racy, upper bound only)   mode 3: loads only
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int J = 16384, JT = 3 * J - 2, I0 = 1024, D = 4;

__global__ void fill(float* t, size_t n, uint32_t* tab) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)(i * 2654435761u);
    t[i] = (float)((int)(h >> 8) - (1 << 23)) / (float)(1 << 23);
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D * 3 * I0; i += gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)((i + 17) * 2246822519u);
    h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
    tab[i] = (h % J) | ((h >> 31) << 31);
  }
}

template <int MODE, int NV>
__global__ void __launch_bounds__(512, 1) scatter(const float* __restrict__ t, const uint32_t* __restrict__ tab,
                                                  uint64_t fibers, int* out) {
  extern __shared__ int sk[];
  const int d = blockIdx.x % D;
  const int chunk = blockIdx.x / D, nchunk = gridDim.x / D;
  const uint32_t* tb = tab + d * 3 * I0;
  for (int b = threadIdx.x; b < JT; b += blockDim.x) sk[b] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t e0[NV][4];
#pragma unroll
  for (int j = 0; j < NV; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k) e0[j][k] = tb[(lane + 32 * j) * 4 + k];
  __syncthreads();
  int ovf = 0;
  const uint64_t per = (fibers + nchunk - 1) / nchunk;
  const uint64_t fb = chunk * per, fe = min(fibers, fb + per);
  for (uint64_t f = fb + warp; f < fe; f += nw) {
    const uint32_t i1 = f % 1024, i2 = f / 1024;
    const uint32_t e1 = __ldg(tb + I0 + i1), e2 = __ldg(tb + 2 * I0 + i2);
    const uint32_t c = (e1 & 0x7fffffff) + (e2 & 0x7fffffff);
    const uint32_t sb = (e1 ^ e2) & 0x80000000u;
    float4 v[NV];
    const float4* src = reinterpret_cast<const float4*>(t + f * I0);
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = __ldcs(src + lane + 32 * j);
    if (MODE == 3) {
      float s = 0;
#pragma unroll
      for (int j = 0; j < NV; ++j) s += v[j].x + v[j].y + v[j].z + v[j].w;
      if (s == 12345.f) out[0] = 1;
      continue;
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const float* x = reinterpret_cast<const float*>(&v[j]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t e = e0[j][k];
        const uint32_t idx = (e & 0x7fffffff) + c;
        const float val = __uint_as_float(__float_as_uint(x[k]) ^ ((e ^ sb) & 0x80000000u));
        if (MODE == 0) {
          atomicAdd(reinterpret_cast<float*>(sk) + idx, val);
        } else if (MODE == 1) {
          const int q = __float2int_rn(val * 1048576.f);
          asm volatile("red.shared.add.s32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(sk + idx)), "r"(q));
        } else if (MODE == 5) {  // same instruction stream, conflict-free banks (upper bound)
          const int q = __float2int_rn(val * 1048576.f);
          const uint32_t cf = ((idx & ~31u) | lane) % JT;
          const int old = atomicAdd(sk + cf, q);
          ovf |= (old ^ (old + q)) & (q ^ (old + q));
        } else if (MODE == 4) {
          const int q = __float2int_rn(val * 1048576.f);
          const int old = atomicAdd(sk + idx, q);
          ovf |= (old ^ (old + q)) & (q ^ (old + q));
        } else {
          reinterpret_cast<float*>(sk)[idx] += val;
        }
      }
    }
  }
  if (__syncthreads_or(ovf < 0) && threadIdx.x == 0) out[0] = -1;
  for (int b = threadIdx.x; b < JT; b += blockDim.x) out[(size_t)blockIdx.x * JT + b] = sk[b];
}

template <int MODE>
int run(const char* name, const float* t, const uint32_t* tab, int* out, int sms) {
  auto k = scatter<MODE, 8>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, JT * 4));
  const uint64_t fibers = 1024ull * 1024;
  for (int w = 0; w < 2; ++w) k<<<sms / 4 * 4, 512, JT * 4>>>(t, tab, fibers, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int w = 0; w < 5; ++w) k<<<sms / 4 * 4, 512, JT * 4>>>(t, tab, fibers, out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("%-34s %.3f ms  (%.1f%% of 655.7us HBM roofline)\n", name, ms, 65.57 / ms);
  return 0;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t n = size_t(1) << 30;
  float* t;
  uint32_t* tab;
  int* out;
  CK(cudaMalloc(&t, n * 4));
  CK(cudaMalloc(&tab, D * 3 * I0 * 4));
  CK(cudaMalloc(&out, (size_t)sms * JT * 4));
  fill<<<sms * 4, 512>>>(t, n, tab);
  CK(cudaDeviceSynchronize());
  run<3>("loads only (4x per family)", t, tab, out, sms);
  run<0>("atomicAdd f32 (CAS)", t, tab, out, sms);
  run<1>("red.shared.add.s32 fixed point", t, tab, out, sms);
  run<2>("plain RMW (racy bound)", t, tab, out, sms);
  run<4>("atom.shared.add.s32 + overflow check", t, tab, out, sms);
  run<5>("same, conflict-free banks (bound)", t, tab, out, sms);
  return 0;
}
