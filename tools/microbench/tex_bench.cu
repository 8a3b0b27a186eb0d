// Probe: do texture fetches of the tensor relieve K1's saturated LSU data pipe?
// Same geometry as scatter_bench (1024^3 fp32, J~=49150, D=4, one family per
// CTA, 148 CTAs x 512 threads, int32 fixed-point atom.shared.add with the
// overflow check), tensor read either with ld.global.nc.L1::no_allocate
// (LSU pipe) or tex1Dfetch<float4> (TEX pipe; 4 texture objects of 1 GiB).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int J = 16384, JT = 3 * J - 2, I0 = 1024, D = 4, NV = 8;
constexpr uint64_t kFibersPerTex = 1ull << 18;  // 2^18 fibers x 4 KiB = 1 GiB

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

struct Tex4 { cudaTextureObject_t o[4]; };

__device__ __forceinline__ float4 ld_na(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

template <bool kTex>
__global__ void __launch_bounds__(512, 1) scatter(const float* __restrict__ t, Tex4 tx,
                                                  const uint32_t* __restrict__ tab,
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
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sk);
  for (uint64_t f = fb + warp; f < fe; f += nw) {
    const uint32_t i1 = f % 1024, i2 = f / 1024;
    const uint32_t e1 = __ldg(tb + I0 + i1), e2 = __ldg(tb + 2 * I0 + i2);
    const uint32_t c = (e1 & 0x7fffffff) + (e2 & 0x7fffffff);
    const uint32_t sb = (e1 ^ e2) & 0x80000000u;
    float4 v[NV];
    if (kTex) {
      const cudaTextureObject_t o = tx.o[f / kFibersPerTex];
      const int off = (int)((f % kFibersPerTex) * 256);
#pragma unroll
      for (int j = 0; j < NV; ++j) v[j] = tex1Dfetch<float4>(o, off + lane + 32 * j);
    } else {
      const float4* src = reinterpret_cast<const float4*>(t + f * I0);
#pragma unroll
      for (int j = 0; j < NV; ++j) v[j] = ld_na(src + lane + 32 * j);
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const float* x = reinterpret_cast<const float*>(&v[j]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t e = e0[j][k];
        const float val = __uint_as_float(__float_as_uint(x[k]) ^ ((e ^ sb) & 0x80000000u));
        const int q = __float2int_rn(val * 1048576.f);
        int old;
        asm volatile("atom.shared.add.s32 %0, [%1], %2;" : "=r"(old) : "r"(base + 4 * ((e & 0x7fffffff) + c)), "r"(q));
        ovf |= (old ^ (old + q)) & (q ^ (old + q));
      }
    }
  }
  if (__syncthreads_or(ovf < 0) && threadIdx.x == 0) out[0] = -1;
  for (int b = threadIdx.x; b < JT; b += blockDim.x) out[(size_t)blockIdx.x * JT + b] = sk[b];
}

template <bool kTex>
int run(const char* name, const float* t, Tex4 tx, const uint32_t* tab, int* out, int sms) {
  auto k = scatter<kTex>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, JT * 4));
  const uint64_t fibers = 1024ull * 1024;
  for (int w = 0; w < 2; ++w) k<<<sms / 4 * 4, 512, JT * 4>>>(t, tx, tab, fibers, out);
  CK(cudaGetLastError());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int w = 0; w < 10; ++w) k<<<sms / 4 * 4, 512, JT * 4>>>(t, tx, tab, fibers, out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-40s %.3f ms\n", name, ms / 10);
  return 0;
}

int main() {
  int sms, texw;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&texw, cudaDevAttrMaxTexture1DLinearWidth, 0));
  printf("max 1D linear texture width: %d texels\n", texw);
  const size_t n = size_t(1) << 30;
  float* t;
  uint32_t* tab;
  int* out;
  CK(cudaMalloc(&t, n * 4));
  CK(cudaMalloc(&tab, D * 3 * I0 * 4));
  CK(cudaMalloc(&out, (size_t)sms * JT * 4));
  fill<<<sms * 4, 512>>>(t, n, tab);
  CK(cudaDeviceSynchronize());
  Tex4 tx;
  for (int i = 0; i < 4; ++i) {
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = t + (size_t)i * (n / 4);
    rd.res.linear.desc = cudaCreateChannelDesc<float4>();
    rd.res.linear.sizeInBytes = n;  // 1 GiB of floats = n/4 * 4 B
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    CK(cudaCreateTextureObject(&tx.o[i], &rd, &td, nullptr));
  }
  run<false>("atom.s32 + check, ld.nc.L1::no_allocate", t, tx, tab, out, sms);
  run<true>("atom.s32 + check, tex1Dfetch<float4>", t, tx, tab, out, sms);
  run<false>("atom.s32 + check, ld.nc.L1::no_allocate", t, tx, tab, out, sms);
  run<true>("atom.s32 + check, tex1Dfetch<float4>", t, tx, tab, out, sms);
  return 0;
}
