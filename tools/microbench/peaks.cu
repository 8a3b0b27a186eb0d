// Peak probes for the rooflines the FCS kernels are reported against
// (profiles/fp64_peak.json; MEASURED_PEAKS.json is driver-owned and has only
// HBM copy bandwidth and the bf16 GEMM rate):
//   * fp64 FMA throughput (DFMA), all SMs, 8 independent chains per thread;
//   * shared-memory load bandwidth (LDS.128, conflict-free);
//   * shared-memory int32 atomic throughput (ATOMS.ADD / red.shared, with and
//     without returned value) with 1, 2, 4, 8 lanes per bank and random banks —
//     the update primitive of K1, as updates per clock per SM;
//   * shared-memory fp64 atomicAdd (the CAS loop the old fp64 K1 used).
// Addresses are held in registers and stepped by immediates (multiples of
// 128 B keep each lane's bank), so the loops issue one memory instruction per
// update and measure the shared-memory pipe, not address arithmetic.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                           \
      return 1;                                                                \
    }                                                                          \
  } while (0)

constexpr int kDfmaIters = 8192;
__global__ void __launch_bounds__(256) dfma_kernel(double* out, double seed) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 1e-9 + k;
  const double m = 0.999999999, c = 1e-12;
  for (int it = 0; it < kDfmaIters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.0) out[0] = s;
}

constexpr int kSmemWords = 49152;  // 192 KB (the c4 sketch size)
constexpr int kIters = 16384;

__global__ void __launch_bounds__(1024, 1) lds_kernel(float* out, unsigned long long* cyc) {
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  for (int i = threadIdx.x; i < kSmemWords; i += blockDim.x) sm[i] = i;
  __syncthreads();
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm4)) + 16u * threadIdx.x;
  float acc = 0.f;
  unsigned long long t0 = clock64();
  for (int it = 0; it < kIters / 8; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float4 v;
      // 1024 threads x 16 B = 16 KB per step; 8 steps cover 128 KB
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                   : "r"(base + k * 16384));
      acc += v.x + v.w;
    }
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 1.2345f) out[0] = acc;
}

// MODE 0: atom.shared.add.s32 (returned value consumed), 1: red.shared.add.s32,
// 2: atom.shared.add.f64-style CAS (atomicAdd(double*)), 3: atom.shared.add.f32 (CAS).
// Lane address: bank chosen by `bankmap` (per lane), row by warp.
template <int MODE>
__global__ void __launch_bounds__(1024, 1) atoms_kernel(const int* __restrict__ bankmap,
                                                        int* out, unsigned long long* cyc) {
  extern __shared__ int smi[];
  for (int i = threadIdx.x; i < kSmemWords; i += blockDim.x) smi[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // word = bank + 32 * (warp * 8 + lane % 8): distinct words, bank from the map
  const uint32_t word = static_cast<uint32_t>(bankmap[lane]) + 32u * (warp * 8 + (lane & 7));
  const uint32_t addr = static_cast<uint32_t>(__cvta_generic_to_shared(smi)) + 4u * word;
  int acc = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < kIters / 8; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      // + k * 32 KB: same bank, different rows (stays inside 192 KB for 1024 threads)
      if (MODE == 0) {
        int old;
        asm volatile("atom.shared.add.s32 %0, [%1], 1;" : "=r"(old) : "r"(addr + k * 8192));
        acc ^= old;
      } else if (MODE == 1) {
        asm volatile("red.shared.add.s32 [%0], 1;" ::"r"(addr + k * 8192));
      } else if (MODE == 2) {
        double* p = reinterpret_cast<double*>(reinterpret_cast<char*>(smi) + ((4u * word) & ~7u) +
                                              (k * 4096 * 4 / 2 % (kSmemWords * 4 - 8)));
        atomicAdd(p, 1.0);
      } else {
        float* p = reinterpret_cast<float*>(reinterpret_cast<char*>(smi) + 4u * word + k * 4096 * 4 / 2);
        atomicAdd(p, 1.0f);
      }
    }
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 12345) out[0] = acc;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const int sms = prop.multiProcessorCount;
  double* dout;
  int* iout;
  float* fout;
  unsigned long long* cyc;
  int* bank_d;
  CK(cudaMalloc(&dout, 64));
  CK(cudaMalloc(&iout, 64));
  CK(cudaMalloc(&fout, 64));
  CK(cudaMalloc(&cyc, sizeof(unsigned long long) * 4096));
  CK(cudaMalloc(&bank_d, 32 * sizeof(int)));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  printf("{\"device\": \"%s\", \"sms\": %d, \"max_clock_mhz\": %.0f", prop.name, sms, clk_khz / 1e3);

  // fp64 FMA peak
  {
    const int grid = sms * 8, threads = 256;
    dfma_kernel<<<grid, threads>>>(dout, 1.0);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      dfma_kernel<<<grid, threads>>>(dout, 1.0 + r);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
    }
    const double flops = 2.0 * grid * threads * 8.0 * kDfmaIters;
    printf(", \"fp64_fma_tflops\": %.3f", flops / (best * 1e-3) / 1e12);
  }
  // Per-SM rates are timed with events over the whole kernel (a warp's own
  // clock64 span under-counts: early-finishing warps) and converted at the
  // SM clock; "_sm_clk_per_kernel" cross-checks with the slowest CTA's cycles.
  auto timed = [&](auto launch, double work_per_sm, const char* name) -> int {
    launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
    }
    printf(", \"%s\": %.3f", name, work_per_sm / (best * 1e-3 * clk_khz * 1e3));
    return 0;
  };
  // LDS.128 bandwidth in bytes / clk / SM
  {
    const size_t smem = kSmemWords * 4;
    CK(cudaFuncSetAttribute(lds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (timed([&] { lds_kernel<<<sms, 1024, smem>>>(fout, cyc); }, 1024.0 * kIters * 16.0,
              "lds128_bytes_per_clk_sm"))
      return 1;
  }
  // shared atomics: lanes per bank 1, 2, 4, 8 and random
  int bankmaps[5][32];
  const int lpb[4] = {1, 2, 4, 8};
  // k lanes per bank: lanes 8q..8q+7 spread over banks l / k (distinct rows)
  for (int m = 0; m < 4; ++m)
    for (int l = 0; l < 32; ++l) bankmaps[m][l] = (l / lpb[m]) % 32;
  uint32_t s = 12345u;
  for (int l = 0; l < 32; ++l) {
    s = s * 1664525u + 1013904223u;
    bankmaps[4][l] = (s >> 16) % 32;
  }
  const char* names[5] = {"1", "2", "4", "8", "random"};
  const size_t smem = kSmemWords * 4;
  auto run_atoms = [&](auto kern, const char* prim) -> int {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int m = 0; m < 5; ++m) {
      CK(cudaMemcpy(bank_d, bankmaps[m], sizeof(bankmaps[m]), cudaMemcpyHostToDevice));
      char name[128];
      snprintf(name, sizeof(name), "%s_lanes_per_bank_%s_updates_per_clk_sm", prim, names[m]);
      if (timed([&] { kern<<<sms, 1024, smem>>>(bank_d, iout, cyc); }, 1024.0 * kIters, name))
        return 1;
    }
    return 0;
  };
  if (run_atoms(atoms_kernel<0>, "atom_s32")) return 1;
  if (run_atoms(atoms_kernel<1>, "red_s32")) return 1;
  if (run_atoms(atoms_kernel<3>, "atomicadd_f32")) return 1;
  if (run_atoms(atoms_kernel<2>, "atomicadd_f64")) return 1;
  printf("}\n");
  return 0;
}
