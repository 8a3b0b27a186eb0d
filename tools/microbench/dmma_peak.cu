// fp64 tensor-core (DMMA, mma.sync.m8n8k4.f64) throughput vs DFMA on one
// B200: all SMs, independent accumulator chains per warp. Prints JSON.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) dmma_kernel(double* out, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void __launch_bounds__(256) dfma_kernel(double* out, double seed) {
  double a[8];
  const double m = 1.0 + 1e-12, c0 = 1e-9;
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed + k;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c0);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps_per_sm : {4, 8, 16, 32}) {
    const int grid = sms * warps_per_sm / 8, threads = 256;
    float best_m = 1e30f, best_f = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      dmma_kernel<<<grid, threads>>>(d, 1.0 + r);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best_m) best_m = ms;
      cudaEventRecord(e0);
      dfma_kernel<<<grid, threads>>>(d, 1.0 + r);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best_f) best_f = ms;
    }
    const double warps = static_cast<double>(grid) * threads / 32;
    const double dmma_flops = warps * kIters * 8 * 8 * 8 * 4 * 2.0;  // m8n8k4 = 256 FMA / warp
    const double dfma_flops = static_cast<double>(grid) * threads * kIters * 8 * 2.0;
    printf("{\"warps_per_sm\": %d, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f}\n", warps_per_sm,
           dmma_flops / (best_m * 1e-3) / 1e12, dfma_flops / (best_f * 1e-3) / 1e12);
  }
  return 0;
}
