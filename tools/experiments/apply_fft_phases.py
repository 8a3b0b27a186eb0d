"""Probe (not for merge): globaltimer stamps inside rfft_of_cs (zero, scatter,
each forward pass, fused last pass) of iuv1_kernel; read with st_probe_phases.
Restore with git checkout of spectral.cu and fft.cuh."""
p = 'paper_2106_13062_b200/csrc/fft.cuh'
s = open(p).read()
s = s.replace('namespace fcs {\n', '''namespace fcs {
__device__ unsigned long long g_ph[1024][16];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PH(k) do { __syncthreads(); if (threadIdx.x == 0) g_ph[blockIdx.x + blockIdx.y * gridDim.x][k] = gtime(); } while (0)
''', 1)
old = '''  for (int p = 0; p + 1 < pl.npass; ++p) {
    fft_dispatch<true>(buf, tw, 1 << kTwLoBits, pl.M, pl.P, pl.radix[p], pl.len[p]);
    __syncthreads();
  }
  pair_group_dispatch<true>(buf, pl, tw);
}'''
assert old in s
s = s.replace(old, '''  for (int p = 0; p + 1 < pl.npass; ++p) {
    fft_dispatch<true>(buf, tw, 1 << kTwLoBits, pl.M, pl.P, pl.radix[p], pl.len[p]);
    __syncthreads();
    PH(3 + p);
  }
  pair_group_dispatch<true>(buf, pl, tw);
  PH(9);
}''', 1)
open(p, 'w').write(s)
p = 'paper_2106_13062_b200/csrc/spectral.cu'
s = open(p).read()
old = '''  zero_slots(buf, pl.P);
  __syncthreads();
  scatter_cs(buf, vec, I, tab);
  __syncthreads();
  fft_forward_post(buf, pl, sm.tw);'''
assert old in s
s = s.replace(old, '''  PH(0);
  zero_slots(buf, pl.P);
  __syncthreads();
  PH(1);
  scatter_cs(buf, vec, I, tab);
  __syncthreads();
  PH(2);
  fft_forward_post(buf, pl, sm.tw);''', 1)
s += '''
extern "C" int st_probe_phases(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, fcs::g_ph, sizeof(fcs::g_ph)) == cudaSuccess ? 0 : 1;
}
'''
open(p, 'w').write(s)
