// Shared pieces of the dense-FCS kernels (fcs_dense.cu, fcs_round.cu).
#pragma once

#include "common.cuh"

namespace fcs {

struct DenseArgs {
  int order;
  int D;
  uint32_t dims[ST_MAX_ORDER];
  uint32_t tab_off[ST_MAX_ORDER];  // start of mode n inside one family's tables
  uint32_t fam_stride;             // sum(dims): distance between families
  uint32_t jt;                     // composed length J~
  uint32_t last_begin;             // first i_{N-1} of this slab
  uint32_t i0_shift;               // mode-0 table shift (order-1 slabs only)
  uint32_t inv_d1;                 // floor(2^32 / dims[1]) for fast division (order 3)
  uint64_t fibers;                 // mode-0 fibers in this slab
  uint64_t fibers_per_chunk;
};

// Offset and sign bit of fiber f (slab-local) for the family at `tab`.
__device__ __forceinline__ void fiber_offset(const DenseArgs& a, const uint32_t* __restrict__ tab,
                                             uint64_t f, uint32_t& c, uint32_t& sbit) {
  c = 0;
  sbit = 0;
  for (int n = 1; n < a.order; ++n) {
    uint64_t i;
    if (n < a.order - 1) {
      i = f % a.dims[n];
      f /= a.dims[n];
    } else {
      i = f + a.last_begin;
    }
    const uint32_t e = __ldg(tab + a.tab_off[n] + i);
    c += e & 0x7fffffffu;
    sbit ^= e & 0x80000000u;
  }
}

template <typename Tacc>
__device__ __forceinline__ Tacc signed_val(Tacc v, uint32_t sbit) {
  return sbit ? -v : v;
}

// One shared-memory compare-and-swap of the bit pattern; true if `desired`
// was stored (the word still held `expected`).
__device__ __forceinline__ bool cas_update(float* p, float expected, float desired) {
  const unsigned e = __float_as_uint(expected);
  return atomicCAS(reinterpret_cast<unsigned*>(p), e, __float_as_uint(desired)) == e;
}
__device__ __forceinline__ bool cas_update(double* p, double expected, double desired) {
  const unsigned long long e = __double_as_longlong(expected);
  return atomicCAS(reinterpret_cast<unsigned long long*>(p), e, __double_as_longlong(desired)) == e;
}

}  // namespace fcs
