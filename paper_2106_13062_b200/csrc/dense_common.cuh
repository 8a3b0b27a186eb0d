// Shared pieces of the dense sketch kernels (fcs_dense.cu).
#pragma once

#include "common.cuh"

namespace fcs {

// A dense sketch launch. The composed bucket of multi-index (i_0..i_{N-1}) is
// sum_n mult[n] * h_n(i_n) with mult[0] = 1:
//   FCS (sketch.cpp:187-201): mult[n] = 1, out length J~ = sum J_n - N + 1;
//   HCS (sketch.cpp:157-173): mult[n] = J_0 * ... * J_{n-1}, out length prod J_n.
struct DenseArgs {
  int order;
  int D;
  uint32_t dims[ST_MAX_ORDER];
  uint32_t tab_off[ST_MAX_ORDER];  // start of mode n inside one family's tables
  uint32_t mult[ST_MAX_ORDER];     // bucket multiplier of mode n (mult[0] = 1)
  uint32_t fam_stride;             // sum(dims): distance between families
  uint32_t jt;                     // output length per family (J~ for FCS)
  uint32_t last_begin;             // first i_{N-1} of this slab
  uint32_t i0_shift;               // mode-0 table shift (order-1 slabs only)
  uint32_t inv_d1;                 // floor(2^32 / dims[1]) for fast division (order 3)
  uint64_t fibers;                 // mode-0 fibers in this slab
  uint64_t fibers_per_chunk;
  // fixed-point kernels with lane-owned entries (fx64 / fx32s): a fiber is
  // 2^lseg segments of seg_len entries (the last one shorter), one warp each
  uint32_t seg_len;
  uint32_t lseg;
  // fx64 with J~ beyond shared memory: the buckets in rparts ranges of rspan,
  // one CTA per (chunk, family, range)
  uint32_t rparts;
  uint32_t rspan;
  uint32_t j0;  // mode-0 hash length (the lane-owned kernels pack mode-0 buckets in 16 bits)
};

// A sparse (COO) sketch launch (fcs_coo.cu).
struct CooArgs {
  uint32_t dims[ST_MAX_ORDER];
  uint32_t tab_off[ST_MAX_ORDER];
  uint32_t fam_stride;
  uint32_t jt;
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
    c += (e & 0x7fffffffu) * a.mult[n];
    sbit ^= e & 0x80000000u;
  }
}

template <typename Tacc>
__device__ __forceinline__ Tacc signed_val(Tacc v, uint32_t sbit) {
  return sbit ? -v : v;
}

}  // namespace fcs
