// prims.cuh -- CTA-level building blocks shared by the kernels: block-wide exclusive sums
// (warp shuffles + one shared-memory word per warp).  Device-wide scans and the radix sort are
// in prims.cu.
#pragma once
#include "h2_internal.cuh"

namespace h2 {

template <int NT>
struct BlockScanSmem {
  int warp_sum[NT / 32];
};

// Exclusive prefix sum of v over the CTA's threads (thread order); *total gets the CTA sum.
// Every thread must call it.  Like any shared-memory scratch, `sm` may be reused only after a
// __syncthreads() that follows the previous call.
template <int NT>
__device__ __forceinline__ int block_excl_sum(int v, int* total, BlockScanSmem<NT>& sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) sm.warp_sum[w] = incl;
  __syncthreads();
  int before = 0, all = 0;
#pragma unroll
  for (int q = 0; q < NT / 32; q++) {
    const int s = sm.warp_sum[q];
    before += q < w ? s : 0;
    all += s;
  }
  *total = all;
  return before + incl - v;
}

}  // namespace h2
