// vol.cuh -- CTA-wide volume-based DataReduct Vol(S, k) (readings C2-C5).
//
//   |S| <= k   : S sorted, de-duplicated (pass-through, C5)
//   otherwise  : m = max{m : m^d <= k}; grid = cell centres of an m^d tensor grid over the tight
//                bounding box of S (C2, C3); for every grid node q the point of S minimising
//                sum_c (x_c - q_c)^2 (operations rounded separately, summed in c order, ties to
//                the lowest index: C4); result sorted and de-duplicated.
// Used by the HiDR sweeps (hidr.cu) and the r calibration (calib.cu).
#pragma once
#include <cfloat>
#include <climits>
#include <cub/block/block_scan.cuh>

#include "h2_internal.cuh"

namespace h2 {

constexpr int kVolTile = 256;
constexpr int kVolSelCap = 4096;  // max budget k (and max |S| for pass-through) a CTA handles

template <int D, int NT>
struct VolSmem {
  double tile[D][kVolTile];
  int tidx[kVolTile];
  double bd[NT];
  int bi[NT];
  int sel[kVolSelCap];
  double lo[D], hi[D], hstep[D];
  double rlo[D][NT / 32], rhi[D][NT / 32];
  typename cub::BlockScan<int, NT>::TempStorage scan;
  int cnt;
};

// bitonic sort of a[0..P), P a power of two, by the whole CTA
template <int NT>
__device__ void cta_bitonic(int* a, int P) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += NT) {
        int l = i ^ j;
        if (l > i) {
          int x = a[i], y = a[l];
          bool up = (i & k) == 0;
          if ((x > y) == up) {
            a[i] = y;
            a[l] = x;
          }
        }
      }
      __syncthreads();
    }
}

// sort sm.sel[0..cnt) and write the distinct values to out; returns the distinct count
template <int D, int NT>
__device__ int cta_sort_unique_write(VolSmem<D, NT>& sm, int cnt, int* out) {
  int P = 1;
  while (P < cnt) P <<= 1;
  for (int i = cnt + threadIdx.x; i < P; i += NT) sm.sel[i] = INT_MAX;
  __syncthreads();
  cta_bitonic<NT>(sm.sel, P);
  int base = 0;
  for (int c0 = 0; c0 < cnt; c0 += NT) {
    int i = c0 + threadIdx.x;
    int keep = (i < cnt) && (i == 0 || sm.sel[i] != sm.sel[i - 1]);
    int pos, agg;
    cub::BlockScan<int, NT>(sm.scan).ExclusiveSum(keep, pos, agg);
    if (keep) out[base + pos] = sm.sel[i];
    base += agg;
    __syncthreads();
  }
  return base;
}

// Acc: __device__ double coord(int pos, int c) const; __device__ int index(int pos) const
template <int D, int NT, class Acc>
__device__ int cta_vol(const Acc& acc, int ns, int k, int* out, VolSmem<D, NT>& sm,
                       unsigned long long* evals = nullptr) {
  const int tid = threadIdx.x;
  if (ns <= 0) return 0;
  if (ns <= k) {
    for (int i = tid; i < ns; i += NT) sm.sel[i] = acc.index(i);
    __syncthreads();
    int c = cta_sort_unique_write<D, NT>(sm, ns, out);
    return c;
  }
  int m = 1;
  for (;;) {
    long long p = 1;
    for (int c = 0; c < D; c++) p *= (m + 1);
    if (p > k) break;
    m++;
  }
  int G = 1;
  for (int c = 0; c < D; c++) G *= m;
  // tight bounding box of S (exact: min/max)
  double lo[D], hi[D];
#pragma unroll
  for (int c = 0; c < D; c++) {
    lo[c] = DBL_MAX;
    hi[c] = -DBL_MAX;
  }
  for (int i = tid; i < ns; i += NT)
#pragma unroll
    for (int c = 0; c < D; c++) {
      double v = acc.coord(i, c);
      lo[c] = fmin(lo[c], v);
      hi[c] = fmax(hi[c], v);
    }
#pragma unroll
  for (int c = 0; c < D; c++)
    for (int o = 16; o > 0; o >>= 1) {
      lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
  if ((tid & 31) == 0)
#pragma unroll
    for (int c = 0; c < D; c++) {
      sm.rlo[c][tid >> 5] = lo[c];
      sm.rhi[c][tid >> 5] = hi[c];
    }
  __syncthreads();
  if (tid < D) {
    double a = DBL_MAX, b = -DBL_MAX;
    for (int w = 0; w < NT / 32; w++) {
      a = fmin(a, sm.rlo[tid][w]);
      b = fmax(b, sm.rhi[tid][w]);
    }
    sm.lo[tid] = a;
    sm.hi[tid] = b;
    sm.hstep[tid] = __ddiv_rn(__dsub_rn(b, a), (double)m);
  }
  __syncthreads();
  // thread -> (grid nodes g0, g0+NT*?, ...) x point slice
  const int nslice = G >= NT ? 1 : NT / G;
  const int gthreads = G >= NT ? NT : G * nslice;
  const bool active = tid < gthreads;
  const int slice = G >= NT ? 0 : tid / G;
  for (int gbase = 0; gbase < G; gbase += (G >= NT ? NT : G)) {
    int g = gbase + (G >= NT ? tid : tid % G);
    bool gact = active && g < G;
    double q[D];
    {
      int rem = g;
#pragma unroll
      for (int c = 0; c < D; c++) {
        int j = rem % m;
        rem /= m;
        q[c] = __dadd_rn(sm.lo[c], __dmul_rn((double)j + 0.5, sm.hstep[c]));
      }
    }
    double best = DBL_MAX;
    int bi = INT_MAX;
    bool have = false;
    for (int t0 = 0; t0 < ns; t0 += kVolTile) {
      int tn = ns - t0 < kVolTile ? ns - t0 : kVolTile;
      __syncthreads();
      for (int i = tid; i < tn; i += NT) {
        sm.tidx[i] = acc.index(t0 + i);
#pragma unroll
        for (int c = 0; c < D; c++) sm.tile[c][i] = acc.coord(t0 + i, c);
      }
      __syncthreads();
      if (gact) {
        for (int p = slice; p < tn; p += nslice) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < D; c++) {
            double df = __dsub_rn(sm.tile[c][p], q[c]);
            s = __dadd_rn(s, __dmul_rn(df, df));
          }
          int ix = sm.tidx[p];
          if (!have || s < best || (s == best && ix < bi)) {
            best = s;
            bi = ix;
            have = true;
          }
        }
      }
    }
    __syncthreads();
    sm.bd[tid] = have ? best : DBL_MAX;
    sm.bi[tid] = have ? bi : INT_MAX;
    __syncthreads();
    if (gact && slice == 0) {
      int gl = G >= NT ? tid : tid % G;
      for (int sl = 1; sl < nslice; sl++) {
        int o = gl + sl * G;
        double s2 = sm.bd[o];
        int i2 = sm.bi[o];
        if (s2 < best || (s2 == best && i2 < bi)) {
          best = s2;
          bi = i2;
        }
      }
      sm.sel[g] = bi;
    }
    __syncthreads();
  }
  if (evals && tid == 0) atomicAdd(evals, (unsigned long long)G * (unsigned long long)ns);
  return cta_sort_unique_write<D, NT>(sm, G, out);
}

}  // namespace h2
