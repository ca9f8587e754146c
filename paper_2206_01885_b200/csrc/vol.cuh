// vol.cuh -- CTA-wide volume-based DataReduct Vol(S, k) (readings C2-C5).
//
//   |S| <= k   : S sorted, de-duplicated (pass-through, C5)
//   otherwise  : m = max{m : m^d <= k}; grid = cell centres of an m^d tensor grid over the tight
//                bounding box of S (C2, C3); for every grid node q the point of S minimising
//                sum_c (x_c - q_c)^2 (operations rounded separately, summed in c order, ties to
//                the lowest index: C4); result sorted and de-duplicated.
// Used by the HiDR sweeps (hidr.cu) and the r calibration (calib.cu).
//
// Shared memory: the point tile (coordinates + indices, one gather per point when S fits one
// tile) and the combine / selection buffers are used in different phases and share storage.
#pragma once
#include <cfloat>
#include <climits>

#include "prims.cuh"

namespace h2 {

constexpr int kVolSelCap = 4096;  // max budget k (and max |S| for pass-through) a CTA handles
constexpr int kVolGPT = 4;        // grid nodes per thread in the argmin
__host__ __device__ constexpr int vol_tile(int D) { return D <= 2 ? 1536 : (D <= 4 ? 768 : 384); }

template <int D, int NT>
struct VolSmem {
  union {
    struct {  // argmin phase
      double x[D][vol_tile(D)];
      int idx[vol_tile(D)];
    } tile;
    struct {  // combine + selection phase
      double bd[kVolGPT][NT];
      int bi[kVolGPT][NT];
      int sel[kVolSelCap];
    } out;
  } u;
  double lo[D], hi[D], hstep[D];
  double rlo[D][NT / 32], rhi[D][NT / 32];
  BlockScanSmem<NT> scan;
};

// bitonic sort of a[0..P), P a power of two, by the whole CTA
template <int NT>
__device__ void cta_bitonic(int* a, int P) {
  // every thread takes compare-exchange pairs (i, i + j) directly: P/2 pairs per stage
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int q = threadIdx.x; q < (P >> 1); q += NT) {
        const int i = ((q & ~(j - 1)) << 1) | (q & (j - 1)), l = i + j;
        const int x = a[i], y = a[l];
        if ((x > y) == ((i & k) == 0)) {
          a[i] = y;
          a[l] = x;
        }
      }
      __syncthreads();
    }
}

// sort sel[0..cnt) and write the distinct values to out; returns the distinct count.
// cnt <= 64: warp 0 sorts two keys per lane with shuffles and compacts with ballots (no CTA
// barrier inside); larger: CTA bitonic sort + block-scan compaction.
template <int NT>
__device__ int cta_sort_unique_write(BlockScanSmem<NT>& scan, int* sel, int cnt,
                                     int* out) {
  __shared__ int s_cnt;
  if (cnt <= 64) {
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int a = lane < cnt ? sel[lane] : INT_MAX;            // element lane
      int b = lane + 32 < cnt ? sel[lane + 32] : INT_MAX;  // element lane + 32
      // bitonic network over 64 elements: position p = lane (a) and lane + 32 (b)
      for (int k = 2; k <= 64; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
          if (j == 32) {  // partner of a is b of the same lane
            const bool up = (lane & k) == 0;
            const int lo = min(a, b), hi = max(a, b);
            a = up ? lo : hi;
            b = up ? hi : lo;
          } else {
            const int pa = __shfl_xor_sync(0xffffffffu, a, j);
            const int pb = __shfl_xor_sync(0xffffffffu, b, j);
            const bool lower = (lane & j) == 0;
            const bool upa = (lane & k) == 0, upb = ((lane + 32) & k) == 0;
            a = (lower == upa) ? min(a, pa) : max(a, pa);
            b = (lower == upb) ? min(b, pb) : max(b, pb);
          }
        }
      // distinct values: a sorted sequence a(0..31), b(0..31)
      const int prev_a = __shfl_up_sync(0xffffffffu, a, 1);  // all lanes execute every shuffle
      const int last_a = __shfl_sync(0xffffffffu, a, 31);
      const int up_b = __shfl_up_sync(0xffffffffu, b, 1);
      const int prev_b = lane == 0 ? last_a : up_b;
      const bool ka = lane < cnt && (lane == 0 || a != prev_a);
      const bool kb = lane + 32 < cnt && b != prev_b;
      const unsigned ba = __ballot_sync(0xffffffffu, ka), bb = __ballot_sync(0xffffffffu, kb);
      const unsigned below = (1u << lane) - 1u;
      if (ka) out[__popc(ba & below)] = a;
      if (kb) out[__popc(ba) + __popc(bb & below)] = b;
      if (lane == 0) s_cnt = __popc(ba) + __popc(bb);
    }
    __syncthreads();
    const int c = s_cnt;
    __syncthreads();
    return c;
  }
  int P = 1;
  while (P < cnt) P <<= 1;
  for (int i = cnt + threadIdx.x; i < P; i += NT) sel[i] = INT_MAX;
  __syncthreads();
  cta_bitonic<NT>(sel, P);
  int base = 0;
  for (int c0 = 0; c0 < cnt; c0 += NT) {
    int i = c0 + threadIdx.x;
    int keep = (i < cnt) && (i == 0 || sel[i] != sel[i - 1]);
    int agg;
    const int pos = block_excl_sum<NT>(keep, &agg, scan);
    if (keep) out[base + pos] = sel[i];
    base += agg;
    __syncthreads();
  }
  return base;
}

// Acc: __device__ double coord(int pos, int c) const; __device__ int index(int pos) const
// part / split > 1 (ns > k): this CTA handles only the grid nodes [part G / split, (part+1) G / split),
// parks their nearest points in out[g] and returns -1; vol_finalize then sorts and de-duplicates.
template <int D, int NT, class Acc>
__device__ int cta_vol(const Acc& acc, int ns, int k, int* out, VolSmem<D, NT>& sm,
                       unsigned long long* evals = nullptr, int part = 0, int split = 1) {
  constexpr int TILE = vol_tile(D);
  constexpr int GPT = kVolGPT;
  const int tid = threadIdx.x;
  if (ns <= 0) return 0;
  if (ns <= k) {
    for (int i = tid; i < ns; i += NT) sm.u.out.sel[i] = acc.index(i);
    __syncthreads();
    return cta_sort_unique_write<NT>(sm.scan, sm.u.out.sel, ns, out);
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
  // stage S into shared memory when it fits one tile (one gather per point); then the tight
  // bounding box (exact: min/max) from shared or global memory
  const bool staged = ns <= TILE;
  if (staged) {
    for (int i = tid; i < ns; i += NT) {
      sm.u.tile.idx[i] = acc.index(i);
#pragma unroll
      for (int c = 0; c < D; c++) sm.u.tile.x[c][i] = acc.coord(i, c);
    }
    __syncthreads();
  }
  double lo[D], hi[D];
#pragma unroll
  for (int c = 0; c < D; c++) {
    lo[c] = DBL_MAX;
    hi[c] = -DBL_MAX;
  }
  for (int i = tid; i < ns; i += NT)
#pragma unroll
    for (int c = 0; c < D; c++) {
      const double v = staged ? sm.u.tile.x[c][i] : acc.coord(i, c);
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
  // thread -> (group of GPT grid nodes) x point slice: each point read from shared memory is
  // compared against GPT grid nodes.  Exact rule (C4): s < best, or s == best and a lower index,
  // written as a rare branch on s <= best.  s = d0^2 + d1^2 + ... with every operation rounded
  // separately (0 + d0^2 == d0^2 exactly, so the sum starts from the first square).
  const int g_lo = (int)((int64_t)G * part / split), g_hi = (int)((int64_t)G * (part + 1) / split);
  const int ngroups = (g_hi - g_lo + GPT - 1) / GPT;
  const int nslice = ngroups >= NT ? 1 : NT / ngroups;
  const int gstride = ngroups >= NT ? NT : ngroups;
  const int slice = ngroups >= NT ? 0 : tid / ngroups;
  const bool active = tid < gstride * nslice;
  for (int gb = 0; gb < ngroups; gb += gstride) {
    if (staged && gb > 0) {  // the combine of the previous group round reused the tile storage
      for (int i = tid; i < ns; i += NT) {
        sm.u.tile.idx[i] = acc.index(i);
#pragma unroll
        for (int c = 0; c < D; c++) sm.u.tile.x[c][i] = acc.coord(i, c);
      }
      __syncthreads();
    }
    const int grp = gb + (ngroups >= NT ? tid : tid % ngroups);
    const bool gact = active && grp < ngroups;
    double q[GPT][D];
    double best[GPT];
    int bi[GPT];
#pragma unroll
    for (int kk = 0; kk < GPT; kk++) {
      int rem = g_lo + grp * GPT + kk;
#pragma unroll
      for (int c = 0; c < D; c++) {
        const int j = rem % m;
        rem /= m;
        q[kk][c] = __dadd_rn(sm.lo[c], __dmul_rn((double)j + 0.5, sm.hstep[c]));
      }
      best[kk] = INFINITY;
      bi[kk] = INT_MAX;
    }
    for (int t0 = 0; t0 < ns; t0 += TILE) {
      const int tn = ns - t0 < TILE ? ns - t0 : TILE;
      if (!staged) {
        __syncthreads();
        for (int i = tid; i < tn; i += NT) {
          sm.u.tile.idx[i] = acc.index(t0 + i);
#pragma unroll
          for (int c = 0; c < D; c++) sm.u.tile.x[c][i] = acc.coord(t0 + i, c);
        }
        __syncthreads();
      }
      if (gact) {
        for (int p = slice; p < tn; p += nslice) {
          double x[D];
#pragma unroll
          for (int c = 0; c < D; c++) x[c] = sm.u.tile.x[c][p];
#pragma unroll
          for (int kk = 0; kk < GPT; kk++) {
            double df = __dsub_rn(x[0], q[kk][0]);
            double s = __dmul_rn(df, df);
#pragma unroll
            for (int c = 1; c < D; c++) {
              df = __dsub_rn(x[c], q[kk][c]);
              s = __dadd_rn(s, __dmul_rn(df, df));
            }
            if (s <= best[kk]) {
              const int ix = sm.u.tile.idx[p];
              if (s < best[kk] || ix < bi[kk]) {
                best[kk] = s;
                bi[kk] = ix;
              }
            }
          }
        }
      }
    }
    // combine the slices of every grid node (same exact rule); the tile is dead from here on
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GPT; kk++) {
      sm.u.out.bd[kk][tid] = best[kk];
      sm.u.out.bi[kk][tid] = bi[kk];
    }
    __syncthreads();
    if (gact && slice == 0) {
#pragma unroll
      for (int kk = 0; kk < GPT; kk++) {
        const int g = g_lo + grp * GPT + kk;
        if (g >= g_hi) break;
        double b = best[kk];
        int ib = bi[kk];
        for (int sl = 1; sl < nslice; sl++) {
          const int o = (grp - gb) + sl * gstride;
          const double s2 = sm.u.out.bd[kk][o];
          const int i2 = sm.u.out.bi[kk][o];
          if (s2 < b || (s2 == b && i2 < ib)) {
            b = s2;
            ib = i2;
          }
        }
        out[g] = ib;  // parked in the output slot (capacity k >= G) until all rounds are done
      }
    }
    __syncthreads();
  }
  if (evals && tid == 0) atomicAdd(evals, (unsigned long long)(g_hi - g_lo) * (unsigned long long)ns);
  if (split > 1) return -1;
  int* sel = sm.u.out.sel;
  for (int g = tid; g < G; g += NT) sel[g] = out[g];
  __syncthreads();
  return cta_sort_unique_write<NT>(sm.scan, sel, G, out);
}

}  // namespace h2
