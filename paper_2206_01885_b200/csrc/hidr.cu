// hidr.cu -- a6/a7: HiDR, Algorithm 1.
//
// Bottom-up (lines 7-13): S_i = X_i at a leaf, S_p = U_{c in ch(p)} X_c^*; X_i^* = Vol(S_i, r1).
// Top-down (lines 14-21): T_i = Y_p^* U (U_{j in IL(i)} X_j^*), Y_root^* = {} (reading D1); a node
// with empty IL still gets T_i = Y_p^* (D2); Y_i^* = Vol(T_i, r2) (empty if T_i is empty).
// Level-synchronous: per level, (1) a size kernel, (2) an exclusive scan, (3) a gather kernel
// writing every node's S_i / T_i index list contiguously (the union is disjoint by the tiling of
// the block partition, so it is a concatenation), (4) one CTA per node runs Vol.
#include <cmath>
#include <vector>

#include "hidr_down.cuh"

namespace h2 {

constexpr int kHidrThreads = 256;

// sizes of S_i (mode 0, bottom-up) or T_i (mode 1, top-down) for the nodes of one level
__global__ void hidr_sizes_kernel(int mode, int base, int count, const int* __restrict__ is_leaf,
                                  const int* __restrict__ nbegin, const int* __restrict__ nend,
                                  const int* __restrict__ first_child, const int* __restrict__ nchild,
                                  const int* __restrict__ parent, const int64_t* __restrict__ il_off,
                                  const int* __restrict__ il_idx, const int* __restrict__ xs_cnt,
                                  const int* __restrict__ ys_cnt, int64_t* sizes) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > count) return;
  if (t == count) {
    sizes[t] = 0;
    return;
  }
  int i = base + t;
  int64_t s = 0;
  if (mode == 0) {
    if (is_leaf[i]) s = nend[i] - nbegin[i];
    else
      for (int c = 0; c < nchild[i]; c++) s += xs_cnt[first_child[i] + c];
  } else {
    s = ys_cnt[parent[i]];
    for (int64_t e = il_off[i]; e < il_off[i + 1]; e++) s += xs_cnt[il_idx[e]];
  }
  sizes[t] = s;
}

// one CTA per node: concatenate the segments of S_i / T_i into list[off[t] ...]
__global__ void __launch_bounds__(kHidrThreads) hidr_gather_kernel(
    int mode, int base, const int64_t* __restrict__ off, const int* __restrict__ is_leaf,
    const int* __restrict__ nbegin, const int* __restrict__ first_child, const int* __restrict__ nchild,
    const int* __restrict__ parent, const int64_t* __restrict__ il_off, const int* __restrict__ il_idx,
    const int* __restrict__ xs_cnt, const int* __restrict__ xs, const int* __restrict__ ys_cnt,
    const int* __restrict__ ys, int r, int* list) {
  __shared__ BlockScanSmem<kHidrThreads> scan;
  const int t = blockIdx.x;
  const int i = base + t;
  int* out = list + off[t];
  const int64_t tot = off[t + 1] - off[t];
  if (mode == 0 && is_leaf[i]) {
    for (int64_t a = threadIdx.x; a < tot; a += blockDim.x) out[a] = nbegin[i] + (int)a;
    return;
  }
  // segments: mode 0 -> children's X^* slots; mode 1 -> Y_p^* slot then X_j^* for j in IL(i)
  int nseg = mode == 0 ? nchild[i] : 1 + (int)(il_off[i + 1] - il_off[i]);
  int pos0 = 0;
  for (int s0 = 0; s0 < nseg; s0 += kHidrThreads) {
    int sidx = s0 + threadIdx.x;
    const int* src = nullptr;
    int cnt = 0;
    if (sidx < nseg) {
      int node;
      if (mode == 0) {
        node = first_child[i] + sidx;
        src = xs + (int64_t)node * r;
        cnt = xs_cnt[node];
      } else if (sidx == 0) {
        node = parent[i];
        src = ys + (int64_t)node * r;
        cnt = ys_cnt[node];
      } else {
        node = il_idx[il_off[i] + sidx - 1];
        src = xs + (int64_t)node * r;
        cnt = xs_cnt[node];
      }
    }
    int agg;
    const int pos = block_excl_sum<kHidrThreads>(cnt, &agg, scan);
    for (int a = 0; a < cnt; a++) out[pos0 + pos + a] = src[a];
    pos0 += agg;
    __syncthreads();
  }
}

struct ListAcc {
  const double* X;
  int64_t n;
  const int* list;
  __device__ __forceinline__ double coord(int pos, int c) const { return X[c * n + list[pos]]; }
  __device__ __forceinline__ int index(int pos) const { return list[pos]; }
};

// `split` CTAs per node (levels with few nodes): each computes a share of the grid nodes; the
// selection is then sorted and de-duplicated by vol_finalize_kernel (one CTA per node).
template <int D>
__global__ void __launch_bounds__(kHidrThreads) hidr_vol_kernel(const double* __restrict__ X, int64_t n, int base,
                                                                 const int64_t* __restrict__ off,
                                                                 const int* __restrict__ list, int r, int* out_cnt,
                                                                 int* out_slots, unsigned long long* evals,
                                                                 int split) {
  __shared__ VolSmem<D, kHidrThreads> sm;
  const int t = blockIdx.x / split, part = blockIdx.x % split;
  const int i = base + t;
  ListAcc acc{X, n, list + off[t]};
  int ns = (int)(off[t + 1] - off[t]);
  if (ns <= r || split == 1) {  // pass-through or a single CTA: the whole selection here
    if (part != 0) return;
    const int c = cta_vol<D, kHidrThreads>(acc, ns, r, out_slots + (int64_t)i * r, sm, evals);
    if (threadIdx.x == 0) out_cnt[i] = c;
    return;
  }
  cta_vol<D, kHidrThreads>(acc, ns, r, out_slots + (int64_t)i * r, sm, evals, part, split);
}

// sort and de-duplicate the grid nodes' nearest points parked in the output slots (split levels)
template <int D>
__global__ void __launch_bounds__(kHidrThreads) vol_finalize_kernel(int base, const int64_t* __restrict__ off,
                                                                    int r, int* out_cnt, int* out_slots) {
  __shared__ int sel[kVolSelCap];
  __shared__ BlockScanSmem<kHidrThreads> scan;
  const int t = blockIdx.x, i = base + t;
  const int ns = (int)(off[t + 1] - off[t]);
  if (ns <= r) return;  // done by the pass-through
  int m = 1;
  for (;;) {
    long long p = 1;
    for (int c = 0; c < D; c++) p *= (m + 1);
    if (p > r) break;
    m++;
  }
  int G = 1;
  for (int c = 0; c < D; c++) G *= m;
  int* out = out_slots + (int64_t)i * r;
  for (int g = threadIdx.x; g < G; g += kHidrThreads) sel[g] = out[g];
  __syncthreads();
  const int c = cta_sort_unique_write<kHidrThreads>(scan, sel, G, out);
  if (threadIdx.x == 0) out_cnt[i] = c;
}

// Farthest point sampling (reading C6), one CTA per node over the gathered list:
// the first point is the one nearest the centre of the tight bounding box (the m = 1 case of Vol,
// the same arithmetic), then, r - 1 times, the point of largest C4 distance to the selected set
// (ties to the lowest index).  mind[] (global scratch, one double per candidate) holds each
// candidate's distance to the selected set, -1 once selected; every round fuses the update by the
// last pick with the next argmax.  O(r |S|) distances per node.
template <int D>
__device__ __forceinline__ double fps_dist(const double* __restrict__ X, int64_t n, int a, const double* z) {
  double df = __dsub_rn(X[a], z[0]);
  double s = __dmul_rn(df, df);
#pragma unroll
  for (int c = 1; c < D; c++) {
    df = __dsub_rn(X[(int64_t)c * n + a], z[c]);
    s = __dadd_rn(s, __dmul_rn(df, df));
  }
  return s;
}

template <int D>
__global__ void __launch_bounds__(kHidrThreads) hidr_fps_kernel(const double* __restrict__ X, int64_t n, int base,
                                                                 const int64_t* __restrict__ off,
                                                                 const int* __restrict__ list, int r, int* out_cnt,
                                                                 int* out_slots, double* mind_all,
                                                                 unsigned long long* evals) {
  constexpr int NT = kHidrThreads, NW = NT / 32;
  __shared__ int sel[kVolSelCap];
  __shared__ BlockScanSmem<NT> scan;
  __shared__ double wv[NW], s_lo[D], s_hi[D], z[D];
  __shared__ double wlo[D][NW], whi[D][NW];
  __shared__ int wi[NW], wp[NW];
  __shared__ int s_pick, s_pos;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = blockIdx.x, i = base + t;
  const int* L = list + off[t];
  const int ns = (int)(off[t + 1] - off[t]);
  double* mind = mind_all + off[t];
  int* out = out_slots + (int64_t)i * r;
  if (ns <= 0) {
    if (tid == 0) out_cnt[i] = 0;
    return;
  }
  if (ns <= r) {  // pass-through (reading C5)
    for (int a = tid; a < ns; a += NT) sel[a] = L[a];
    __syncthreads();
    const int c = cta_sort_unique_write<NT>(scan, sel, ns, out);
    if (tid == 0) out_cnt[i] = c;
    return;
  }
  // tight bounding box (exact min / max) and its centre, as Vol with m = 1
  {
    double lo[D], hi[D];
#pragma unroll
    for (int c = 0; c < D; c++) {
      lo[c] = DBL_MAX;
      hi[c] = -DBL_MAX;
    }
    for (int a = tid; a < ns; a += NT)
#pragma unroll
      for (int c = 0; c < D; c++) {
        const double v = X[(int64_t)c * n + L[a]];
        lo[c] = fmin(lo[c], v);
        hi[c] = fmax(hi[c], v);
      }
#pragma unroll
    for (int c = 0; c < D; c++)
      for (int o = 16; o > 0; o >>= 1) {
        lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
        hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
      }
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < D; c++) {
        wlo[c][warp] = lo[c];
        whi[c][warp] = hi[c];
      }
    __syncthreads();
    if (tid < D) {
      double a = DBL_MAX, b = -DBL_MAX;
      for (int w = 0; w < NW; w++) {
        a = fmin(a, wlo[tid][w]);
        b = fmax(b, whi[tid][w]);
      }
      s_lo[tid] = a;
      s_hi[tid] = b;
      z[tid] = __dadd_rn(a, __dmul_rn(0.5, __ddiv_rn(__dsub_rn(b, a), 1.0)));
    }
    __syncthreads();
  }
  // block arg-extremum of (value, index) over the candidates: sign = +1 max, -1 min; ties -> lowest
  // index; returns through s_pick / s_pos
  auto block_pick = [&](double v, int ix, int ps, double sign) {
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, ix, o), p2 = __shfl_xor_sync(0xffffffffu, ps, o);
      if (sign * v2 > sign * v || (v2 == v && i2 < ix)) {
        v = v2;
        ix = i2;
        ps = p2;
      }
    }
    if (lane == 0) {
      wv[warp] = v;
      wi[warp] = ix;
      wp[warp] = ps;
    }
    __syncthreads();
    if (tid == 0) {
      double bv = wv[0];
      int bi = wi[0], bp = wp[0];
      for (int w = 1; w < NW; w++)
        if (sign * wv[w] > sign * bv || (wv[w] == bv && wi[w] < bi)) {
          bv = wv[w];
          bi = wi[w];
          bp = wp[w];
        }
      s_pick = bi;
      s_pos = bp;
      wv[0] = bv;
    }
    __syncthreads();
  };
  // the seed: nearest to the box centre
  {
    double bv = INFINITY;
    int bix = INT_MAX, bps = -1;
    for (int a = tid; a < ns; a += NT) {
      const double dv = fps_dist<D>(X, n, L[a], z);
      if (dv < bv || (dv == bv && L[a] < bix)) {
        bv = dv;
        bix = L[a];
        bps = a;
      }
    }
    block_pick(bv, bix, bps, -1.0);
  }
  int cnt = 0;
  for (;;) {
    const int pick = s_pick, ppos = s_pos;
    if (tid == 0) {
      sel[cnt] = pick;
      mind[ppos] = -1.0;
    }
    if (tid < D) z[tid] = X[(int64_t)tid * n + pick];
    cnt++;
    __syncthreads();
    if (cnt >= r) break;
    // update by the last pick, then the farthest remaining candidate
    double bv = -1.0;
    int bix = INT_MAX, bps = -1;
    for (int a = tid; a < ns; a += NT) {
      double m = cnt == 1 ? (a == ppos ? -1.0 : INFINITY) : mind[a];
      if (m >= 0.0) {
        const double dv = fps_dist<D>(X, n, L[a], z);
        if (dv < m) m = dv;
        mind[a] = m;
        if (m > bv || (m == bv && L[a] < bix)) {
          bv = m;
          bix = L[a];
          bps = a;
        }
      } else if (cnt == 1) {
        mind[a] = -1.0;
      }
    }
    block_pick(bv, bix, bps, 1.0);
    if (wv[0] < 0.0) break;  // every candidate selected
  }
  if (evals && tid == 0) atomicAdd(evals, (unsigned long long)cnt * (unsigned long long)ns);
  __syncthreads();
  const int c = cta_sort_unique_write<NT>(scan, sel, cnt, out);
  if (tid == 0) out_cnt[i] = c;
}

// Surface-based DataReduct (reading C7, d = 2 or 3): reference points
// c + (gamma w) u on three ellipsoids about the centre c of the tight bounding box (w = its widths),
// the unit directions u and gammas from h->surf_dirs (computed once on the host with the C math
// library, as the oracle does); for every reference point the nearest candidate (C4, ties -> lowest
// index).  One CTA per node, a thread per reference point over all candidates (warp-uniform
// candidate loads).  O(r |S|) distances per node.
template <int D>
__global__ void __launch_bounds__(kHidrThreads) hidr_surface_kernel(const double* __restrict__ X, int64_t n,
                                                                     int base, const int64_t* __restrict__ off,
                                                                     const int* __restrict__ list, int r,
                                                                     const double* __restrict__ dirs, int nq,
                                                                     int* out_cnt, int* out_slots,
                                                                     unsigned long long* evals) {
  constexpr int NT = kHidrThreads, NW = NT / 32;
  __shared__ int sel[kVolSelCap];
  __shared__ BlockScanSmem<NT> scan;
  __shared__ double wlo[D][NW], whi[D][NW], s_cen[D], s_w[D];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = blockIdx.x, i = base + t;
  const int* L = list + off[t];
  const int ns = (int)(off[t + 1] - off[t]);
  int* out = out_slots + (int64_t)i * r;
  if (ns <= 0) {
    if (tid == 0) out_cnt[i] = 0;
    return;
  }
  if (ns <= r) {  // pass-through (reading C5)
    for (int a = tid; a < ns; a += NT) sel[a] = L[a];
    __syncthreads();
    const int c = cta_sort_unique_write<NT>(scan, sel, ns, out);
    if (tid == 0) out_cnt[i] = c;
    return;
  }
  {
    double lo[D], hi[D];
#pragma unroll
    for (int c = 0; c < D; c++) {
      lo[c] = DBL_MAX;
      hi[c] = -DBL_MAX;
    }
    for (int a = tid; a < ns; a += NT)
#pragma unroll
      for (int c = 0; c < D; c++) {
        const double v = X[(int64_t)c * n + L[a]];
        lo[c] = fmin(lo[c], v);
        hi[c] = fmax(hi[c], v);
      }
#pragma unroll
    for (int c = 0; c < D; c++)
      for (int o = 16; o > 0; o >>= 1) {
        lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
        hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
      }
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < D; c++) {
        wlo[c][warp] = lo[c];
        whi[c][warp] = hi[c];
      }
    __syncthreads();
    if (tid < D) {
      double a = DBL_MAX, b = -DBL_MAX;
      for (int w = 0; w < NW; w++) {
        a = fmin(a, wlo[tid][w]);
        b = fmax(b, whi[tid][w]);
      }
      const double w = __dsub_rn(b, a);
      s_w[tid] = w;
      s_cen[tid] = __dadd_rn(a, __dmul_rn(0.5, __ddiv_rn(w, 1.0)));
    }
    __syncthreads();
  }
  for (int g = tid; g < nq; g += NT) {
    const double* u = dirs + (int64_t)g * (D + 1);
    double q[D];
#pragma unroll
    for (int c = 0; c < D; c++) q[c] = __dadd_rn(s_cen[c], __dmul_rn(__dmul_rn(u[D], s_w[c]), u[c]));
    double best = INFINITY;
    int bi = INT_MAX;
    for (int a = 0; a < ns; a++) {
      const int idx = L[a];
      double df = __dsub_rn(X[idx], q[0]);
      double sd = __dmul_rn(df, df);
#pragma unroll
      for (int c = 1; c < D; c++) {
        df = __dsub_rn(X[(int64_t)c * n + idx], q[c]);
        sd = __dadd_rn(sd, __dmul_rn(df, df));
      }
      if (sd < best || (sd == best && idx < bi)) {
        best = sd;
        bi = idx;
      }
    }
    sel[g] = bi;
  }
  if (evals && tid == 0) atomicAdd(evals, (unsigned long long)nq * (unsigned long long)ns);
  __syncthreads();
  const int c = cta_sort_unique_write<NT>(scan, sel, nq, out);
  if (tid == 0) out_cnt[i] = c;
}

static void launch_fps(int d, unsigned grid, cudaStream_t s, const double* X, int64_t n, int base,
                       const int64_t* off, const int* list, int r, int* cnt, int* slots, double* mind,
                       unsigned long long* ev) {
  switch (d) {
#define H2_FPS_CASE(DD) \
  case DD:              \
    hidr_fps_kernel<DD><<<grid, kHidrThreads, 0, s>>>(X, n, base, off, list, r, cnt, slots, mind, ev); break;
    H2_FPS_CASE(1) H2_FPS_CASE(2) H2_FPS_CASE(3) H2_FPS_CASE(4)
    H2_FPS_CASE(5) H2_FPS_CASE(6) H2_FPS_CASE(7) H2_FPS_CASE(8)
#undef H2_FPS_CASE
  }
}

static void launch_vol(int d, unsigned count, cudaStream_t s, const double* X, int64_t n, int base,
                       const int64_t* off, const int* list, int r, int* cnt, int* slots, unsigned long long* ev) {
  // few nodes: several CTAs per node (at least 64 grid nodes each) so a level fills the machine
  long long G = 1;
  {
    int m = 1;
    for (;;) {
      long long p = 1;
      for (int c = 0; c < d; c++) p *= (m + 1);
      if (p > r) break;
      m++;
    }
    for (int c = 0; c < d; c++) G *= m;
  }
  int split = (int)((4LL * 148 + count - 1) / count);
  const int smax = (int)(G / 64);
  if (split > smax) split = smax;
  if (split < 1) split = 1;
  const unsigned grid = count * (unsigned)split;
  switch (d) {
#define H2_VOL_CASE(DD)                                                                                   \
  case DD:                                                                                                \
    hidr_vol_kernel<DD><<<grid, kHidrThreads, 0, s>>>(X, n, base, off, list, r, cnt, slots, ev, split);      \
    if (split > 1) vol_finalize_kernel<DD><<<count, kHidrThreads, 0, s>>>(base, off, r, cnt, slots);     \
    break;
    H2_VOL_CASE(1) H2_VOL_CASE(2) H2_VOL_CASE(3) H2_VOL_CASE(4)
    H2_VOL_CASE(5) H2_VOL_CASE(6) H2_VOL_CASE(7) H2_VOL_CASE(8)
#undef H2_VOL_CASE
  }
}

static void launch_sel_box(h2_handle* h, int base, int count, const int* cnt, const int* slots, double* box,
                           float* boxf, double* xyz) {
  const unsigned grid = (unsigned)((count * 32LL + 255) / 256);
  switch (h->d) {
#define H2_BOX_CASE(DD) \
  case DD: sel_box_kernel<DD><<<grid, 256, 0, h->stream>>>(base, count, cnt, slots, h->r, h->X, h->n, box, boxf, xyz); break;
    H2_BOX_CASE(1) H2_BOX_CASE(2) H2_BOX_CASE(3) H2_BOX_CASE(4)
    H2_BOX_CASE(5) H2_BOX_CASE(6) H2_BOX_CASE(7) H2_BOX_CASE(8)
#undef H2_BOX_CASE
  }
  H2_CHECK_LAUNCH();
  h->gpu_launches += 1;
}

// pruned down level; false when the group boxes do not fit shared memory (brute-force path then)
static bool hidr_down_level_pruned(h2_handle* h, int l, unsigned long long* ev, unsigned long long* ev_done) {
  const LevelRange lr = level_range(h, l);
  const int base = lr.begin, count = lr.end - lr.begin;
  const int ngmax = (h->csp + 1 + 31) / 32;
  // group boxes + the segments' node ids, or the aliased selection buffer (next power of two >= r)
  size_t sel_bytes = sizeof(int);
  while (sel_bytes < sizeof(int) * (size_t)h->r) sel_bytes <<= 1;
  size_t smem = sizeof(float) * 2 * h->d * (size_t)ngmax + sizeof(int) * (size_t)(h->csp + 1);
  if (smem < sel_bytes) smem = sel_bytes;
  if (smem > (size_t)kDownSmemMax) return false;
  cudaStream_t s = h->stream;
  switch (h->d) {
#define H2_DOWN_CASE(DD)                                                                                         \
  case DD: {                                                                                                     \
        H2_CUDA_TRY(cudaFuncSetAttribute(hidr_down_kernel<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                                       kDownSmemMax));                                                           \
    hidr_down_kernel<DD><<<count, kDownThreads, smem, s>>>(h->X, h->n, base, h->r, h->parent, h->il_off,           \
                                                           h->il_idx, h->xs, h->xbox, h->ybox, h->xboxf, h->yboxf,        \
                                                           h->ys_cnt, h->ys, h->xs_xyz, h->ys_xyz, ev, ev_done);                       \
  } break;
    H2_DOWN_CASE(1) H2_DOWN_CASE(2) H2_DOWN_CASE(3) H2_DOWN_CASE(4)
    H2_DOWN_CASE(5) H2_DOWN_CASE(6) H2_DOWN_CASE(7) H2_DOWN_CASE(8)
#undef H2_DOWN_CASE
  }
  H2_CHECK_LAUNCH();
  h->gpu_launches += 1;
  return true;
}

// `pre`: a buffer known to hold the level's gathered candidate lists (hidr_up's bound), so the
// level needs no host readback of their total and the up sweep is issued without a synchronisation
static void hidr_level(h2_handle* h, int mode, int l, unsigned long long* ev, int* pre = nullptr) {
  cudaStream_t s = h->stream;
  const LevelRange lr = level_range(h, l);
  int base = lr.begin, count = lr.end - lr.begin;
  if (count == 0) return;
  Scratch sizes(sizeof(int64_t) * (count + 1), s), off(sizeof(int64_t) * (count + 1), s);
  hidr_sizes_kernel<<<(count + 1 + 255) / 256, 256, 0, s>>>(mode, base, count, h->is_leaf, h->nbegin, h->nend,
                                                             h->first_child, h->nchild, h->parent, h->il_off,
                                                             h->il_idx, h->xs_cnt, h->ys_cnt, sizes.as<int64_t>());
  scan_excl_i64(sizes.as<int64_t>(), off.as<int64_t>(), count + 1, s);
  H2_CHECK_LAUNCH();
  const bool bounded = pre && h->reduct == H2_REDUCT_VOLUME;
  const int64_t total = bounded ? 0 : read1(off.as<int64_t>() + count, s);
  Scratch list;
  if (!bounded) list = Scratch(sizeof(int) * (total > 0 ? total : 1), s);
  int* const lp = bounded ? pre : list.as<int>();  // (`pre` is not owned: hidr_up releases it)
  hidr_gather_kernel<<<count, kHidrThreads, 0, s>>>(mode, base, off.as<int64_t>(), h->is_leaf, h->nbegin,
                                                    h->first_child, h->nchild, h->parent, h->il_off, h->il_idx,
                                                    h->xs_cnt, h->xs, h->ys_cnt, h->ys, h->r, lp);
  H2_CHECK_LAUNCH();
  if (h->reduct == H2_REDUCT_SURFACE) {
    const int nq = (int)(h->surf_dirs_n);
    if (h->d == 2)
      hidr_surface_kernel<2><<<count, kHidrThreads, 0, s>>>(h->X, h->n, base, off.as<int64_t>(), lp,
                                                            h->r, h->surf_dirs, nq, mode == 0 ? h->xs_cnt : h->ys_cnt,
                                                            mode == 0 ? h->xs : h->ys, ev);
    else
      hidr_surface_kernel<3><<<count, kHidrThreads, 0, s>>>(h->X, h->n, base, off.as<int64_t>(), lp,
                                                            h->r, h->surf_dirs, nq, mode == 0 ? h->xs_cnt : h->ys_cnt,
                                                            mode == 0 ? h->xs : h->ys, ev);
  } else if (h->reduct == H2_REDUCT_FPS) {
    Scratch mind(sizeof(double) * (total > 0 ? total : 1), s);
    launch_fps(h->d, count, s, h->X, h->n, base, off.as<int64_t>(), lp, h->r,
               mode == 0 ? h->xs_cnt : h->ys_cnt, mode == 0 ? h->xs : h->ys, mind.as<double>(), ev);
  } else {
    launch_vol(h->d, count, s, h->X, h->n, base, off.as<int64_t>(), lp, h->r,
               mode == 0 ? h->xs_cnt : h->ys_cnt, mode == 0 ? h->xs : h->ys, ev);
  }
  H2_CHECK_LAUNCH();
  h->gpu_launches += 3;
  if (mode == 0) launch_sel_box(h, base, count, h->xs_cnt, h->xs, h->xbox, h->xboxf, h->xs_xyz);
  else launch_sel_box(h, base, count, h->ys_cnt, h->ys, h->ybox, h->yboxf, h->ys_xyz);
}

// reading C7: the surface reference directions (unit vector + gamma per point, k = r points dealt
// round-robin to the three ellipsoids), computed with the host C math library
static void make_surface_dirs(h2_handle* h) {
  const int d = h->d, k = h->r;
  const double gam[3] = {0.3, 0.6, 1.2};
  std::vector<double> u;
  for (int e = 0; e < 3; e++) {
    const int M = k / 3 + (e < k % 3 ? 1 : 0);
    for (int j = 0; j < M; j++) {
      if (d == 2) {
        const double t = 2.0 * M_PI * (double)j / (double)M;
        u.push_back(cos(t));
        u.push_back(sin(t));
      } else {
        const double z = 1.0 - (2.0 * (double)j + 1.0) / (double)M;
        const double rho = sqrt(1.0 - z * z);
        const double f = (double)j * (M_PI * (3.0 - sqrt(5.0)));
        u.push_back(rho * cos(f));
        u.push_back(rho * sin(f));
        u.push_back(z);
      }
      u.push_back(gam[e]);
    }
  }
  h->surf_dirs_n = (int64_t)(u.size() / (size_t)(d + 1));
  h->surf_dirs = halloc<double>(h, u.size() > 0 ? u.size() : 1);
  if (!u.empty())
    H2_CUDA_TRY(cudaMemcpyAsync(h->surf_dirs, u.data(), sizeof(double) * u.size(), cudaMemcpyHostToDevice,
                                h->stream));
  H2_CUDA_TRY(cudaStreamSynchronize(h->stream));  // u is a host temporary
}

void hidr_up(h2_handle* h) {
  if (h->r > kVolSelCap) throw Error{H2_ERR_INVALID_ARG, "r exceeds the supported budget 4096"};
  if (h->reduct == H2_REDUCT_SURFACE) make_surface_dirs(h);
  h->xs_cnt = halloc<int>(h, h->nnodes);
  h->xs = halloc<int>(h, (size_t)h->nnodes * h->r);
  h->ys_cnt = halloc<int>(h, h->nnodes);
  h->ys = halloc<int>(h, (size_t)h->nnodes * h->r);
  h->xbox = halloc<double>(h, (size_t)h->nnodes * kBox);
  h->ybox = halloc<double>(h, (size_t)h->nnodes * kBox);
  h->xboxf = halloc<float>(h, (size_t)h->nnodes * kBoxF);
  h->yboxf = halloc<float>(h, (size_t)h->nnodes * kBoxF);
  h->xs_xyz = halloc<double>(h, (size_t)h->nnodes * h->r * h->d);
  h->ys_xyz = halloc<double>(h, (size_t)h->nnodes * h->r * h->d);
  H2_CUDA_TRY(cudaMemsetAsync(h->ys_cnt, 0, sizeof(int) * h->nnodes, h->stream));
  Scratch ev(sizeof(unsigned long long), h->stream);
  H2_CUDA_TRY(cudaMemsetAsync(ev.p, 0, sizeof(unsigned long long), h->stream));
  // The up sweep's candidate sets S_i: a leaf's points or the children's X_c^* (<= r each), so a
  // level's lists hold at most n + count * (2^d) * r indices.  One buffer of the largest bound
  // serves every level (stream-ordered), when it is modest; else each level reads its total back.
  int64_t bound = 0;
  for (int l = 0; l <= h->depth; l++) {
    const LevelRange lr = level_range(h, l);
    const int64_t ch = h->d >= 8 ? 256 : (1LL << h->d);
    const int64_t b = (int64_t)h->n + (int64_t)(lr.end - lr.begin) * ch * h->r;
    bound = b > bound ? b : bound;
  }
  const bool use_bound = h->reduct == H2_REDUCT_VOLUME && bound * (int64_t)sizeof(int) <= ((int64_t)512 << 20);
  Scratch pre(use_bound ? sizeof(int) * (size_t)bound : 0, h->stream);
  for (int l = h->depth; l >= 0; l--) {
    hidr_level(h, 0, l, ev.as<unsigned long long>(), use_bound ? pre.as<int>() : nullptr);
    if (h->nranks > 1 && l == h->cut) {
      // sharded: every rank's X^* of the levels >= cut, then their boxes (hidr_down.cuh)
      exchange_slots(h, h->xs_cnt, h->xs);
      for (int m = h->cut; m <= h->depth; m++) {
        const int b = h->lvl_start[m], c = h->lvl_start[m + 1] - b;
        if (c > 0) launch_sel_box(h, b, c, h->xs_cnt, h->xs, h->xbox, h->xboxf, h->xs_xyz);
      }
    }
  }
  defer_stat(h, kStatHidrUp, ev.p, sizeof(unsigned long long));
}

void hidr_down(h2_handle* h) {
  Scratch ev(sizeof(unsigned long long), h->stream);
  H2_CUDA_TRY(cudaMemsetAsync(ev.p, 0, sizeof(unsigned long long), h->stream));
  Scratch evd(sizeof(unsigned long long), h->stream);
  H2_CUDA_TRY(cudaMemsetAsync(evd.p, 0, sizeof(unsigned long long), h->stream));
  // the root's Y^* is empty (reading D1): its box is the empty box
  launch_sel_box(h, 0, 1, h->ys_cnt, h->ys, h->ybox, h->yboxf, h->ys_xyz);
  for (int l = 1; l <= h->depth; l++) {
    const LevelRange lr = level_range(h, l);
    const int base = lr.begin, count = lr.end - lr.begin;
    if (count == 0) continue;
    if (h->hidr_prune && h->reduct == H2_REDUCT_VOLUME &&
        hidr_down_level_pruned(h, l, ev.as<unsigned long long>(), evd.as<unsigned long long>()))
      launch_sel_box(h, base, count, h->ys_cnt, h->ys, h->ybox, h->yboxf, h->ys_xyz);
    else
      hidr_level(h, 1, l, ev.as<unsigned long long>());
  }
  defer_stat(h, kStatHidrDown, ev.p, sizeof(unsigned long long));
  defer_stat(h, kStatHidrDone, evd.p, sizeof(unsigned long long));
}

}  // namespace h2
