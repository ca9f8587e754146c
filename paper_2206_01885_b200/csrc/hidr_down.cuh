// hidr_down.cuh -- selection boxes and the pruned exact top-down Vol of HiDR (a7; Algorithm 1
// lines 14-21; Vol as in vol.cuh, readings C2-C5).  Included by hidr.cu.
#pragma once
#include "vol.cuh"

namespace h2 {

// ------------------------------------------------------------------------------------------
// Selection boxes: the tight bounding box of every node's X_i^* (after its up level) and Y_i^*
// (after its down level): box[i * kBox + c] = lo_c, box[i * kBox + D + c] = hi_c and the selection
// size at box[i * kBox + 2D] (one load gives the top-down search a segment's box and count); an
// empty selection gets lo = +inf, hi = -inf.  The same pass packs the selection's coordinates per
// slot, coordinate-major, xyz[(i D + c) r + a], so the top-down search reads a segment's points
// with coalesced loads instead of an index load and D scattered loads per point.  One warp per
// node.  min / max are exact, so the union of the segment boxes is the bounding box of T_i bit for
// bit.  A float copy of each box, rounded outward (lo down, hi up, so it contains the double box),
// with the count, serves the pruning tests (boxf[i * kBoxF + ...], same layout).
// ------------------------------------------------------------------------------------------
constexpr int kBox = 2 * kMaxD + 2;
constexpr int kBoxF = 20;  // floats per node: 2 kMaxD + 1 rounded up to whole float4s

template <int D>
__global__ void sel_box_kernel(int base, int count, const int* __restrict__ cnt, const int* __restrict__ slots, int r,
                               const double* __restrict__ X, int64_t n, double* __restrict__ box,
                               float* __restrict__ boxf, double* __restrict__ xyz) {
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (w >= count) return;
  const int i = base + w;
  const int c = cnt[i];
  double lo[D], hi[D];
#pragma unroll
  for (int k = 0; k < D; k++) {
    lo[k] = INFINITY;
    hi[k] = -INFINITY;
  }
  for (int a = lane; a < c; a += 32) {
    const int idx = slots[(int64_t)i * r + a];
#pragma unroll
    for (int k = 0; k < D; k++) {
      const double v = X[k * n + idx];
      xyz[((int64_t)i * D + k) * r + a] = v;
      lo[k] = fmin(lo[k], v);
      hi[k] = fmax(hi[k], v);
    }
  }
#pragma unroll
  for (int k = 0; k < D; k++)
    for (int o = 16; o > 0; o >>= 1) {
      lo[k] = fmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < D; k++) {
      box[(int64_t)i * kBox + k] = lo[k];
      box[(int64_t)i * kBox + D + k] = hi[k];
    }
    box[(int64_t)i * kBox + 2 * D] = (double)c;
#pragma unroll
    for (int k = 0; k < D; k++) {
      boxf[(int64_t)i * kBoxF + k] = __double2float_rd(lo[k]);
      boxf[(int64_t)i * kBoxF + D + k] = __double2float_ru(hi[k]);
    }
    boxf[(int64_t)i * kBoxF + 2 * D] = (float)c;
  }
}

// ------------------------------------------------------------------------------------------
// Pruned exact top-down Vol.  Same result as the brute-force argmin of cta_vol, bit for bit.
// T_i is the union of segments -- Y_p^* and X_j^* for j in IL(i) -- whose bounding boxes are
// known.  The point distance s(x) = sum_c fl(fl(x_c - q_c)^2) (fp64, each operation rounded to
// nearest, c order) is within a factor (1 +- 11 * 2^-53) of the exact sum of squares.  The box
// tests run in fp32 with directed rounding on the outward-rounded float boxes and on q rounded
// down (qd) and up (qu):
//   lb(q,B) = rd(sum_c rd(g_c^2)) * (1 - 2^-20), g_c = max(0, rd(lo_c - qu_c), rd(qd_c - hi_c))
//   ub(q,B) = ru(sum_c ru(u_c^2)) * (1 + 2^-20), u_c = max(ru(hi_c - qd_c), ru(qu_c - lo_c))
// so lb <= s(x) <= ub for every x in B: each step only moves the bound away from the exact value,
// and the slack covers the fp64 rounding of s.  A segment is skipped only when lb > delta, delta
// an upper bound of the best s found so far (an evaluated s or the ub of a non-empty box), so the
// minimiser and every tie with it are always evaluated; ties go to the lowest index (reading C4)
// as in the brute-force kernel.  fp32 max / min / directed-rounding add and multiply are single
// instructions (the fp64 max is a compare plus selects).
// Segments are grouped 32 at a time (one per lane); the group boxes live in shared memory.
// One CTA per node, one warp per grid node.
// ------------------------------------------------------------------------------------------
constexpr int kDownThreads = 256;
constexpr int kDownWarps = kDownThreads / 32;
constexpr int kDownSmemMax = 96 * 1024;
constexpr float kLbSlack = 0x1.ffffep-1f;  // 1 - 2^-20
constexpr float kUbSlack = 0x1.00001p+0f;  // 1 + 2^-20

template <int D>
__device__ __forceinline__ float box_lb(const float* qd, const float* qu, const float* lo, const float* hi) {
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < D; c++) {
    const float g = fmaxf(fmaxf(__fsub_rd(lo[c], qu[c]), __fsub_rd(qd[c], hi[c])), 0.f);
    s = __fadd_rd(s, __fmul_rd(g, g));
  }
  return __fmul_rd(s, kLbSlack);
}

template <int D>
__device__ __forceinline__ float box_ub(const float* qd, const float* qu, const float* lo, const float* hi) {
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < D; c++) {
    const float u = fmaxf(__fsub_ru(hi[c], qd[c]), __fsub_ru(qu[c], lo[c]));
    s = __fadd_ru(s, __fmul_ru(u, u));
  }
  return __fmul_ru(s, kUbSlack);
}

// the warp minimum of v >= 0 (or +inf) in one instruction: non-negative floats order like their bits
__device__ __forceinline__ float warp_min_f(float v) {
  return __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(v)));
}

// An upper bound of the warp minimum of v >= 0 (distances) in ONE instruction: high words of
// non-negative doubles order like the doubles, so the least high word with an all-ones low word
// bounds the minimum from above (at most 2^-20 relative above it).  The pruning only needs
// delta >= the true best; the result is warp-uniform.  +inf stays +inf.
__device__ __forceinline__ double warp_min_ub(double v) {
  const unsigned hi = __reduce_min_sync(0xffffffffu, (unsigned)__double2hiint(v));
  return hi >= 0x7FF00000u ? INFINITY : __hiloint2double((int)hi, (int)0xFFFFFFFFu);
}

template <int D>
__global__ void __launch_bounds__(kDownThreads, D <= 2 ? 5 : 4) hidr_down_kernel(
    const double* __restrict__ X, int64_t n, int base, int r, const int* __restrict__ parent,
    const int64_t* __restrict__ il_off, const int* __restrict__ il_idx,
    const int* __restrict__ xs, const double* __restrict__ xbox, const double* __restrict__ ybox,
    const float* __restrict__ xboxf, const float* __restrict__ yboxf, int* ys_cnt,
    int* ys, const double* __restrict__ xs_xyz, const double* __restrict__ ys_xyz, unsigned long long* evals_alg,
    unsigned long long* evals_done) {
  // dynamic shared memory: during the search, the group boxes (float, outward: lo at
  // gbox[g*2D + c], hi at gbox[g*2D + D + c]) and the segments' node ids; before and after it,
  // the selection buffer `sel` (pass-through gather, final sort) aliased onto the same space
  extern __shared__ float gbox[];
  int* const sel = reinterpret_cast<int*>(gbox);
  __shared__ BlockScanSmem<kDownThreads> scan;
  __shared__ double wlo[D][kDownWarps], whi[D][kDownWarps];
  __shared__ long long wcnt[kDownWarps];
  __shared__ double s_lo[D], s_hi[D], s_h[D];
  __shared__ long long s_tot;
  __shared__ int s_fill;
  const int i = base + blockIdx.x, p = parent[i];
  const int64_t e0 = il_off[i];
  const int nseg = 1 + (int)(il_off[i + 1] - e0);
  const int ng = (nseg + 31) >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
  int* out = ys + (int64_t)i * r;
  const int* yp = ys + (int64_t)p * r;
  // segment s: 0 = Y_p^*, s >= 1 = X_j^* of the (s-1)-th entry of IL(i)
  int* const seg_nd = reinterpret_cast<int*>(gbox + ng * 2 * D);  // filled in phase 1
  auto seg_node = [&](int s) { return s == 0 ? p : il_idx[e0 + s - 1]; };
  auto seg_box = [&](int s, int nd) { return (s == 0 ? ybox : xbox) + (int64_t)nd * kBox; };
  auto seg_slots = [&](int s, int nd) { return s == 0 ? yp : xs + (int64_t)nd * r; };
  auto seg_xyz = [&](int s, int nd) { return (s == 0 ? ys_xyz : xs_xyz) + (int64_t)nd * r * D; };
  // a segment's float box and count in whole float4 loads
  auto load_segf = [&](int s, int& nd, float* blo, float* bhi) {
    nd = seg_nd[s];
    const float4* b = reinterpret_cast<const float4*>((s == 0 ? yboxf : xboxf) + (int64_t)nd * kBoxF);
    constexpr int NV = (2 * D + 1 + 3) / 4;
    float v[4 * NV];
#pragma unroll
    for (int k = 0; k < NV; k++) {
      const float4 t = __ldg(b + k);
      v[4 * k] = t.x;
      v[4 * k + 1] = t.y;
      v[4 * k + 2] = t.z;
      v[4 * k + 3] = t.w;
    }
#pragma unroll
    for (int c = 0; c < D; c++) {
      blo[c] = v[c];
      bhi[c] = v[D + c];
    }
    return (int)v[2 * D];
  };
  // a segment's box and count: lo, hi, |segment| (one contiguous run of 2D + 1 doubles)
  auto load_seg = [&](int s, int& nd, double* blo, double* bhi) {
    nd = seg_node(s);
    const double* b = seg_box(s, nd);
#pragma unroll
    for (int c = 0; c < D; c++) {
      blo[c] = b[c];
      bhi[c] = b[D + c];
    }
    return (int)b[2 * D];
  };

  // 1. group boxes, bbox(T_i), |T_i|
  double tlo[D], thi[D];
#pragma unroll
  for (int c = 0; c < D; c++) {
    tlo[c] = INFINITY;
    thi[c] = -INFINITY;
  }
  long long tcnt = 0;
  for (int g = warp; g < ng; g += kDownWarps) {
    const int s = g * 32 + lane;
    double blo[D], bhi[D];
#pragma unroll
    for (int c = 0; c < D; c++) {
      blo[c] = INFINITY;
      bhi[c] = -INFINITY;
    }
    int cnt = 0;
    if (s < nseg) {
      int nd;
      cnt = load_seg(s, nd, blo, bhi);
      seg_nd[s] = nd;
    }
#pragma unroll
    for (int c = 0; c < D; c++)
      for (int o = 16; o > 0; o >>= 1) {
        blo[c] = fmin(blo[c], __shfl_xor_sync(0xffffffffu, blo[c], o));
        bhi[c] = fmax(bhi[c], __shfl_xor_sync(0xffffffffu, bhi[c], o));
      }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < D; c++) {
        gbox[g * 2 * D + c] = __double2float_rd(blo[c]);
        gbox[g * 2 * D + D + c] = __double2float_ru(bhi[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < D; c++) {
      tlo[c] = fmin(tlo[c], blo[c]);
      thi[c] = fmax(thi[c], bhi[c]);
    }
    tcnt += cnt;
  }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < D; c++) {
      wlo[c][warp] = tlo[c];
      whi[c][warp] = thi[c];
    }
    wcnt[warp] = tcnt;
  }
  if (tid == 0) s_fill = 0;
  __syncthreads();
  if (tid == 0) {
    long long t = 0;
    for (int w = 0; w < kDownWarps; w++) t += wcnt[w];
    s_tot = t;
  }
  if (tid < D) {
    double a = INFINITY, b = -INFINITY;
    for (int w = 0; w < kDownWarps; w++) {
      a = fmin(a, wlo[tid][w]);
      b = fmax(b, whi[tid][w]);
    }
    s_lo[tid] = a;
    s_hi[tid] = b;
  }
  __syncthreads();
  const long long tot = s_tot;
  if (tot == 0) {
    if (tid == 0) ys_cnt[i] = 0;
    return;
  }
  if (tot <= r) {  // pass-through (reading C5): gather, sort, de-duplicate
    for (int s = tid; s < nseg; s += kDownThreads) {
      const int nd = seg_node(s);
      const int cnt = (int)seg_box(s, nd)[2 * D];
      if (cnt > 0) {
        const int pos = atomicAdd(&s_fill, cnt);
        const int* src = seg_slots(s, nd);
        for (int a = 0; a < cnt; a++) sel[pos + a] = src[a];
      }
    }
    __syncthreads();
    const int c = cta_sort_unique_write<kDownThreads>(scan, sel, (int)tot, out);
    if (tid == 0) ys_cnt[i] = c;
    return;
  }
  // 2. the grid: the same arithmetic as cta_vol
  int m = 1;
  for (;;) {
    long long pw = 1;
    for (int c = 0; c < D; c++) pw *= (m + 1);
    if (pw > r) break;
    m++;
  }
  int G = 1;
  for (int c = 0; c < D; c++) G *= m;
  if (tid < D) s_h[tid] = __ddiv_rn(__dsub_rn(s_hi[tid], s_lo[tid]), (double)m);
  __syncthreads();
  // 3. one warp per grid node
  unsigned long long done = 0;
  // grid nodes are taken dynamically (their search costs differ): a CTA-local counter
  if (tid == 0) s_fill = kDownWarps;
  __syncthreads();
  for (int g = warp; g < G;) {
    double q[D];
    {
      int rem = g;
#pragma unroll
      for (int c = 0; c < D; c++) {
        const int j = rem % m;
        rem /= m;
        q[c] = __dadd_rn(s_lo[c], __dmul_rn((double)j + 0.5, s_h[c]));
      }
    }
    float qd[D], qu[D];
#pragma unroll
    for (int c = 0; c < D; c++) {
      qd[c] = __double2float_rd(q[c]);
      qu[c] = __double2float_ru(q[c]);
    }
    // pass A: delta = min over the non-empty groups of ub; g0 = a group attaining it
    float ua = INFINITY;
    int g0 = -1;
    for (int gg = lane; gg < ng; gg += 32) {
      const float* b = gbox + gg * 2 * D;
      if (b[0] <= b[D]) {
        const float u = box_ub<D>(qd, qu, b, b + D);
        if (u < ua) {
          ua = u;
          g0 = gg;
        }
      }
    }
    {  // any attaining group will do; the highest-numbered lane's, uniform
      const float um = warp_min_f(ua);
      const unsigned who = __ballot_sync(0xffffffffu, ua == um && g0 >= 0);
      g0 = who ? __shfl_sync(0xffffffffu, g0, 31 - __clz(who)) : -1;
      ua = um;
    }
    double dl = (double)ua;
    double best = INFINITY;
    int bi = INT_MAX;
    auto eval_point = [&](const double* px, int idx) {  // px: coordinate c at px[c * r]
      double df = __dsub_rn(px[0], q[0]);
      double sd = __dmul_rn(df, df);
#pragma unroll
      for (int c = 1; c < D; c++) {
        df = __dsub_rn(px[c * r], q[c]);
        sd = __dadd_rn(sd, __dmul_rn(df, df));
      }
      if (sd < best || (sd == best && idx < bi)) {
        best = sd;
        bi = idx;
      }
    };
    // A group: lane t holds segment gg*32+t.  The passing segment with the least lower bound is
    // evaluated first (it tightens delta); the others that still pass are then evaluated together,
    // their points flattened over the lanes so every load of an iteration is independent.
    auto process_group = [&](int gg) {
      const int s = gg * 32 + lane;
      int nd = 0, cnt = 0;
      float lbs = INFINITY, u = INFINITY;
      if (s < nseg) {
        float blo[D], bhi[D];
        cnt = load_segf(s, nd, blo, bhi);
        if (cnt > 0) {
          lbs = box_lb<D>(qd, qu, blo, bhi);
          u = box_ub<D>(qd, qu, blo, bhi);
        }
      }
      dl = fmin(dl, (double)warp_min_f(u));
      bool pass = cnt > 0 && (double)lbs <= dl;
      const unsigned key = pass ? __float_as_uint(lbs) : 0xFFFFFFFFu;
      const unsigned kmin = __reduce_min_sync(0xffffffffu, key);
      if (kmin == 0xFFFFFFFFu) return;
      {
        const int t = __ffs(__ballot_sync(0xffffffffu, key == kmin)) - 1;
        const int ct = __shfl_sync(0xffffffffu, cnt, t);
        const int ndt = __shfl_sync(0xffffffffu, nd, t);
        const int* sl = seg_slots(gg * 32 + t, ndt);
        const double* px = seg_xyz(gg * 32 + t, ndt);
        for (int a = lane; a < ct; a += 32) eval_point(px + a, sl[a]);
        done += (unsigned long long)ct;
        dl = fmin(dl, warp_min_ub(best));
        if (lane == t) pass = false;
      }
      pass = pass && (double)lbs <= dl;
      // flattened remainder: inclusive prefix of the passing counts over the lanes
      int incl = pass ? cnt : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      const int excl = incl - (pass ? cnt : 0);
      for (int a0 = 0; a0 < total; a0 += 32) {
        const int a = a0 + lane;
        int t = 0;  // the lane whose range holds a: the number of lanes with incl <= a
#pragma unroll
        for (int bb = 16; bb > 0; bb >>= 1)
          if (__shfl_sync(0xffffffffu, incl, t + bb - 1) <= a) t += bb;
        const int off = a - __shfl_sync(0xffffffffu, excl, t & 31);
        const int ndt = __shfl_sync(0xffffffffu, nd, t & 31);
        if (a < total) eval_point(seg_xyz(gg * 32 + t, ndt) + off, seg_slots(gg * 32 + t, ndt)[off]);
      }
      done += (unsigned long long)total;
      dl = fmin(dl, warp_min_ub(best));
    };
    if (g0 >= 0) process_group(g0);
    // the other groups, best-first (least lower bound) within each run of 32
    for (int gg0 = 0; gg0 < ng; gg0 += 32) {
      const int gg = gg0 + lane;
      bool cand = false;
      float lbg = INFINITY;
      if (gg < ng && gg != g0) {
        const float* b = gbox + gg * 2 * D;
        lbg = box_lb<D>(qd, qu, b, b + D);
        cand = (double)lbg <= dl;
      }
      for (;;) {
        const unsigned key = (cand && (double)lbg <= dl) ? __float_as_uint(lbg) : 0xFFFFFFFFu;
        const unsigned kmin = __reduce_min_sync(0xffffffffu, key);
        if (kmin == 0xFFFFFFFFu) break;
        const int t = __ffs(__ballot_sync(0xffffffffu, key == kmin)) - 1;
        if (lane == t) cand = false;
        process_group(gg0 + t);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob < best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (lane == 0) out[g] = bi;  // parked in the output slot (capacity r >= G)
    int nxt = 0;
    if (lane == 0) nxt = atomicAdd(&s_fill, 1);
    g = __shfl_sync(0xffffffffu, nxt, 0);
  }
  if (lane == 0 && evals_done) atomicAdd(evals_done, done);
  if (tid == 0 && evals_alg) atomicAdd(evals_alg, (unsigned long long)G * (unsigned long long)tot);
  __syncthreads();
  for (int g = tid; g < G; g += kDownThreads) sel[g] = out[g];
  __syncthreads();
  const int c = cta_sort_unique_write<kDownThreads>(scan, sel, G, out);
  if (tid == 0) ys_cnt[i] = c;
}

}  // namespace h2
