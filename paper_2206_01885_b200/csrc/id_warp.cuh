// id_warp.cuh -- a8 for levels with many small nodes: ONE WARP per node, no CTA barrier.
//
// The ID of one node (Algorithm 2 lines 10-12; getBasis = CPQR of A^T = K(Xbar_i, Y_i^*)^T, Eqs.(4.1)-
// (4.4) P:570-604; readings F1-F3) is a chain of k dependent pivot steps.  A CTA per node spends
// every step in CTA barriers and cross-warp reductions; with thousands of nodes per level it is
// faster to give each node one warp and run many nodes per SM: a lane owns the columns
// lane, lane + 32, ... (its residual norms and positions in registers), every step is one warp
// shuffle argmax, a broadcast read of the pivot column, and each lane's update of its own columns
// (the Householder dot, update and recomputed residual norm in one pass over the column).
// Same algorithm and rules as cta_cpqr (cpqr.cuh): largest residual norm, ties to the lowest
// position (a position map instead of column swaps), stop when the norm < tol |R11|, row t joins R
// and leaves the residual norm.  A^T lives in the warp's shared-memory slot, column-major with an
// odd leading dimension (the 32 lanes' rows fall in distinct bank pairs).
#pragma once
#include <climits>

#include "h2_internal.cuh"

namespace h2 {

constexpr int kIdWarpMaxCols = 8;    // columns per lane: nx <= 256
constexpr int kIdWarpPerCta = 2;     // warps (nodes) per CTA
constexpr int kIdWarpMaxBytes = 110 * 1024;  // a node's slot (two per CTA within 227 KB)
__host__ __device__ __forceinline__ int id_warp_ld(int ny) { return ny | 1; }
// a node's shared-memory slot: A^T (ld x nx) + Xbar (nx ints) + the position map (nx ints)
__host__ __device__ __forceinline__ int64_t id_warp_bytes(int ny, int nx) {
  return 8LL * id_warp_ld(ny) * nx + 8LL * nx + 16;
}

template <int D>
__global__ void __launch_bounds__(32 * kIdWarpPerCta) id_kernel_warp(
    int base, const int* __restrict__ list, int nlist, int slot_doubles, int kid, double p2, double tol,
    const double* __restrict__ Xf, const double* __restrict__ X, int64_t n, int r, const int* __restrict__ is_leaf,
    const int* __restrict__ nbegin, const int* __restrict__ first_child, const int* __restrict__ nchild,
    const int* __restrict__ ys_cnt, const int* __restrict__ ys, const int* __restrict__ xbar_n,
    const int64_t* __restrict__ uoff, double* U, int* kout, int* sk, unsigned long long* evals) {
  constexpr unsigned kFull = 0xffffffffu;
  extern __shared__ double sh[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int li = blockIdx.x * kIdWarpPerCta + w;
  if (li >= nlist) return;  // (warp-uniform)
  const int t_ = list[li];
  const int i = base + t_;
  const int nx = xbar_n[i], ny = ys_cnt[i];
  const int ld = id_warp_ld(ny);
  double* M = sh + (int64_t)w * slot_doubles;
  int* xb = reinterpret_cast<int*>(M + (int64_t)ld * nx);
  int* col_at = xb + nx;
  // Xbar_i: the leaf's points or the children's skeletons in child order
  if (is_leaf[i]) {
    for (int b = lane; b < nx; b += 32) xb[b] = nbegin[i] + b;
  } else {
    int o = 0;
    for (int c = 0; c < nchild[i]; c++) {
      const int ch = first_child[i] + c;
      const int kc = kout[ch];
      for (int a = lane; a < kc; a += 32) xb[o + a] = sk[(int64_t)ch * r + a];
      o += kc;
    }
  }
  for (int b = lane; b < nx; b += 32) col_at[b] = b;
  __syncwarp();
  // A^T column b = K(Xbar[b], Y^*[:]) by its owner lane (the column point in registers, the rows'
  // points broadcast), and the column's norm
  const int* yv = ys + (int64_t)i * r;
  double nrm[kIdWarpMaxCols];
  int pos[kIdWarpMaxCols];
#pragma unroll
  for (int j = 0; j < kIdWarpMaxCols; j++) {
    const int c = lane + 32 * j;
    nrm[j] = -1.0;
    pos[j] = INT_MAX;
    if (c < nx) {
      double xr[D];
#pragma unroll
      for (int q = 0; q < D; q++) xr[q] = Xf[q * n + xb[c]];
      double* col = M + (int64_t)ld * c;
      double s0 = 0.0, s1 = 0.0;
      for (int a = 0; a < ny; a++) {
        const int ya = yv[a];
        double sq = 0.0, dt = 0.0;
#pragma unroll
        for (int q = 0; q < D; q++) {
          const double yc = X[q * n + ya], df = xr[q] - yc;
          sq = fma(df, df, sq);
          dt = fma(xr[q], yc, dt);
        }
        const double v = kid == H2_KERNEL_COSDOT ? kernel_cosdot(dt) : kernel_s(kid, p2, sq);
        col[a] = v;
        if (a & 1) s1 += v * v;
        else s0 += v * v;
      }
      nrm[j] = s0 + s1;
      pos[j] = c;
    }
  }
  __syncwarp();
  const int kmax = ny < nx ? ny : nx;
  double r11 = 0.0;
  int k = 0;
  for (int t = 0; t < kmax; t++) {
    // pivot: the largest residual norm among positions >= t, ties to the lowest position
    double bv = -1.0;
    int bp = INT_MAX, bc = -1;
#pragma unroll
    for (int j = 0; j < kIdWarpMaxCols; j++)
      if (pos[j] != INT_MAX && pos[j] >= t && (nrm[j] > bv || (nrm[j] == bv && pos[j] < bp))) {
        bv = nrm[j];
        bp = pos[j];
        bc = lane + 32 * j;
      }
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(kFull, bv, o);
      const int p2_ = __shfl_xor_sync(kFull, bp, o), c2 = __shfl_xor_sync(kFull, bc, o);
      if (v2 > bv || (v2 == bv && p2_ < bp)) {
        bv = v2;
        bp = p2_;
        bc = c2;
      }
    }
    const double nrm_p = bv > 0.0 ? sqrt(bv) : 0.0;
    if (t == 0) {
      r11 = nrm_p;
      if (r11 == 0.0) break;
    }
    if (bc < 0 || nrm_p < tol * r11) break;
    const int p = bc, posp = bp;
    const int ct = col_at[t];
    const double* colp = M + (int64_t)ld * p;
    const double x0 = colp[t];
    const double alpha = x0 >= 0.0 ? -nrm_p : nrm_p;
    const double vhead = x0 - alpha;
    const double vtv = vhead * vhead + (bv - x0 * x0);  // |v|^2: row t replaced, rows > t unchanged
    // positions: the pivot moves to t, the column at t to the pivot's old position
#pragma unroll
    for (int j = 0; j < kIdWarpMaxCols; j++) {
      const int c = lane + 32 * j;
      if (c == p) pos[j] = t;
      else if (c == ct) pos[j] = posp;
    }
    // each lane: its columns at positions > t -- reflector and recomputed residual norm
#pragma unroll
    for (int j = 0; j < kIdWarpMaxCols; j++) {
      if (pos[j] == INT_MAX || pos[j] <= t) continue;
      double* col = M + (int64_t)ld * (lane + 32 * j);
      double nn = 0.0;
      if (vtv > 0.0) {
        double s0 = vhead * col[t], s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int a = t + 1;
        for (; a + 3 < ny; a += 4) {
          s0 += colp[a] * col[a];
          s1 += colp[a + 1] * col[a + 1];
          s2 += colp[a + 2] * col[a + 2];
          s3 += colp[a + 3] * col[a + 3];
        }
        for (; a < ny; a++) s0 += colp[a] * col[a];
        const double f = 2.0 * ((s0 + s1) + (s2 + s3)) / vtv;
        col[t] -= f * vhead;
        double n1 = 0.0;
        a = t + 1;
        for (; a + 1 < ny; a += 2) {
          const double u0 = col[a] - f * colp[a], u1 = col[a + 1] - f * colp[a + 1];
          col[a] = u0;
          col[a + 1] = u1;
          nn += u0 * u0;
          n1 += u1 * u1;
        }
        for (; a < ny; a++) {
          const double u0 = col[a] - f * colp[a];
          col[a] = u0;
          nn += u0 * u0;
        }
        nn += n1;
      } else {
        for (int a = t + 1; a < ny; a++) nn += col[a] * col[a];
      }
      nrm[j] = nn;
    }
    __syncwarp();  // every lane has read the pivot column and col_at[t]
    if (lane == 0) {
      M[t + (int64_t)ld * p] = alpha;  // R[t, t]; the pivot's rows below t are never read again
      col_at[posp] = ct;
      col_at[t] = p;
    }
    __syncwarp();
    k = t + 1;
  }
  __syncwarp();
  // T = R11^{-1} R12 on the own non-skeleton columns (positions >= k), R11 through the map
#pragma unroll
  for (int j = 0; j < kIdWarpMaxCols; j++) {
    if (pos[j] == INT_MAX || pos[j] < k) continue;
    double* col = M + (int64_t)ld * (lane + 32 * j);
    for (int a = k - 1; a >= 0; a--) {
      double s = col[a];
      for (int l = a + 1; l < k; l++) s -= M[a + (int64_t)ld * col_at[l]] * col[l];
      col[a] = s / M[a + (int64_t)ld * col_at[a]];
    }
  }
  __syncwarp();
  // outputs: k, the skeleton (pivot order), U (nx x k column-major): identity on the skeleton rows
  double* Ui = U + uoff[t_];
  for (int a = lane; a < k; a += 32) sk[(int64_t)i * r + a] = xb[col_at[a]];
#pragma unroll
  for (int j = 0; j < kIdWarpMaxCols; j++) {
    const int c = lane + 32 * j;
    if (pos[j] == INT_MAX) continue;
    const bool skel = pos[j] < k;
    for (int tt = 0; tt < k; tt++)
      Ui[c + (int64_t)nx * tt] = skel ? (pos[j] == tt ? 1.0 : 0.0) : M[tt + (int64_t)ld * c];
  }
  if (lane == 0) {
    kout[i] = k;
    atomicAdd(evals, (unsigned long long)nx * ny);
  }
}

}  // namespace h2
