// cpqr_panel.cuh -- panel-blocked column-pivoted Householder QR for the interpolative decomposition
// (getBasis, Eqs.(4.1)-(4.4); readings F1-F3), one CTA per node.
//
// Same pivot rule and stop rule as cta_cpqr (cpqr.cuh): at step t the pivot is the column of largest
// residual norm (ties -> lowest current position), and the factorisation stops when that norm is
// < tol * |R11|.  What changes is how the trailing matrix is kept up to date (the delayed update of
// LAPACK's dlaqps):
//   * within a panel of NB steps the trailing columns are NOT rewritten: A = A0 - V F^T, with V the
//     panel's Householder vectors (stored in place below the pivots' diagonals) and F (ncols x NB,
//     shared memory, Fs[l * nx + c]);
//   * per step: the pivot column is brought up to date (a_p = a0_p - V F_p^T), its reflector built,
//     and one GEMV pass over the trailing columns gives the new F column
//     f_j = tau (A0^T v_j - F (V^T v_j)) and the final R row t = A0[t,:] - V[t,:] F^T; the residual
//     norms are downdated (nrm -= R_tc^2);
//   * at the end of the panel one pass applies A -= V F^T to the rows below it and recomputes every
//     residual norm exactly.  A panel also ends early when a downdated norm lost more than ~8
//     digits against its last exact value (dgeqp3's guard), so the downdated norms used for the
//     pivot choice and the stop test keep ~1e-8 relative accuracy or better.
// Per step that is one read of the trailing block (plus a full read/write once per panel) instead
// of the unblocked algorithm's read + read/write, and three CTA barriers instead of seven.  Columns
// never move: a position map (col_at / pos) replaces the swaps, with the tie rule on positions kept.
//
// Threads: groups of G (a power of two <= 32) threads per column; group q owns the physical
// columns q, q + NT/G, ... (at most RMAX of them); within a group thread g takes rows g, g + G, ...
// M is column-major with leading dimension ld (>= ny; ld = G mod 16 makes the shared-memory
// accesses of a warp conflict-free).
//
// On return (k = rank): col_at[l] = the physical column at pivot position l; for l < k, column
// col_at[l] rows 0..l hold R11[0:l+1, l]; for positions c >= k, column col_at[c] rows 0..k-1 hold
// T[:, c] = R11^{-1} R12 (so column col_at[c] ~= sum_t T[t, c] column col_at[t]).
#pragma once
#include <climits>

#include "h2_internal.cuh"

namespace h2 {

template <int NT, int NB>
struct PanelSmem {
  double wval[NT / 32];   // per-warp candidate: residual norm^2 (-1: none)
  double tot[NB + 1];
  int wpos[NT / 32], wcol[NT / 32];
  double xt;  // x_t of the pivot column (row t)
  int vcol[NB];  // physical columns of the panel's reflectors
  int flag;   // a downdated norm tripped the guard: end the panel
};

// leading dimension for group size G: the smallest ld >= ny that is an odd multiple of G for G <= 8
// (the G-row segments of the 32 / G columns a warp reads then fall in distinct shared-memory bank
// pairs: every bank serves exactly two of the warp's 32 doubles); any ld for G >= 16
__host__ __device__ __forceinline__ int panel_ld(int ny, int G) {
  if (G >= 16) return ny;
  int ld = (ny + G - 1) / G;
  if ((ld & 1) == 0) ld++;
  return ld * G;
}
// rows of padding panel_ld adds: < 2G (G <= 8)
// group size: the largest power of two <= 32 with nx * G <= NT (1 when nx > NT)
__host__ __device__ __forceinline__ int panel_group(int nx, int NT) {
  int G = 1;
  while (G < 32 && (int64_t)nx * (2 * G) <= NT) G *= 2;
  return G;
}

constexpr double kPanelGuard = 1e-8;  // downdated / exact norm^2 below this: recompute (dgeqp3: sqrt(eps))

// Fs: NB * nx doubles of scratch (shared memory; the delayed-update coefficients F[c, l] at Fs[l*nx+c])
template <int NT, int NB, int RMAX>
__device__ int cta_cpqr_panel(double* __restrict__ M, const int ld, const int ny, const int nx, const double tol,
                              const int G, int* __restrict__ col_at, double* __restrict__ Fs,
                              PanelSmem<NT, NB>& sm) {
  constexpr int NW = NT / 32;
  constexpr unsigned kFull = 0xffffffffu;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = tid / G, g = tid - grp * G;
  const int ngrp = NT / G;
  double nrm[RMAX], ref[RMAX];
  int pos[RMAX];
  for (int b = tid; b < nx; b += NT) col_at[b] = b;
  // exact initial norms
#pragma unroll
  for (int r = 0; r < RMAX; r++) {
    const int c = grp + r * ngrp;
    const bool act = c < nx;
    double s = 0.0, s1 = 0.0;
    if (act) {
      const double* col = M + (int64_t)ld * c;
      int i = g;
      for (; i + G < ny; i += 2 * G) {
        s += col[i] * col[i];
        s1 += col[i + G] * col[i + G];
      }
      for (; i < ny; i += G) s += col[i] * col[i];
    }
    s += s1;
    for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    nrm[r] = act ? s : -1.0;
    ref[r] = s;
    pos[r] = act ? c : INT_MAX;
  }
  // publishes this warp's candidate: the largest residual norm among positions >= tmin, ties to
  // the lowest position
  auto publish = [&](int tmin) {
    double bv = -1.0;
    int bp = INT_MAX, bc = -1;
#pragma unroll
    for (int r = 0; r < RMAX; r++)
      if (pos[r] >= tmin && pos[r] != INT_MAX && (nrm[r] > bv || (nrm[r] == bv && pos[r] < bp))) {
        bv = nrm[r];
        bp = pos[r];
        bc = grp + r * ngrp;
      }
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(kFull, bv, o);
      const int p2 = __shfl_xor_sync(kFull, bp, o);
      const int c2 = __shfl_xor_sync(kFull, bc, o);
      if (v2 > bv || (v2 == bv && p2 < bp)) {
        bv = v2;
        bp = p2;
        bc = c2;
      }
    }
    if (lane == 0) {
      sm.wval[warp] = bv;
      sm.wpos[warp] = bp;
      sm.wcol[warp] = bc;
    }
  };
  publish(0);
  if (tid == 0) sm.flag = 0;
  __syncthreads();
  const int kmax = ny < nx ? ny : nx;
  double r11 = 0.0;
  int k = 0, j = 0;
  const int* vcol = sm.vcol;
  for (int t = 0; t < kmax; t++) {
    // ---- end of a panel: A[t:, trailing] -= V F^T, exact residual norms --------------------------
    if (j == NB || (j > 0 && sm.flag)) {
#pragma unroll
      for (int r = 0; r < RMAX; r++) {
        const int c = grp + r * ngrp;
        const bool act = pos[r] >= t && pos[r] != INT_MAX;
        if (!__any_sync(kFull, act)) continue;
        double s = 0.0;
        if (act) {
          double* col = M + (int64_t)ld * c;
          double fc[NB];
          int vc[NB];
#pragma unroll
          for (int l = 0; l < NB; l++) {
            fc[l] = l < j ? Fs[l * nx + c] : 0.0;
            vc[l] = l < j ? vcol[l] : 0;
          }
          double s1 = 0.0;
          int i = t + g;
          for (; i + G < ny; i += 2 * G) {
            double a = col[i], b = col[i + G];
#pragma unroll
            for (int l = 0; l < NB; l++)
              if (l < j) {
                const double* vl = M + (int64_t)ld * vc[l];
                a -= vl[i] * fc[l];
                b -= vl[i + G] * fc[l];
              }
            col[i] = a;
            col[i + G] = b;
            s += a * a;
            s1 += b * b;
          }
          for (; i < ny; i += G) {
            double a = col[i];
#pragma unroll
            for (int l = 0; l < NB; l++)
              if (l < j) a -= M[i + (int64_t)ld * vc[l]] * fc[l];
            col[i] = a;
            s += a * a;
          }
          s += s1;
        }
        for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
        if (act) {
          nrm[r] = s;
          ref[r] = s;
        }
      }
      j = 0;
      publish(t);
      __syncthreads();
      if (tid == 0) sm.flag = 0;  // every thread has read the flag (before the barrier above)
    }
    // ---- the pivot: the best of the warps' candidates ---------------------------------------------
    double bv = -1.0;
    int bp = INT_MAX, bc = -1;
#pragma unroll
    for (int w = 0; w < NW; w++) {
      const double v = sm.wval[w];
      const int p = sm.wpos[w];
      if (v > bv || (v == bv && p < bp)) {
        bv = v;
        bp = p;
        bc = sm.wcol[w];
      }
    }
    const double nrm_p = bv > 0.0 ? sqrt(bv) : 0.0;
    if (t == 0) {
      r11 = nrm_p;
      if (r11 == 0.0) break;
    }
    if (bc < 0 || nrm_p < tol * r11) break;
    const int p = bc, posp = bp;
    const int ct = col_at[t];  // the column at position t moves to the pivot's position
    const double* fpp = Fs + p;  // F[p, l] at fpp[l * nx]
    // ---- the pivot column brought up to date: x = a0_p - V F_p^T (rows >= t), then (one warp per
    // quantity, in parallel) |x|^2 and the dots (V^T x)_l ------------------------------------------
    double* colp = M + (int64_t)ld * p;
    for (int i = t + tid; i < ny; i += NT) {
      double x0 = colp[i], x1 = 0.0;
#pragma unroll
      for (int l = 0; l < NB; l += 2) {
        if (l < j) x0 -= M[i + (int64_t)ld * vcol[l]] * fpp[l * nx];
        if (l + 1 < j) x1 -= M[i + (int64_t)ld * vcol[l + 1]] * fpp[(l + 1) * nx];
      }
      const double x = x0 + x1;
      colp[i] = x;
      if (i == t) sm.xt = x;
    }
    __syncthreads();
    for (int qq = warp; qq <= j; qq += NW) {  // quantity q < j: (V^T x)_q over rows >= t; q = j: |x|^2
      const double* a = qq == j ? colp : M + (int64_t)ld * vcol[qq];
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int i = t + lane;
      for (; i + 96 < ny; i += 128) {
        s0 += a[i] * colp[i];
        s1 += a[i + 32] * colp[i + 32];
        s2 += a[i + 64] * colp[i + 64];
        s3 += a[i + 96] * colp[i + 96];
      }
      for (; i < ny; i += 32) s0 += a[i] * colp[i];
      double sq = (s0 + s1) + (s2 + s3);
      for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(kFull, sq, o);
      if (lane == 0) sm.tot[qq == j ? NB : qq] = sq;
    }
    __syncthreads();
    // ---- the reflector H = I - tau v v^T, v = x - alpha e_t ---------------------------------------
    const double n2 = sm.tot[NB], xt = sm.xt;
    const double alpha = xt >= 0.0 ? -sqrt(n2) : sqrt(n2);
    const double vhead = xt - alpha;
    const double vtv = n2 - xt * xt + vhead * vhead;
    const double tau = vtv > 0.0 ? 2.0 / vtv : 0.0;
    // positions: the pivot moves to t, the column at t to the pivot's old position
#pragma unroll
    for (int r = 0; r < RMAX; r++) {
      const int c = grp + r * ngrp;
      if (c == p) pos[r] = t;
      else if (c == ct) pos[r] = posp;
    }
    // ---- one pass over the trailing columns: F column j, the final R row t, downdated norms -------
    bool trip = false;
#pragma unroll
    for (int r = 0; r < RMAX; r++) {
      const int c = grp + r * ngrp;
      const bool act = pos[r] > t && pos[r] != INT_MAX;
      if (!__any_sync(kFull, act)) continue;
      double s = 0.0, at = 0.0;
      if (act) {
        const double* col = M + (int64_t)ld * c;
        at = col[t];
        double s1 = 0.0, s2 = 0.0, s3 = 0.0;
        s = g == 0 ? vhead * at : 0.0;
        int i = t + 1 + g;
        for (; i + 3 * G < ny; i += 4 * G) {
          s += colp[i] * col[i];
          s1 += colp[i + G] * col[i + G];
          s2 += colp[i + 2 * G] * col[i + 2 * G];
          s3 += colp[i + 3 * G] * col[i + 3 * G];
        }
        for (; i < ny; i += G) s += colp[i] * col[i];
        s = (s + s1) + (s2 + s3);
      }
      for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
      if (act) {
        double corr = 0.0, rt = at;
#pragma unroll
        for (int l = 0; l < NB; l++)
          if (l < j) {
            const double f = Fs[l * nx + c];
            const double vt = M[t + (int64_t)ld * vcol[l]];  // V[t, l]
            corr += (sm.tot[l] - alpha * vt) * f;            // (V^T v_j)_l: row t of v_j is vhead
            rt -= vt * f;
          }
        const double fj = tau * (s - corr);
        rt -= vhead * fj;
        if (g == 0) {
          Fs[j * nx + c] = fj;
          M[t + (int64_t)ld * c] = rt;
        }
        double nn = nrm[r] - rt * rt;
        nn = nn > 0.0 ? nn : 0.0;
        nrm[r] = nn;
        trip |= nn < kPanelGuard * ref[r];
      }
    }
    if (tid == 0) {
      colp[t] = alpha;  // R[t, t]
      col_at[posp] = ct;
      col_at[t] = p;
      sm.vcol[j] = p;  // v_j lives below the diagonal of column p
    }
    if (trip) sm.flag = 1;
    j++;
    k = t + 1;
    publish(t + 1);
    __syncthreads();
  }
  __syncthreads();
  // T = R11^{-1} R12 by back substitution (one thread per column of R12), R11 through the map
  for (int cpos = k + tid; cpos < nx; cpos += NT) {
    double* col = M + (int64_t)ld * col_at[cpos];
    for (int a = k - 1; a >= 0; a--) {
      double s = col[a];
      for (int l = a + 1; l < k; l++) s -= M[a + (int64_t)ld * col_at[l]] * col[l];
      col[a] = s / M[a + (int64_t)ld * col_at[a]];
    }
  }
  __syncthreads();
  return k;
}

}  // namespace h2
