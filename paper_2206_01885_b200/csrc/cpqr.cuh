// cpqr.cuh -- CTA-wide column-pivoted Householder QR interpolative decomposition (getBasis,
// PAPER.md Eqs.(4.1)-(4.4); readings F1-F3).
//
// M (rows x cols, column-major, ld = rows) is held in global memory (L2-resident for the block
// sizes of this method).  Per step t: residual column norms (recomputed, fused into the previous
// step's update) -> pivot = largest norm, ties to the lowest position -> stop if
// norm < tol * |R11| -> column swap -> Householder reflector -> one warp per trailing column
// applies it and recomputes that column's residual norm.  On return M[0:k,0:k] = R11,
// M[0:k,k:cols] = T = R11^{-1} R12 (so column piv[c] ~= sum_t T[t,c] column piv[t]).
#pragma once
#include <climits>

#include "h2_internal.cuh"

namespace h2 {

template <int NT>
struct CpqrSmem {
  double rd[NT / 32];
  int ri[NT / 32];
  double bc_d[2];
  int bc_i[2];
};

template <int NT>
__device__ __forceinline__ double cta_sum(double v, CpqrSmem<NT>& sm) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sm.rd[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < NT / 32; w++) s += sm.rd[w];
  return s;
}

// v: scratch of `rows` doubles (shared or global); nrm2, piv: `cols` entries (global ok)
template <int NT>
__device__ int cta_cpqr(double* __restrict__ M, int rows, int cols, double tol, int* __restrict__ piv,
                        double* __restrict__ nrm2, double* __restrict__ v, CpqrSmem<NT>& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  for (int j = tid; j < cols; j += NT) piv[j] = j;
  for (int j = warp; j < cols; j += NW) {
    const double* col = M + (int64_t)rows * j;
    double s = 0.0;
    for (int i = lane; i < rows; i += 32) s += col[i] * col[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) nrm2[j] = s;
  }
  __syncthreads();
  const int kmax = rows < cols ? rows : cols;
  double r11 = 0.0;
  int k = 0;
  for (int t = 0; t < kmax; t++) {
    // argmax of the residual norms over positions >= t (ties -> lowest position)
    double best = -1.0;
    int bj = INT_MAX;
    for (int j = t + tid; j < cols; j += NT) {
      double x = sqrt(nrm2[j]);
      if (x > best) {
        best = x;
        bj = j;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      double b2 = __shfl_xor_sync(0xffffffffu, best, o);
      int j2 = __shfl_xor_sync(0xffffffffu, bj, o);
      if (b2 > best || (b2 == best && j2 < bj)) {
        best = b2;
        bj = j2;
      }
    }
    if (lane == 0) {
      sm.rd[warp] = best;
      sm.ri[warp] = bj;
    }
    __syncthreads();
    if (tid == 0) {
      double b = sm.rd[0];
      int j = sm.ri[0];
      for (int w = 1; w < NW; w++)
        if (sm.rd[w] > b || (sm.rd[w] == b && sm.ri[w] < j)) {
          b = sm.rd[w];
          j = sm.ri[w];
        }
      sm.bc_d[0] = b;
      sm.bc_i[0] = j;
    }
    __syncthreads();
    const double nrm = sm.bc_d[0];
    const int p = sm.bc_i[0];
    if (t == 0) {
      r11 = nrm;
      if (r11 == 0.0) break;
    }
    if (nrm < tol * r11) break;
    if (p != t) {
      double* ct = M + (int64_t)rows * t;
      double* cp = M + (int64_t)rows * p;
      for (int i = tid; i < rows; i += NT) {
        double a = ct[i];
        ct[i] = cp[i];
        cp[i] = a;
      }
      if (tid == 0) {
        int tp = piv[t];
        piv[t] = piv[p];
        piv[p] = tp;
        nrm2[p] = nrm2[t];
      }
    }
    __syncthreads();
    double* ct = M + (int64_t)rows * t;
    const double x0 = ct[t];
    const double alpha = x0 >= 0.0 ? -nrm : nrm;
    double part = 0.0;
    for (int i = t + tid; i < rows; i += NT) {
      double vi = i == t ? x0 - alpha : ct[i];
      v[i] = vi;
      part += vi * vi;
    }
    const double vtv = cta_sum<NT>(part, sm);  // includes the syncs that publish v
    __syncthreads();
    if (vtv > 0.0) {
      for (int j = t + 1 + warp; j < cols; j += NW) {
        double* col = M + (int64_t)rows * j;
        // four rows per lane in flight (independent loads and partial sums): the column is in
        // L2 / HBM, so memory-level parallelism sets the pace
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int i = t + lane;
        for (; i + 96 < rows; i += 128) {
          const double c0 = col[i], c1 = col[i + 32], c2 = col[i + 64], c3 = col[i + 96];
          s0 += v[i] * c0;
          s1 += v[i + 32] * c1;
          s2 += v[i + 64] * c2;
          s3 += v[i + 96] * c3;
        }
        for (; i < rows; i += 32) s0 += v[i] * col[i];
        double s = (s0 + s1) + (s2 + s3);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const double f = 2.0 * s / vtv;
        double n0 = 0.0, n1 = 0.0, n2 = 0.0, n3 = 0.0;
        i = t + lane;
        for (; i + 96 < rows; i += 128) {
          const double a0 = col[i] - f * v[i], a1 = col[i + 32] - f * v[i + 32];
          const double a2 = col[i + 64] - f * v[i + 64], a3 = col[i + 96] - f * v[i + 96];
          col[i] = a0;
          col[i + 32] = a1;
          col[i + 64] = a2;
          col[i + 96] = a3;
          if (i > t) n0 += a0 * a0;  // only row t itself is excluded (it joins R)
          n1 += a1 * a1;
          n2 += a2 * a2;
          n3 += a3 * a3;
        }
        for (; i < rows; i += 32) {
          const double a = col[i] - f * v[i];
          col[i] = a;
          if (i > t) n0 += a * a;
        }
        double nn = (n0 + n1) + (n2 + n3);
        for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
        if (lane == 0) nrm2[j] = nn;
      }
    } else {
      for (int j = t + 1 + warp; j < cols; j += NW) {
        double* col = M + (int64_t)rows * j;
        double nn = 0.0;
        for (int i = t + 1 + lane; i < rows; i += 32) nn += col[i] * col[i];
        for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
        if (lane == 0) nrm2[j] = nn;
      }
    }
    __syncthreads();
    // the pivot column joins R: row t = alpha; its rows below t are never read again (the back
    // substitution and T read rows < k of R11 / R12 only), so they are left as they are
    if (tid == 0) ct[t] = alpha;
    k = t + 1;
    __syncthreads();
  }
  __syncthreads();
  // T = R11^{-1} R12 by back substitution (one thread per column of R12)
  for (int c = k + tid; c < cols; c += NT) {
    double* col = M + (int64_t)rows * c;
    for (int i = k - 1; i >= 0; i--) {
      double s = col[i];
      for (int l = i + 1; l < k; l++) s -= M[i + (int64_t)rows * l] * col[l];
      col[i] = s / M[i + (int64_t)rows * i];
    }
  }
  __syncthreads();
  return k;
}

// ---- shared-memory variant: M row-major (M[i*ld + j]), thread-per-column ownership ----------
// Same algorithm and tie rules as cta_cpqr.  Per step: (1) every thread scans the residual norms
// of its own columns, a warp argmax, the warps' winners are combined redundantly by every thread
// (one barrier); (2) warp 0 swaps the pivot column in, builds the Householder vector and v^T v
// (one barrier); (3) each thread applies the reflector to its columns and recomputes their
// residual norms (one barrier).  Used when the block fits in shared memory.
template <int NT>
struct CpqrRmSmem {
  double wb[NT / 32];
  int wj[NT / 32];
  double vtv;
};

template <int NT>
__device__ __forceinline__ void cta_cpqr_rm_argmax(const double* __restrict__ nrm2, int t, int nx,
                                                   CpqrRmSmem<NT>& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double best = -1.0;
  int bj = INT_MAX;
  for (int j = t + tid; j < nx; j += NT) {
    const double x = sqrt(nrm2[j]);
    if (x > best) {
      best = x;
      bj = j;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double b2 = __shfl_xor_sync(0xffffffffu, best, o);
    const int j2 = __shfl_xor_sync(0xffffffffu, bj, o);
    if (b2 > best || (b2 == best && j2 < bj)) {
      best = b2;
      bj = j2;
    }
  }
  if (lane == 0) {
    sm.wb[warp] = best;
    sm.wj[warp] = bj;
  }
}

// Two barriers per step: the warps' argmax candidates for step t+1 are published at the end of
// step t's update (each thread owns its columns, so it scans the norms it just computed), the
// barrier closing the update also publishes them.
template <int NT>
__device__ int cta_cpqr_rm(double* __restrict__ M, int ny, int nx, int ld, double tol, int* __restrict__ piv,
                           double* __restrict__ nrm2, double* __restrict__ v, CpqrRmSmem<NT>& sm) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = tid; j < nx; j += NT) {
    piv[j] = j;
    double s = 0.0;
    for (int i = 0; i < ny; i++) s += M[i * ld + j] * M[i * ld + j];
    nrm2[j] = s;
  }
  cta_cpqr_rm_argmax<NT>(nrm2, 0, nx, sm);  // each thread scans only the norms it wrote
  __syncthreads();
  const int kmax = ny < nx ? ny : nx;
  double r11 = 0.0;
  int k = 0;
  for (int t = 0; t < kmax; t++) {
    double nrm = sm.wb[0];
    int p = sm.wj[0];
#pragma unroll
    for (int w = 1; w < NW; w++)
      if (sm.wb[w] > nrm || (sm.wb[w] == nrm && sm.wj[w] < p)) {
        nrm = sm.wb[w];
        p = sm.wj[w];
      }
    if (t == 0) {
      r11 = nrm;
      if (r11 == 0.0) break;
    }
    if (nrm < tol * r11) break;
    if (warp == 0) {
      // swap columns t <-> p, Householder vector of the new column t (rows t..ny-1)
      const double x0 = M[t * ld + p];
      const double alpha = x0 >= 0.0 ? -nrm : nrm;
      __syncwarp();  // every lane has read x0 before row t is rewritten
      double part = 0.0;
      for (int i = lane; i < ny; i += 32) {
        const double a = M[i * ld + p];
        if (p != t) M[i * ld + p] = M[i * ld + t];
        double vi = 0.0;
        if (i > t) vi = a;
        else if (i == t) vi = x0 - alpha;
        if (i >= t) {
          v[i] = vi;
          part += vi * vi;
          M[i * ld + t] = i == t ? alpha : 0.0;
        } else {
          M[i * ld + t] = a;
        }
      }
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0) {
        sm.vtv = part;
        const int tp = piv[t];
        piv[t] = piv[p];
        piv[p] = tp;
        nrm2[p] = nrm2[t];
      }
    }
    __syncthreads();  // (every thread read this step's winners before it)
    const double vtv = sm.vtv;
    for (int j = t + 1 + tid; j < nx; j += NT) {
      // independent partial sums (4-way) break the serial FMA chains
      double nn0 = 0.0, nn1 = 0.0;
      if (vtv > 0.0) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int i = t;
        for (; i + 3 < ny; i += 4) {
          s0 += v[i] * M[i * ld + j];
          s1 += v[i + 1] * M[(i + 1) * ld + j];
          s2 += v[i + 2] * M[(i + 2) * ld + j];
          s3 += v[i + 3] * M[(i + 3) * ld + j];
        }
        for (; i < ny; i++) s0 += v[i] * M[i * ld + j];
        const double f = 2.0 * ((s0 + s1) + (s2 + s3)) / vtv;
        const double a0 = M[t * ld + j] - f * v[t];  // row t joins R, not the residual norm
        M[t * ld + j] = a0;
        i = t + 1;
        for (; i + 1 < ny; i += 2) {
          const double a = M[i * ld + j] - f * v[i], b = M[(i + 1) * ld + j] - f * v[i + 1];
          M[i * ld + j] = a;
          M[(i + 1) * ld + j] = b;
          nn0 += a * a;
          nn1 += b * b;
        }
        for (; i < ny; i++) {
          const double a = M[i * ld + j] - f * v[i];
          M[i * ld + j] = a;
          nn0 += a * a;
        }
      } else {
        for (int i = t + 1; i < ny; i++) nn0 += M[i * ld + j] * M[i * ld + j];
      }
      nrm2[j] = nn0 + nn1;
    }
    k = t + 1;
    cta_cpqr_rm_argmax<NT>(nrm2, t + 1, nx, sm);  // next step's candidates (own columns only)
    __syncthreads();
  }
  __syncthreads();
  // T = R11^{-1} R12 by back substitution (one thread per column of R12)
  for (int c = k + tid; c < nx; c += NT) {
    for (int i = k - 1; i >= 0; i--) {
      double s = M[i * ld + c];
      for (int l = i + 1; l < k; l++) s -= M[i * ld + l] * M[l * ld + c];
      M[i * ld + c] = s / M[i * ld + i];
    }
  }
  __syncthreads();
  return k;
}

}  // namespace h2
