// calib.cu -- a5: r1 = r2 = r from the tolerance (Algorithm 2 line 2).
//
// Readings (E1-E6): r1 = r2 = r; for every level l holding an admissible pair, box
// width w = W 2^-l; Z1 = 256 SplitMix64 points in [0,w]^d, Z2 = the same construction shifted by
// w/tau in every coordinate (the Eq.(2.1) boundary); for m = 1, 2, ...: Z2* = Vol(Z2, m^d), ID of
// K(Z1, Z2*) at tolerance 1e-3 eps, e = ||K(Z1,Z2) - U K(Z1^,Z2)||_F / ||K(Z1,Z2)||_F; the level's
// budget is the first m^d with e < 1e-2 eps, or m^d >= 256 (pass-through); r = max over levels.
// All (level, m) trials run as one batched launch: one CTA per trial.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "cpqr.cuh"
#include "cpqr_panel.cuh"
#include "vol.cuh"

namespace h2 {

constexpr int kCalThreads = 256;
constexpr int N = kCalibPoints;

struct CalWork {  // per-trial global workspace
  double Z1[N * kMaxD], Z2[N * kMaxD];
  double M[N * N];
  double Ks[N * N];
  double nrm2[N], v[N];
  int piv[N], sel[N];
  int ns, k;  // |Z2^*| and the ID rank, passed between the trial's launches
  int panel;  // 1: the panel CPQR ran (columns never moved: position c is physical column piv[c])
  double pnum[8], pden[8];  // the error's partial sums per column slice (calib_err_kernel)
  int lv;     // the trial's virtual level (calib_cpqr_cluster_kernel's cancellation test)
};
constexpr int kErrSlices = 8;  // CTAs per trial of the error evaluation: N / 8 = 32 columns each

// k-th SplitMix64 output of the stream seeded with `seed` (counter form of the sequential
// generator: state_k = seed + (k+1) * golden gamma)
__device__ __forceinline__ unsigned long long splitmix_at(unsigned long long seed, unsigned long long k) {
  unsigned long long z = seed + (k + 1ULL) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// kappa(x, y) for two point-major points of a trial
template <int D>
__device__ __forceinline__ double calib_kernel(int kid, double p2, const double* x, const double* y) {
  if (kid == H2_KERNEL_COSDOT) {
    double t = 0.0;
    for (int c = 0; c < D; c++) t = fma(x[c], y[c], t);
    return kernel_cosdot(t);
  }
  double s = 0.0;
  for (int c = 0; c < D; c++) {
    const double df = x[c] - y[c];
    s = fma(df, df, s);
  }
  return kernel_s(kid, p2, s);
}

struct PtAcc {
  const double* Z;
  int d;
  __device__ __forceinline__ double coord(int pos, int c) const { return Z[pos * d + c]; }
  __device__ __forceinline__ int index(int pos) const { return pos; }
};

// A trial runs as three launches over the batch: prep (Z1, Z2, Vol(Z2, m^d), the block M; 256
// threads), the CPQR ID of M (1024 threads: the block lives in global memory / L2 and the steps are
// latency-bound, so more columns in flight), and the error of the interpolation (256 threads).
// the shift of H2_KERNEL_MQSHIFT (kappa's first argument is x + a, or x - a for the transposed
// kernel of the column bases: reading E7)
struct CalShift {
  double a[kMaxD];
};

// A trial's level field is a VIRTUAL level: l for kappa, l + 32 for the transposed kernel kappa^T(x,
// y) = kappa(y, x) of a non-symmetric build (its column bases); the points are those of level l.
template <int D>
__global__ void __launch_bounds__(kCalThreads) calib_prep_kernel(int kid, double p2, double tau,
                                                                 const double* __restrict__ wl,
                                                                 const int* __restrict__ lv, const int* __restrict__ mv,
                                                                 const int* __restrict__ skip_level, CalShift sh,
                                                                 CalWork* work) {
  __shared__ VolSmem<D, kCalThreads> vsm;
  __shared__ int s_ns;
  const int tid = threadIdx.x;
  CalWork& W = work[blockIdx.x];
  long long Gm = 1;
  for (int c = 0; c < D; c++) Gm *= mv[blockIdx.x];
  // skipped: the level already passed at a smaller m, or m^d >= N (passes by definition, so its
  // error is never needed)
  if ((skip_level && skip_level[lv[blockIdx.x]]) || Gm >= N) {
    if (tid == 0) W.ns = -1;
    return;
  }
  const double w = wl[blockIdx.x];
  const int level = lv[blockIdx.x] & 31, m = mv[blockIdx.x];
  const double sgn = lv[blockIdx.x] >= 32 ? -1.0 : 1.0;
  const unsigned long long seed = kCalibSeed + (unsigned long long)level;
  const double shift = __ddiv_rn(w, tau);
  for (int e = tid; e < N * D; e += kCalThreads) {
    double u1 = (double)(splitmix_at(seed, e) >> 11) * 0x1.0p-53;
    double u2 = (double)(splitmix_at(seed, N * D + e) >> 11) * 0x1.0p-53;
    // Z1 is every kernel evaluation's first argument: for the shifted multiquadric it is stored
    // shifted by +-a (the points themselves are only used through the kernel)
    W.Z1[e] = __dmul_rn(u1, w) + (kid == H2_KERNEL_MQSHIFT ? sgn * sh.a[e % D] : 0.0);
    W.Z2[e] = __dadd_rn(__dmul_rn(u2, w), shift);
  }
  __syncthreads();
  long long G = 1;
  for (int c = 0; c < D; c++) G *= m;
  if (G >= N) {
    for (int i = tid; i < N; i += kCalThreads) W.sel[i] = i;
    if (tid == 0) s_ns = N;
  } else {
    PtAcc acc{W.Z2, D};
    int c = cta_vol<D, kCalThreads>(acc, N, (int)G, W.sel, vsm);
    if (tid == 0) s_ns = c;
  }
  __syncthreads();
  const int ns = s_ns;
  if (tid == 0) {
    W.ns = ns;
    W.lv = lv[blockIdx.x];
  }
  // M = K(Z1, Z2*)^T : ns x N column-major (columns = Z1 candidates)
  for (int e = tid; e < ns * N; e += kCalThreads) {
    int a = e % ns, b = e / ns;
    W.M[e] = calib_kernel<D>(kid, p2, W.Z1 + b * D, W.Z2 + W.sel[a] * D);
  }
}

constexpr int kCalCpqrThreads = 1024;
constexpr int kCalPanelNb = 8;
// the trial's ID: the panel-blocked CPQR (cpqr_panel.cuh; 4 threads per column of the 256 Z1
// candidates) or, with H2_CAL_PANEL=0, the unblocked one (cpqr.cuh)
__global__ void __launch_bounds__(kCalCpqrThreads) calib_cpqr_kernel(double eps, int use_panel, CalWork* work) {
  __shared__ CpqrSmem<kCalCpqrThreads> csm;
  __shared__ PanelSmem<kCalCpqrThreads, kCalPanelNb> psm;
  __shared__ double sv[N];
  __shared__ double Fs[kCalPanelNb * N];
  CalWork& W = work[blockIdx.x];
  if (W.ns < 0) return;  // skipped trial
  const int k = use_panel ? cta_cpqr_panel<kCalCpqrThreads, kCalPanelNb, 1>(W.M, W.ns, W.ns, N, 1e-3 * eps, 4, W.piv,
                                                                            Fs, psm)
                          : cta_cpqr<kCalCpqrThreads>(W.M, W.ns, N, 1e-3 * eps, W.piv, W.nrm2, sv, csm);
  if (threadIdx.x == 0) {
    W.k = k;
    W.panel = use_panel;
  }
}

// The trial's ID on a thread-block cluster (default; H2_CAL_CLUSTER=0 restores the one-CTA kernel
// above): M (ns x 256) is too large for one SM's shared memory and on one SM every pivot step
// re-reads it from L2 (the one-CTA kernel is L2-latency- and barrier-bound: ~10 us per step).
// Here kCalCl CTAs each hold kCalClW = 256 / kCalCl consecutive columns (Z1 candidates) in shared
// memory, column-major, for the whole factorisation.  The algorithm and tie rule of cta_cpqr
// (unblocked Householder, residual norms recomputed after every update, pivot = largest norm, ties
// to the lowest position, stop when it is < tol * |R11|), with a position map instead of column
// swaps.  One cluster barrier per pivot step: after it every CTA reads the CTAs' candidates (DSMEM)
// and picks the same pivot, reads the pivot column straight from its owner's shared memory, builds
// the Householder vector (the same arithmetic in every CTA) and updates its own live columns.  The
// owner writes the pivot's diagonal alpha only after the next barrier (the others read the column
// until then).  At the end the slices go back to W.M and T = R11^{-1} R12 is formed column by column
// from R11 in global memory.  Output as the panel kernel's (W.panel = 1): columns in place,
// W.piv[position] = physical column.
constexpr int kCalCl = 8;                    // CTAs per trial (portable cluster size)
constexpr int kCalClNT = 256;
constexpr int kCalClW = N / kCalCl;          // columns per CTA (= 32: one lane per column in publish)
static_assert(kCalClW == 32, "one lane per own column");
struct CalClCand {
  double x;   // sqrt of the residual norm^2 (-1: no live column)
  int pos;    // position in the pivot order
  int j;      // physical column
  int abort;  // (rank 0's candidate) the trial is cancelled
};
// dynamic shared memory: the slice (ns x kCalClW) + v (ns); ns < N
constexpr int kCalClSmem = (int)sizeof(double) * (N * kCalClW + N);

__global__ void __cluster_dims__(kCalCl, 1, 1) __launch_bounds__(kCalClNT) calib_cpqr_cluster_kernel(double eps,
                                                                                                    CalWork* work,
                                                                                                    const int* cancel) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  constexpr int NT = kCalClNT, NW = NT / 32, WC = kCalClW;
  CalWork& W = work[blockIdx.x / kCalCl];
  const int ns = W.ns;
  if (ns < 0) return;  // a skipped trial: every CTA of the cluster leaves (no cluster barrier reached)
  const int q = (int)cl.block_rank(), j0 = q * WC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double tol = 1e-3 * eps;
  extern __shared__ double sh[];
  double* Ms = sh;               // own columns: Ms[a + ns * jl] = M[a, j0 + jl]
  double* v = Ms + ns * WC;      // Householder vector (rows t..ns-1)
  __shared__ double nrm2[WC];
  __shared__ int pos[WC];        // own column -> position
  __shared__ int col_at[N];      // position -> physical column (replicated in every CTA)
  __shared__ CalClCand cand[2];  // this CTA's candidate by step parity (read by every CTA)
  __shared__ CalClCand best_s;
  __shared__ CpqrSmem<NT> csm;
  for (int e = tid; e < ns * WC; e += NT) Ms[e] = W.M[(int64_t)ns * j0 + e];
  for (int b = tid; b < N; b += NT) col_at[b] = b;
  if (tid < WC) pos[tid] = j0 + tid;
  __syncthreads();
  for (int jl = warp; jl < WC; jl += NW) {
    const double* col = Ms + ns * jl;
    double s = 0.0;
    for (int a = lane; a < ns; a += 32) s += col[a] * col[a];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) nrm2[jl] = s;
  }
  __syncthreads();
  auto publish = [&](int tt) {  // lane jl = own column jl
    if (warp == 0) {
      const int ps = pos[lane];
      double bx = ps >= tt ? sqrt(nrm2[lane]) : -1.0;
      int bp = ps >= tt ? ps : INT_MAX, bj = ps >= tt ? j0 + lane : -1;
      for (int o = 16; o > 0; o >>= 1) {
        const double x2 = __shfl_xor_sync(0xffffffffu, bx, o);
        const int p2_ = __shfl_xor_sync(0xffffffffu, bp, o);
        const int j2 = __shfl_xor_sync(0xffffffffu, bj, o);
        if (x2 > bx || (x2 == bx && p2_ < bp)) {
          bx = x2;
          bp = p2_;
          bj = j2;
        }
      }
      // cancellation (speculative phase 1, calibrate_begin): the trial's level passed in phase 0.
      // Rank 0 alone reads the flag, so every CTA of the cluster takes the same decision.
      int ab = 0;
      if (cancel && q == 0 && lane == 0) ab = *reinterpret_cast<const volatile int*>(cancel + W.lv);
      if (lane == 0) cand[tt & 1] = CalClCand{bx, bp, bj, ab};
    }
  };
  publish(0);
  const int kmax = ns < N ? ns : N;
  double r11 = 0.0;
  int k = 0;
  bool aborted = false;
  int pend_jl = -1, pend_row = 0;
  double pend_alpha = 0.0;
  for (int tt = 0; tt < kmax; tt++) {
    cl.sync();  // candidates published, the previous step's updates done, its pivot column read
    if (pend_jl >= 0 && tid == 0) Ms[ns * pend_jl + pend_row] = pend_alpha;
    pend_jl = -1;
    if (warp == 0) {
      CalClCand c{-1.0, INT_MAX, -1, 0};
      if (lane < kCalCl) c = *cl.map_shared_rank(&cand[tt & 1], lane);
      const int ab = __shfl_sync(0xffffffffu, c.abort, 0);
      for (int o = 16; o > 0; o >>= 1) {
        const double x2 = __shfl_xor_sync(0xffffffffu, c.x, o);
        const int p2_ = __shfl_xor_sync(0xffffffffu, c.pos, o);
        const int j2 = __shfl_xor_sync(0xffffffffu, c.j, o);
        if (x2 > c.x || (x2 == c.x && p2_ < c.pos)) c = CalClCand{x2, p2_, j2, 0};
      }
      c.abort = ab;
      if (lane == 0) best_s = c;
    }
    __syncthreads();
    const CalClCand b = best_s;
    const double nrm = b.x;
    if (b.abort) {
      aborted = true;
      break;
    }
    if (tt == 0) {
      r11 = nrm;
      if (r11 == 0.0) break;
    }
    if (b.j < 0 || nrm < tol * r11) break;
    const int p = b.j, owner = p / WC;
    const double* src = cl.map_shared_rank(Ms, owner) + ns * (p - owner * WC);  // DSMEM
    const double x0 = src[tt];
    const double alpha = x0 >= 0.0 ? -nrm : nrm;
    double part = 0.0;
    for (int a = tt + tid; a < ns; a += NT) {
      const double vi = a == tt ? x0 - alpha : src[a];
      v[a] = vi;
      part += vi * vi;
    }
    const double vtv = cta_sum<NT>(part, csm);  // its barriers publish v
    if (q == owner) {
      pend_jl = p - j0;
      pend_row = tt;
      pend_alpha = alpha;
    }
    if (tid == 0) {  // position map: the column at position tt moves to the pivot's position
      const int jt = col_at[tt];
      col_at[b.pos] = jt;
      col_at[tt] = p;
      if (jt >= j0 && jt < j0 + WC) pos[jt - j0] = b.pos;
      if (p >= j0 && p < j0 + WC) pos[p - j0] = tt;
    }
    __syncthreads();
    for (int jl = warp; jl < WC; jl += NW) {  // own live columns: reflector, residual norm (rows > tt)
      if (pos[jl] <= tt) continue;
      double* col = Ms + ns * jl;
      double nn = 0.0;
      if (vtv > 0.0) {
        double s0 = 0.0, s1 = 0.0;
        int a = tt + lane;
        for (; a + 32 < ns; a += 64) {
          s0 += v[a] * col[a];
          s1 += v[a + 32] * col[a + 32];
        }
        for (; a < ns; a += 32) s0 += v[a] * col[a];
        double sd = s0 + s1;
        for (int o = 16; o > 0; o >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, o);
        const double f = 2.0 * sd / vtv;
        for (a = tt + lane; a < ns; a += 32) {
          const double x = col[a] - f * v[a];
          col[a] = x;
          if (a > tt) nn += x * x;
        }
      } else {
        for (int a = tt + 1 + lane; a < ns; a += 32) nn += col[a] * col[a];
      }
      for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
      if (lane == 0) nrm2[jl] = nn;
    }
    k = tt + 1;
    __syncthreads();
    publish(tt + 1);
  }
  if (pend_jl >= 0 && tid == 0) Ms[ns * pend_jl + pend_row] = pend_alpha;
  __syncthreads();
  for (int e = tid; e < ns * WC; e += NT) W.M[(int64_t)ns * j0 + e] = Ms[e];
  cl.sync();  // every R column in global memory, visible cluster-wide; no DSMEM read after this
  // T = R11^{-1} R12 for the own columns at positions >= k, column-oriented back substitution:
  // for l = k-1..0: x_l /= R_ll; x_a -= R_al x_l (a < l).  The diagonal is staged in shared memory
  // and a warp takes its (up to WC / NW) columns together, so every R11 column is loaded once per
  // warp (lanes over its rows, one step ahead: the loads do not depend on x) instead of once per
  // column behind a dependent load of the diagonal.  The same operations in the same order per entry.
  if (aborted) k = 0;  // a cancelled trial: rank 0, no T (its pass flag is never used)
  constexpr int CPW = WC / NW;         // own columns per warp
  double* diag = Ms;                   // k (the slice's space is free after the write-back)
  double* xall = Ms + N;               // [own column jl][row a], k <= ns < N rows each
  for (int l = tid; l < k; l += NT) diag[l] = W.M[l + (int64_t)ns * col_at[l]];
  for (int e = tid; e < WC * k; e += NT) {
    const int jl = e / k, a = e - jl * k;
    if (pos[jl] >= k) xall[jl * N + a] = W.M[a + (int64_t)ns * (j0 + jl)];
  }
  __syncthreads();
  if (k > 0) {
    bool mine[CPW];
    bool any = false;
#pragma unroll
    for (int c = 0; c < CPW; c++) {
      mine[c] = pos[warp + NW * c] >= k;
      any |= mine[c];
    }
    if (any) {
      constexpr int RPL = N / 32;  // rows per lane
      double r[RPL], rn[RPL];
      auto load_col = [&](int l, double (&dst)[RPL]) {
        const double* Rl = W.M + (int64_t)ns * col_at[l];
#pragma unroll
        for (int u = 0; u < RPL; u++) {
          const int a = lane + 32 * u;
          dst[u] = a < l ? Rl[a] : 0.0;
        }
      };
      load_col(k - 1, r);
      for (int l = k - 1; l >= 0; l--) {
        if (l > 0) load_col(l - 1, rn);
        const double dl = diag[l];
        double xl[CPW];
#pragma unroll
        for (int c = 0; c < CPW; c++) {
          xl[c] = 0.0;
          if (!mine[c]) continue;
          double* xw = xall + (warp + NW * c) * N;
          xl[c] = xw[l] / dl;
#pragma unroll
          for (int u = 0; u < RPL; u++) {
            const int a = lane + 32 * u;
            if (a < l) xw[a] -= r[u] * xl[c];
          }
        }
        __syncwarp();  // every lane has read x_l before it is overwritten
        if (lane == 0)
#pragma unroll
          for (int c = 0; c < CPW; c++)
            if (mine[c]) xall[(warp + NW * c) * N + l] = xl[c];
        __syncwarp();
#pragma unroll
        for (int u = 0; u < RPL; u++) r[u] = rn[u];
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < WC * k; e += NT) {
    const int jl = e / k, a = e - jl * k;
    if (pos[jl] >= k) W.M[a + (int64_t)ns * (j0 + jl)] = xall[jl * N + a];
  }
  if (q == 0) {
    for (int b = tid; b < N; b += NT) W.piv[b] = col_at[b];
    if (tid == 0) {
      W.k = k;
      W.panel = 1;
    }
  }
}

// H2_CAL_CLUSTER=0 (A/B knob, read once): the one-CTA trial ID kernel instead of the cluster one
static int cal_cluster() {
  static const int v = [] {
    const char* e = getenv("H2_CAL_CLUSTER");
    return e ? atoi(e) : 1;
  }();
  return v;
}

// Ks[t][e] = K(Z1[piv[t]], Z2[e]) for the k skeleton rows
template <int D>
__global__ void __launch_bounds__(kCalThreads) calib_ks_kernel(int kid, double p2, CalWork* work) {
  CalWork& W = work[blockIdx.x];
  if (W.ns < 0) return;
  const int k = W.k;
  for (int x = threadIdx.x; x < k * N; x += kCalThreads) {
    const int t = x / N, e = x % N;
    W.Ks[x] = calib_kernel<D>(kid, p2, W.Z1 + W.piv[t] * D, W.Z2 + e * D);
  }
}

// Error of one trial, kErrSlices CTAs per trial: slice q takes the 32 columns (pivoted positions)
// [32 q, 32 q + 32) x all N points of Z2.  A warp owns 4 columns (the same for all its lanes:
// T and M loads are broadcasts) and a lane 8 points: a 4 x 8 register tile, 32 FMAs per 12 loads
// in the k-long inner product U K^.  Partial sums per slice; calib_final_kernel adds them in a
// fixed order.
template <int D>
__global__ void __launch_bounds__(kCalThreads) calib_err_kernel(int kid, double p2, CalWork* work) {
  __shared__ CpqrSmem<kCalThreads> csm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  CalWork& W = work[blockIdx.x / kErrSlices];
  if (W.ns < 0) return;
  const int q = blockIdx.x % kErrSlices;
  const int ns = W.ns, k = W.k;
  constexpr int CPW = 4, EPL = N / 32;  // columns per warp, points per lane
  const int c0 = q * (N / kErrSlices) + warp * CPW;
  double num = 0.0, den = 0.0;
  double kv[CPW][EPL];
#pragma unroll
  for (int j = 0; j < CPW; j++) {
    const int row = W.piv[c0 + j];
#pragma unroll
    for (int u = 0; u < EPL; u++) {
      const int e = lane + 32 * u;
      kv[j][u] = calib_kernel<D>(kid, p2, W.Z1 + row * D, W.Z2 + e * D);
      den += kv[j][u] * kv[j][u];
    }
  }
  if (c0 + CPW > k) {  // some of the warp's columns are outside the skeleton: K - U K^
    double ap[CPW][EPL];
#pragma unroll
    for (int j = 0; j < CPW; j++)
#pragma unroll
      for (int u = 0; u < EPL; u++) ap[j][u] = 0.0;
    for (int t = 0; t < k; t++) {
      double tm[CPW], ks[EPL];
#pragma unroll
      for (int j = 0; j < CPW; j++) tm[j] = W.M[t + ns * (W.panel ? W.piv[c0 + j] : c0 + j)];
#pragma unroll
      for (int u = 0; u < EPL; u++) ks[u] = W.Ks[t * N + lane + 32 * u];
#pragma unroll
      for (int j = 0; j < CPW; j++)
#pragma unroll
        for (int u = 0; u < EPL; u++) ap[j][u] = fma(tm[j], ks[u], ap[j][u]);
    }
#pragma unroll
    for (int j = 0; j < CPW; j++)
      if (c0 + j >= k)
#pragma unroll
        for (int u = 0; u < EPL; u++) {
          const double df = kv[j][u] - ap[j][u];
          num += df * df;
        }
  }
  num = cta_sum<kCalThreads>(num, csm);
  den = cta_sum<kCalThreads>(den, csm);
  if (tid == 0) {
    W.pnum[q] = num;
    W.pden[q] = den;
  }
}

__global__ void calib_final_kernel(double eps, const int* __restrict__ mv, int d, CalWork* work, double* err,
                                   int* pass) {
  const int t = blockIdx.x;  // one thread per trial
  CalWork& W = work[t];
  long long G = 1;
  for (int c = 0; c < d; c++) G *= mv[t];
  if (W.ns < 0) {  // skipped: a pass-through trial (m^d >= N) passes, a skipped level's never counts
    err[t] = G >= N ? 0.0 : -1.0;
    pass[t] = G >= N;
    return;
  }
  double num = 0.0, den = 0.0;
  for (int q = 0; q < kErrSlices; q++) {
    num += W.pnum[q];
    den += W.pden[q];
  }
  const double e = den > 0.0 ? sqrt(num) / sqrt(den) : 0.0;
  err[t] = e;
  pass[t] = (e < 1e-2 * eps) || G >= N;
}

__global__ void level_has_il_kernel(int nnodes, const int* __restrict__ level, const int64_t* __restrict__ il_off,
                                    int* has) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nnodes && il_off[i + 1] > il_off[i]) has[level[i]] = 1;
}

// Page-locked host staging for the trial parameters and pass flags (per host thread; slot 0 =
// phase 0, slot 1 = phase 1): asynchronous copies to / from pageable memory would make the host
// wait for the trials and serialise phase 0 with the lists.
static char* pinned_slot(int slot, size_t bytes) {
  thread_local char* p[2] = {nullptr, nullptr};
  thread_local size_t cap[2] = {0, 0};
  if (cap[slot] < bytes) {
    if (p[slot]) cudaFreeHost(p[slot]);
    p[slot] = nullptr;
    cap[slot] = 0;
    const size_t c = std::max<size_t>(bytes, 64 << 10);
    H2_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&p[slot]), c));
    cap[slot] = c;
  }
  return p[slot];
}

// H2_CAL_PANEL=0 (A/B knob, read once): the unblocked CPQR in the calibration trials
static int cal_panel() {
  static const int v = [] {
    const char* e = getenv("H2_CAL_PANEL");
    return e ? atoi(e) : 1;
  }();
  return v;
}

// One batch of (level, m) trials on stream s; the per-trial pass flags land in job.pass_h
// (page-locked) once the stream has reached the end of the batch.
static void launch_trials(h2_handle* h, cudaStream_t s, int slot, const std::vector<double>& wl,
                          const std::vector<int>& lv, const std::vector<int>& mv, const int* skip_level,
                          CalibSet& job, const int* cancel = nullptr) {
  const int T = (int)wl.size();
  job.T = T;
  if (T == 0) return;
  const int d = h->d;
  const double p2 = kernel_p2(h->kid, h->kp);
  CalShift sh{};
  for (int c = 0; c < d; c++) sh.a[c] = h->kpa[c];
  const int batch = 256;
  job.work = Scratch(sizeof(CalWork) * (T < batch ? T : batch), s);
  job.params = Scratch(sizeof(double) * T + sizeof(int) * 2 * T, s);
  job.outs = Scratch(sizeof(double) * T + sizeof(int) * T, s);
  double* dw = job.params.as<double>();
  int* dl = reinterpret_cast<int*>(dw + T);
  int* dm = dl + T;
  double* derr = job.outs.as<double>();
  int* dpass = reinterpret_cast<int*>(derr + T);
  const size_t in_bytes = sizeof(double) * T + sizeof(int) * 2 * T;
  char* hin = pinned_slot(slot, in_bytes + sizeof(int) * T);
  std::memcpy(hin, wl.data(), sizeof(double) * T);
  std::memcpy(hin + sizeof(double) * T, lv.data(), sizeof(int) * T);
  std::memcpy(hin + sizeof(double) * T + sizeof(int) * T, mv.data(), sizeof(int) * T);
  H2_CUDA_TRY(cudaMemcpyAsync(dw, hin, in_bytes, cudaMemcpyHostToDevice, s));
  if (cal_cluster())
    H2_CUDA_TRY(cudaFuncSetAttribute(calib_cpqr_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kCalClSmem));
  for (int b0 = 0; b0 < T; b0 += batch) {
    int nb = T - b0 < batch ? T - b0 : batch;
    switch (d) {
#define H2_CAL_CASE(DD)                                                                                   \
  case DD:                                                                                                \
    calib_prep_kernel<DD><<<nb, kCalThreads, 0, s>>>(h->kid, p2, h->tau, dw + b0, dl + b0, dm + b0,         \
                                                     skip_level, sh, job.work.as<CalWork>());              \
    if (cal_cluster()) calib_cpqr_cluster_kernel<<<nb * kCalCl, kCalClNT, kCalClSmem, s>>>(h->id_tol,        \
                                                                                job.work.as<CalWork>(),    \
                                                                                cancel);                   \
    else calib_cpqr_kernel<<<nb, kCalCpqrThreads, 0, s>>>(h->id_tol, cal_panel(), job.work.as<CalWork>());  \
    calib_ks_kernel<DD><<<nb, kCalThreads, 0, s>>>(h->kid, p2, job.work.as<CalWork>());                    \
    calib_err_kernel<DD><<<nb * kErrSlices, kCalThreads, 0, s>>>(h->kid, p2, job.work.as<CalWork>());        \
    break;
      H2_CAL_CASE(1) H2_CAL_CASE(2) H2_CAL_CASE(3) H2_CAL_CASE(4)
      H2_CAL_CASE(5) H2_CAL_CASE(6) H2_CAL_CASE(7) H2_CAL_CASE(8)
#undef H2_CAL_CASE
    }
    calib_final_kernel<<<nb, 1, 0, s>>>(h->id_tol, dm + b0, d, job.work.as<CalWork>(), derr + b0, dpass + b0);
    H2_CHECK_LAUNCH();
    h->gpu_launches += 5;
  }
  job.pass_h = reinterpret_cast<int*>(hin + in_bytes);
  H2_CUDA_TRY(cudaMemcpyAsync(job.pass_h, dpass, sizeof(int) * T, cudaMemcpyDeviceToHost, s));
  job.lv = lv;
  job.mv = mv;
}

// passed[lv[t]] = 1 for every passing trial t of phase 0 (benign same-value races).
__global__ void level_passed_kernel(int T, const int* __restrict__ lv, const int* __restrict__ pass, int* passed) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T && pass[t]) passed[lv[t]] = 1;
}

static long long grid_size(int d, int m) {
  long long G = 1;
  for (int c = 0; c < d; c++) G *= m;
  return G;
}

// Issued right after the tree (a1-a3) on the stream `s`, overlapping a4 -- a trial depends only on
// the level's box width W 2^-l, not on the lists.  Phase 0: the trials with m^d <= 64 for EVERY level
// 1..depth.  Phase 1 (speculative): the trials with m^d > 64 for every level.  d <= 2: after phase 0
// on `s`, each exiting at once when a phase-0 trial of its level passed.  d >= 3 (at most two
// computed trials per level: m^d < N = 256 stops at m = 6): on `s2`, concurrently with phase 0, and
// calibrate_end waits for it only when some level needs it (H2_CAL_MERGE=0, A/B knob: the d <= 2
// order for every d).  calibrate_end keeps the levels that hold an admissible pair; levels without
// one cost trials but never decide r.
void calibrate_begin(h2_handle* h, cudaStream_t s, cudaStream_t s2, CalibJob& job) {
  job.stream = s;
  job.stream2 = s2;
  std::vector<double> wl, wl1;
  std::vector<int> lv, mv, lv1, mv1;
  for (int o = 0; o < (h->nonsym ? 2 : 1); o++)  // o = 1: the transposed kernel (reading E7)
    for (int l = 1; l <= h->depth; l++)
      for (int m = 1;; m++) {
        const long long G = grid_size(h->d, m);
        const bool p0 = G <= 64 || m == 1;
        (p0 ? wl : wl1).push_back(ldexp(h->W, -l));
        (p0 ? lv : lv1).push_back(l + 32 * o);
        (p0 ? mv : mv1).push_back(m);
        if (G >= N) break;
      }
  static const bool split_env = [] {
    const char* e = getenv("H2_CAL_MERGE");
    return e ? atoi(e) != 0 : true;
  }();
  job.split = split_env && h->d >= 3 && !wl1.empty() && s2 != nullptr;
  // (a previous build's unawaited phase 1 may still own the page-locked slot 1)
  if (s2) H2_CUDA_TRY(cudaStreamSynchronize(s2));
  job.passed = Scratch(sizeof(int) * 64, s);
  H2_CUDA_TRY(cudaMemsetAsync(job.passed.p, 0, sizeof(int) * 64, s));
  if (job.split) {  // phase 1 reads `passed` (its cancellation flags): only after the clear above
    cudaEvent_t clr;
    H2_CUDA_TRY(cudaEventCreateWithFlags(&clr, cudaEventDisableTiming));
    H2_CUDA_TRY(cudaEventRecord(clr, s));
    H2_CUDA_TRY(cudaStreamWaitEvent(s2, clr, 0));
    cudaEventDestroy(clr);
  }
  launch_trials(h, s, 0, wl, lv, mv, nullptr, job.p0);
  if (job.split) {
    // the speculative phase 1 runs concurrently with phase 0; a phase-1 trial whose level passed
    // in phase 0 stops at its next pivot step (the flags land as phase 0 ends), so an unneeded
    // phase 1 does not keep the SMs busy into the next stages or the next build
    if (job.p0.T > 0) {
      const int* dl = reinterpret_cast<const int*>(job.p0.params.as<double>() + job.p0.T);
      const int* dpass = reinterpret_cast<const int*>(job.p0.outs.as<double>() + job.p0.T);
      level_passed_kernel<<<(job.p0.T + 127) / 128, 128, 0, s>>>(job.p0.T, dl, dpass, job.passed.as<int>());
      H2_CHECK_LAUNCH();
      h->gpu_launches += 1;
    }
    launch_trials(h, s2, 1, wl1, lv1, mv1, nullptr, job.p1, job.passed.as<int>());
  } else if (!wl1.empty()) {
    if (job.p0.T > 0) {
      const int* dl = reinterpret_cast<const int*>(job.p0.params.as<double>() + job.p0.T);
      const int* dpass = reinterpret_cast<const int*>(job.p0.outs.as<double>() + job.p0.T);
      level_passed_kernel<<<(job.p0.T + 127) / 128, 128, 0, s>>>(job.p0.T, dl, dpass, job.passed.as<int>());
      H2_CHECK_LAUNCH();
      h->gpu_launches += 1;
    }
    launch_trials(h, s, 1, wl1, lv1, mv1, job.passed.as<int>(), job.p1);
  }
  job.active = true;
}

// r = max over the levels holding an admissible pair of the first passing m^d (phase 0, then phase 1).
int calibrate_end(h2_handle* h, CalibJob& job) {
  cudaStream_t s = h->stream;
  Scratch hasd(sizeof(int) * 64, s);
  H2_CUDA_TRY(cudaMemsetAsync(hasd.p, 0, sizeof(int) * 64, s));
  level_has_il_kernel<<<(h->nnodes + 255) / 256, 256, 0, s>>>(h->nnodes, h->level, h->il_off, hasd.as<int>());
  H2_CHECK_LAUNCH();
  h->gpu_launches += 1;
  int has[64];
  if (h->nranks > 1) {  // sharded lists hold the rank's own rows: a level has a pair on SOME rank
    Scratch all(sizeof(int) * 64 * h->nranks, s);
    comm_allgather(h->comm, hasd.p, all.p, sizeof(int) * 64, s);
    std::vector<int> v((size_t)64 * h->nranks);
    H2_CUDA_TRY(cudaMemcpyAsync(v.data(), all.p, sizeof(int) * v.size(), cudaMemcpyDeviceToHost, s));
    comm_sync(h->comm, s);
    for (int l = 0; l < 64; l++) {
      has[l] = 0;
      for (int q = 0; q < h->nranks; q++) has[l] |= v[(size_t)q * 64 + l];
    }
  } else {
    H2_CUDA_TRY(cudaMemcpyAsync(has, hasd.p, sizeof(int) * 64, cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaStreamSynchronize(s));
  }
  if (job.active) H2_CUDA_TRY(cudaStreamSynchronize(job.stream));
  std::vector<int> chosen(64, 0);  // per virtual level (l, l + 32)
  // trials of a level are in increasing m: keep the first pass
  auto take = [&](CalibSet& set) {
    for (int t = 0; t < set.T; t++)
      if (set.pass_h[t] && !chosen[set.lv[t]]) chosen[set.lv[t]] = set.mv[t];
  };
  take(job.p0);
  // the split phase 1 is awaited only when a level holding a pair has no passing phase-0 trial (all
  // phase-0 trials of every level are in job.p0, so its passes are final)
  bool awaited = !job.split;
  if (job.split)
    for (int t = 0; t < job.p1.T && !awaited; t++)
      if (has[job.p1.lv[t] & 31] && !chosen[job.p1.lv[t]]) awaited = true;
  if (job.split && awaited) H2_CUDA_TRY(cudaStreamSynchronize(job.stream2));
  if (awaited) take(job.p1);
  // release the buffers on h->stream (ordered after the synchronisation above); an unawaited phase 1
  // releases its own on stream2 (the pool reuses them only after stream2 has passed the release)
  for (CalibSet* set : {&job.p0, &job.p1}) {
    const cudaStream_t rs = (set == &job.p1 && !awaited) ? job.stream2 : s;
    set->work.s = set->params.s = set->outs.s = rs;
    set->work = Scratch();
    set->params = Scratch();
    set->outs = Scratch();
  }
  job.passed.s = (job.split && !awaited) ? job.stream2 : s;  // (an unawaited phase 1 still reads it)
  job.passed = Scratch();
  job.active = false;
  int r = 1;
  for (int l = 1; l <= h->depth; l++)
    for (int vl : {l, l + 32})
      if (has[l] && chosen[vl]) r = (int)std::max<long long>(r, grid_size(h->d, chosen[vl]));
  return r;
}

CalibJob::~CalibJob() {
  if (active && stream) cudaStreamSynchronize(stream);  // error path: the trials may still run
  if (active && stream2) cudaStreamSynchronize(stream2);
}

}  // namespace h2
