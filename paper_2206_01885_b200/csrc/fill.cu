// fill.cu -- a9/a10: coupling blocks B_ij = K(X^_i, X^_j) over the admissible pairs and dense
// nearfield blocks K(X_i, X_j) over the leaf nearfield pairs (Algorithm 2, PAPER.md P:496-503;
// reading G1).  Symmetric kernels: only i < j (coupling) and i <= j (nearfield) are stored, each
// block row-major, blocks concatenated in CSR pair order.
//
// The fill is FP64 / HBM-write bound (8 B stored per kernel evaluation).
//  * nearfield (a10): the block space is cut into warp UNITS of one block (a row chunk x up to
//    32*CW columns, ~kWarpUnitEntries entries); a persistent grid of warps walks the units.  A lane
//    keeps CW column points in registers, rows are broadcast, stores of a row are coalesced and
//    streaming; no CTA barrier is involved, so the loop is the kernel evaluation itself.  Big and
//    small blocks are balanced alike (unit -> pair map precomputed).
//  * coupling (a9): k_i x k_j blocks are small (ranks <= r): one warp per pair, lanes over columns
//    (column skeleton coordinates in registers), rows broadcast.
#include <climits>
#include <cstdlib>

#include "h2_internal.cuh"

namespace h2 {

constexpr int kFillThreads = 256;
#ifndef H2_NF_THREADS
#define H2_NF_THREADS 128
#endif
// threads of a nearfield-fill CTA; the per-SM register budget is kept (MINB scaled): smaller CTAs
// let a concurrent main-stream CTA displace less of an SM's fill work
constexpr int kNfThreads = H2_NF_THREADS;
constexpr int kNfScale = 256 / kNfThreads;

// ---- symmetric-once pair lists over the CSR ----------------------------------------------------
// a pair is stored (and applied by the matvec) by the rank owning its row: nbegin[i] in [p_lo, p_hi).
// Symmetric: i < j (coupling), i <= j (nearfield); non-symmetric: every ordered pair (the column
// ranks kc of the coupling blocks are the column-basis ranks).
// a warp per CSR row (grid-stride over rows), lanes over the row's entries: the row is known
// without a per-entry binary search over the offsets (round 2: the search's dependent loads made
// these two kernels ~0.2-0.4 ms per list on configs[1] and configs[4])
// flag[e] = 1 when CSR entry e is a stored pair, size[e] its block's entry count (0 otherwise)
__global__ void pair_flag_kernel(int mode, int nonsym, int nnodes, int64_t m, const int64_t* __restrict__ off,
                                 const int* __restrict__ idx, const int* __restrict__ k, const int* __restrict__ kc,
                                 const int* __restrict__ nbegin, const int* __restrict__ nend, int p_lo, int p_hi,
                                 int64_t* flag, int64_t* size) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (w0 == 0 && lane == 0) flag[m] = size[m] = 0;
  for (int64_t i = w0; i < nnodes; i += nw) {
    const int64_t e0 = off[i], e1 = off[i + 1];
    if (e0 == e1) continue;
    const bool own = nbegin[i] >= p_lo && nbegin[i] < p_hi;
    const bool ki = mode != 0 || k[i] > 0;
    const int64_t si = mode == 0 ? (int64_t)k[i] : (int64_t)(nend[i] - nbegin[i]);
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const int j = idx[e];
      const bool f = own && (mode == 0 ? ((nonsym || j > i) && ki && kc[j] > 0) : (nonsym || j >= i));
      flag[e] = f;
      size[e] = f ? si * (mode == 0 ? (int64_t)kc[j] : (int64_t)(nend[j] - nbegin[j])) : 0;
    }
  }
}

// pairs[pos[e]] = (i, j) and voff[pos[e]] = the scanned size of every stored CSR entry e; voff[np] = total
__global__ void pair_emit_kernel(int nnodes, int64_t m, const int64_t* __restrict__ off,
                                 const int* __restrict__ idx, const int64_t* __restrict__ pos,
                                 const int64_t* __restrict__ spos, int2* pairs, int64_t* voff) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (w0 == 0 && lane == 0) voff[pos[m]] = spos[m];
  for (int64_t i = w0; i < nnodes; i += nw) {
    const int64_t e0 = off[i], e1 = off[i + 1];
    if (e0 == e1) continue;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const int64_t o = pos[e];
      if (pos[e + 1] == o) continue;
      pairs[o] = make_int2((int)i, idx[e]);
      voff[o] = spos[e];
    }
  }
}

// ---- nearfield units (warp-level) ------------------------------------------------------------
// A unit is (pair, row chunk, column chunk) of one block and is processed by ONE warp, without
// CTA barriers: lane l owns the columns c0 + l + 32 s (s < CW), whose coordinates stay in
// registers; rows are streamed with warp-uniform (broadcast) loads; slot s stores at a fixed
// offset of 256 s bytes from the lane's row pointer.  The inner loop is the kernel evaluation.
__host__ __device__ constexpr int warp_slots(int D) { return D <= 2 ? 8 : (D <= 3 ? 5 : (D <= 5 ? 3 : 2)); }

// H2_FILL_VARIANT (tuning knob, read once): selects the (slots, clamp, min blocks) instantiation of the
// D = 2 nearfield kernel; 0 = default (8 slots, 6 CTAs of 128 threads per SM at 80 registers: round 2
// measured config 4 builds of 18.9 ms against 19.7 for the round-1 default, variant 7, at 124 registers
// and 4 CTAs per SM -- more resident warps hide the fill's latency, and each main-stream CTA displaces
// a smaller share of an SM's fill throughput).
static int nf_variant() {
  static const int v = [] {
    const char* e = getenv("H2_FILL_VARIANT");
    return e ? atoi(e) : 0;
  }();
  return v;
}
static int nf_slots(int d) {
  if (d != 2) return warp_slots(d);
  const int v = nf_variant();
  switch (v) {  // the column slots CW of each variant's instantiation (launch_fill_kid)
    case 1: case 2: return 4;
    case 3: return 6;
    case 5: return 2;
    default: return 8;
  }
}


__global__ void nf_units_kernel(int wc, int64_t np, const int2* __restrict__ pairs, const int* __restrict__ nbegin,
                                const int* __restrict__ nend, int64_t* units) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= np; p += (int64_t)gridDim.x * blockDim.x) {
    if (p == np) {
      units[p] = 0;
      continue;
    }
    int2 pr = pairs[p];
    int R, nrb, ncb;
    unit_shape(nend[pr.x] - nbegin[pr.x], nend[pr.y] - nbegin[pr.y], wc, R, nrb, ncb);
    units[p] = (int64_t)nrb * ncb;
  }
}

// matvec items (matvec.cu): one per column chunk of a nearfield block, covering all its rows
__global__ void nf_items_kernel(int wc, int64_t np, const int2* __restrict__ pairs, const int* __restrict__ nbegin,
                                const int* __restrict__ nend, int64_t* items) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= np; p += (int64_t)gridDim.x * blockDim.x)
    items[p] = p == np ? 0 : (int64_t)((nend[pairs[p].y] - nbegin[pairs[p].y] + wc - 1) / wc);
}

__global__ void unit_map_kernel(int64_t np, const int64_t* __restrict__ uoff, int* umap) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np; p += (int64_t)gridDim.x * blockDim.x)
    for (int64_t u = uoff[p]; u < uoff[p + 1]; u++) umap[u] = (int)p;
}

// one unit's rows [r0, r1) over NS column slots: NS independent evaluation chains per row, no
// control flow between them (so the compiler interleaves them), next row's point prefetched.
// Coordinates are pre-scaled (kernel_cscale), so sq is the kernel's own argument.
template <int D, int KID, int NS, bool CL>
__device__ __forceinline__ void nf_unit_rows(const double* __restrict__ xr, int64_t n, const double (&xb)[8][D],
                                             bool last_ok, int r0, int r1, int nj, double* o,
                                             const double* __restrict__ tab) {
  double xa[D];
#pragma unroll
  for (int c = 0; c < D; c++) xa[c] = xr[c * n + r0];  // warp-uniform address: one broadcast
  for (int row = r0; row < r1; row++, o += nj) {
    double xn[D];
    const int rn = row + 1 < r1 ? row + 1 : row;
#pragma unroll
    for (int c = 0; c < D; c++) xn[c] = xr[c * n + rn];
    double v[NS];
#pragma unroll
    for (int s = 0; s < NS; s++) {
      if constexpr (KID == H2_KERNEL_COSDOT) {  // cos(x . y) on unscaled coordinates (cs = 1)
        double dt = 0.0;
#pragma unroll
        for (int c = 0; c < D; c++) dt = fma(xa[c], xb[s][c], dt);
        v[s] = kernel_cosdot(dt);
      } else {
        double sq = kFillBias;
#pragma unroll
        for (int c = 0; c < D; c++) {
          const double df = xa[c] - xb[s][c];
          sq = fma(df, df, sq);
        }
        v[s] = kernel_fill<KID, CL>(sq, tab);
      }
    }
#pragma unroll
    for (int s = 0; s < NS; s++)  // slots before the last are full (see nslot)
      if (s < NS - 1 || last_ok) __stcs(o + 32 * s, v[s]);
#pragma unroll
    for (int c = 0; c < D; c++) xa[c] = xn[c];
  }
}

// MINB: minimum resident CTAs per SM of 256 threads' worth (scaled by kNfScale); MINB >= 10 means
// MINB / 10 CTAs of kNfThreads directly (the register-capped variants of H2_FILL_VARIANT 6-8)
template <int D, int KID, int CW, int CL, int MINB>
__global__ void __launch_bounds__(kNfThreads, MINB >= 10 ? MINB / 10 : MINB * kNfScale) nf_fill_kernel(int64_t nunits, const int* __restrict__ umap,
                                                                     const int64_t* __restrict__ uoff,
                                                                     const int2* __restrict__ pairs,
                                                                     const int64_t* __restrict__ voff,
                                                                     const int* __restrict__ nbegin,
                                                                     const int* __restrict__ nend,
                                                                     const double* __restrict__ X,
                                                                     const double* __restrict__ Xr, int64_t n,
                                                                     double* __restrict__ out, int upc,
                                                                     unsigned long long* ctl) {
  static_assert(CW >= 1 && CW <= 8, "1..8 column slots");
  constexpr int WC = 32 * CW;
  __shared__ double tab[kFillTab];
  for (int e = threadIdx.x; e < kFillTab; e += kNfThreads) tab[e] = kExp2Tab2048[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // Work is taken by warps in chunks of upc consecutive units from a global counter (ctl[0]).
  // While the main stream's level kernels still run (ctl[1] == 0) a warp does one chunk and
  // exits, so fill CTAs are short-lived and free their SM slots quickly; once the main stream has
  // passed a9 (it sets ctl[1]) the resident warps keep taking chunks until the work is done and
  // the CTAs launched after that find the counter exhausted and leave at once.
  const int64_t nchunks = (nunits + upc - 1) / upc;
  for (;;) {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(ctl, 1ull);
    c = __shfl_sync(0xffffffffu, c, 0);
    if ((int64_t)c >= nchunks) break;
    const int64_t u_end = ((int64_t)c + 1) * upc < nunits ? ((int64_t)c + 1) * upc : nunits;
  for (int64_t u = (int64_t)c * upc; u < u_end; u++) {
    const int p = umap[u];
    const int2 pr = pairs[p];
    const int bi = nbegin[pr.x], bj = nbegin[pr.y];
    const int ni = nend[pr.x] - bi, nj = nend[pr.y] - bj;
    int R, nrb, ncb;
    unit_shape(ni, nj, WC, R, nrb, ncb);
    const int loc = (int)(u - uoff[p]);
    const int rb = loc / ncb, cb = loc - rb * ncb;
    const int r0 = rb * R, c0 = cb * WC;
    const int r1 = ni < r0 + R ? ni : r0 + R;
    double xb[8][D];

#pragma unroll
    for (int s = 0; s < 8; s++) {
      const int col = c0 + lane + 32 * s;
      const bool ok = s < CW && col < nj;
#pragma unroll
      for (int c = 0; c < D; c++) xb[s][c] = ok ? X[c * n + bj + col] : 0.0;
    }
    double* o = out + voff[p] + (int64_t)r0 * nj + c0 + lane;
    const double* xr = Xr + bi;  // rows: kappa's first argument (= X but for the shifted multiquadric)
    int nslot = (nj - c0 + 31) >> 5;  // warp-uniform: slots with at least one column
    if (nslot > CW) nslot = CW;
    const bool last_ok = c0 + lane + 32 * (nslot - 1) < nj;  // only the last slot can be partial
    switch (nslot) {
      case 1: nf_unit_rows<D, KID, 1, CL != 0>(xr, n, xb, last_ok, r0, r1, nj, o, tab); break;
      case 2: nf_unit_rows<D, KID, (CW < 2 ? CW : 2), CL != 0>(xr, n, xb, last_ok, r0, r1, nj, o, tab); break;
      case 3: nf_unit_rows<D, KID, (CW < 3 ? CW : 3), CL != 0>(xr, n, xb, last_ok, r0, r1, nj, o, tab); break;
      case 4: nf_unit_rows<D, KID, (CW < 4 ? CW : 4), CL != 0>(xr, n, xb, last_ok, r0, r1, nj, o, tab); break;
      case 5: nf_unit_rows<D, KID, (CW < 5 ? CW : 5), CL != 0>(xr, n, xb, last_ok, r0, r1, nj, o, tab); break;
      case 6: nf_unit_rows<D, KID, (CW < 6 ? CW : 6), CL != 0>(xr, n, xb, last_ok, r0, r1, nj, o, tab); break;
      case 7: nf_unit_rows<D, KID, (CW < 7 ? CW : 7), CL != 0>(xr, n, xb, last_ok, r0, r1, nj, o, tab); break;
      default: nf_unit_rows<D, KID, CW, CL != 0>(xr, n, xb, last_ok, r0, r1, nj, o, tab); break;
    }
  }
    if (*reinterpret_cast<volatile unsigned long long*>(ctl + 1) == 0) break;
  }
}

// ---- coupling: S warps per 32 consecutive pairs, entries flattened -----------------------------
// Coupling blocks are small (k_i x k_j, ranks of a few to a few tens), so per-pair work is a
// chain of dependent loads (pair -> ranks, offset -> skeleton indices -> coordinates).  A group of
// 32 consecutive pairs is taken by S warps at once: lane t of each loads pair t's metadata (one
// round of latency for all 32), a warp scan gives the pairs' entry prefix, then warp `sl` of the
// S walks every S-th 32-entry row of the group's concatenated entries -- which are also
// consecutive in the output (blocks are stored in pair order), so every store instruction writes
// 256 contiguous bytes -- each lane gathering its entry's two skeleton points (L2-resident) and
// evaluating the kernel.  S (host: ~256 entries per warp) sets how many independent dependent-load
// chains are in flight: with one warp per group a group of ~8K entries was a 256-step serial chain
// and the whole fill a few thousand such chains (latency-bound, ~1 TB/s).
template <int D, int KID>
__global__ void __launch_bounds__(kFillThreads) cp_fill_kernel(int64_t np, const int2* __restrict__ pairs,
                                                               const int64_t* __restrict__ voff,
                                                               const int* __restrict__ k, const int* __restrict__ sk,
                                                               const int* __restrict__ kc,
                                                               const int* __restrict__ skc, int r,
                                                               const double* __restrict__ Xf,
                                                               const double* __restrict__ X, int64_t n,
                                                               double cs, int S, double* __restrict__ out) {
  __shared__ double tab[kFillTab];
  for (int e = threadIdx.x; e < kFillTab; e += blockDim.x) tab[e] = kExp2Tab2048[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nunits = ((np + 31) >> 5) * S;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t us = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; us < nunits; us += nw) {
    const int64_t u = us / S;
    const int sl = (int)(us - u * S);
    const int64_t p = (u << 5) + lane;
    int pi = 0, pj = 0, ki = 0, kj = 0;
    if (p < np) {
      const int2 pr = pairs[p];
      pi = pr.x;
      pj = pr.y;
      ki = k[pi];
      kj = kc[pj];
    }
    int sz = ki * kj, pre = sz;  // inclusive scan of the pairs' sizes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += v;
    }
    const int total = __shfl_sync(0xffffffffu, pre, 31);
    pre -= sz;  // exclusive
    double* o = out + voff[u << 5];
    for (int e0 = 32 * sl; e0 < total; e0 += 32 * S) {  // warp-uniform trip count: every shuffle is converged
      const int e = e0 + lane;
      // this entry's pair: the largest q with pre[q] <= e (size-0 pairs never win)
      int q = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int cand = q + step;
        const int pc = __shfl_sync(0xffffffffu, pre, cand & 31);
        if (cand < 32 && pc <= e) q = cand;
      }
      const int pre_q = __shfl_sync(0xffffffffu, pre, q);
      const int i_q = __shfl_sync(0xffffffffu, pi, q), j_q = __shfl_sync(0xffffffffu, pj, q);
      const int kj_q = __shfl_sync(0xffffffffu, kj, q);
      if (e >= total) continue;
      const int loc = e - pre_q, row = loc / kj_q, col = loc - row * kj_q;
      // B_ij = K(X^_i^(row), X^_j^(col)): rows from the row skeletons (first argument, Xf), columns
      // from the column skeletons (the same arrays on the symmetric path)
      const int a = sk[(int64_t)i_q * r + row], b = skc[(int64_t)j_q * r + col];
      if constexpr (KID == H2_KERNEL_COSDOT) {
        double dt = 0.0;
#pragma unroll
        for (int c = 0; c < D; c++) dt = fma(Xf[c * n + a], X[c * n + b], dt);
        __stcs(o + e, kernel_cosdot(dt));
      } else {
        double sq = kFillBias;
#pragma unroll
        for (int c = 0; c < D; c++) {
          const double df = Xf[c * n + a] * cs - X[c * n + b] * cs;
          sq = fma(df, df, sq);
        }
        __stcs(o + e, kernel_fill<KID, true>(sq, tab));
      }
    }
  }
}

// coordinates pre-scaled by kernel_cscale for the nearfield fill (SoA, like h->X)
__global__ void scale_coords_kernel(int64_t m, const double* __restrict__ X, double cs, double* __restrict__ Xs) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
    Xs[t] = X[t] * cs;
}

// H2_NF_UPW (tuning knob, read once): nearfield units per chunk (see nf_fill_kernel).  The
// nearfield fill runs CONCURRENTLY with the HiDR / ID stages (api.cu), on a low-priority stream;
// while they run, a fill warp does one chunk and its CTA retires (~0.05 ms), so the latency-bound
// level kernels of the high-priority stream get SM slots quickly; after a9 the fill CTAs persist.
static int nf_units_per_warp() {
  static const int v = [] {
    const char* e = getenv("H2_NF_UPW");
    const int u = e ? atoi(e) : 8;
    return u > 0 ? u : 8;
  }();
  return v;
}

// H2_NF_SMEM (tuning knob, read once): dynamic shared memory requested by (and unused in) the
// nearfield kernel, to cap how many of its CTAs an SM holds and leave room for the concurrent
// level kernels of the main stream.
static int nf_smem_reserve() {
  static const int v = [] {
    const char* e = getenv("H2_NF_SMEM");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <class K, class... A>
static void launch_nf(K kernel, unsigned g, cudaStream_t s, A... args) {
  const int sm = nf_smem_reserve();
  if (sm > 48 * 1024) H2_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  kernel<<<g, kNfThreads, sm, s>>>(args...);
}

template <int KID>
static void launch_fill_kid(const h2_handle* h, cudaStream_t s, int mode, int64_t nwork, int64_t np, const int* umap,
                            const int64_t* uoff, const int2* pairs, const int64_t* voff, const double* Xs,
                            const double* Xrs, double cs, double* out, unsigned long long* ctl) {
  if (mode == 1) {
    const bool clamp = fill_needs_clamp(h->kid, h->d, h->W, cs);
    const int upw = nf_units_per_warp();
    constexpr int wpc = kNfThreads / 32;
    const int64_t blocks = (nwork + wpc * upw - 1) / (wpc * upw);  // one chunk per warp
    unsigned g = (unsigned)(blocks < ((int64_t)1 << 30) ? blocks : ((int64_t)1 << 30));
#define H2_NF_ARGS nwork, umap, uoff, pairs, voff, h->nbegin, h->nend, Xs, Xrs, h->n, out, upw, ctl
    switch (h->d) {
      case 2:
        switch (nf_variant()) {  // tuning variants of the D = 2 kernel (CW, clamp, MINB)
          case 1: launch_nf(nf_fill_kernel<2, KID, 4, 1, 4>, g, s, H2_NF_ARGS); break;
          case 2: launch_nf(nf_fill_kernel<2, KID, 4, 1, 2>, g, s, H2_NF_ARGS); break;
          case 3: launch_nf(nf_fill_kernel<2, KID, 6, 1, 2>, g, s, H2_NF_ARGS); break;
          case 4: launch_nf(nf_fill_kernel<2, KID, 8, 1, 1>, g, s, H2_NF_ARGS); break;
          case 5: launch_nf(nf_fill_kernel<2, KID, 2, 1, 4>, g, s, H2_NF_ARGS); break;
          case 6: launch_nf(nf_fill_kernel<2, KID, 8, 0, 50>, g, s, H2_NF_ARGS); break;  // 5 CTAs/SM, 96 regs
          case 7: launch_nf(nf_fill_kernel<2, KID, 8, 0, 2>, g, s, H2_NF_ARGS); break;   // round 1: 4 CTAs/SM, 124 regs
          case 8: launch_nf(nf_fill_kernel<2, KID, 8, 0, 70>, g, s, H2_NF_ARGS); break;  // 7 CTAs/SM, 72 regs
          case 9: launch_nf(nf_fill_kernel<2, KID, 8, 0, 80>, g, s, H2_NF_ARGS); break;  // 8 CTAs/SM, 64 regs
          default:  // 8 slots, 6 CTAs of 128 threads per SM (80 registers, no spill): round 2's measured best
            if (clamp) launch_nf(nf_fill_kernel<2, KID, 8, 1, 60>, g, s, H2_NF_ARGS);
            else launch_nf(nf_fill_kernel<2, KID, 8, 0, 60>, g, s, H2_NF_ARGS);
            break;
        }
        break;
#define H2_NF_CASE(DD) \
  case DD:             \
    launch_nf(nf_fill_kernel<DD, KID, warp_slots(DD), 1, 2>, g, s, H2_NF_ARGS); break;
      H2_NF_CASE(1) H2_NF_CASE(3) H2_NF_CASE(4)
      H2_NF_CASE(5) H2_NF_CASE(6) H2_NF_CASE(7) H2_NF_CASE(8)
#undef H2_NF_CASE
#undef H2_NF_ARGS
    }
  } else {
    // S warps per 32 pairs (~256 entries per warp), 8 warps per CTA
    const int64_t groups = (np + 31) / 32;
    const int64_t epg = (h->cp_entries + groups - 1) / groups;
    static const int64_t epw = [] {  // H2_CP_EPW (tuning knob): target entries per warp
      const char* e = getenv("H2_CP_EPW");
      const long long v = e ? atoll(e) : 256;
      return (int64_t)(v > 0 ? v : 256);
    }();
    const int S = (int)(epg / epw < 1 ? 1 : (epg / epw > 64 ? 64 : epg / epw));
    const int64_t blocks = (groups * S + 7) / 8;
    // skeleton coordinates: the points, or the Chebyshev nodes of the interpolation baseline
    const double* cXf = h->Xq ? h->Xq : h->Xf;
    const double* cX = h->Xq ? h->Xq : h->X;
    const int64_t cn = h->Xq ? h->nq : h->n;
    unsigned g = (unsigned)(blocks < ((int64_t)1 << 30) ? blocks : ((int64_t)1 << 30));
    switch (h->d) {
#define H2_CP_CASE(DD)                                                                                        \
  case DD:                                                                                                    \
    cp_fill_kernel<DD, KID><<<g, kFillThreads, 0, s>>>(np, pairs, voff, h->k, h->sk, h->k_col, h->sk_col, h->r,  \
                                                       cXf, cX, cn, cs, S, out);                               \
    break;
      H2_CP_CASE(1) H2_CP_CASE(2) H2_CP_CASE(3) H2_CP_CASE(4)
      H2_CP_CASE(5) H2_CP_CASE(6) H2_CP_CASE(7) H2_CP_CASE(8)
#undef H2_CP_CASE
    }
  }
}

static void launch_fill(const h2_handle* h, cudaStream_t s, int mode, int64_t nwork, int64_t np, const int* umap,
                        const int64_t* uoff, const int2* pairs, const int64_t* voff, const double* Xs,
                        const double* Xrs, double* out, unsigned long long* ctl = nullptr) {
  if (nwork < 1) return;
  const double cs = kernel_cscale(h->kid, h->kp);
#define H2_FILL_KID(K) launch_fill_kid<K>(h, s, mode, nwork, np, umap, uoff, pairs, voff, Xs, Xrs, cs, out, ctl)
  switch (h->kid) {
    case H2_KERNEL_COULOMB: H2_FILL_KID(H2_KERNEL_COULOMB); break;
    case H2_KERNEL_GAUSSIAN: H2_FILL_KID(H2_KERNEL_GAUSSIAN); break;
    case H2_KERNEL_MATERN32: H2_FILL_KID(H2_KERNEL_MATERN32); break;
    case H2_KERNEL_LAPLACE: H2_FILL_KID(H2_KERNEL_LAPLACE); break;
    case H2_KERNEL_BUMP: H2_FILL_KID(H2_KERNEL_BUMP); break;
    case H2_KERNEL_MQSHIFT: H2_FILL_KID(H2_KERNEL_MQSHIFT); break;
    default: H2_FILL_KID(H2_KERNEL_COSDOT); break;
  }
#undef H2_FILL_KID
}

// builds the symmetric-once pair list of one class (CSR order) with entry offsets, on stream s
static void make_pairs(h2_handle* h, cudaStream_t s, int mode, int64_t& np, int2*& pairs, int64_t*& voff,
                       int64_t& entries) {
  const int nn = h->nnodes;
  const int64_t* off = mode == 0 ? h->il_off : h->nf_off;
  const int* idx = mode == 0 ? h->il_idx : h->nf_idx;
  const int64_t m = mode == 0 ? h->n_il : h->n_nf;
  // flags and block sizes per CSR entry, both scanned, the two totals read back at once: the pair
  // count and the entry count (one host synchronisation), then the pairs and their offsets
  Scratch fs(sizeof(int64_t) * 2 * (m + 1), s), ps(sizeof(int64_t) * 2 * (m + 1), s);
  int64_t *flag = fs.as<int64_t>(), *size = flag + (m + 1);
  int64_t *pos = ps.as<int64_t>(), *spos = pos + (m + 1);
  pair_flag_kernel<<<grid_for((int64_t)nn * 32, 256), 256, 0, s>>>(mode, h->nonsym, nn, m, off, idx, h->k, h->k_col,
                                                                   h->nbegin, h->nend, h->p_lo, h->p_hi, flag, size);
  scan_excl_i64(flag, pos, m + 1, s);
  scan_excl_i64(size, spos, m + 1, s);
  H2_CHECK_LAUNCH();
  {
    thread_local int64_t* tot = nullptr;  // page-locked, per host thread
    if (!tot) H2_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&tot), 2 * sizeof(int64_t)));
    H2_CUDA_TRY(cudaMemcpyAsync(tot, pos + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaMemcpyAsync(tot + 1, spos + m, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaStreamSynchronize(s));
    np = tot[0];
    entries = tot[1];
  }
  pairs = halloc<int2>(h, np);
  voff = halloc<int64_t>(h, np + 1);
  pair_emit_kernel<<<grid_for((int64_t)nn * 32, 256), 256, 0, s>>>(nn, m, off, idx, pos, spos, pairs, voff);
  H2_CHECK_LAUNCH();
  h->gpu_launches += 2;  // + the scans (prims.cu counts its own launches)
}

static int64_t pool_available() {
  size_t fr = 0, tot = 0;
  H2_CUDA_TRY(cudaMemGetInfo(&fr, &tot));
  return (int64_t)fr + (int64_t)cached_free_bytes();
}

static int64_t store_budget(int64_t budget) { return budget > 0 ? budget : pool_available() - ((int64_t)4 << 30); }

// a10, issued right after the lists (it needs only the tree and the nearfield list) on the side
// stream `side`, which first waits for everything already queued on h->stream.  Storage policy
// AUTO stores the nearfield class first when it fits the budget (it is the class a matvec
// re-evaluates at the highest cost per entry), then the coupling class in what remains.
void fill_nearfield_begin(h2_handle* h, cudaStream_t side, int storage, int64_t budget, NfJob& job) {
  job.side = side;
  H2_CUDA_TRY(cudaEventCreateWithFlags(&job.forked, cudaEventDisableTiming));
  H2_CUDA_TRY(cudaEventCreateWithFlags(&job.done, cudaEventDisableTiming));
  if (h->timing) {
    H2_CUDA_TRY(cudaEventCreate(&job.t0));
    H2_CUDA_TRY(cudaEventCreate(&job.t1));
  }
  H2_CUDA_TRY(cudaEventRecord(job.forked, h->stream));
  H2_CUDA_TRY(cudaStreamWaitEvent(side, job.forked, 0));
  make_pairs(h, side, 1, h->n_np, h->np_pairs, h->np_off, h->np_entries);
  const int64_t nb = h->np_entries * 8;
  const bool store_np = storage == H2_STORE_ALL || (storage == H2_STORE_AUTO && nb <= store_budget(budget));
  if (store_np) {
    h->np_val = halloc<double>(h, h->np_entries + 2);  // +2: the matvec's 16-byte-aligned bulk copies
    h->np_stored = 1;
    job.stored_bytes = nb;
  }
  int64_t nunits = 0;
  if (store_np && h->n_np > 0) {
    const int64_t np = h->n_np;
    // the fill's units and the matvec's items per pair, both scanned, one readback of the totals
    Scratch units(sizeof(int64_t) * 2 * (np + 1), side);
    int64_t* items = units.as<int64_t>() + (np + 1);
    h->nf_wc = 32 * nf_slots(h->d);
    h->nf_uoff = halloc_on<int64_t>(h, np + 1, side);
    h->nf_ioff = halloc_on<int64_t>(h, np + 1, side);
    nf_units_kernel<<<grid_for(np + 1, 256), 256, 0, side>>>(h->nf_wc, np, h->np_pairs, h->nbegin, h->nend,
                                                             units.as<int64_t>());
    nf_items_kernel<<<grid_for(np + 1, 256), 256, 0, side>>>(h->nf_wc, np, h->np_pairs, h->nbegin, h->nend, items);
    scan_excl_i64(units.as<int64_t>(), h->nf_uoff, np + 1, side);
    scan_excl_i64(items, h->nf_ioff, np + 1, side);
    H2_CHECK_LAUNCH();
    {
      thread_local int64_t* tot = nullptr;  // page-locked, per host thread
      if (!tot) H2_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&tot), 2 * sizeof(int64_t)));
      H2_CUDA_TRY(cudaMemcpyAsync(tot, h->nf_uoff + np, sizeof(int64_t), cudaMemcpyDeviceToHost, side));
      H2_CUDA_TRY(cudaMemcpyAsync(tot + 1, h->nf_ioff + np, sizeof(int64_t), cudaMemcpyDeviceToHost, side));
      H2_CUDA_TRY(cudaStreamSynchronize(side));
      nunits = tot[0];
      h->nf_nitems = tot[1];
    }
    h->nf_nunits = nunits;
    h->nf_umap = halloc_on<int>(h, nunits > 0 ? nunits : 1, side);
    unit_map_kernel<<<grid_for(np, 256), 256, 0, side>>>(np, h->nf_uoff, h->nf_umap);
    h->nf_imap = halloc_on<int>(h, h->nf_nitems > 0 ? h->nf_nitems : 1, side);
    unit_map_kernel<<<grid_for(np, 256), 256, 0, side>>>(np, h->nf_ioff, h->nf_imap);
    H2_CHECK_LAUNCH();
    h->gpu_launches += 4;
  }
  if (h->timing) H2_CUDA_TRY(cudaEventRecord(job.t0, side));
  if (nunits > 0) {
    const int64_t m = (int64_t)h->n * h->d;
    const bool shifted = h->Xf != h->X;  // the rows' coordinates differ (shifted multiquadric)
    job.xs = Scratch(sizeof(double) * (size_t)m * (shifted ? 2 : 1), side);
    scale_coords_kernel<<<grid_for(m, 256), 256, 0, side>>>(m, h->X, kernel_cscale(h->kid, h->kp), job.xs.as<double>());
    if (shifted)
      scale_coords_kernel<<<grid_for(m, 256), 256, 0, side>>>(m, h->Xf, kernel_cscale(h->kid, h->kp),
                                                              job.xs.as<double>() + m);
    // chunk counter + "main stream past a9" flag (set at once when the fill runs on the main stream)
    job.ctl = Scratch(2 * sizeof(unsigned long long), side);
    H2_CUDA_TRY(cudaMemsetAsync(job.ctl.p, 0, 2 * sizeof(unsigned long long), side));
    if (side == h->stream) H2_CUDA_TRY(cudaMemsetAsync(job.ctl.as<unsigned long long>() + 1, 1, 1, side));
    launch_fill(h, side, 1, nunits, h->n_np, h->nf_umap, h->nf_uoff, h->np_pairs, h->np_off, job.xs.as<double>(),
                job.xs.as<double>() + (shifted ? m : 0), h->np_val, job.ctl.as<unsigned long long>());
    h->gpu_launches += 1;
    H2_CHECK_LAUNCH();
    h->gpu_launches += 1;
  }
  if (h->timing) H2_CUDA_TRY(cudaEventRecord(job.t1, side));
  H2_CUDA_TRY(cudaEventRecord(job.done, side));
  job.active = true;
}

// a9 on h->stream (needs the skeletons of the ID sweep)
void fill_coupling(h2_handle* h, int storage, int64_t budget, const NfJob& job) {
  cudaStream_t s = h->stream;
  make_pairs(h, s, 0, h->n_cp, h->cp_pairs, h->cp_off, h->cp_entries);
  const int64_t cb = h->cp_entries * 8;
  const bool store_cp = storage == H2_STORE_ALL || (storage == H2_STORE_AUTO && cb <= store_budget(budget) -
                                                                                    (budget > 0 ? job.stored_bytes : 0));
  cudaEvent_t ev[2];
  if (h->timing)
    for (auto& e : ev) H2_CUDA_TRY(cudaEventCreate(&e));
  if (store_cp) {
    h->cp_val = halloc<double>(h, h->cp_entries);
    h->cp_stored = 1;
  }
  if (h->timing) H2_CUDA_TRY(cudaEventRecord(ev[0], s));
  if (store_cp && h->n_cp > 0) {
    launch_fill(h, s, 0, h->n_cp, h->n_cp, nullptr, nullptr, h->cp_pairs, h->cp_off, h->X, h->Xf, h->cp_val);
    H2_CHECK_LAUNCH();
    h->gpu_launches += 1;
  }
  // the main stream is past its level kernels: the concurrent nearfield fill may keep its SMs
  if (job.ctl.p && job.side != s)
    H2_CUDA_TRY(cudaMemsetAsync(static_cast<unsigned long long*>(job.ctl.p) + 1, 1, 1, s));
  if (h->timing) {
    H2_CUDA_TRY(cudaEventRecord(ev[1], s));
    H2_CUDA_TRY(cudaEventSynchronize(ev[1]));
    float a = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    h->stage_ms[6] = a;
    for (auto& e : ev) cudaEventDestroy(e);
  }
}

// joins the side stream into h->stream; the nearfield scratch is released on h->stream after
// the join (so no later allocation ever waits on the fill)
void fill_nearfield_join(h2_handle* h, NfJob& job) {
  if (!job.active) return;
  H2_CUDA_TRY(cudaStreamWaitEvent(h->stream, job.done, 0));
  job.xs.s = h->stream;
  job.xs = Scratch();
  job.ctl.s = h->stream;
  job.ctl = Scratch();
  job.active = false;
}

void NfJob::finish_timing(h2_handle* h) {
  if (h->timing && t0 && t1) {
    float b = 0;
    if (cudaEventElapsedTime(&b, t0, t1) == cudaSuccess) h->stage_ms[7] = b;
  }
}

NfJob::~NfJob() {
  if (active && side) cudaStreamSynchronize(side);  // error path: nothing may still use the scratch
  for (cudaEvent_t e : {forked, done, t0, t1})
    if (e) cudaEventDestroy(e);
}

// ---- sampled reads of stored entries for the parity tests ----------------------------------
__global__ void sample_kernel(int64_t count, const int32_t* kind, const int64_t* pair, const int64_t* entry,
                              const int2* cpp, const int64_t* cpo, const double* cpv, const int2* npp,
                              const int64_t* npo, const double* npv, const int* nbegin, const int* nend,
                              const int* k, const int* sk, const int* kc, const int* skc, int r, double* val,
                              int32_t* rp, int32_t* cp) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < count; s += (int64_t)gridDim.x * blockDim.x) {
    int md = kind[s];
    int64_t p = pair[s], e = entry[s];
    int2 pr = md == 0 ? cpp[p] : npp[p];
    int nj = md == 0 ? kc[pr.y] : nend[pr.y] - nbegin[pr.y];
    int row = (int)(e / nj), col = (int)(e % nj);
    val[s] = md == 0 ? cpv[cpo[p] + e] : npv[npo[p] + e];
    rp[s] = md == 0 ? sk[(int64_t)pr.x * r + row] : nbegin[pr.x] + row;
    cp[s] = md == 0 ? skc[(int64_t)pr.y * r + col] : nbegin[pr.y] + col;
  }
}

void sample_blocks(const h2_handle* h, int64_t count, const int32_t* kind, const int64_t* pair, const int64_t* entry,
                   double* value, int32_t* row_pt, int32_t* col_pt) {
  cudaStream_t s = h->stream;
  for (int64_t q = 0; q < count; q++) {
    if (kind[q] == 0 && (!h->cp_stored || pair[q] < 0 || pair[q] >= h->n_cp))
      throw Error{H2_ERR_INVALID_ARG, "coupling sample out of range or not stored"};
    if (kind[q] == 1 && (!h->np_stored || pair[q] < 0 || pair[q] >= h->n_np))
      throw Error{H2_ERR_INVALID_ARG, "nearfield sample out of range or not stored"};
    if (kind[q] != 0 && kind[q] != 1) throw Error{H2_ERR_INVALID_ARG, "sample kind must be 0 or 1"};
  }
  Scratch in(count * (4 + 8 + 8) + 64, s), out(count * (8 + 4 + 4) + 64, s);
  int32_t* dk = in.as<int32_t>();
  int64_t* dp = reinterpret_cast<int64_t*>(in.as<char>() + ((count * 4 + 15) / 16) * 16);
  int64_t* de = dp + count;
  double* dv = out.as<double>();
  int32_t* dr = reinterpret_cast<int32_t*>(dv + count);
  int32_t* dc = dr + count;
  H2_CUDA_TRY(cudaMemcpyAsync(dk, kind, 4 * count, cudaMemcpyHostToDevice, s));
  H2_CUDA_TRY(cudaMemcpyAsync(dp, pair, 8 * count, cudaMemcpyHostToDevice, s));
  H2_CUDA_TRY(cudaMemcpyAsync(de, entry, 8 * count, cudaMemcpyHostToDevice, s));
  sample_kernel<<<grid_for(count, 256), 256, 0, s>>>(count, dk, dp, de, h->cp_pairs, h->cp_off, h->cp_val,
                                                     h->np_pairs, h->np_off, h->np_val, h->nbegin, h->nend, h->k,
                                                     h->sk, h->k_col, h->sk_col, h->r, dv, dr, dc);
  H2_CHECK_LAUNCH();
  H2_CUDA_TRY(cudaMemcpyAsync(value, dv, 8 * count, cudaMemcpyDeviceToHost, s));
  H2_CUDA_TRY(cudaMemcpyAsync(row_pt, dr, 4 * count, cudaMemcpyDeviceToHost, s));
  H2_CUDA_TRY(cudaMemcpyAsync(col_pt, dc, 4 * count, cudaMemcpyDeviceToHost, s));
  H2_CUDA_TRY(cudaStreamSynchronize(s));
}

}  // namespace h2
