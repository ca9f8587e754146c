// matvec.cu -- y = K~ x with the four-pass H^2 product:
//   upward    z^_i = U_i^T x_i at leaves, z^_p = sum_c R_c^T z^_c      (levels deepest -> 1)
//   coupling  y^_i += B_ij z^_j and y^_j += B_ij^T z^_i, i < j            (stored or on the fly)
//   downward  y^_c += R_c y^_p, then y_i += U_i y^_i at leaves          (levels 1 -> deepest)
//   nearfield y_i += D_ij x_j and y_j += D_ij^T x_i, i <= j              (stored or on the fly)
// Accumulation uses fp64 atomics (order-dependent rounding only).  Used for accuracy checks.
#include <cstdlib>

#include "h2_internal.cuh"

namespace h2 {

constexpr int kMvThreads = 128;

__global__ void permute_in_kernel(const double* __restrict__ x, const int* __restrict__ perm, int64_t n, double* xt) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    xt[t] = x[perm[t]];
}

__global__ void add_kernel(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    b[t] += a[t];
}

// y[perm[t]] = yt[t] + yf[t]: the nearfield and the farfield contributions (tree order)
__global__ void permute_out_kernel(const double* __restrict__ yt, const double* __restrict__ yf,
                                   const int* __restrict__ perm, int64_t n, double* y) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    y[perm[t]] = yt[t] + yf[t];
}

__global__ void up_kernel(int base, int r, const int* __restrict__ is_leaf, const int* __restrict__ nbegin,
                          const int* __restrict__ first_child, const int* __restrict__ nchild,
                          const int* __restrict__ k, const int* __restrict__ xbar_n, const int* __restrict__ child_off,
                          const int64_t* __restrict__ u_off, const double* __restrict__ U,
                          const double* __restrict__ xt, double* zh) {
  const int i = base + blockIdx.x;
  const int ki = k[i];
  if (ki == 0) return;
  const int nx = xbar_n[i];
  const double* Ui = U + u_off[i];
  for (int c = threadIdx.x; c < ki; c += blockDim.x) {
    const double* col = Ui + (int64_t)nx * c;
    double s = 0.0;
    if (is_leaf[i]) {
      const double* xi = xt + nbegin[i];
      for (int a = 0; a < nx; a++) s += col[a] * xi[a];
    } else {
      for (int cc = 0; cc < nchild[i]; cc++) {
        int ch = first_child[i] + cc;
        const double* z = zh + (int64_t)ch * r;
        const int o = child_off[ch];
        for (int a = 0; a < k[ch]; a++) s += col[o + a] * z[a];
      }
    }
    zh[(int64_t)i * r + c] = s;
  }
}

template <int D>
__device__ __forceinline__ double kval(int kid, double p2, const double* __restrict__ Xf,
                                       const double* __restrict__ X, int64_t n, int a, int b) {
  return kernel_pts<D>(kid, p2, Xf, X, n, a, b);
}

// B_ij = K(X^_i^(row), X^_j^(col)) (stored or evaluated): y^_i += B z^_j, and for a symmetric build
// (sym: pairs stored once) also y^_j += B^T z^_i
template <int D>
__global__ void coupling_kernel(int64_t np, const int2* __restrict__ pairs, const int64_t* __restrict__ voff,
                                const double* __restrict__ B, int kid, double p2, const double* __restrict__ Xf,
                                const double* __restrict__ X, int64_t n, const int* __restrict__ k,
                                const int* __restrict__ sk, const int* __restrict__ kc, const int* __restrict__ skc,
                                int r, int sym, const double* __restrict__ zh, double* yh) {
  for (int64_t p = blockIdx.x; p < np; p += gridDim.x) {
    const int2 pr = pairs[p];
    const int i = pr.x, j = pr.y, ki = k[i], kj = kc[j];
    const double* Bp = B ? B + voff[p] : nullptr;
    const int* si = sk + (int64_t)i * r;
    const int* sj = skc + (int64_t)j * r;
    const double* zi = zh + (int64_t)i * r;
    const double* zj = zh + (int64_t)j * r;
    for (int a = threadIdx.x; a < ki; a += blockDim.x) {  // y^_i += B z^_j
      double s = 0.0;
      for (int b = 0; b < kj; b++)
        s += (Bp ? Bp[(int64_t)a * kj + b] : kval<D>(kid, p2, Xf, X, n, si[a], sj[b])) * zj[b];
      atomicAdd(yh + (int64_t)i * r + a, s);
    }
    if (sym)
      for (int b = threadIdx.x; b < kj; b += blockDim.x) {  // y^_j += B^T z^_i
        double s = 0.0;
        for (int a = 0; a < ki; a++)
          s += (Bp ? Bp[(int64_t)a * kj + b] : kval<D>(kid, p2, Xf, X, n, si[a], sj[b])) * zi[a];
        atomicAdd(yh + (int64_t)j * r + b, s);
      }
  }
}

// stored coupling blocks (k_i x k_j, small): warp per pair, lanes over columns, rows in chunks of
// 8 (eight independent loads in flight); the row dots of a chunk are warp-reduced by a transposing
// butterfly (lane l ends with row l & 7: one atomic per row) and the column contributions kept in
// registers (one atomic per column per pair): every entry read once, coalesced along the row
__global__ void __launch_bounds__(256) coupling_mv_kernel(int64_t np, const int2* __restrict__ pairs,
                                                          const int64_t* __restrict__ voff, const double* __restrict__ B,
                                                          const int* __restrict__ k, const int* __restrict__ kc, int r,
                                                          int sym, const double* __restrict__ zh, double* yh) {
  constexpr int RC = 8;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // the warp takes 32 consecutive pairs at a time; their metadata is loaded in one round (lane t
  // holds pair p0 + t) and broadcast by shuffles, so no pair waits on its own dependent loads
  for (int64_t p0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 32; p0 < np; p0 += nw * 32) {
    const int64_t pl = p0 + lane;
    int mi = 0, mj = 0, mki = 0, mkj = 0;
    long long mvo = 0;
    if (pl < np) {
      const int2 pr = pairs[pl];
      mi = pr.x;
      mj = pr.y;
      mvo = voff[pl];
      mki = k[mi];
      mkj = kc[mj];
    }
    const int cnt = np - p0 < 32 ? (int)(np - p0) : 32;
    for (int t = 0; t < cnt; t++) {
      const int i = __shfl_sync(0xffffffffu, mi, t), j = __shfl_sync(0xffffffffu, mj, t);
      const int ki = __shfl_sync(0xffffffffu, mki, t), kj = __shfl_sync(0xffffffffu, mkj, t);
      const double* Bp = B + __shfl_sync(0xffffffffu, mvo, t);
      const double* zi = zh + (int64_t)i * r;
      const double* zj = zh + (int64_t)j * r;
      double* yi = yh + (int64_t)i * r;
      double* yj = yh + (int64_t)j * r;
      for (int c0 = 0; c0 < kj; c0 += 32) {
        const int col = c0 + lane;
        const bool ok = col < kj;
        const double zc = ok ? zj[col] : 0.0;
        double acc = 0.0;
        for (int a0 = 0; a0 < ki; a0 += RC) {
          double v[RC], part[RC];
#pragma unroll
          for (int u = 0; u < RC; u++) v[u] = ok && a0 + u < ki ? Bp[(int64_t)(a0 + u) * kj + col] : 0.0;
#pragma unroll
          for (int u = 0; u < RC; u++) {
            part[u] = v[u] * zc;
            acc = fma(v[u], a0 + u < ki ? zi[a0 + u] : 0.0, acc);
          }
#pragma unroll
          for (int u = 0; u < RC; u++) {
            part[u] += __shfl_xor_sync(0xffffffffu, part[u], 16);
            part[u] += __shfl_xor_sync(0xffffffffu, part[u], 8);
          }
#pragma unroll
          for (int o = 4, w = 4; o > 0; o >>= 1, w >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int q = 0; q < w; q++) {
              const double lo = part[q], hi = part[q + w];
              part[q] = (up ? hi : lo) + __shfl_xor_sync(0xffffffffu, up ? lo : hi, o);
            }
          }
          if (lane < RC && a0 + lane < ki) atomicAdd(yi + a0 + lane, part[0]);
        }
        if (ok && sym) atomicAdd(yj + col, acc);  // y^_j += B^T z^_i (symmetric-once storage)
      }
    }
  }
}

// leaf outputs only for leaves whose first point lies in [p_lo, p_hi) (sharded: the row owner)
__global__ void down_kernel(int base, int r, const int* __restrict__ is_leaf, const int* __restrict__ nbegin,
                            const int* __restrict__ parent, const int* __restrict__ k, const int* __restrict__ xbar_n,
                            const int* __restrict__ child_off, const int64_t* __restrict__ u_off,
                            const double* __restrict__ U, int p_lo, int p_hi, double* yh, double* yt) {
  const int i = base + blockIdx.x;
  const int ki = k[i];
  if (ki == 0) return;
  const int p = parent[i];
  double* yi = yh + (int64_t)i * r;
  if (p >= 0 && k[p] > 0) {
    const int nxp = xbar_n[p], kp = k[p], o = child_off[i];
    const double* Up = U + u_off[p];
    const double* yp = yh + (int64_t)p * r;
    for (int a = threadIdx.x; a < ki; a += blockDim.x) {
      double s = 0.0;
      for (int t = 0; t < kp; t++) s += Up[o + a + (int64_t)nxp * t] * yp[t];
      yi[a] += s;
    }
  }
  __syncthreads();
  if (is_leaf[i] && nbegin[i] >= p_lo && nbegin[i] < p_hi) {
    const int nx = xbar_n[i];
    const double* Ui = U + u_off[i];
    for (int a = threadIdx.x; a < nx; a += blockDim.x) {
      double s = 0.0;
      for (int t = 0; t < ki; t++) s += Ui[a + (int64_t)nx * t] * yi[t];
      yt[nbegin[i] + a] += s;
    }
  }
}

template <int D>
__global__ void nearfield_kernel(int64_t np, const int2* __restrict__ pairs, const int64_t* __restrict__ voff,
                                 const double* __restrict__ Dv, int kid, double p2, const double* __restrict__ Xf,
                                 const double* __restrict__ X, int64_t n, const int* __restrict__ nbegin,
                                 const int* __restrict__ nend, int sym, const double* __restrict__ xt, double* yt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t p = blockIdx.x; p < np; p += gridDim.x) {
    const int2 pr = pairs[p];
    const int i = pr.x, j = pr.y;
    const int bi = nbegin[i], bj = nbegin[j], ni = nend[i] - bi, nj = nend[j] - bj;
    const double* Dp = Dv ? Dv + voff[p] : nullptr;
    for (int a = warp; a < ni; a += nw) {  // y_i += D x_j (warp per row, coalesced)
      double s = 0.0;
      for (int b = lane; b < nj; b += 32)
        s += (Dp ? Dp[(int64_t)a * nj + b] : kval<D>(kid, p2, Xf, X, n, bi + a, bj + b)) * xt[bj + b];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) atomicAdd(yt + bi + a, s);
    }
    if (sym && i != j)
      for (int b = threadIdx.x; b < nj; b += blockDim.x) {  // y_j += D^T x_i
        double s = 0.0;
        for (int a = 0; a < ni; a++)
          s += (Dp ? Dp[(int64_t)a * nj + b] : kval<D>(kid, p2, Xf, X, n, bi + a, bj + b)) * xt[bi + a];
        atomicAdd(yt + bj + b, s);
      }
  }
}

// ---- stored nearfield blocks: one pass over each entry, both directions ---------------------
// Warp per ITEM: one 32 CW-column slice of one nearfield block (a 32 CW SPLIT-column chunk is
// split over SPLIT warps), all rows.  Lane l owns the columns c0 + l + 32 s: x_j of those columns
// and the D^T x_i accumulators stay in registers for the whole block (flushed with one atomic per
// column), each row contributes one FMA per entry to the row partial and one to the column
// accumulator; the entries stream once with coalesced 256-byte loads issued PF rows ahead.  The
// row partials of 16 rows are summed across the warp by a transposing butterfly (31 shuffles;
// lane l ends with row l & 15), one atomic per row.  Diagonal blocks (i = j) are stored whole and
// only multiply forward.
template <int CW, int SPLIT>
__global__ void __launch_bounds__(256, 2) nf_matvec_kernel(int64_t nitems, const int* __restrict__ imap,
                                                           const int64_t* __restrict__ ioff,
                                                           const int2* __restrict__ pairs,
                                                           const int64_t* __restrict__ voff,
                                                           const int* __restrict__ nbegin, const int* __restrict__ nend,
                                                           const double* __restrict__ Dv, const double* __restrict__ xt,
                                                           double* yt, int kMvPfRows,
                                                           unsigned long long* ctr, int sym) {
  constexpr int WC = 32 * CW * SPLIT, G = 16, PF = CW >= 3 ? 4 : 8;
  static_assert(G % PF == 0, "the prefetch ring must wrap with the row groups");
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // items in grid-stride order, or (ctr != nullptr) taken dynamically by whole warps
  auto next = [&](int64_t cur) -> int64_t {
    if (!ctr) return cur + nw;
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ctr, 1ULL);
    return (int64_t)__shfl_sync(0xffffffffu, t, 0);
  };
  const int64_t v0 = ctr ? next(0) : (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  for (int64_t v = v0; v < nitems * SPLIT; v = next(v)) {
    const int64_t it = v / SPLIT;
    const int half = (int)(v - it * SPLIT);
    const int p = imap[it];
    const int2 pr = pairs[p];
    const bool diag = !sym || pr.x == pr.y;  // forward only (non-symmetric: every block is stored)
    const int bi = nbegin[pr.x], bj = nbegin[pr.y];
    const int ni = nend[pr.x] - bi, nj = nend[pr.y] - bj;
    const int c0 = (int)(it - ioff[p]) * WC + half * 32 * CW;
    if (c0 >= nj) continue;  // warp-uniform: an empty slice of a narrow last chunk
    double xj[CW], acc[CW];
    bool ok[CW];
#pragma unroll
    for (int s = 0; s < CW; s++) {
      const int col = c0 + lane + 32 * s;
      ok[s] = col < nj;
      xj[s] = ok[s] ? xt[bj + col] : 0.0;
      acc[s] = 0.0;
    }
    const double* Db = Dv + voff[p] + c0;
    const double* Dp = Db + lane;
    // L2 prefetch of rows [a, a + G) of the slice, kMvPfRows rows ahead of their use: the register
    // ring holds only PF rows, so HBM would see too few bytes in flight per warp; prefetches hold no
    // registers.  A slice spanning whole rows is one contiguous range (128-byte lines over the
    // lanes); otherwise lane l takes row a + (l & 15) and every second line from l >> 4.
    const bool contig = c0 == 0 && nj <= 32 * CW;
    const int wbytes = 8 * (nj - c0 < 32 * CW ? nj - c0 : 32 * CW);
    auto prefetch_rows = [&](int a, int a_end) {
      if (a_end > ni) a_end = ni;
      if (a >= a_end) return;
      if (contig) {
        const uintptr_t b = reinterpret_cast<uintptr_t>(Db + (int64_t)a * nj) & ~(uintptr_t)127;
        const uintptr_t e = reinterpret_cast<uintptr_t>(Db + (int64_t)a_end * nj);
        for (uintptr_t q = b + 128 * lane; q < e; q += 32 * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
      } else {
        const int row = a + (lane & 15);
        if (row < a_end) {
          const uintptr_t b = reinterpret_cast<uintptr_t>(Db + (int64_t)row * nj);
          for (int o = 128 * (lane >> 4); o < wbytes + 128; o += 256)
            asm volatile("prefetch.global.L2 [%0];" ::"l"((b & ~(uintptr_t)127) + o));
        }
      }
    };
    if (kMvPfRows > 0) prefetch_rows(0, kMvPfRows + G);
    auto load_row = [&](int a, double (&b)[CW], double& xa) {
      if (a < ni) {  // warp-uniform
        const double* row = Dp + (int64_t)a * nj;
#pragma unroll
        for (int s = 0; s < CW; s++) b[s] = ok[s] ? __ldcs(row + 32 * s) : 0.0;
        xa = diag ? 0.0 : xt[bi + a];
      } else {
#pragma unroll
        for (int s = 0; s < CW; s++) b[s] = 0.0;
        xa = 0.0;
      }
    };
    // a continuous ring: row a lives in buf[a % PF] from PF rows before its use (across groups)
    double buf[PF][CW], xbuf[PF];
#pragma unroll
    for (int q = 0; q < PF; q++) load_row(q, buf[q], xbuf[q]);
    for (int a0 = 0; a0 < ni; a0 += G) {
      if (kMvPfRows > 0) prefetch_rows(a0 + kMvPfRows + G, a0 + kMvPfRows + 2 * G);
      double part[G];
#pragma unroll
      for (int q = 0; q < G; q++) {
        double pq = 0.0;
#pragma unroll
        for (int s = 0; s < CW; s++) {
          pq = fma(buf[q % PF][s], xj[s], pq);
          acc[s] = fma(buf[q % PF][s], xbuf[q % PF], acc[s]);
        }
        part[q] = pq;
        load_row(a0 + q + PF, buf[q % PF], xbuf[q % PF]);
      }
      // lanes l and l ^ 16 first add up, then the transposing butterfly over 16 rows: after the
      // step with offset o a lane keeps the half of its rows selected by bit o of its lane id
#pragma unroll
      for (int q = 0; q < G; q++) part[q] += __shfl_xor_sync(0xffffffffu, part[q], 16);
#pragma unroll
      for (int o = 8, w = 8; o > 0; o >>= 1, w >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int q = 0; q < w; q++) {
          const double lo = part[q], hi = part[q + w];
          const double send = up ? lo : hi, keep = up ? hi : lo;
          part[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (lane < 16 && a0 + lane < ni) atomicAdd(yt + bi + a0 + lane, part[0]);
    }
    if (!diag)
#pragma unroll
      for (int s = 0; s < CW; s++)
        if (ok[s]) atomicAdd(yt + bj + c0 + lane + 32 * s, acc[s]);
  }
}

// ---- stored nearfield blocks, bulk-staged (opt-in variant, H2_MV_BULK=1) ----------------------
// A CTA walks its nearfield units with a two-deep ring of shared-memory buffers: one elected
// thread arms an mbarrier with the unit's byte count and issues cp.async.bulk copies (the TMA
// bulk engine: a unit of a block with nj <= 32 CW columns is ONE contiguous range; wider blocks
// copy row by row) of the NEXT unit while the CTA computes the current one from shared memory.
// Nothing is staged through registers, so HBM sees up to two units (2 x ~32 KB) in flight per
// CTA without the register cost of a deep software prefetch.  Compute: warp w takes rows
// r0 + w, r0 + w + 8, ...; lanes over columns; row sums by warp shuffles (one atomic per row),
// the D^T x_i column partials reduced across the 8 warps in shared memory (one atomic per column
// per unit).  Diagonal blocks multiply forward only.
// Buffer: a contiguous unit takes <= kWarpUnitEntries + 2 doubles; a row-wise unit R = 4096 / WC rows
// of stride mv_row_stride(nc) <= WC + 2, at most 64 x 66 = 4224 doubles (CW = 2).
constexpr int kMvBulkThreads = 256, kMvBulkWarps = kMvBulkThreads / 32, kMvBulkBuf = 4224;

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done)
                 : "r"(a), "r"(parity)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

struct MvUnit {
  int pi, pj, bi, bj, r0, r1, c0, nc, nj;
  int64_t base;  // global index (doubles) of the unit's first entry
  bool contig;   // nj <= WC: the unit's rows are one contiguous range
};

template <int WC>
__device__ __forceinline__ MvUnit mv_unit(int64_t u, const int* __restrict__ umap, const int64_t* __restrict__ uoff,
                                          const int2* __restrict__ pairs, const int64_t* __restrict__ voff,
                                          const int* __restrict__ nbegin, const int* __restrict__ nend) {
  MvUnit m;
  const int p = umap[u];
  const int2 pr = pairs[p];
  m.pi = pr.x;
  m.pj = pr.y;
  m.bi = nbegin[pr.x];
  m.bj = nbegin[pr.y];
  const int ni = nend[pr.x] - m.bi;
  m.nj = nend[pr.y] - m.bj;
  int R, nrb, ncb;
  unit_shape(ni, m.nj, WC, R, nrb, ncb);
  const int loc = (int)(u - uoff[p]);
  const int rb = loc / ncb, cb = loc - rb * ncb;
  m.r0 = rb * R;
  m.r1 = ni < m.r0 + R ? ni : m.r0 + R;
  m.c0 = cb * WC;
  m.nc = m.nj - m.c0 < WC ? m.nj - m.c0 : WC;
  m.base = voff[p] + (int64_t)m.r0 * m.nj + m.c0;
  m.contig = m.nj <= WC;
  return m;
}

// row stride of a row-wise staged unit: even (every row copy lands 16-byte aligned) and >= nc + 2
// (a copy starts at the even global index below the row and spans at most nc + 2 doubles)
__device__ __forceinline__ int mv_row_stride(int nc) { return ((nc + 1) & ~1) + 2; }

// shared-memory position of (row a - r0, column b - c0) of a staged unit; copies start at an
// even global index (16-byte alignment), hence the +1 when the range starts odd
__device__ __forceinline__ int mv_pos(const MvUnit& m, int ra, int cb) {
  if (m.contig) return (int)(m.base & 1) + ra * m.nj + cb;
  const int64_t rs = m.base + (int64_t)ra * m.nj;
  return ra * mv_row_stride(m.nc) + (int)(rs & 1) + cb;
}

template <int WC>
__device__ __forceinline__ void mv_issue(const MvUnit& m, const double* __restrict__ Dv, double* buf, uint64_t* bar) {
  if (m.contig) {
    const int64_t s0 = m.base & ~1LL, e = m.base + (int64_t)(m.r1 - m.r0) * m.nj;
    const unsigned bytes = (unsigned)(((e - s0 + 1) & ~1LL) * 8);
    mbar_expect_tx(bar, bytes);
    bulk_g2s(buf, Dv + s0, bytes, bar);
  } else {
    unsigned total = 0;
    for (int ra = 0; ra < m.r1 - m.r0; ra++) {
      const int64_t rs = m.base + (int64_t)ra * m.nj;
      total += (unsigned)((((rs + m.nc) - (rs & ~1LL) + 1) & ~1LL) * 8);
    }
    mbar_expect_tx(bar, total);
    for (int ra = 0; ra < m.r1 - m.r0; ra++) {
      const int64_t rs = m.base + (int64_t)ra * m.nj;
      const unsigned bytes = (unsigned)((((rs + m.nc) - (rs & ~1LL) + 1) & ~1LL) * 8);
      bulk_g2s(buf + ra * mv_row_stride(m.nc), Dv + (rs & ~1LL), bytes, bar);
    }
  }
}

template <int CW>
__global__ void __launch_bounds__(kMvBulkThreads) nf_matvec_bulk_kernel(
    int64_t nunits, const int* __restrict__ umap, const int64_t* __restrict__ uoff, const int2* __restrict__ pairs,
    const int64_t* __restrict__ voff, const int* __restrict__ nbegin, const int* __restrict__ nend,
    const double* __restrict__ Dv, const double* __restrict__ xt, double* yt, int sym) {
  constexpr int WC = 32 * CW;
  extern __shared__ double sm[];  // buf[2][kMvBulkBuf], red[kMvBulkWarps][WC]
  __shared__ __align__(8) uint64_t bar[2];
  double* red = sm + 2 * kMvBulkBuf;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int64_t u = blockIdx.x;
  if (tid == 0 && u < nunits) mv_issue<WC>(mv_unit<WC>(u, umap, uoff, pairs, voff, nbegin, nend), Dv, sm, &bar[0]);
  for (int k = 0; u < nunits; k++, u += gridDim.x) {
    const int cur = k & 1;
    const int64_t un = u + gridDim.x;
    if (tid == 0 && un < nunits) {  // the other buffer was released by the barrier ending step k-1
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mv_issue<WC>(mv_unit<WC>(un, umap, uoff, pairs, voff, nbegin, nend), Dv, sm + (cur ^ 1) * kMvBulkBuf,
                   &bar[cur ^ 1]);
    }
    const MvUnit m = mv_unit<WC>(u, umap, uoff, pairs, voff, nbegin, nend);
    const bool diag = !sym || m.pi == m.pj;
    const double* buf = sm + cur * kMvBulkBuf;
    double xj[CW], acc[CW];
#pragma unroll
    for (int s = 0; s < CW; s++) {
      const int cb = lane + 32 * s;
      xj[s] = cb < m.nc ? xt[m.bj + m.c0 + cb] : 0.0;
      acc[s] = 0.0;
    }
    mbar_wait(&bar[cur], (unsigned)((k >> 1) & 1));
    for (int ra = w; ra < m.r1 - m.r0; ra += kMvBulkWarps) {
      const double xa = diag ? 0.0 : xt[m.bi + m.r0 + ra];
      const int p0 = mv_pos(m, ra, 0);
      double part = 0.0;
#pragma unroll
      for (int s = 0; s < CW; s++) {
        const int cb = lane + 32 * s;
        const double dv = cb < m.nc ? buf[p0 + cb] : 0.0;
        part = fma(dv, xj[s], part);
        acc[s] = fma(dv, xa, acc[s]);
      }
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0) atomicAdd(yt + m.bi + m.r0 + ra, part);
    }
    if (!diag) {
#pragma unroll
      for (int s = 0; s < CW; s++) red[w * WC + lane + 32 * s] = acc[s];
    }
    __syncthreads();  // buffer `cur` consumed, column partials published
    if (!diag)
      for (int cb = tid; cb < m.nc; cb += kMvBulkThreads) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < kMvBulkWarps; q++) t += red[q * WC + cb];
        atomicAdd(yt + m.bj + m.c0 + cb, t);
      }
    __syncthreads();  // red free for the next unit
  }
}

// H2_MV_BULK=1 (A/B knob, read once): the bulk-staged nearfield kernel instead of the
// register-prefetch one (measured slower on config 4: 24.7 vs 14 ms -- the per-unit metadata
// chain delays the next copy)
static bool mv_bulk() {
  static const bool v = [] {
    const char* e = getenv("H2_MV_BULK");
    return e && atoi(e) != 0;
  }();
  return v;
}

// H2_MV_PF (A/B knob, read once): the nearfield matvec's L2 prefetch distance in rows beyond the
// current 16-row group (0 = no prefetch)
static int mv_pf_rows() {
  static const int v = [] {
    const char* e = getenv("H2_MV_PF");
    return e ? atoi(e) : 16;
  }();
  return v;
}

static int mv_order() {
  static const int v = [] {
    const char* e = getenv("H2_MV_ORDER");
    return e ? atoi(e) : 0;
  }();
  return v;
}

static bool mv_dyn() {
  static const bool v = [] {
    const char* e = getenv("H2_MV_DYN");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

template <int D>
static void launch_far_near(const h2_handle* h, double p2, const double* zh, double* yh, const double* xt, double* yt,
                            int which, cudaStream_t s) {
  if (which == 0 && h->n_cp > 0 && h->cp_stored) {
    const int64_t blocks = (h->n_cp + 255) / 256;  // 8 warps x 32 pairs
    const unsigned g = (unsigned)(blocks < 148 * 16 ? blocks : 148 * 16);
    coupling_mv_kernel<<<g, 256, 0, s>>>(h->n_cp, h->cp_pairs, h->cp_off, h->cp_val, h->k, h->k_col, h->r,
                                         !h->nonsym, zh, yh);
  } else if (which == 0 && h->n_cp > 0) {
    unsigned g = (unsigned)(h->n_cp < 148 * 64 ? h->n_cp : 148 * 64);
    coupling_kernel<D><<<g, kMvThreads, 0, s>>>(h->n_cp, h->cp_pairs, h->cp_off, h->cp_stored ? h->cp_val : nullptr,
                                                h->kid, p2, h->Xq ? h->Xq : h->Xf, h->Xq ? h->Xq : h->X,
                                                h->Xq ? h->nq : (int64_t)h->n, h->k, h->sk, h->k_col, h->sk_col, h->r,
                                                !h->nonsym, zh, yh);
  }
  if (which == 1 && h->n_np > 0 && h->np_stored && h->nf_nunits > 0) {
    const int cw = h->nf_wc / 32;
    const int64_t blocks = (2 * h->nf_nitems + 7) / 8;  // (split items: up to two warps per item)
    unsigned g = (unsigned)(blocks < 148 * 16 ? blocks : 148 * 16);
    if (mv_bulk()) {
      const int smem = (int)(sizeof(double) * (2 * kMvBulkBuf + kMvBulkWarps * 32 * cw));
      const unsigned gb = (unsigned)(h->nf_nunits < 148 * 2 ? h->nf_nunits : 148 * 2);
      switch (cw) {
#define H2_NFMVB_CASE(C)                                                                                         \
  case C:                                                                                                        \
    H2_CUDA_TRY(cudaFuncSetAttribute(nf_matvec_bulk_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                     200 * 1024));                                                               \
    nf_matvec_bulk_kernel<C><<<gb, kMvBulkThreads, smem, s>>>(h->nf_nunits, h->nf_umap, h->nf_uoff, h->np_pairs,  \
                                                              h->np_off, h->nbegin, h->nend, h->np_val, xt, yt,  \
                                                              !h->nonsym);                                       \
    break;
        H2_NFMVB_CASE(2) H2_NFMVB_CASE(3) H2_NFMVB_CASE(4) H2_NFMVB_CASE(5) H2_NFMVB_CASE(6) H2_NFMVB_CASE(8)
#undef H2_NFMVB_CASE
        default: throw Error{H2_ERR_INTERNAL, "nearfield matvec: unexpected unit width"};
      }
      return;
    }
    // H2_MV_DYN (default 1): one resident wave (2 CTAs per SM) taking items from a counter
    Scratch ctr_s;
    unsigned long long* ctr = nullptr;
    if (mv_dyn()) {
      ctr_s = Scratch(sizeof(unsigned long long), s);
      ctr = ctr_s.as<unsigned long long>();
      H2_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s));
      if (g > 148 * 2) g = 148 * 2;
    }
    switch (cw) {
#define H2_NFMV_CASE(C, CWW, SP)                                                                              \
  case C:                                                                                                    \
    nf_matvec_kernel<CWW, SP><<<g, 256, 0, s>>>(h->nf_nitems, h->nf_imap, h->nf_ioff, h->np_pairs, h->np_off,     \
                                                h->nbegin, h->nend, h->np_val, xt, yt, mv_pf_rows(), ctr,     \
                                                !h->nonsym);                                                  \
    break;
      H2_NFMV_CASE(2, 2, 1) H2_NFMV_CASE(3, 3, 1) H2_NFMV_CASE(4, 4, 1) H2_NFMV_CASE(5, 5, 1)
      H2_NFMV_CASE(6, 3, 2) H2_NFMV_CASE(8, 4, 2)
#undef H2_NFMV_CASE
      default: throw Error{H2_ERR_INTERNAL, "nearfield matvec: unexpected unit width"};
    }
  } else if (which == 1 && h->n_np > 0) {
    unsigned g = (unsigned)(h->n_np < 148 * 64 ? h->n_np : 148 * 64);
    nearfield_kernel<D><<<g, kMvThreads, 0, s>>>(h->n_np, h->np_pairs, h->np_off, h->np_stored ? h->np_val : nullptr,
                                                 h->kid, p2, h->Xf, h->X, h->n, h->nbegin, h->nend, !h->nonsym, xt, yt);
  }
}

static void far_near(const h2_handle* h, double p2, const double* zh, double* yh, const double* xt, double* yt,
                     int which, cudaStream_t s) {
  switch (h->d) {
#define H2_MV_CASE(DD) \
  case DD:             \
    launch_far_near<DD>(h, p2, zh, yh, xt, yt, which, s); break;
    H2_MV_CASE(1) H2_MV_CASE(2) H2_MV_CASE(3) H2_MV_CASE(4)
    H2_MV_CASE(5) H2_MV_CASE(6) H2_MV_CASE(7) H2_MV_CASE(8)
#undef H2_MV_CASE
  }
}

// Sharded handles (shard.cu): the upward pass runs on the owned subtrees, the z^ of the levels
// >= cut are summed over the ranks (each node is non-zero on its owner only), and the levels
// above the cut are then computed by every rank; coupling and nearfield apply the rank's own
// (row-owned) blocks in both directions, so y^ and y are partial sums completed by allreduces.
// The nearfield pass (xt -> yt, by far the most bytes) depends only on the permuted input, so it
// runs on a second stream concurrently with the farfield chain (up -> coupling -> down, xt -> yf);
// the two outputs are added in the final permutation.
void matvec(const h2_handle* h, const double* x, double* y) {
  cudaStream_t s = h->stream;
  const int64_t n = h->n;
  const int nn = h->nnodes, r = h->r;
  const bool sharded = h->nranks > 1;
  Scratch xt(sizeof(double) * n, s), yt(sizeof(double) * n, s), yf(sizeof(double) * n, s),
      zh(sizeof(double) * (size_t)nn * r, s), yh(sizeof(double) * (size_t)nn * r, s);
  H2_CUDA_TRY(cudaMemsetAsync(yt.p, 0, sizeof(double) * n, s));
  H2_CUDA_TRY(cudaMemsetAsync(yf.p, 0, sizeof(double) * n, s));
  H2_CUDA_TRY(cudaMemsetAsync(yh.p, 0, sizeof(double) * (size_t)nn * r, s));
  H2_CUDA_TRY(cudaMemsetAsync(zh.p, 0, sizeof(double) * (size_t)nn * r, s));
  permute_in_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, h->perm, n, xt.as<double>());
  const double p2 = kernel_p2(h->kid, h->kp);
  // nearfield on the build's lowest-priority stream, forked after permute_in: its short CTAs yield
  // SM slots to the farfield chain's level kernels on `s` as they retire
  // H2_MV_ORDER=1 (A/B knob): the farfield chain first, then the nearfield pass, on one stream
  const bool far_first = mv_order() == 1;
  cudaStream_t ns = h->low && !far_first ? h->low : s;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  if (ns != s) {
    for (auto& e : ev) H2_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    H2_CUDA_TRY(cudaEventRecord(ev[0], s));
    H2_CUDA_TRY(cudaStreamWaitEvent(ns, ev[0], 0));
  }
  if (!far_first) far_near(h, p2, zh.as<double>(), yh.as<double>(), xt.as<double>(), yt.as<double>(), 1, ns);
  if (ns != s) H2_CUDA_TRY(cudaEventRecord(ev[1], ns));
  auto up = [&](int l) {
    const LevelRange lr = level_range(h, l);
    if (lr.end > lr.begin)
      up_kernel<<<lr.end - lr.begin, kMvThreads, 0, s>>>(lr.begin, r, h->is_leaf, h->nbegin, h->first_child,
                                                         h->nchild, h->k_col, h->xbar_col_n, h->child_off_col,
                                                         h->u_off_col, h->V, xt.as<double>(), zh.as<double>());
  };
  const int cut = sharded ? (h->cut > 1 ? h->cut : 1) : 1;
  for (int l = h->depth; l >= cut; l--) up(l);
  if (sharded) comm_allreduce_sum(h->comm, zh.as<double>(), zh.as<double>(), (int64_t)nn * r, s);
  for (int l = cut - 1; l >= 1; l--) up(l);
  far_near(h, p2, zh.as<double>(), yh.as<double>(), xt.as<double>(), yt.as<double>(), 0, s);
  if (sharded) comm_allreduce_sum(h->comm, yh.as<double>(), yh.as<double>(), (int64_t)nn * r, s);
  for (int l = 1; l <= h->depth; l++) {
    const LevelRange lr = level_range(h, l);
    if (lr.end > lr.begin)
      down_kernel<<<lr.end - lr.begin, kMvThreads, 0, s>>>(lr.begin, r, h->is_leaf, h->nbegin, h->parent, h->k,
                                                           h->xbar_n, h->child_off, h->u_off, h->U, h->p_lo, h->p_hi,
                                                           yh.as<double>(), yf.as<double>());
  }
  if (far_first) far_near(h, p2, zh.as<double>(), yh.as<double>(), xt.as<double>(), yt.as<double>(), 1, s);
  if (ns != s) H2_CUDA_TRY(cudaStreamWaitEvent(s, ev[1], 0));
  if (sharded) {
    add_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, yf.as<double>(), yt.as<double>());
    H2_CUDA_TRY(cudaMemsetAsync(yf.p, 0, sizeof(double) * n, s));
    comm_allreduce_sum(h->comm, yt.as<double>(), yt.as<double>(), n, s);
  }
  permute_out_kernel<<<grid_for(n, 256), 256, 0, s>>>(yt.as<double>(), yf.as<double>(), h->perm, n, y);
  H2_CHECK_LAUNCH();
  if (sharded) comm_sync(h->comm, s);
  else H2_CUDA_TRY(cudaStreamSynchronize(s));
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
}

}  // namespace h2
