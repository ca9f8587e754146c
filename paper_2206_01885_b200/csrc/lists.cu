// lists.cu -- a4: interaction and nearfield lists by a level-synchronous dual traversal.
//
// Eq.(2.1): diam(X_i) + diam(X_j) <= 2 tau |a_i - a_j|, with the cell
// diagonal as diameter (reading B1), equality admissible (B2), pair-of-parents interaction lists
// (B3) and cross-level pairs on adaptive trees (B4).  The frontier of candidate pairs
// starts at (root, root); each step classifies every pair: admissible -> IL, both leaves -> NF,
// otherwise expand the non-leaf side (both sides when neither is a leaf).  A sharded build keeps
// only its own rows (RowFilter): per-rank lists, the single-GPU lists restricted to those rows.
#include <climits>
#include <cstdlib>
#include <vector>

#include "vol.cuh"

namespace h2 {

// exact-integer admissibility in units of the finer cell (same operation order as DESIGN.md B)
__device__ __forceinline__ bool admissible(const int* __restrict__ cell, int nnodes, int d, int i, int li, int j,
                                           int lj, double tau2) {
  int lf = li > lj ? li : lj;
  long long wi = 1LL << (lf - li), wj = 1LL << (lf - lj);
  double S = 0.0;
  for (int c = 0; c < d; c++) {
    long long Ai = (2LL * cell[(int64_t)c * nnodes + i] + 1) * wi;
    long long Aj = (2LL * cell[(int64_t)c * nnodes + j] + 1) * wj;
    double df = (double)(Ai - Aj);
    S = __dadd_rn(S, __dmul_rn(df, df));
  }
  double w = (double)(wi + wj);
  double lhs = __dmul_rn((double)d, __dmul_rn(w, w));
  return lhs <= __dmul_rn(tau2, S);
}

// ---- one traversal step in two launches ----------------------------------------------------
// Tiles of kTravTile frontier pairs (each thread kTravIPT consecutive pairs).  trav_count:
// classify every pair (far -> IL, both leaves -> NF, else expand), per-tile counts of the three
// outputs, and their totals (atomics) for the host to size the outputs.  trav_emit: the same
// classification again, each tile's offsets = the sums of the tiles before it plus an in-tile
// exclusive scan (thread-blocked, so the output order is the frontier order), and the writes.
// Two pairs per thread (round 2; was 8): an expanded pair's child block (up to 2^d x 2^d writes)
// is written by its thread alone, so fewer pairs per thread shorten the serial write chains
// (lists stage config 2 3.07 -> 2.5 ms, config 4 1.32 -> 1.10, config 5 7.2 -> 5.7).
constexpr int kTravThreads = 256, kTravIPT = 2, kTravTile = kTravThreads * kTravIPT;

// Sharded builds: a rank keeps only the pairs whose row node it needs -- every node above the cut
// level, and its own contiguous range at each level >= cut (shard.cu).  The children of a dropped
// row are never needed either, so the frontier it would have grown is dropped with it.
// Nearfield rows are needed only by the rank that stores them (a leaf whose first point lies in its
// point range [p_lo, p_hi), fill.cu), also above the cut.
struct RowFilter {
  int on, cut, p_lo, p_hi;
  int lo[32], hi[32];
  const int* nbegin;
};

__device__ __forceinline__ void trav_classify(const int2 pr, const int* __restrict__ cell, int nnodes, int d,
                                              double tau2, const int* __restrict__ level,
                                              const int* __restrict__ is_leaf, const int* __restrict__ nchild,
                                              const RowFilter& rf, long long& a, long long& b, long long& c) {
  const int i = pr.x, j = pr.y;
  a = b = c = 0;
  if (rf.on) {
    const int li = level[i];
    if (li >= rf.cut && (i < rf.lo[li] || i >= rf.hi[li])) return;
  }
  if (admissible(cell, nnodes, d, i, level[i], j, level[j], tau2)) {
    a = 1;
  } else {
    const int li = is_leaf[i], lj = is_leaf[j];
    if (li && lj) b = !rf.on || (rf.nbegin[i] >= rf.p_lo && rf.nbegin[i] < rf.p_hi);
    else c = (long long)(li ? 1 : nchild[i]) * (lj ? 1 : nchild[j]);
  }
}

__global__ void __launch_bounds__(kTravThreads) trav_count_kernel(const int2* __restrict__ fr, int64_t nf,
                                                                  const int* __restrict__ cell, int nnodes, int d,
                                                                  double tau2, const int* __restrict__ level,
                                                                  const int* __restrict__ is_leaf,
                                                                  const int* __restrict__ nchild, RowFilter rf,
                                                                  long long* __restrict__ tile_sum,
                                                                  unsigned long long* totals,
                                                                  unsigned long long* __restrict__ ej,
                                                                  unsigned long long* __restrict__ ex,
                                                                  int64_t* __restrict__ rs, int64_t* __restrict__ re) {
  __shared__ long long red[3][kTravThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t base = blockIdx.x * (int64_t)kTravTile + (int64_t)tid * kTravIPT;
  long long sa = 0, sb = 0, sc = 0;
  for (int k = 0; k < kTravIPT; k++) {
    if (base + k >= nf) break;
    long long a, b, c;
    const int2 pr = fr[base + k];
    trav_classify(pr, cell, nnodes, d, tau2, level, is_leaf, nchild, rf, a, b, c);
    sa += a;
    sb += b;
    sc += c;
    if (ej) {  // ordered emission: the pair's packed expansion counts (trav_emit_kernel)
      unsigned long long vj = 0, vx = 0;
      if (c) {
        const int li = is_leaf[pr.x], lj = is_leaf[pr.y];
        vj = lj ? (1ULL << 32) : (unsigned long long)nchild[pr.y];
        vx = li ? ((unsigned long long)c << 32) : (unsigned long long)c;
      }
      ej[base + k] = vj;
      ex[base + k] = vx;
      // the row blocks (the frontier is sorted by row)
      const int64_t f = base + k;
      if (f == 0 || fr[f - 1].x != pr.x) rs[pr.x] = f;
      if (f == nf - 1 || fr[f + 1].x != pr.x) re[pr.x] = f + 1;
    }
  }
  if (ej && blockIdx.x == 0 && tid == 0) {
    ej[nf] = 0;
    ex[nf] = 0;
  }
  for (int o = 16; o > 0; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
    sc += __shfl_xor_sync(0xffffffffu, sc, o);
  }
  if (lane == 0) {
    red[0][w] = sa;
    red[1][w] = sb;
    red[2][w] = sc;
  }
  __syncthreads();
  if (tid < 3) {
    long long t = 0;
    for (int q = 0; q < kTravThreads / 32; q++) t += red[tid][q];
    tile_sum[(int64_t)tid * gridDim.x + blockIdx.x] = t;
    atomicAdd(totals + tid, (unsigned long long)t);
  }
}

__global__ void __launch_bounds__(kTravThreads) trav_emit_kernel(
    const int2* __restrict__ fr, int64_t nf, const int* __restrict__ cell, int nnodes, int d, double tau2,
    const int* __restrict__ level, const int* __restrict__ is_leaf, const int* __restrict__ nchild,
    const int* __restrict__ first_child, RowFilter rf, const long long* __restrict__ tile_pre,
    unsigned long long* il, int64_t il_base, unsigned long long* nl, int64_t nl_base, int2* next,
    const int64_t* __restrict__ rs, const int64_t* __restrict__ re, const unsigned long long* __restrict__ Ej,
    const unsigned long long* __restrict__ Ex) {
  __shared__ long long wsum[3][kTravThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int ntiles = gridDim.x;
  // offsets of this tile: tile_pre is the exclusive prefix sum of the channel-major tile sums, so
  // channel c's offset is tile_pre[c ntiles + tile] - tile_pre[c ntiles]
  const long long pa = tile_pre[blockIdx.x];
  const long long pb = tile_pre[ntiles + blockIdx.x] - tile_pre[ntiles];
  const long long pc = tile_pre[2 * ntiles + blockIdx.x] - tile_pre[2 * ntiles];
  // this thread's pairs: classification and thread totals
  const int64_t base = blockIdx.x * (int64_t)kTravTile + (int64_t)tid * kTravIPT;
  long long ca[kTravIPT], cb[kTravIPT], cc[kTravIPT];
  long long ta = 0, tb = 0, tc = 0;
#pragma unroll
  for (int k = 0; k < kTravIPT; k++) {
    ca[k] = cb[k] = cc[k] = 0;
    if (base + k < nf)
      trav_classify(fr[base + k], cell, nnodes, d, tau2, level, is_leaf, nchild, rf, ca[k], cb[k], cc[k]);
    ta += ca[k];
    tb += cb[k];
    tc += cc[k];
  }
  // in-tile exclusive scan of the thread totals (warp scan + warp sums)
  long long ia = ta, ib = tb, ic = tc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long ua = __shfl_up_sync(0xffffffffu, ia, o), ub = __shfl_up_sync(0xffffffffu, ib, o),
                    uc = __shfl_up_sync(0xffffffffu, ic, o);
    if (lane >= o) {
      ia += ua;
      ib += ub;
      ic += uc;
    }
  }
  if (lane == 31) {
    wsum[0][w] = ia;
    wsum[1][w] = ib;
    wsum[2][w] = ic;
  }
  __syncthreads();
  long long oa = pa + ia - ta, ob = pb + ib - tb, oc = pc + ic - tc;
#pragma unroll
  for (int q = 0; q < kTravThreads / 32; q++) {
    oa += q < w ? wsum[0][q] : 0;
    ob += q < w ? wsum[1][q] : 0;
    oc += q < w ? wsum[2][q] : 0;
  }
#pragma unroll
  for (int k = 0; k < kTravIPT; k++) {
    if (base + k >= nf) break;
    const int2 pr = fr[base + k];
    const int i = pr.x, j = pr.y;
    if (ca[k]) {
      il[il_base + oa] = ((unsigned long long)i << 32) | (unsigned)j;
    } else if (cb[k]) {
      nl[nl_base + ob] = ((unsigned long long)i << 32) | (unsigned)j;
    } else if (cc[k]) {  // (a pair a sharded rank drops has no output at all)
      const int li = is_leaf[i], lj = is_leaf[j];
      const int ci = li ? 1 : nchild[i], cj = lj ? 1 : nchild[j];
      const int fi = li ? i : first_child[i], fj = lj ? j : first_child[j];
      if (Ej) {  // ordered emission (see build_lists)
        constexpr unsigned long long kLo = 0xffffffffULL;
        const int64_t f = base + k, f0 = rs[i], f1 = re[i];
        const unsigned long long E0 = Ej[f0], E1 = Ej[f1], Ef = Ej[f];
        const unsigned long long X0 = Ex[f0] - Ex[0], XT = Ex[nf] - Ex[0];  // (Ex carries the ej total)
        const int64_t SL = (int64_t)((E1 >> 32) - (E0 >> 32)), SN = (int64_t)((E1 & kLo) - (E0 & kLo));
        const int64_t inrow = lj ? (int64_t)((Ef >> 32) - (E0 >> 32)) : SL + (int64_t)((Ef & kLo) - (E0 & kLo));
        const int64_t rb = li ? (int64_t)(X0 >> 32) : (int64_t)(XT >> 32) + (int64_t)(X0 & kLo);
        for (int a = 0; a < ci; a++)
          for (int b = 0; b < cj; b++) next[rb + (int64_t)a * (SL + SN) + inrow + b] = make_int2(fi + a, fj + b);
      } else {
        for (int a = 0; a < ci; a++)
          for (int b = 0; b < cj; b++) next[oc + (int64_t)a * cj + b] = make_int2(fi + a, fj + b);
      }
    }
    oa += ca[k];
    ob += cb[k];
    oc += cc[k];
  }
}

// ---- ordered emission ------------------------------------------------------------------------
// With the frontier sorted by (row, column), every step's IL / NF output (the classified pairs in
// frontier order) is sorted too, and so is the next frontier when the expansions are placed in this
// order: first the blocks of leaf rows (they keep their id, a level <= t), then the children of the
// non-leaf rows (level t + 1), each group in row order; inside a child row's block, the leaf columns
// (kept) before the children of the non-leaf columns, each in frontier order.  Node ids ascend with
// the level and, within a level, with the parent, so every one of these runs is ascending.  A pair's
// position: its row block [rs, re) (the rows are contiguous), the packed prefixes Ej (leaf-column
// pairs << 32 | children of non-leaf columns) and Ex (leaf-row expansions << 32 | non-leaf-row
// expansions) over the frontier.
// CSR of an ordered emission.  The keys are the steps' sorted segments (segment s = [b[s], b[s+1]));
// a row's entries of later steps have larger columns (deeper levels), so each row is its runs (one
// per segment at most) in segment order.  csr_runs: per (segment, row) the run start rsA, its length
// lenA (two atomic adds: -start at the start, end + 1 at the end) and its first / last columns, and
// `bad` when a column is not above its predecessor in the run.  csr_rows: per row, lenA turned into
// the prefix over the segments, the total count, and `bad` when a run does not start above the
// previous run's last column (then the per-row sort runs).  csr_place: every entry to off[row] +
// prefix + its offset in the run.
constexpr int kMaxSeg = 64;
struct SegBounds {
  int64_t b[kMaxSeg + 1];
  int n;
};
__device__ __forceinline__ int seg_of(const SegBounds& sb, int64_t e) {
  int lo = 0, hi = sb.n - 1;  // the last s with b[s] <= e
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (sb.b[mid] <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}
__global__ void csr_runs_kernel(const unsigned long long* __restrict__ keys, int64_t m, SegBounds sb, int nn,
                                int64_t* rsA, long long* lenA, int* firstA, int* lastA, int* bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int sg = seg_of(sb, e);
    const unsigned long long k = keys[e];
    const unsigned row = (unsigned)(k >> 32);
    const int col = (int)(k & 0xffffffffULL);
    const int64_t x = (int64_t)sg * nn + row;
    const bool start = e == sb.b[sg] || (unsigned)(keys[e - 1] >> 32) != row;
    const bool end = e == sb.b[sg + 1] - 1 || (unsigned)(keys[e + 1] >> 32) != row;
    if (start) {
      rsA[x] = e;
      firstA[x] = col;
      atomicAdd(reinterpret_cast<unsigned long long*>(&lenA[x]), (unsigned long long)(-(long long)e));  // (mod 2^64)
    } else if ((int)(keys[e - 1] & 0xffffffffULL) >= col) {
      *bad = 1;
    }
    if (end) {
      lastA[x] = col;
      atomicAdd(reinterpret_cast<unsigned long long*>(&lenA[x]), (unsigned long long)e + 1ULL);
    }
  }
}
__global__ void csr_rows_kernel(int nn, int nseg, long long* lenA, const int* __restrict__ firstA,
                                const int* __restrict__ lastA, int64_t* cnt, int* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  long long acc = 0;
  int prev = -1;
  for (int sg = 0; sg < nseg; sg++) {
    const int64_t x = (int64_t)sg * nn + i;
    const long long l = lenA[x];
    lenA[x] = acc;
    if (l > 0) {
      if (acc > 0 && firstA[x] <= prev) *bad = 1;
      prev = lastA[x];
    }
    acc += l;
  }
  cnt[i] = acc;
}
__global__ void csr_place_kernel(const unsigned long long* __restrict__ keys, int64_t m, SegBounds sb, int nn,
                                 const int64_t* __restrict__ rsA, const long long* __restrict__ preA,
                                 const int64_t* __restrict__ off, int* idx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int sg = seg_of(sb, e);
    const unsigned long long k = keys[e];
    const unsigned row = (unsigned)(k >> 32);
    const int64_t x = (int64_t)sg * nn + row;
    idx[off[row] + preA[x] + (e - rsA[x])] = (int)(k & 0xffffffffULL);
  }
}

// ---- CSR from the unordered (i << 32 | j) pairs: counting sort by row, then each row sorted --
__global__ void row_hist_kernel(const unsigned long long* __restrict__ keys, int64_t m, unsigned long long* cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[keys[e] >> 32], 1ULL);
}

__global__ void row_scatter_kernel(const unsigned long long* __restrict__ keys, int64_t m,
                                   const int64_t* __restrict__ off, int* fill, int* idx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[e];
    const int i = (int)(k >> 32);
    idx[off[i] + atomicAdd(&fill[i], 1)] = (int)(k & 0xffffffffULL);
  }
}

// one CTA per row: a row of <= 64 entries is sorted by warp 0 with shuffles (two per lane, no
// barrier), a longer one by a shared-memory bitonic network of its own power-of-two size
constexpr int kRowSortThreads = 512;
__global__ void __launch_bounds__(kRowSortThreads) row_sort_kernel(const int64_t* __restrict__ off, int* idx) {
  extern __shared__ int rs[];
  const int64_t b = off[blockIdx.x];
  const int len = (int)(off[blockIdx.x + 1] - b);
  if (len <= 1) return;
  int* row = idx + b;
  if (len <= 64) {
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    int a = lane < len ? row[lane] : INT_MAX, c = lane + 32 < len ? row[lane + 32] : INT_MAX;
    for (int k = 2; k <= 64; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        if (j == 32) {
          const bool up = (lane & k) == 0;
          const int lo = min(a, c), hi = max(a, c);
          a = up ? lo : hi;
          c = up ? hi : lo;
        } else {
          const int pa = __shfl_xor_sync(0xffffffffu, a, j), pc = __shfl_xor_sync(0xffffffffu, c, j);
          const bool lower = (lane & j) == 0;
          const bool upa = (lane & k) == 0, upc = ((lane + 32) & k) == 0;
          a = (lower == upa) ? min(a, pa) : max(a, pa);
          c = (lower == upc) ? min(c, pc) : max(c, pc);
        }
      }
    if (lane < len) row[lane] = a;
    if (lane + 32 < len) row[lane + 32] = c;
    return;
  }
  int P = 128;
  while (P < len) P <<= 1;
  for (int t = threadIdx.x; t < P; t += kRowSortThreads) rs[t] = t < len ? row[t] : INT_MAX;
  __syncthreads();
  cta_bitonic<kRowSortThreads>(rs, P);
  for (int t = threadIdx.x; t < len; t += kRowSortThreads) row[t] = rs[t];
}

__global__ void max_row_kernel(const int64_t* __restrict__ off, int nnodes, int* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nnodes) atomicMax(out, (int)(off[i + 1] - off[i]));
}

// growable device array of T
template <class T>
struct Grow {
  T* p = nullptr;
  int64_t cap = 0;
  cudaStream_t s;
  explicit Grow(cudaStream_t st) : s(st) {}
  ~Grow() {
    if (p) dev_free(p, s);
  }
  void ensure(int64_t need, int64_t used) {
    if (need <= cap) return;
    int64_t nc = need > 2 * cap ? need : 2 * cap;
    T* np = static_cast<T*>(dev_alloc(sizeof(T) * nc, s));
    if (p && used > 0) H2_CUDA_TRY(cudaMemcpyAsync(np, p, sizeof(T) * used, cudaMemcpyDeviceToDevice, s));
    if (p) dev_free(p, s);
    p = np;
    cap = nc;
  }
};

static void to_csr(h2_handle* h, unsigned long long* keys, int64_t m, int64_t*& off, int*& idx) {
  cudaStream_t s = h->stream;
  const int nn = h->nnodes;
  off = halloc<int64_t>(h, nn + 1);
  idx = halloc<int>(h, m);
  Scratch cnt(sizeof(int64_t) * (nn + 1), s), fill(sizeof(int) * nn, s), mx(sizeof(int), s);
  H2_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(int64_t) * (nn + 1), s));
  H2_CUDA_TRY(cudaMemsetAsync(fill.p, 0, sizeof(int) * nn, s));
  H2_CUDA_TRY(cudaMemsetAsync(mx.p, 0, sizeof(int), s));
  if (m > 0) row_hist_kernel<<<grid_for(m, 256), 256, 0, s>>>(keys, m, cnt.as<unsigned long long>());
  scan_excl_i64(cnt.as<int64_t>(), off, nn + 1, s);
  if (m == 0) return;
  row_scatter_kernel<<<grid_for(m, 256), 256, 0, s>>>(keys, m, off, fill.as<int>(), idx);
  max_row_kernel<<<(nn + 255) / 256, 256, 0, s>>>(off, nn, mx.as<int>());
  H2_CHECK_LAUNCH();
  const int maxlen = read1(mx.as<int>(), s);
  int P = 128;
  while (P < maxlen) P <<= 1;
  const size_t smem = sizeof(int) * (size_t)P;
  if (smem > 200 * 1024) throw Error{H2_ERR_INTERNAL, "list row longer than the row sort supports"};
  // one constant value: concurrent builds on other host threads set the same attribute
  H2_CUDA_TRY(cudaFuncSetAttribute(row_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  row_sort_kernel<<<nn, kRowSortThreads, smem, s>>>(off, idx);
  H2_CHECK_LAUNCH();
  h->gpu_launches += 4;
}

// CSR of an ordered emission (csr_*_kernel): `seg` = the keys' step boundaries.  Device flags and
// the longest row land in out4[0..1] (read by the caller in one synchronisation); a flagged list is
// then sorted per row (csr_fix).
static void to_csr_ordered(h2_handle* h, unsigned long long* keys, int64_t m, const std::vector<int64_t>& seg,
                           int64_t*& off, int*& idx, int* out2) {
  cudaStream_t s = h->stream;
  const int nn = h->nnodes;
  off = halloc<int64_t>(h, nn + 1);
  idx = halloc<int>(h, m);
  SegBounds sb{};
  sb.n = 0;
  for (size_t t = 0; t + 1 < seg.size(); t++)  // (empty segments dropped; at most kMaxSeg kept)
    if (seg[t + 1] > seg[t]) {
      if (sb.n == kMaxSeg) throw Error{H2_ERR_INTERNAL, "lists: more traversal steps than the CSR pass supports"};
      sb.b[sb.n++] = seg[t];
    }
  sb.b[sb.n] = m;
  const int nseg = sb.n > 0 ? sb.n : 1;
  Scratch cnt(sizeof(int64_t) * (nn + 1), s);
  H2_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(int64_t) * (nn + 1), s));
  if (m == 0) {
    scan_excl_i64(cnt.as<int64_t>(), off, nn + 1, s);
    max_row_kernel<<<(nn + 255) / 256, 256, 0, s>>>(off, nn, out2 + 1);
    H2_CHECK_LAUNCH();
    h->gpu_launches += 1;
    return;
  }
  const size_t sn = (size_t)nseg * nn;
  Scratch ws(sn * (8 + 8 + 4 + 4), s);
  int64_t* rsA = ws.as<int64_t>();
  long long* lenA = reinterpret_cast<long long*>(rsA + sn);
  int* firstA = reinterpret_cast<int*>(lenA + sn);
  int* lastA = firstA + sn;
  H2_CUDA_TRY(cudaMemsetAsync(lenA, 0, sizeof(long long) * sn, s));
  csr_runs_kernel<<<grid_for(m, 256), 256, 0, s>>>(keys, m, sb, nn, rsA, lenA, firstA, lastA, out2);
  csr_rows_kernel<<<(nn + 255) / 256, 256, 0, s>>>(nn, nseg, lenA, firstA, lastA, cnt.as<int64_t>(), out2);
  scan_excl_i64(cnt.as<int64_t>(), off, nn + 1, s);
  csr_place_kernel<<<grid_for(m, 256), 256, 0, s>>>(keys, m, sb, nn, rsA, lenA, off, idx);
  max_row_kernel<<<(nn + 255) / 256, 256, 0, s>>>(off, nn, out2 + 1);
  H2_CHECK_LAUNCH();
  h->gpu_launches += 4;
}

// the per-row sort of a CSR whose ordering check failed (maxlen = its longest row)
static void csr_fix(h2_handle* h, const int64_t* off, int* idx, int maxlen) {
  cudaStream_t s = h->stream;
  int P = 128;
  while (P < maxlen) P <<= 1;
  const size_t smem = sizeof(int) * (size_t)P;
  if (smem > 200 * 1024) throw Error{H2_ERR_INTERNAL, "list row longer than the row sort supports"};
  H2_CUDA_TRY(cudaFuncSetAttribute(row_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  row_sort_kernel<<<h->nnodes, kRowSortThreads, smem, s>>>(off, idx);
  H2_CHECK_LAUNCH();
  h->gpu_launches += 1;
}

// H2_LISTS_ORDERED=0 (A/B knob): the unordered emission, atomic scatter + per-row sort
static bool lists_ordered() {
  static const bool v = [] {
    const char* e = getenv("H2_LISTS_ORDERED");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

void build_lists(h2_handle* h) {
  cudaStream_t s = h->stream;
  const double tau2 = h->tau * h->tau;
  RowFilter rf{};  // sharded: this rank's rows only (shard_plan ran before)
  if (h->nranks > 1) {
    if (h->depth >= 32) throw Error{H2_ERR_INTERNAL, "sharded lists: depth beyond the row filter"};
    rf.on = 1;
    rf.cut = h->cut;
    rf.p_lo = h->p_lo;
    rf.p_hi = h->p_hi;
    rf.nbegin = h->nbegin;
    for (int l = 0; l <= h->depth; l++) {
      const LevelRange lr = level_range(h, l);
      rf.lo[l] = lr.begin;
      rf.hi[l] = lr.end;
    }
  }
  Grow<int2> fa(s), fb(s);
  Grow<unsigned long long> il(s), nl(s);
  fa.ensure(1, 0);
  int2 root = make_int2(0, 0);
  H2_CUDA_TRY(cudaMemcpyAsync(fa.p, &root, sizeof(int2), cudaMemcpyHostToDevice, s));
  int64_t nf = 1, nil = 0, nnl = 0;
  const bool ordered = lists_ordered();
  std::vector<int64_t> il_seg{0}, nl_seg{0};  // the steps' output boundaries (ordered emission)
  Scratch rsre(ordered ? sizeof(int64_t) * 2 * (size_t)h->nnodes : 0, s);
  int64_t* rs = ordered ? rsre.as<int64_t>() : nullptr;
  int64_t* re = ordered ? rs + h->nnodes : nullptr;
  unsigned long long* tot_h = nullptr;  // page-locked totals (per host thread, reused)
  {
    thread_local unsigned long long* pinned = nullptr;
    if (!pinned) H2_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&pinned), 4 * sizeof(unsigned long long)));
    tot_h = pinned;
  }
  while (nf > 0) {
    const int64_t ntiles = (nf + kTravTile - 1) / kTravTile;
    Scratch ts(sizeof(long long) * 3 * ntiles + sizeof(unsigned long long) * 4, s), tp(sizeof(long long) * 3 * ntiles, s);
    unsigned long long* tot_d = reinterpret_cast<unsigned long long*>(ts.as<long long>() + 3 * ntiles);
    H2_CUDA_TRY(cudaMemsetAsync(tot_d, 0, 3 * sizeof(unsigned long long), s));
    // ordered emission: the row blocks, the packed per-pair counts and their prefixes (nf + 1: the
    // last entry is the total)
    // [ej (nf + 1) | ex (nf + 1)] scanned as ONE array: Ex = the second half minus its first entry
    // (the ej total; packed halves subtract exactly)
    Scratch ejx(ordered ? sizeof(unsigned long long) * 4 * (size_t)(nf + 1) : 0, s);
    unsigned long long *ej = nullptr, *ex = nullptr, *Ej = nullptr, *Ex = nullptr;
    if (ordered) {
      ej = ejx.as<unsigned long long>();
      ex = ej + (nf + 1);
      Ej = ex + (nf + 1);
      Ex = Ej + (nf + 1);
    }
    trav_count_kernel<<<(unsigned)ntiles, kTravThreads, 0, s>>>(fa.p, nf, h->cell, h->nnodes, h->d, tau2, h->level,
                                                                 h->is_leaf, h->nchild, rf, ts.as<long long>(), tot_d,
                                                                 ej, ex, rs, re);
    H2_CHECK_LAUNCH();
    scan_excl_i64(reinterpret_cast<const int64_t*>(ts.as<long long>()), tp.as<int64_t>(), 3 * ntiles, s);
    if (ordered)
      scan_excl_i64(reinterpret_cast<const int64_t*>(ej), reinterpret_cast<int64_t*>(Ej), 2 * (nf + 1), s);
    H2_CUDA_TRY(cudaMemcpyAsync(tot_h, tot_d, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaStreamSynchronize(s));
    const int64_t tot[3] = {(int64_t)tot_h[0], (int64_t)tot_h[1], (int64_t)tot_h[2]};
    if (ordered && tot[2] >= (1LL << 31))  // (the packed 32-bit halves of Ej / Ex)
      throw Error{H2_ERR_INTERNAL, "lists: traversal frontier beyond 2^31 pairs"};
    il.ensure(nil + tot[0], nil);
    nl.ensure(nnl + tot[1], nnl);
    fb.ensure(tot[2] > 0 ? tot[2] : 1, 0);
    trav_emit_kernel<<<(unsigned)ntiles, kTravThreads, 0, s>>>(fa.p, nf, h->cell, h->nnodes, h->d, tau2, h->level,
                                                                h->is_leaf, h->nchild, h->first_child, rf,
                                                                tp.as<long long>(), il.p, nil, nl.p, nnl, fb.p, rs, re,
                                                                Ej, Ex);
    H2_CHECK_LAUNCH();
    h->gpu_launches += 2;
    nil += tot[0];
    nnl += tot[1];
    il_seg.push_back(nil);
    nl_seg.push_back(nnl);
    nf = tot[2];
    std::swap(fa.p, fb.p);
    std::swap(fa.cap, fb.cap);
  }
  h->n_il = nil;
  h->n_nf = nnl;
  if (ordered) {  // flags and longest rows of both lists in one readback (csp = the longest IL row)
    Scratch fl(sizeof(int) * 4, s);
    H2_CUDA_TRY(cudaMemsetAsync(fl.p, 0, sizeof(int) * 4, s));
    to_csr_ordered(h, il.p, nil, il_seg, h->il_off, h->il_idx, fl.as<int>());
    to_csr_ordered(h, nl.p, nnl, nl_seg, h->nf_off, h->nf_idx, fl.as<int>() + 2);
    int hf[4];
    H2_CUDA_TRY(cudaMemcpyAsync(hf, fl.p, sizeof(hf), cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaStreamSynchronize(s));
    if (hf[0]) csr_fix(h, h->il_off, h->il_idx, hf[1]);
    if (hf[2]) csr_fix(h, h->nf_off, h->nf_idx, hf[3]);
    h->csp = hf[1];
    return;
  }
  to_csr(h, il.p, nil, h->il_off, h->il_idx);
  to_csr(h, nl.p, nnl, h->nf_off, h->nf_idx);
  Scratch mx(sizeof(int), s);
  H2_CUDA_TRY(cudaMemsetAsync(mx.p, 0, sizeof(int), s));
  max_row_kernel<<<(h->nnodes + 255) / 256, 256, 0, s>>>(h->il_off, h->nnodes, mx.as<int>());
  H2_CHECK_LAUNCH();
  h->gpu_launches += 1;
  h->csp = read1(mx.as<int>(), s);
}

}  // namespace h2
