// tree.cu -- a1-a3: bounding box, Morton quantisation, radix sort, level-order tree nodes.
//
// PAPER.md P:108-113 (adaptive partition "until no more than m = O(1) points"), Fig. partition
// P:115-124.  Readings: A1 root box = cube about the bbox centre; A2 half-open cells
// defined by quantisation, clamped at the top; A3 L = min(30, floor(63/d)) key bits per dimension,
// a leaf at depth L may exceed q; A4 order (Morton key, original index), level-order ids.
#include <cfloat>

#include "h2_internal.cuh"

namespace h2 {

// ---- a1: bounding box (min/max are order-free, so the two-pass reduction is exact) ----------
__global__ void bbox_partial_kernel(const double* __restrict__ pts, int64_t n, int d, double* part,
                                    int* nonfinite) {
  __shared__ double slo[kMaxD][256], shi[kMaxD][256];
  double lo[kMaxD], hi[kMaxD];
  for (int c = 0; c < d; c++) {
    lo[c] = DBL_MAX;
    hi[c] = -DBL_MAX;
  }
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int c = 0; c < d; c++) {
      double v = pts[i * d + c];
      if (!isfinite(v)) bad = true;
      lo[c] = fmin(lo[c], v);
      hi[c] = fmax(hi[c], v);
    }
  }
  if (bad) atomicOr(nonfinite, 1);
  for (int c = 0; c < d; c++) {
    slo[c][threadIdx.x] = lo[c];
    shi[c][threadIdx.x] = hi[c];
  }
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int c = 0; c < d; c++) {
        slo[c][threadIdx.x] = fmin(slo[c][threadIdx.x], slo[c][threadIdx.x + s]);
        shi[c][threadIdx.x] = fmax(shi[c][threadIdx.x], shi[c][threadIdx.x + s]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int c = 0; c < d; c++) {
      part[(blockIdx.x * 2) * kMaxD + c] = slo[c][0];
      part[(blockIdx.x * 2 + 1) * kMaxD + c] = shi[c][0];
    }
}

__global__ void bbox_final_kernel(const double* part, int nparts, int d, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;  // 32 * kMaxD threads: warp w = coordinate w
  if (w < d) {
    double lo = DBL_MAX, hi = -DBL_MAX;
    for (int b = lane; b < nparts; b += 32) {
      lo = fmin(lo, part[(b * 2) * kMaxD + w]);
      hi = fmax(hi, part[(b * 2 + 1) * kMaxD + w]);
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      out[w] = lo;
      out[kMaxD + w] = hi;
    }
  }
}

// ---- a1: quantise + Morton interleave (dimension c of bit b at key bit d*b + c) --------------
// The root box (reading A1) is derived here from the device bbox with the host's operation order
// (no contraction), so no host round trip precedes the quantisation; build_tree repeats it on the
// host for h->W / h->rlo once the tree's first synchronisation has passed.  The digit histograms
// of the radix sort's passes are counted on the fly (prims.cu, onesweep).
__device__ __forceinline__ unsigned long long spread_bits(unsigned long long x, int d, int L) {
  if (d == 1) return x;
  if (d == 2) {  // bit b -> 2b
    x &= 0xffffffffULL;
    x = (x | (x << 16)) & 0x0000ffff0000ffffULL;
    x = (x | (x << 8)) & 0x00ff00ff00ff00ffULL;
    x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0fULL;
    x = (x | (x << 2)) & 0x3333333333333333ULL;
    return (x | (x << 1)) & 0x5555555555555555ULL;
  }
  if (d == 3) {  // bit b -> 3b (21 bits)
    x &= 0x1fffffULL;
    x = (x | (x << 32)) & 0x1f00000000ffffULL;
    x = (x | (x << 16)) & 0x1f0000ff0000ffULL;
    x = (x | (x << 8)) & 0x100f00f00f00f00fULL;
    x = (x | (x << 4)) & 0x10c30c30c30c30c3ULL;
    return (x | (x << 2)) & 0x1249249249249249ULL;
  }
  unsigned long long k = 0;
  for (int b = 0; b < L; b++) k |= ((x >> b) & 1ULL) << (d * b);
  return k;
}

__global__ void __launch_bounds__(256) quantize_kernel(const double* __restrict__ pts, int64_t n, int d,
                                                       const double* __restrict__ box, int L, int passes,
                                                       unsigned long long* keys, int* idx, unsigned* hist) {
  __shared__ unsigned sh[8][256];
  __shared__ double s_rlo[kMaxD], s_sc;
  for (int t = threadIdx.x; t < 8 * 256; t += blockDim.x) (&sh[0][0])[t] = 0;
  if (threadIdx.x == 0) {
    double W = 0.0;
    for (int c = 0; c < d; c++) {
      const double wc = __dsub_rn(box[kMaxD + c], box[c]);
      if (wc > W) W = wc;
    }
    for (int c = 0; c < d; c++)
      s_rlo[c] = __dsub_rn(__dmul_rn(__dadd_rn(box[c], box[kMaxD + c]), 0.5), __dmul_rn(W, 0.5));
    s_sc = L > 0 && W > 0.0 ? __ddiv_rn(ldexp(1.0, L), W) : -1.0;  // -1: no key bits (W == 0)
  }
  __syncthreads();
  const long long cmax = L > 0 ? (1LL << L) - 1 : 0;
  const double sc = s_sc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long key = 0;
    if (sc > 0.0) {
      for (int c = 0; c < d; c++) {
        double f = floor(__dmul_rn(__dsub_rn(pts[i * d + c], s_rlo[c]), sc));
        long long cell = f < 0.0 ? 0 : (f > (double)cmax ? cmax : (long long)f);
        key |= spread_bits((unsigned long long)cell, d, L) << c;
      }
    }
    keys[i] = key;
    idx[i] = (int)i;
    for (int p = 0; p < passes; p++) atomicAdd(&sh[p][(key >> (8 * p)) & 255ULL], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < passes * 256; t += blockDim.x) {
    const unsigned v = (&sh[0][0])[t];
    if (v) atomicAdd(hist + t, v);
  }
}

// gather tree-order SoA coordinates X[c*n + t] = pts[perm[t]*d + c]
__global__ void gather_soa_kernel(const double* __restrict__ pts, const int* __restrict__ perm, int64_t n, int d,
                                  double* X) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = (int64_t)perm[t] * d;
    for (int c = 0; c < d; c++) X[c * n + t] = pts[o + c];
  }
}

// ---- a3: level-by-level node construction -------------------------------------------------
// The points are sorted by key, so the children of a node [b, e) at level l are the runs of its
// points with equal child digit (key >> d(L - l - 1)) & (2^d - 1), in digit order -- level-order
// ids with key order inside a level.  Per level: one thread per (node, digit) finds the digit's
// run by two binary searches inside the node's range (O(nodes 2^d log n), not O(n)); a prefix
// sum over the existence flags numbers the children; a third kernel writes them.
__device__ __forceinline__ int digit_lower_bound(const unsigned long long* __restrict__ key, int b, int e, int sh,
                                                 unsigned mask, unsigned g) {
  while (b < e) {  // first position in [b, e) whose digit is >= g (digits are non-decreasing)
    const int mid = (b + e) >> 1;
    if ((unsigned)((key[mid] >> sh) & mask) < g) b = mid + 1;
    else e = mid;
  }
  return b;
}

__global__ void split_count_kernel(const unsigned long long* __restrict__ key, int lb, int count, int d, int sh,
                                   const int* __restrict__ nbegin, const int* __restrict__ nend,
                                   const int* __restrict__ is_leaf, int64_t* exists, int2* range) {
  const int64_t nd = (int64_t)1 << d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= count * nd;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t == count * nd) {
      exists[t] = 0;
      continue;
    }
    const int i = lb + (int)(t >> d);
    const unsigned g = (unsigned)(t & (nd - 1));
    int lo = 0, hi = 0;
    if (!is_leaf[i]) {
      const unsigned mask = (unsigned)(nd - 1);
      lo = digit_lower_bound(key, nbegin[i], nend[i], sh, mask, g);
      hi = g + 1 < nd ? digit_lower_bound(key, lo, nend[i], sh, mask, g + 1) : nend[i];
    }
    exists[t] = hi > lo;
    range[t] = make_int2(lo, hi);
  }
}

__global__ void split_create_kernel(int lb, int count, int d, int base, int lvl, int q, int L,
                                    const int64_t* __restrict__ pos, const int2* __restrict__ range, int* level,
                                    int* nbegin, int* nend, int* parent, int* is_leaf, int* first_child,
                                    int* nchild) {
  const int64_t nd = (int64_t)1 << d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count * nd;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = lb + (int)(t >> d);
    const int64_t t0 = t & ~(nd - 1);  // the node's digit 0
    if ((t & (nd - 1)) == 0) {         // one thread per parent: its child count and first child
      const int nc = (int)(pos[t0 + nd] - pos[t0]);
      nchild[i] = nc;
      first_child[i] = nc > 0 ? base + (int)pos[t0] : -1;
    }
    if (pos[t + 1] == pos[t]) continue;  // this digit has no point
    const int id = base + (int)pos[t];
    const int2 rg = range[t];
    level[id] = lvl;
    nbegin[id] = rg.x;
    nend[id] = rg.y;
    parent[id] = i;
    is_leaf[id] = !(rg.y - rg.x > q && lvl < L);
    first_child[id] = -1;
    nchild[id] = 0;
  }
}

__global__ void root_init_kernel(int n, int q, int L, int* level, int* nbegin, int* nend, int* parent, int* is_leaf,
                                 int* first_child, int* nchild) {
  level[0] = 0;
  nbegin[0] = 0;
  nend[0] = n;
  parent[0] = -1;
  is_leaf[0] = !(n > q && L > 0);
  first_child[0] = -1;
  nchild[0] = 0;
}

// integer cell coordinates of every node at its own level (de-interleaved key prefix)
__global__ void cells_kernel(int nnodes, int d, int L, const int* __restrict__ level, const int* __restrict__ nbegin,
                             const unsigned long long* __restrict__ key, int* cell, int* nleaves,
                             const int* __restrict__ is_leaf) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnodes) return;
  int li = level[i];
  unsigned long long pre = li > 0 ? key[nbegin[i]] >> (d * (L - li)) : 0ULL;
  for (int c = 0; c < d; c++) {
    int v = 0;
    for (int b = 0; b < li; b++) v |= (int)((pre >> (d * b + c)) & 1ULL) << b;
    cell[(int64_t)c * nnodes + i] = v;
  }
  if (is_leaf[i]) atomicAdd(nleaves, 1);
}

static void grow_nodes(h2_handle* h, int& cap, int need) {
  if (need <= cap) return;
  int ncap = need > 2 * cap ? need : 2 * cap;
  int** arrs[7] = {&h->level, &h->nbegin, &h->nend, &h->parent, &h->first_child, &h->nchild, &h->is_leaf};
  for (int a = 0; a < 7; a++) {
    int* np = halloc<int>(h, ncap);
    if (*arrs[a]) {
      if (h->nnodes > 0)
        H2_CUDA_TRY(cudaMemcpyAsync(np, *arrs[a], sizeof(int) * h->nnodes, cudaMemcpyDeviceToDevice, h->stream));
      hfree(h, *arrs[a]);
    }
    *arrs[a] = np;
  }
  cap = ncap;
}

void build_tree(h2_handle* h, const double* pts) {
  cudaStream_t s = h->stream;
  const int64_t n = h->n;
  const int d = h->d;
  // a1 bounding box
  const int nparts = (int)grid_for(n, 256, 148 * 2);
  Scratch part(sizeof(double) * nparts * 2 * kMaxD + sizeof(double) * 2 * kMaxD + 64 + sizeof(unsigned) * 8 * 256, s);
  double* dpart = part.as<double>();
  double* dbox = dpart + nparts * 2 * kMaxD;
  int* dbad = reinterpret_cast<int*>(dbox + 2 * kMaxD);
  unsigned* dhist = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(dbad) + 64);
  H2_CUDA_TRY(cudaMemsetAsync(dbad, 0, 64 + sizeof(unsigned) * 8 * 256, s));
  bbox_partial_kernel<<<nparts, 256, 0, s>>>(pts, n, d, dpart, dbad);
  bbox_final_kernel<<<1, 32 * kMaxD, 0, s>>>(dpart, nparts, d, dbox);
  H2_CHECK_LAUNCH();
  h->gpu_launches += 2;
  // the box and the non-finite flag reach the host with the tree's first synchronisation below
  thread_local double* box = nullptr;  // page-locked, per host thread
  if (!box) H2_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&box), sizeof(double) * (2 * kMaxD + 1)));
  H2_CUDA_TRY(cudaMemcpyAsync(box, dbox, sizeof(double) * 2 * kMaxD + sizeof(int), cudaMemcpyDeviceToHost, s));
  h->L = 63 / d < 30 ? 63 / d : 30;
  const int Lq = h->L;  // W == 0 (every point equal) gives L = 0 below; the keys are then all 0 either way

  // a1 quantise, a2 stable radix sort by (key, original index)
  Scratch kin(sizeof(unsigned long long) * n, s), iin(sizeof(int) * n, s);
  h->key = halloc<unsigned long long>(h, n);
  h->perm = halloc<int>(h, n);
  const int end_bit = d * Lq > 0 ? d * Lq : 1;
  const int passes = (end_bit + 7) / 8;
  quantize_kernel<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(pts, n, d, dbox, Lq, passes, kin.as<unsigned long long>(),
                                                            iin.as<int>(), dhist);
  H2_CHECK_LAUNCH();
  h->gpu_launches += 1;
  sort_pairs_u64_i32(kin.as<unsigned long long>(), h->key, iin.as<int>(), h->perm, n, end_bit, s, dhist);
  h->X = halloc<double>(h, (size_t)n * d);
  gather_soa_kernel<<<grid_for(n, 256), 256, 0, s>>>(pts, h->perm, n, d, h->X);
  H2_CHECK_LAUNCH();
  h->gpu_launches += 1;
  bool box_read = false;
  auto read_box = [&]() {  // after a stream synchronisation
    if (box_read) return;
    box_read = true;
    int bad;
    memcpy(&bad, box + 2 * kMaxD, sizeof(int));
    if (bad) throw Error{H2_ERR_NONFINITE, "a coordinate is NaN or Inf"};
    double W = 0.0;
    for (int c = 0; c < d; c++)
      if (box[kMaxD + c] - box[c] > W) W = box[kMaxD + c] - box[c];
    h->W = W;
    for (int c = 0; c < d; c++) h->rlo[c] = (box[c] + box[kMaxD + c]) * 0.5 - W * 0.5;
  };

  // a3 level-order nodes
  int cap = 0;
  h->nnodes = 0;
  grow_nodes(h, cap, (int)(n / (h->q > 1 ? h->q : 1)) * 2 + 64);
  int L = Lq;
  root_init_kernel<<<1, 1, 0, s>>>((int)n, h->q, L, h->level, h->nbegin, h->nend, h->parent, h->is_leaf,
                                   h->first_child, h->nchild);
  h->gpu_launches += 1;
  h->nnodes = 1;
  h->lvl_start.assign(1, 0);
  h->lvl_start.push_back(1);
  int l = 0;
  const int64_t nd = (int64_t)1 << d;
  while (l < L) {
    const int lb = h->lvl_start[l], count = h->lvl_start[l + 1] - lb;
    const int64_t m = count * nd;
    Scratch ex(sizeof(int64_t) * (m + 1), s), pos(sizeof(int64_t) * (m + 1), s), rg(sizeof(int2) * (m + 1), s);
    split_count_kernel<<<grid_for(m + 1, 256), 256, 0, s>>>(h->key, lb, count, d, d * (L - l - 1), h->nbegin, h->nend,
                                                           h->is_leaf, ex.as<int64_t>(), rg.as<int2>());
    scan_excl_i64(ex.as<int64_t>(), pos.as<int64_t>(), m + 1, s);
    H2_CHECK_LAUNCH();
    h->gpu_launches += 1;
    const int total = (int)read1(pos.as<int64_t>() + m, s);
    read_box();
    if (h->W == 0.0) {  // every point equal: no key bits, the root is the only node (a leaf)
      h->L = L = 0;
      root_init_kernel<<<1, 1, 0, s>>>((int)n, h->q, 0, h->level, h->nbegin, h->nend, h->parent, h->is_leaf,
                                       h->first_child, h->nchild);
      h->gpu_launches += 1;
      break;
    }
    if (total == 0) break;
    grow_nodes(h, cap, h->nnodes + total);
    split_create_kernel<<<grid_for(m, 256), 256, 0, s>>>(lb, count, d, h->nnodes, l + 1, h->q, L, pos.as<int64_t>(),
                                                        rg.as<int2>(), h->level, h->nbegin, h->nend, h->parent,
                                                        h->is_leaf, h->first_child, h->nchild);
    H2_CHECK_LAUNCH();
    h->gpu_launches += 1;
    h->nnodes += total;
    h->lvl_start.push_back(h->nnodes);
    l++;
  }
  h->depth = (int)h->lvl_start.size() - 2;
  h->cell = halloc<int>(h, (size_t)h->nnodes * d);
  Scratch nl(sizeof(int), s);
  H2_CUDA_TRY(cudaMemsetAsync(nl.p, 0, sizeof(int), s));
  cells_kernel<<<(h->nnodes + 255) / 256, 256, 0, s>>>(h->nnodes, d, L, h->level, h->nbegin, h->key, h->cell,
                                                       nl.as<int>(), h->is_leaf);
  H2_CHECK_LAUNCH();
  h->gpu_launches += 1;
  h->nleaves = read1(nl.as<int>(), s);
  read_box();
}

}  // namespace h2
