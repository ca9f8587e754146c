// tree.cu -- a1-a3: bounding box, Morton quantisation, radix sort, level-order tree nodes.
//
// PAPER.md P:108-113 (adaptive partition "until no more than m = O(1) points"), Fig. partition
// P:115-124.  Readings: A1 root box = cube about the bbox centre; A2 half-open cells
// defined by quantisation, clamped at the top; A3 L = min(30, floor(63/d)) key bits per dimension,
// a leaf at depth L may exceed q; A4 order (Morton key, original index), level-order ids.
#include <cfloat>

#include "h2_internal.cuh"

namespace h2 {

struct DArr {
  double v[kMaxD];
};

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
  int c = threadIdx.x;
  if (c >= d) return;
  double lo = DBL_MAX, hi = -DBL_MAX;
  for (int b = 0; b < nparts; b++) {
    lo = fmin(lo, part[(b * 2) * kMaxD + c]);
    hi = fmax(hi, part[(b * 2 + 1) * kMaxD + c]);
  }
  out[c] = lo;
  out[kMaxD + c] = hi;
}

// ---- a1: quantise + Morton interleave (dimension c of bit b at key bit d*b + c) --------------
__global__ void quantize_kernel(const double* __restrict__ pts, int64_t n, int d, DArr rlo, double s, int L,
                                long long cmax, unsigned long long* keys, int* idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long key = 0;
    if (L > 0) {
      for (int c = 0; c < d; c++) {
        double f = floor(__dmul_rn(__dsub_rn(pts[i * d + c], rlo.v[c]), s));
        long long cell = f < 0.0 ? 0 : (f > (double)cmax ? cmax : (long long)f);
        for (int b = 0; b < L; b++) key |= (unsigned long long)((cell >> b) & 1) << (d * b + c);
      }
    }
    keys[i] = key;
    idx[i] = (int)i;
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
// flag[p] = 1 iff point p starts a child of its (non-leaf) level-l node at level l+1
__global__ void level_flags_kernel(const unsigned long long* __restrict__ key, const int* __restrict__ nid, int64_t n,
                                   const int* __restrict__ is_leaf, const int* __restrict__ nbegin, int sh,
                                   int* flag, int* nid_next) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int i = nid[p];
    if (i < 0 || is_leaf[i]) {
      flag[p] = 0;
      nid_next[p] = -1;
      continue;
    }
    flag[p] = (p == nbegin[i]) || ((key[p] >> sh) != (key[p - 1] >> sh));
  }
}

__global__ void level_create_kernel(const int* __restrict__ nid, const int* __restrict__ flag,
                                    const int* __restrict__ cnt, int64_t n, const int* __restrict__ is_leaf,
                                    int base, int lvl, int* nid_next, int* level, int* nbegin, int* nend,
                                    int* parent) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int i = nid[p];
    if (i < 0 || is_leaf[i]) continue;
    int id = base + cnt[p] - 1;
    nid_next[p] = id;
    if (flag[p]) {
      nbegin[id] = (int)p;
      parent[id] = i;
      level[id] = lvl;
    }
    if (p == n - 1 || nid[p + 1] != i || flag[p + 1]) nend[id] = (int)(p + 1);
  }
}

__global__ void level_finalize_kernel(int base, int count, int q, int lvl, int L, const int* __restrict__ nbegin,
                                      const int* __restrict__ nend, const int* __restrict__ parent, int* is_leaf,
                                      int* first_child, int* nchild) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  int id = base + t;
  int c = nend[id] - nbegin[id];
  is_leaf[id] = !(c > q && lvl < L);
  first_child[id] = -1;
  nchild[id] = 0;
  int p = parent[id];
  if (nbegin[id] == nbegin[p]) first_child[p] = id;
  atomicAdd(&nchild[p], 1);
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
  Scratch part(sizeof(double) * nparts * 2 * kMaxD + sizeof(double) * 2 * kMaxD + 64, s);
  double* dpart = part.as<double>();
  double* dbox = dpart + nparts * 2 * kMaxD;
  int* dbad = reinterpret_cast<int*>(dbox + 2 * kMaxD);
  H2_CUDA_TRY(cudaMemsetAsync(dbad, 0, sizeof(int), s));
  bbox_partial_kernel<<<nparts, 256, 0, s>>>(pts, n, d, dpart, dbad);
  bbox_final_kernel<<<1, 32, 0, s>>>(dpart, nparts, d, dbox);
  H2_CHECK_LAUNCH();
  h->gpu_launches += 2;
  double box[2 * kMaxD + 1];
  H2_CUDA_TRY(cudaMemcpyAsync(box, dbox, sizeof(double) * 2 * kMaxD + sizeof(int), cudaMemcpyDeviceToHost, s));
  H2_CUDA_TRY(cudaStreamSynchronize(s));
  int bad;
  memcpy(&bad, box + 2 * kMaxD, sizeof(int));
  if (bad) throw Error{H2_ERR_NONFINITE, "a coordinate is NaN or Inf"};
  double W = 0.0;
  for (int c = 0; c < d; c++)
    if (box[kMaxD + c] - box[c] > W) W = box[kMaxD + c] - box[c];
  h->W = W;
  DArr rlo;
  for (int c = 0; c < kMaxD; c++) rlo.v[c] = 0.0;
  for (int c = 0; c < d; c++) rlo.v[c] = h->rlo[c] = (box[c] + box[kMaxD + c]) * 0.5 - W * 0.5;
  h->L = 63 / d < 30 ? 63 / d : 30;
  if (W == 0.0) h->L = 0;
  const int L = h->L;
  const double sc = L > 0 ? ldexp(1.0, L) / W : 0.0;
  const long long cmax = L > 0 ? (1LL << L) - 1 : 0;

  // a1 quantise, a2 stable radix sort by (key, original index)
  Scratch kin(sizeof(unsigned long long) * n, s), iin(sizeof(int) * n, s);
  h->key = halloc<unsigned long long>(h, n);
  h->perm = halloc<int>(h, n);
  quantize_kernel<<<grid_for(n, 256), 256, 0, s>>>(pts, n, d, rlo, sc, L, cmax, kin.as<unsigned long long>(),
                                                   iin.as<int>());
  H2_CHECK_LAUNCH();
  h->gpu_launches += 1;
  int end_bit = d * L > 0 ? d * L : 1;
  sort_pairs_u64_i32(kin.as<unsigned long long>(), h->key, iin.as<int>(), h->perm, n, end_bit, s);
  h->X = halloc<double>(h, (size_t)n * d);
  gather_soa_kernel<<<grid_for(n, 256), 256, 0, s>>>(pts, h->perm, n, d, h->X);
  H2_CHECK_LAUNCH();
  h->gpu_launches += 1;

  // a3 level-order nodes
  int cap = 0;
  h->nnodes = 0;
  grow_nodes(h, cap, (int)(n / (h->q > 1 ? h->q : 1)) * 2 + 64);
  root_init_kernel<<<1, 1, 0, s>>>((int)n, h->q, L, h->level, h->nbegin, h->nend, h->parent, h->is_leaf,
                                   h->first_child, h->nchild);
  h->gpu_launches += 1;
  h->nnodes = 1;
  h->lvl_start.assign(1, 0);
  h->lvl_start.push_back(1);
  Scratch nid_a(sizeof(int) * n, s), nid_b(sizeof(int) * n, s), flag(sizeof(int) * n, s), cnt(sizeof(int) * n, s);
  H2_CUDA_TRY(cudaMemsetAsync(nid_a.p, 0, sizeof(int) * n, s));
  int l = 0;
  while (l < L) {
    int sh = d * (L - l - 1);
    level_flags_kernel<<<grid_for(n, 256), 256, 0, s>>>(h->key, nid_a.as<int>(), n, h->is_leaf, h->nbegin, sh,
                                                        flag.as<int>(), nid_b.as<int>());
    H2_CHECK_LAUNCH();
    scan_incl_i32(flag.as<int>(), cnt.as<int>(), n, s);
    h->gpu_launches += 1;
    int total = read1(cnt.as<int>() + n - 1, s);
    if (total == 0) break;
    grow_nodes(h, cap, h->nnodes + total);
    level_create_kernel<<<grid_for(n, 256), 256, 0, s>>>(nid_a.as<int>(), flag.as<int>(), cnt.as<int>(), n,
                                                         h->is_leaf, h->nnodes, l + 1, nid_b.as<int>(), h->level,
                                                         h->nbegin, h->nend, h->parent);
    level_finalize_kernel<<<(total + 255) / 256, 256, 0, s>>>(h->nnodes, total, h->q, l + 1, L, h->nbegin, h->nend,
                                                             h->parent, h->is_leaf, h->first_child, h->nchild);
    H2_CHECK_LAUNCH();
    h->gpu_launches += 2;
    h->nnodes += total;
    h->lvl_start.push_back(h->nnodes);
    std::swap(nid_a, nid_b);
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
}

}  // namespace h2
