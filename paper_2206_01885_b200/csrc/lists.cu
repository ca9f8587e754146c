// lists.cu -- a4: interaction and nearfield lists by a level-synchronous dual traversal.
//
// Eq.(2.1): diam(X_i) + diam(X_j) <= 2 tau |a_i - a_j|, with the cell
// diagonal as diameter (reading B1), equality admissible (B2), pair-of-parents interaction lists
// (B3) and cross-level pairs on adaptive trees (B4).  The frontier of candidate pairs
// starts at (root, root); each step classifies every pair: admissible -> IL, both leaves -> NF,
// otherwise expand the non-leaf side (both sides when neither is a leaf).
#include "h2_internal.cuh"

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

// classify: kind 0 far, 1 near, 2 expand; counts for the three output streams
__global__ void classify_kernel(const int2* __restrict__ fr, int64_t nf, const int* __restrict__ cell, int nnodes,
                                int d, double tau2, const int* __restrict__ level, const int* __restrict__ is_leaf,
                                const int* __restrict__ nchild, int64_t* cfar, int64_t* cnear, int64_t* cexp) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nf; e += (int64_t)gridDim.x * blockDim.x) {
    int2 pr = fr[e];
    int i = pr.x, j = pr.y;
    int64_t a = 0, b = 0, c = 0;
    if (admissible(cell, nnodes, d, i, level[i], j, level[j], tau2)) {
      a = 1;
    } else {
      int li = is_leaf[i], lj = is_leaf[j];
      if (li && lj) b = 1;
      else c = (int64_t)(li ? 1 : nchild[i]) * (lj ? 1 : nchild[j]);
    }
    cfar[e] = a;
    cnear[e] = b;
    cexp[e] = c;
  }
}

__global__ void emit_kernel(const int2* __restrict__ fr, int64_t nf, const int64_t* __restrict__ ofar,
                            const int64_t* __restrict__ onear, const int64_t* __restrict__ oexp,
                            const int* __restrict__ is_leaf, const int* __restrict__ first_child,
                            const int* __restrict__ nchild, unsigned long long* il, int64_t il_base,
                            unsigned long long* nl, int64_t nl_base, int2* next) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nf; e += (int64_t)gridDim.x * blockDim.x) {
    int2 pr = fr[e];
    int i = pr.x, j = pr.y;
    unsigned long long key = ((unsigned long long)i << 32) | (unsigned)j;
    if (ofar[e + 1] != ofar[e]) {
      il[il_base + ofar[e]] = key;
    } else if (onear[e + 1] != onear[e]) {
      nl[nl_base + onear[e]] = key;
    } else {
      int li = is_leaf[i], lj = is_leaf[j];
      int ci = li ? 1 : nchild[i], cj = lj ? 1 : nchild[j];
      int fi = li ? i : first_child[i], fj = lj ? j : first_child[j];
      int64_t o = oexp[e];
      for (int a = 0; a < ci; a++)
        for (int b = 0; b < cj; b++) next[o + (int64_t)a * cj + b] = make_int2(fi + a, fj + b);
    }
  }
}

// (i << 32 | j) -> (i << bits | j): the sort then needs 2 bits key bits instead of 32 + bits
__global__ void repack_kernel(unsigned long long* keys, int64_t m, int bits) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[e];
    keys[e] = ((k >> 32) << bits) | (k & 0xffffffffULL);
  }
}

__global__ void row_count_kernel(const unsigned long long* __restrict__ keys, int64_t m, int bits,
                                 unsigned long long* cnt, int* idx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long k = keys[e];
    atomicAdd(&cnt[k >> bits], 1ULL);
    idx[e] = (int)(k & ((1ULL << bits) - 1ULL));
  }
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
  int bits = 1;
  while ((1LL << bits) <= h->nnodes) bits++;
  Scratch sorted(sizeof(unsigned long long) * (m > 0 ? m : 1), s);
  if (m > 0) {
    repack_kernel<<<grid_for(m, 256), 256, 0, s>>>(keys, m, bits);
    sort_keys_u64(keys, sorted.as<unsigned long long>(), m, 2 * bits, s);
  }
  off = halloc<int64_t>(h, h->nnodes + 1);
  idx = halloc<int>(h, m);
  Scratch cnt(sizeof(int64_t) * (h->nnodes + 1), s);
  H2_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(int64_t) * (h->nnodes + 1), s));
  if (m > 0)
    row_count_kernel<<<grid_for(m, 256), 256, 0, s>>>(sorted.as<unsigned long long>(), m, bits,
                                                      cnt.as<unsigned long long>(), idx);
  scan_excl_i64(cnt.as<int64_t>(), off, h->nnodes + 1, s);
  H2_CHECK_LAUNCH();
  h->gpu_launches += 2;
}

void build_lists(h2_handle* h) {
  cudaStream_t s = h->stream;
  const double tau2 = h->tau * h->tau;
  Grow<int2> fa(s), fb(s);
  Grow<unsigned long long> il(s), nl(s);
  fa.ensure(1, 0);
  int2 root = make_int2(0, 0);
  H2_CUDA_TRY(cudaMemcpyAsync(fa.p, &root, sizeof(int2), cudaMemcpyHostToDevice, s));
  int64_t nf = 1, nil = 0, nnl = 0;
  while (nf > 0) {
    Scratch c3(sizeof(int64_t) * 3 * (nf + 1), s), o3(sizeof(int64_t) * 3 * (nf + 1), s);
    int64_t *cfar = c3.as<int64_t>(), *cnear = cfar + nf + 1, *cexp = cnear + nf + 1;
    int64_t *ofar = o3.as<int64_t>(), *onear = ofar + nf + 1, *oexp = onear + nf + 1;
    classify_kernel<<<grid_for(nf, 256), 256, 0, s>>>(fa.p, nf, h->cell, h->nnodes, h->d, tau2, h->level,
                                                      h->is_leaf, h->nchild, cfar, cnear, cexp);
    H2_CUDA_TRY(cudaMemsetAsync(cfar + nf, 0, sizeof(int64_t), s));
    H2_CUDA_TRY(cudaMemsetAsync(cnear + nf, 0, sizeof(int64_t), s));
    H2_CUDA_TRY(cudaMemsetAsync(cexp + nf, 0, sizeof(int64_t), s));
    scan_excl_i64(cfar, ofar, nf + 1, s);
    scan_excl_i64(cnear, onear, nf + 1, s);
    scan_excl_i64(cexp, oexp, nf + 1, s);
    H2_CHECK_LAUNCH();
    h->gpu_launches += 1;
    int64_t tot[3];
    H2_CUDA_TRY(cudaMemcpyAsync(&tot[0], ofar + nf, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaMemcpyAsync(&tot[1], onear + nf, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaMemcpyAsync(&tot[2], oexp + nf, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaStreamSynchronize(s));
    il.ensure(nil + tot[0], nil);
    nl.ensure(nnl + tot[1], nnl);
    fb.ensure(tot[2] > 0 ? tot[2] : 1, 0);
    emit_kernel<<<grid_for(nf, 256), 256, 0, s>>>(fa.p, nf, ofar, onear, oexp, h->is_leaf, h->first_child, h->nchild,
                                                  il.p, nil, nl.p, nnl, fb.p);
    H2_CHECK_LAUNCH();
    h->gpu_launches += 1;
    nil += tot[0];
    nnl += tot[1];
    nf = tot[2];
    std::swap(fa.p, fb.p);
    std::swap(fa.cap, fb.cap);
  }
  h->n_il = nil;
  h->n_nf = nnl;
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
