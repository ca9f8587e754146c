// idsweep.cu -- a8: bottom-up skeleton sweep, Algorithm 2 lines 10-14.
//
// For every non-root node with Y_i^* != {} (level by level, deepest first):
//   Xbar_i = X_i at a leaf, the concatenation of the children's X^_c (child order) otherwise;
//   A = K(Xbar_i, Y_i^*) generated directly into the CTA's workspace as A^T (|Y^*| x |Xbar|);
//   CPQR ID of A^T (cpqr.cuh) -> k_i, X^_i = Xbar_i[piv[0:k]], U_i = P [I; T^T] (|Xbar| x k);
//   for a parent, the rows of U_i belonging to child c are the transfer matrix R_c.
// Symmetric kernels: V = U, W = R (reading F6).
#include "cpqr.cuh"

namespace h2 {

// global-memory path: one CTA per node; blocks of >= kIdBigBlock bytes get 1024 threads (they are
// L2-latency-bound: more columns in flight), smaller ones 256 (more CTAs per SM)
constexpr int kIdBigBlock = 256 << 10;
constexpr int kIdSmemThreads = 128;
constexpr int kIdSmemMax = 100 * 1024;  // dynamic shared memory budget of the shared-memory path

// shared-memory size classes: nodes are launched per class so small nodes get high occupancy;
// the bounds are ~228 KB / {9, 7, 6, 5, 4, 3, 2} CTAs per SM (minus the static part)
constexpr int kIdClasses = 7;
__host__ __device__ __forceinline__ int id_class_bound(int c) {
  return c == 0 ? 24 * 1024 : c == 1 ? 31 * 1024 : c == 2 ? 36 * 1024 : c == 3 ? 44 * 1024
       : c == 4 ? 55 * 1024 : c == 5 ? 74 * 1024 : kIdSmemMax;
}
__host__ __device__ __forceinline__ int id_class(int64_t bytes) {
  int c = 0;
  while (c < kIdClasses - 1 && bytes > id_class_bound(c)) c++;
  return c;
}

// shared-memory footprint of one node's ID: M (ny x nx) + nrm2 (nx) + v (ny) + piv, Xbar (2 nx ints)
// (+ staged coordinates of Xbar and Y^*: 8 (nx + ny) d bytes, + the exp table)
__host__ __device__ __forceinline__ int64_t id_smem_bytes(int ny, int nx, int d) {
  return 8LL * ((int64_t)ny * nx + nx + ny) + 8LL * nx + 8LL * d * (nx + ny) + 512;
}
// the lean layout of the one-CTA-per-SM class: no staged coordinates (the block generation reads
// them from global memory / L1)
constexpr int kIdLeanThreads = 512;
constexpr int kIdLeanMax = 226 * 1024;  // dynamic shared memory of that class (+ the small static part)
constexpr int kIdLean = kIdClasses;      // its class number
__host__ __device__ __forceinline__ int64_t id_smem_bytes_lean(int ny, int nx) {
  return 8LL * ((int64_t)ny * nx + nx + ny) + 8LL * nx + 512;
}
// Layout of a shared-memory block: row-major with a thread per column (cta_cpqr_rm) unless the
// block is tall enough that a warp per column (cta_cpqr, column-major) takes fewer serial steps:
// per pivot step ~ceil(nx / NT) * ny smem accesses per thread against ceil(nx / (NT/32)) *
// (ny / 32 + ~24 for the two warp reductions).
__host__ __device__ __forceinline__ bool id_tall(int ny, int nx, int nt) {
  const int64_t rm = (int64_t)((nx + nt - 1) / nt) * ny;
  const int64_t cm = (int64_t)((nx + nt / 32 - 1) / (nt / 32)) * (ny / 32 + 24);
  return cm < rm;
}
// the node's class: 0..kIdClasses-1 (staged, <= kIdSmemMax), kIdLean, or -1 (global-memory path)
__host__ __device__ __forceinline__ int id_smem_class(int ny, int nx, int d) {
  const int64_t b = id_smem_bytes(ny, nx, d);
  if (b <= kIdSmemMax) return id_class(b);
  return id_smem_bytes_lean(ny, nx) <= kIdLeanMax ? kIdLean : -1;
}

// per node of one level: |Xbar| (and child offsets), workspace and U sizes
__global__ void id_sizes_kernel(int base, int count, int d, const int* __restrict__ is_leaf, const int* __restrict__ nbegin,
                                const int* __restrict__ nend, const int* __restrict__ first_child,
                                const int* __restrict__ nchild, const int* __restrict__ ys_cnt,
                                const int* __restrict__ k, int* xbar_n, int* child_off, int64_t* wsz, int64_t* usz,
                                int* smax) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > count) return;
  if (t == count) {
    wsz[t] = 0;
    usz[t] = 0;
    return;
  }
  int i = base + t;
  int ny = ys_cnt[i];
  int nx = 0;
  if (is_leaf[i]) {
    nx = nend[i] - nbegin[i];
  } else {
    for (int c = 0; c < nchild[i]; c++) {
      int ch = first_child[i] + c;
      child_off[ch] = nx;
      nx += k[ch];
    }
  }
  if (ny == 0) nx = 0;
  xbar_n[i] = nx;
  int mn = nx < ny ? nx : ny;
  // workspace: M (ny*nx doubles) + nrm2 (nx) + v (ny) + piv/xbar (2*nx ints, as doubles)
  const int cls = id_smem_class(ny, nx, d);
  wsz[t] = nx > 0 && cls < 0 ? (int64_t)ny * nx + nx + ny + nx + 2 : 0;
  usz[t] = (int64_t)nx * mn;
  if (nx > 0 && cls >= 0)
    atomicMax(smax + cls, (int)(cls == kIdLean ? id_smem_bytes_lean(ny, nx) : id_smem_bytes(ny, nx, d)));
}

template <int kIdThreads>
__global__ void __launch_bounds__(kIdThreads) id_kernel(
    int base, int kid, double p2, double tol, const double* __restrict__ X, int64_t n, int d, int r,
    const int* __restrict__ is_leaf, const int* __restrict__ nbegin, const int* __restrict__ first_child,
    const int* __restrict__ nchild, const int* __restrict__ ys_cnt, const int* __restrict__ ys,
    const int* __restrict__ xbar_n, const int64_t* __restrict__ woff, double* work, const int64_t* __restrict__ uoff,
    double* U, int* kout, int* sk, unsigned long long* evals, int64_t min_block, int64_t max_block) {
  __shared__ CpqrSmem<kIdThreads> csm;
  // the Householder vector in shared memory for the big-block variant (ny <= r <= 4096, the budget
  // cap); the 256-thread variant keeps it in its global workspace (more CTAs per SM)
  __shared__ double sv[kIdThreads >= 1024 ? 4096 : 1];
  const int t = blockIdx.x;
  const int i = base + t;
  const int nx = xbar_n[i];
  const int ny = ys_cnt[i];
  const int tid = threadIdx.x;
  if (nx == 0) {
    if (tid == 0) kout[i] = 0;
    return;
  }
  if (id_smem_class(ny, nx, d) >= 0) return;  // handled by id_kernel_smem
  const int64_t blk = 8LL * nx * ny;
  if (blk < min_block || blk >= max_block) return;  // the other thread-count variant
  double* M = work + woff[t];
  double* nrm2 = M + (int64_t)ny * nx;
  double* v = nrm2 + nx;
  int* piv = reinterpret_cast<int*>(v + ny);
  int* xb = piv + nx;
  // Xbar_i (tree-order point indices)
  if (is_leaf[i]) {
    for (int b = tid; b < nx; b += kIdThreads) xb[b] = nbegin[i] + b;
  } else {
    // children's skeletons in child order; child c's rows start at sum_{c'<c} k_c'
    int o = 0;
    for (int c = 0; c < nchild[i]; c++) {
      int ch = first_child[i] + c;
      int kc = kout[ch];
      for (int a = tid; a < kc; a += kIdThreads) xb[o + a] = sk[(int64_t)ch * r + a];
      o += kc;
    }
  }
  __syncthreads();
  // A^T: M[a + ny*b] = K(Xbar[b], Y^*[a]), Y^* ascending
  const int* yv = ys + (int64_t)i * r;
  for (int64_t e = tid; e < (int64_t)ny * nx; e += kIdThreads) {
    int a = (int)(e % ny), b = (int)(e / ny);
    M[e] = kernel_pts_d(kid, p2, X, n, d, xb[b], yv[a]);
  }
  __syncthreads();
  const int k = cta_cpqr<kIdThreads>(M, ny, nx, tol, piv, nrm2, kIdThreads >= 1024 ? sv : v, csm);
  // outputs: k, skeleton (pivot order), U (nx x k column-major)
  double* Ui = U + uoff[t];
  for (int a = tid; a < k; a += kIdThreads) sk[(int64_t)i * r + a] = xb[piv[a]];
  for (int64_t e = tid; e < (int64_t)nx * k; e += kIdThreads) {
    int c = (int)(e % nx), tt = (int)(e / nx);
    double val = c < k ? (c == tt ? 1.0 : 0.0) : M[tt + (int64_t)ny * c];
    Ui[piv[c] + (int64_t)nx * tt] = val;
  }
  if (tid == 0) {
    kout[i] = k;
    atomicAdd(evals, (unsigned long long)nx * ny);
  }
}

// shared-memory path: the whole block and the CPQR live in shared memory (cpqr.cuh, row-major).
// NT = kIdSmemThreads for the staged classes (several CTAs per SM), kIdLeanThreads for the lean
// one-CTA-per-SM class (coordinates read from global memory, no staging).
template <int D, int NT>
__global__ void __launch_bounds__(NT) id_kernel_smem(
    int base, int kid, double p2, double tol, const double* __restrict__ X, int64_t n, int d_unused, int r,
    const int* __restrict__ is_leaf, const int* __restrict__ nbegin, const int* __restrict__ first_child,
    const int* __restrict__ nchild, const int* __restrict__ ys_cnt, const int* __restrict__ ys,
    const int* __restrict__ xbar_n, const int64_t* __restrict__ uoff, double* U, int* kout, int* sk,
    unsigned long long* evals, int cls) {
  extern __shared__ double sh[];
  __shared__ CpqrRmSmem<NT> csm;
  __shared__ CpqrSmem<NT> csm_cm;
  constexpr bool kLean = NT == kIdLeanThreads;
  const int i = base + blockIdx.x;
  const int nx = xbar_n[i];
  const int ny = ys_cnt[i];
  const int tid = threadIdx.x;
  if (nx == 0) return;
  {  // cls < 0: every node of the staged classes (merged launch)
    const int nc = id_smem_class(ny, nx, D);
    if (kLean ? nc != kIdLean : (nc < 0 || nc == kIdLean || (cls >= 0 && nc != cls))) return;
  }
  double* M = sh;
  double* nrm2 = M + (int64_t)ny * nx;
  double* v = nrm2 + nx;
  double* cx = v + ny;                      // Xbar coordinates, [c * nx + b] (staged classes)
  double* cy = cx + D * nx;                 // Y^* coordinates, [c * ny + a]
  double* tab = kLean ? v + ny : cy + D * ny;  // exp table
  int* piv = reinterpret_cast<int*>(tab + 64);
  int* xb = piv + nx;
  if (tid < 64) tab[tid] = kExp2Tab64[tid];
  if (is_leaf[i]) {
    for (int b = tid; b < nx; b += NT) xb[b] = nbegin[i] + b;
  } else {
    int o = 0;
    for (int c = 0; c < nchild[i]; c++) {
      const int ch = first_child[i] + c;
      const int kc = kout[ch];
      for (int a = tid; a < kc; a += NT) xb[o + a] = sk[(int64_t)ch * r + a];
      o += kc;
    }
  }
  const int* yv = ys + (int64_t)i * r;
  if (!kLean) {
    for (int a = tid; a < ny; a += NT)
#pragma unroll
      for (int c = 0; c < D; c++) cy[c * ny + a] = X[c * n + yv[a]];
    __syncthreads();
    for (int b = tid; b < nx; b += NT)
#pragma unroll
      for (int c = 0; c < D; c++) cx[c * nx + b] = X[c * n + xb[b]];
  }
  __syncthreads();
  const bool tall = id_tall(ny, nx, NT);
  auto coord_x = [&](int c, int b) { return kLean ? X[c * n + xb[b]] : cx[c * nx + b]; };
  auto coord_y = [&](int c, int a) { return kLean ? X[c * n + yv[a]] : cy[c * ny + a]; };
  int k;
  if (!tall) {
    // A^T row-major: M[a*nx + b] = K(Xbar[b], Y^*[a]), Y^* ascending; thread per column b, the
    // column's point in registers, rows' points broadcast from shared memory (or L1)
    for (int b = tid; b < nx; b += NT) {
      double xr[D];
#pragma unroll
      for (int c = 0; c < D; c++) xr[c] = coord_x(c, b);
      for (int a = 0; a < ny; a++) {
        double sq = 0.0, dt = 0.0;
#pragma unroll
        for (int c = 0; c < D; c++) {
          const double yc = coord_y(c, a), df = xr[c] - yc;
          sq = fma(df, df, sq);
          dt = fma(xr[c], yc, dt);
        }
        M[a * nx + b] = kid == H2_KERNEL_COSDOT ? kernel_cosdot(dt) : kernel_s(kid, p2, sq, tab);
      }
    }
    __syncthreads();
    k = cta_cpqr_rm<NT>(M, ny, nx, nx, tol, piv, nrm2, v, csm);
  } else {
    // tall block (few candidates, many farfield rows): A^T column-major, M[a + ny*b], and the
    // warp-per-column CPQR of cpqr.cuh on shared memory
    for (int e = tid; e < ny * nx; e += NT) {
      const int a = e % ny, b = e / ny;
      double sq = 0.0, dt = 0.0;
#pragma unroll
      for (int c = 0; c < D; c++) {
        const double xc = coord_x(c, b), yc = coord_y(c, a), df = xc - yc;
        sq = fma(df, df, sq);
        dt = fma(xc, yc, dt);
      }
      M[e] = kid == H2_KERNEL_COSDOT ? kernel_cosdot(dt) : kernel_s(kid, p2, sq, tab);
    }
    __syncthreads();
    k = cta_cpqr<NT>(M, ny, nx, tol, piv, nrm2, v, csm_cm);
  }
  double* Ui = U + uoff[blockIdx.x];
  for (int a = tid; a < k; a += NT) sk[(int64_t)i * r + a] = xb[piv[a]];
  for (int e = tid; e < nx * k; e += NT) {
    const int c = e % nx, tt = e / nx;
    const double val = c < k ? (c == tt ? 1.0 : 0.0) : (tall ? M[tt + ny * c] : M[tt * nx + c]);
    Ui[piv[c] + (int64_t)nx * tt] = val;
  }
  if (tid == 0) {
    kout[i] = k;
    atomicAdd(evals, (unsigned long long)nx * ny);
  }
}

__global__ void uoff_scatter_kernel(int base, int count, const int64_t* __restrict__ off, int64_t shift,
                                    int64_t* u_off) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) u_off[base + t] = shift + off[t];
}

__global__ void kmax_kernel(int nnodes, const int* __restrict__ k, int* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nnodes) atomicMax(out, k[i]);
}

void id_sweep(h2_handle* h) {
  cudaStream_t s = h->stream;
  const int nn = h->nnodes;
  h->k = halloc<int>(h, nn);
  h->sk = halloc<int>(h, (size_t)nn * h->r);
  h->xbar_n = halloc<int>(h, nn);
  h->child_off = halloc<int>(h, nn);
  h->u_off = halloc<int64_t>(h, nn + 1);
  H2_CUDA_TRY(cudaMemsetAsync(h->k, 0, sizeof(int) * nn, s));
  H2_CUDA_TRY(cudaMemsetAsync(h->xbar_n, 0, sizeof(int) * nn, s));
  H2_CUDA_TRY(cudaMemsetAsync(h->child_off, 0, sizeof(int) * nn, s));
  H2_CUDA_TRY(cudaMemsetAsync(h->u_off, 0, sizeof(int64_t) * (nn + 1), s));
  const double p2 = kernel_p2(h->kid, h->kp);
  Scratch ev(sizeof(unsigned long long), s);
  H2_CUDA_TRY(cudaMemsetAsync(ev.p, 0, sizeof(unsigned long long), s));
  // U arena grows level by level (sizes depend on the children's ranks)
  double* U = nullptr;
  int64_t ucap = 0, uused = 0;
  bool exchanged = h->nranks == 1;
  for (int l = h->depth; l >= 1; l--) {
    if (!exchanged && l < h->cut) {  // sharded: every rank's skeletons of the levels >= cut
      exchange_slots(h, h->k, h->sk);
      exchanged = true;
    }
    const LevelRange lr = level_range(h, l);
    int base = lr.begin, count = lr.end - lr.begin;
    if (count == 0) continue;
    Scratch sz(sizeof(int64_t) * 2 * (count + 1) + 4 * (kIdClasses + 1), s), off(sizeof(int64_t) * 2 * (count + 1), s);
    int* smax = reinterpret_cast<int*>(sz.as<int64_t>() + 2 * (count + 1));  // one max per class (+ lean)
    H2_CUDA_TRY(cudaMemsetAsync(smax, 0, (kIdClasses + 1) * sizeof(int), s));
    int64_t *wsz = sz.as<int64_t>(), *usz = wsz + count + 1;
    int64_t *woff = off.as<int64_t>(), *uo = woff + count + 1;
    id_sizes_kernel<<<(count + 1 + 255) / 256, 256, 0, s>>>(base, count, h->d, h->is_leaf, h->nbegin, h->nend,
                                                            h->first_child, h->nchild, h->ys_cnt, h->k, h->xbar_n,
                                                            h->child_off, wsz, usz, smax);
    scan_excl_i64(wsz, woff, count + 1, s);
    scan_excl_i64(usz, uo, count + 1, s);
    H2_CHECK_LAUNCH();
    int64_t tot[2];
    int smem_bytes[kIdClasses + 1] = {0};
    H2_CUDA_TRY(cudaMemcpyAsync(&tot[0], woff + count, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaMemcpyAsync(&tot[1], uo + count, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaMemcpyAsync(smem_bytes, smax, (kIdClasses + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaStreamSynchronize(s));
    if (uused + tot[1] > ucap) {
      int64_t nc = uused + tot[1];
      if (nc < 2 * ucap) nc = 2 * ucap;
      double* nu = static_cast<double*>(dev_alloc(sizeof(double) * (nc > 0 ? nc : 1), s));
      if (U && uused > 0) H2_CUDA_TRY(cudaMemcpyAsync(nu, U, sizeof(double) * uused, cudaMemcpyDeviceToDevice, s));
      if (U) dev_free(U, s);
      U = nu;
      ucap = nc;
    }
    uoff_scatter_kernel<<<(count + 255) / 256, 256, 0, s>>>(base, count, uo, uused, h->u_off);
    Scratch work(sizeof(double) * (tot[0] > 0 ? tot[0] : 1), s);
    if (tot[0] > 0) {  // some node's block exceeds the shared-memory path: global-memory CPQR
      // the two thread-count variants run concurrently on auxiliary streams (disjoint nodes)
      cudaStream_t sa = h->aux[0] ? h->aux[0] : s, sb = h->aux[1] ? h->aux[1] : s;
      cudaEvent_t gev[3];
      for (auto& e : gev) H2_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      H2_CUDA_TRY(cudaEventRecord(gev[0], s));
      H2_CUDA_TRY(cudaStreamWaitEvent(sa, gev[0], 0));
      H2_CUDA_TRY(cudaStreamWaitEvent(sb, gev[0], 0));
      id_kernel<256><<<count, 256, 0, sa>>>(base, h->kid, p2, h->id_tol, h->X, h->n, h->d, h->r, h->is_leaf,
                                           h->nbegin, h->first_child, h->nchild, h->ys_cnt, h->ys, h->xbar_n, woff,
                                           work.as<double>(), h->u_off + base, U, h->k, h->sk,
                                           ev.as<unsigned long long>(), 0, kIdBigBlock);
      id_kernel<1024><<<count, 1024, 0, sb>>>(base, h->kid, p2, h->id_tol, h->X, h->n, h->d, h->r, h->is_leaf,
                                             h->nbegin, h->first_child, h->nchild, h->ys_cnt, h->ys, h->xbar_n, woff,
                                             work.as<double>(), h->u_off + base, U, h->k, h->sk,
                                             ev.as<unsigned long long>(), kIdBigBlock, INT64_MAX);
      H2_CHECK_LAUNCH();
      H2_CUDA_TRY(cudaEventRecord(gev[1], sa));
      H2_CUDA_TRY(cudaEventRecord(gev[2], sb));
      H2_CUDA_TRY(cudaStreamWaitEvent(s, gev[1], 0));
      H2_CUDA_TRY(cudaStreamWaitEvent(s, gev[2], 0));
      for (auto& e : gev) cudaEventDestroy(e);
      h->gpu_launches += 2;
    }
    // Small levels: one launch for all classes (sized by the largest): the class launches of a
    // level run one after the other, and with few nodes each costs a node's full CPQR latency.
    // Merged when the level fits in about two waves at the largest class's occupancy.
    int smax_all = 0, ncls = 0;
    for (int cls = 0; cls < kIdClasses; cls++) {
      smax_all = smem_bytes[cls] > smax_all ? smem_bytes[cls] : smax_all;
      ncls += smem_bytes[cls] > 0;
    }
    const int per_sm = smax_all > 0 ? (228 * 1024) / (smax_all + 1024) : 0;
    const bool merge = ncls > 1 && count <= 2 * 148 * (per_sm > 0 ? per_sm : 1);
    // the class launches of a level are independent (disjoint nodes): they run concurrently on the
    // build's auxiliary streams, joined back into the main stream before the next level
    int launches[kIdClasses + 2], nl = 0;
    if (merge) launches[nl++] = -1;
    else
      for (int cls = 0; cls < kIdClasses; cls++)
        if (smem_bytes[cls] > 0) launches[nl++] = cls;
    if (smem_bytes[kIdLean] > 0) launches[nl++] = kIdLean;
    int used = 0;
    cudaEvent_t lev_ev[h2_handle::kAux + 1];
    const bool fan = nl > 1 && h->aux[0] != nullptr;
    if (fan) {
      for (auto& e : lev_ev) H2_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      H2_CUDA_TRY(cudaEventRecord(lev_ev[h2_handle::kAux], s));
    }
    for (int li = 0; li < nl; li++) {
      const int cls = launches[li];
      const int smem = cls < 0 ? smax_all : smem_bytes[cls];
      if (smem == 0) continue;
      cudaStream_t cs = s;
      if (fan) {
        const int a = used % h2_handle::kAux;
        cs = h->aux[a];
        if (used < h2_handle::kAux) H2_CUDA_TRY(cudaStreamWaitEvent(cs, lev_ev[h2_handle::kAux], 0));
        used++;
      }
      const bool lean = cls == kIdLean;
      switch (h->d) {
#define H2_ID_CASE(DD)                                                                                          \
  case DD:                                                                                                      \
    if (lean) {                                                                                                 \
      H2_CUDA_TRY(cudaFuncSetAttribute(id_kernel_smem<DD, kIdLeanThreads>,                                      \
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kIdLeanMax));               \
      id_kernel_smem<DD, kIdLeanThreads><<<count, kIdLeanThreads, smem, cs>>>(                                  \
          base, h->kid, p2, h->id_tol, h->X, h->n, h->d, h->r, h->is_leaf, h->nbegin, h->first_child,           \
          h->nchild, h->ys_cnt, h->ys, h->xbar_n, h->u_off + base, U, h->k, h->sk, ev.as<unsigned long long>(), \
          cls);                                                                                                 \
    } else {                                                                                                    \
      H2_CUDA_TRY(cudaFuncSetAttribute(id_kernel_smem<DD, kIdSmemThreads>,                                      \
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kIdSmemMax));               \
      id_kernel_smem<DD, kIdSmemThreads><<<count, kIdSmemThreads, smem, cs>>>(                                  \
          base, h->kid, p2, h->id_tol, h->X, h->n, h->d, h->r, h->is_leaf, h->nbegin, h->first_child,           \
          h->nchild, h->ys_cnt, h->ys, h->xbar_n, h->u_off + base, U, h->k, h->sk, ev.as<unsigned long long>(), \
          cls);                                                                                                 \
    }                                                                                                           \
    break;
        H2_ID_CASE(1) H2_ID_CASE(2) H2_ID_CASE(3) H2_ID_CASE(4)
        H2_ID_CASE(5) H2_ID_CASE(6) H2_ID_CASE(7) H2_ID_CASE(8)
#undef H2_ID_CASE
      }
      H2_CHECK_LAUNCH();
      h->gpu_launches += 1;
    }
    if (fan) {
      for (int a = 0; a < h2_handle::kAux && a < used; a++) {
        H2_CUDA_TRY(cudaEventRecord(lev_ev[a], h->aux[a]));
        H2_CUDA_TRY(cudaStreamWaitEvent(s, lev_ev[a], 0));
      }
      for (auto& e : lev_ev) cudaEventDestroy(e);
    }
    h->gpu_launches += 2;
    uused += tot[1];  // u_off[] holds global offsets into the arena
  }
  if (!exchanged) exchange_slots(h, h->k, h->sk);
  h->U = U ? U : static_cast<double*>(dev_alloc(8, s));
  h->allocs.push_back(h->U);
  h->u_total = uused;
  H2_CUDA_TRY(cudaMemcpyAsync(h->u_off + nn, &h->u_total, sizeof(int64_t), cudaMemcpyHostToDevice, s));
  Scratch km(sizeof(int), s);
  H2_CUDA_TRY(cudaMemsetAsync(km.p, 0, sizeof(int), s));
  kmax_kernel<<<(nn + 255) / 256, 256, 0, s>>>(nn, h->k, km.as<int>());
  H2_CHECK_LAUNCH();
  h->kmax = read1(km.as<int>(), s);
  h->id_kernel_evals = (int64_t)read1(ev.as<unsigned long long>(), s);
}

}  // namespace h2
