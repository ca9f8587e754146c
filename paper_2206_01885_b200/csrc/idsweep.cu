// idsweep.cu -- a8: bottom-up skeleton sweep, Algorithm 2 lines 10-14.
//
// For every non-root node with Y_i^* != {} (level by level, deepest first):
//   Xbar_i = X_i at a leaf, the concatenation of the children's X^_c (child order) otherwise;
//   A = K(Xbar_i, Y_i^*) generated directly into the CTA's workspace as A^T (|Y^*| x |Xbar|);
//   CPQR ID of A^T (cpqr.cuh) -> k_i, X^_i = Xbar_i[piv[0:k]], U_i = P [I; T^T] (|Xbar| x k);
//   for a parent, the rows of U_i belonging to child c are the transfer matrix R_c.
// Symmetric kernels: V = U, W = R (reading F6).
#include <cooperative_groups.h>

#include <cstdlib>

#include "cpqr.cuh"
#include "cpqr_panel.cuh"
#include "id_warp.cuh"

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

constexpr int kIdPanelNb = 8;  // panel width of the blocked CPQR (cpqr_panel.cuh)
// rows the panel CPQR's leading dimension adds for a node of nx columns on NT threads (panel_ld)
__host__ __device__ __forceinline__ int id_pad_rows(int nx, int nt) {
  const int G = panel_group(nx, nt);
  return G <= 8 ? 2 * G - 1 : 0;
}
__host__ __device__ __forceinline__ bool id_tall(int ny, int nx, int nt);
// the panel-blocked CPQR runs a node of a shared-memory class on NT threads when the block is tall
// (the column-major layout; wide blocks keep the row-major thread-per-column CPQR) and its columns
// fit the thread groups (cpqr_panel.cuh: at most RMAX columns per group)
__host__ __device__ __forceinline__ int id_panel_rmax(int nt) { return nt >= 512 ? 4 : 2; }
__host__ __device__ __forceinline__ bool id_panel(int ny, int nx, int nt) {
  return id_tall(ny, nx, nt) && (int64_t)nx * panel_group(nx, nt) <= (int64_t)nt * id_panel_rmax(nt);
}
// doubles a node's block and CPQR scratch take: M (+ the panel's padding rows and F) + nrm2 + v
__host__ __device__ __forceinline__ int64_t id_block_doubles(int ny, int nx, int nt) {
  return id_panel(ny, nx, nt) ? (int64_t)(ny + id_pad_rows(nx, nt)) * nx + kIdPanelNb * nx + nx + ny
                              : (int64_t)ny * nx + nx + ny;
}
// shared-memory footprint of one node's ID: block + scratch + piv, Xbar (2 nx ints) (+ staged
// coordinates of Xbar and Y^*: 8 (nx + ny) d bytes, + the exp table)
__host__ __device__ __forceinline__ int64_t id_smem_bytes(int ny, int nx, int d) {
  return 8LL * id_block_doubles(ny, nx, 128) + 8LL * nx + 8LL * d * (nx + ny) + 512;
}
// the lean layout of the one-CTA-per-SM class: no staged coordinates (the block generation reads
// them from global memory / L1)
constexpr int kIdLeanThreads = 512;
constexpr int kIdLeanMax = 226 * 1024;  // dynamic shared memory of that class (+ the small static part)
constexpr int kIdLean = kIdClasses;      // its class number
__host__ __device__ __forceinline__ int64_t id_smem_bytes_lean(int ny, int nx, int nt = 512) {
  return 8LL * id_block_doubles(ny, nx, nt) + 8LL * nx + 512;
}
// The mid class (class kIdMid = kIdClasses - 1): blocks between the staged classes and the lean one
// (e.g. configs[1]'s 64 x ~208 leaves: 115 KB staged, 108 KB lean) run with the lean layout on 256
// threads, two CTAs per SM, instead of one 512-thread CTA per SM (a wide block's row-major CPQR has a
// thread per column, so 512 threads leave most idle while the SM holds a single node)
constexpr int kIdMid = kIdClasses - 1;
constexpr int kIdMidThreads = 256;
constexpr int kIdMidMax = 110 * 1024;
__host__ __device__ __forceinline__ int id_class_threads(int c);
// what a lean (or mid) node asks for: its footprint plus staged coordinates when both fit the class
__host__ __device__ __forceinline__ int64_t id_lean_request(int ny, int nx, int d, int nt = 512) {
  const int64_t cap = nt >= 512 ? kIdLeanMax : kIdMidMax;
  const int64_t b = id_smem_bytes_lean(ny, nx, nt), bs = b + 8LL * d * (nx + ny);
  return bs <= cap ? bs : b;
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
// the node's class: 0..kIdMid-1 (staged, <= id_class_bound(kIdMid - 1)), kIdMid (lean layout, 256
// threads, <= kIdMidMax), kIdLean, or -1 (global-memory path)
__host__ __device__ __forceinline__ int id_smem_class(int ny, int nx, int d) {
  const int64_t b = id_smem_bytes(ny, nx, d);
  if (b <= id_class_bound(kIdMid - 1)) return id_class(b);
  if (id_smem_bytes_lean(ny, nx, kIdMidThreads) <= kIdMidMax) return kIdMid;
  return id_smem_bytes_lean(ny, nx) <= kIdLeanMax ? kIdLean : -1;
}
__host__ __device__ __forceinline__ int id_class_threads(int c) {
  return c == kIdLean ? kIdLeanThreads : c == kIdMid ? kIdMidThreads : kIdSmemThreads;
}

// The largest blocks (>= kIdClusterMin entries) take the cluster path (id_kernel_cluster): on one
// SM the global-memory CPQR of such a block is bound by that SM's L2 / HBM bandwidth (tens of ms for
// the biggest blocks of configs[4]), so a thread-block cluster of CS CTAs spreads its columns over CS
// SMs.  cs = the cluster size the device runs (16, else 8; 0 disables the path); cl_min = the
// block-entry threshold.
constexpr int kIdClThreads = 512;
constexpr int kIdClMaxNx = 8192;  // the cluster kernel's shared memory (~20 nx + 8 r bytes) stays < 200 KB
__host__ __device__ __forceinline__ bool id_big(int ny, int nx, int d, int cs, int64_t cl_min) {
  return cs >= 2 && nx >= 4 * cs && nx <= kIdClMaxNx && (int64_t)ny * nx >= cl_min && id_smem_class(ny, nx, d) < 0;
}

// per node of one level: |Xbar| (and child offsets), workspace and U sizes
__global__ void id_sizes_kernel(int base, int count, int d, const int* __restrict__ is_leaf, const int* __restrict__ nbegin,
                                const int* __restrict__ nend, const int* __restrict__ first_child,
                                const int* __restrict__ nchild, const int* __restrict__ ys_cnt,
                                const int* __restrict__ k, int* xbar_n, int* child_off, int64_t* wsz, int64_t* usz,
                                int* smax, int cs, int64_t cl_min, int* cl_cnt, int* cl_list, int* id_path,
                                int warp_level, int* wp_cnt, int* wp_list, int* lcnt, int* lists) {
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
  // levels with many nodes: the small ones take the warp-per-node path (id_warp.cuh)
  if (warp_level && nx > 0 && nx <= 32 * kIdWarpMaxCols && id_warp_bytes(ny, nx) <= kIdWarpMaxBytes) {
    wp_list[atomicAdd(wp_cnt, 1)] = t;
    atomicMax(wp_cnt + 1, (int)id_warp_bytes(ny, nx));
    id_path[i] = 11;
    wsz[t] = 0;
    usz[t] = (int64_t)nx * mn;
    return;
  }
  // workspace: M (ny*nx doubles) + nrm2 (nx) + v (ny) + piv/xbar (2*nx ints, as doubles)
  const int cls = id_smem_class(ny, nx, d);
  const bool big = nx > 0 && id_big(ny, nx, d, cs, cl_min);
  if (big) {
    cl_list[atomicAdd(cl_cnt, 1)] = t;
    atomicMax(smax + kIdClasses + 1, nx);  // the cluster kernel's shared memory is sized by it
  }
  // cluster path: M (column slices) + the staged candidate columns (2 parities x CS x ny)
  wsz[t] = big ? (int64_t)ny * (((nx + cs - 1) / cs) * cs) + 2LL * cs * ny
         : nx > 0 && cls < 0 ? (int64_t)ny * nx + kIdPanelNb * nx + nx + ny + nx + 2 : 0;
  usz[t] = (int64_t)nx * mn;
  // the code path (H2_EXPORT_ID_PATH): 0..6 staged shared-memory classes, 7 lean class, 8 global
  // memory (256 threads), 9 global memory (1024 threads), 10 thread-block cluster, 11 warp per node,
  // -1 none
  id_path[i] = nx == 0 ? -1 : big ? 10 : cls >= 0 ? cls : (8LL * nx * ny < kIdBigBlock ? 8 : 9);
  if (nx > 0 && cls >= 0) {
    atomicMax(smax + cls, (int)(cls >= kIdMid ? id_lean_request(ny, nx, d, id_class_threads(cls))
                                              : id_smem_bytes(ny, nx, d)));
    // which instantiations the class needs: bit 0 unblocked / row-major nodes, bit 1 panel nodes
    const int pk = id_panel(ny, nx, id_class_threads(cls)) ? 1 : 0;
    atomicOr(smax + kIdClasses + 2 + cls, pk ? 2 : 1);
    // the launch lists: per (class, kind), and per kind over all staged classes (merged launch)
    const int li = cls * 2 + pk;
    lists[(int64_t)li * count + atomicAdd(lcnt + li, 1)] = t;
    if (cls < kIdMid) {  // (the mid class has its own thread count: never merged)
      const int lm = 2 * (kIdClasses + 1) + pk;
      lists[(int64_t)lm * count + atomicAdd(lcnt + lm, 1)] = t;
    }
  }
}

// dynamic shared memory of the global-memory path: F of the panel CPQR (NB x nx, nx <= NT RMAX / 4)
constexpr int kIdGlobalFs = 4096;

template <int kIdThreads>
__global__ void __launch_bounds__(kIdThreads) id_kernel(
    int base, int kid, double p2, double tol, const double* __restrict__ Xf, const double* __restrict__ X, int64_t n,
    int d, int r,
    const int* __restrict__ is_leaf, const int* __restrict__ nbegin, const int* __restrict__ first_child,
    const int* __restrict__ nchild, const int* __restrict__ ys_cnt, const int* __restrict__ ys,
    const int* __restrict__ xbar_n, const int64_t* __restrict__ woff, double* work, const int64_t* __restrict__ uoff,
    double* U, int* kout, int* sk, unsigned long long* evals, int64_t min_block, int64_t max_block, int cs,
    int64_t cl_min, int use_panel, const int* __restrict__ id_path) {
  __shared__ CpqrSmem<kIdThreads> csm;
  constexpr int kNbG = kIdThreads >= 1024 ? 4 : kIdPanelNb;  // (64 registers per thread at 1024)
  __shared__ PanelSmem<kIdThreads, kNbG> psm;
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
  if (id_path[i] == 11) return;  // id_kernel_warp
  if (id_smem_class(ny, nx, d) >= 0 || id_big(ny, nx, d, cs, cl_min)) return;  // id_kernel_smem / _cluster
  const int64_t blk = 8LL * nx * ny;
  if (blk < min_block || blk >= max_block) return;  // the other thread-count variant
  // the panel-blocked CPQR with at least 4 threads per column (32-byte sectors of L2), when the
  // columns fit RMAX rounds of thread groups; else the warp-per-column one
  constexpr int kRmaxG = kIdThreads >= 1024 ? 2 : 4;
  const int Gp = panel_group(nx, kIdThreads);
  const int G = Gp < 4 ? 4 : Gp;
  const bool panel = (use_panel & 4) && (int64_t)nx * G <= (int64_t)kIdThreads * kRmaxG;
  double* M = work + woff[t];
  // the panel's delayed-update coefficients in shared memory (kIdGlobalFs doubles: nx <= NT RMAX / 4)
  extern __shared__ double Fs[];
  double* nrm2 = M + (int64_t)ny * nx + kIdPanelNb * nx;
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
    M[e] = kernel_pts_d(kid, p2, Xf, X, n, d, xb[b], yv[a]);
  }
  __syncthreads();
  const int k = panel ? cta_cpqr_panel<kIdThreads, kNbG, kRmaxG>(M, ny, ny, nx, tol, G, piv, Fs, psm)
                      : cta_cpqr<kIdThreads>(M, ny, nx, tol, piv, nrm2, kIdThreads >= 1024 ? sv : v, csm);
  // outputs: k, skeleton (pivot order), U (nx x k column-major)
  double* Ui = U + uoff[t];
  for (int a = tid; a < k; a += kIdThreads) sk[(int64_t)i * r + a] = xb[piv[a]];
  for (int64_t e = tid; e < (int64_t)nx * k; e += kIdThreads) {
    int c = (int)(e % nx), tt = (int)(e / nx);
    double val = c < k ? (c == tt ? 1.0 : 0.0) : M[tt + (int64_t)ny * (panel ? piv[c] : c)];
    Ui[piv[c] + (int64_t)nx * tt] = val;
  }
  if (tid == 0) {
    kout[i] = k;
    atomicAdd(evals, (unsigned long long)nx * ny);
  }
}

// Cluster path (id_big): a thread-block cluster of CS CTAs per node; CTA q owns the columns
// [q w, q w + w), w = ceil(nx / CS), of A^T in the node's global workspace (column-major, ld = ny).
// Columns never move: the pivot order lives in a position map replicated in every CTA (col_at) and
// in each CTA's `pos` of its own columns.  One cluster barrier per pivot step: after it every CTA
// reads the CTAs' candidates (largest residual norm, ties to the lowest position; DSMEM) and picks
// the same pivot p; it reads column p from the owner's staged copy (global, double-buffered by step
// parity, written before the barrier: L2 serves the CS readers), builds the Householder vector and
// v^T v itself (the same arithmetic in every CTA), applies it to its own live columns, recomputes
// their residual norms and stages its next candidate.  The pivot column is not written in that
// phase (others read its staged copy); its diagonal alpha is stored after the next barrier, its rows
// below the diagonal are never read again.  The algorithm and tie rule of cta_cpqr.
struct IdClCand {
  double x;  // sqrt of the residual norm^2 (-1: no live column)
  int pos;   // position in the pivot order
  int j;     // column index in Xbar
};

__global__ void __launch_bounds__(kIdClThreads) id_kernel_cluster(
    int base, const int* __restrict__ list, int kid, double p2, double tol, const double* __restrict__ Xf,
    const double* __restrict__ X, int64_t n,
    int d, int r, const int* __restrict__ is_leaf, const int* __restrict__ nbegin,
    const int* __restrict__ first_child, const int* __restrict__ nchild, const int* __restrict__ ys_cnt,
    const int* __restrict__ ys, const int* __restrict__ xbar_n, const int64_t* __restrict__ woff, double* work,
    const int64_t* __restrict__ uoff, double* U, int* kout, int* sk, unsigned long long* evals) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  constexpr int NT = kIdClThreads, NW = NT / 32;
  const int CS = (int)cl.num_blocks(), q = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = list[blockIdx.x / CS];
  const int i = base + t;
  const int nx = xbar_n[i], ny = ys_cnt[i];
  const int w = (nx + CS - 1) / CS, j0 = q * w;
  const int wl = nx - j0 < 0 ? 0 : (nx - j0 < w ? nx - j0 : w);  // live width of this CTA's slice
  extern __shared__ double sh[];
  double* v = sh;                       // Householder vector (ny)
  double* nrm2 = v + ny;                // residual norms^2 of the own columns (w)
  double* tab = nrm2 + w;               // exp table (64)
  int* col_at = reinterpret_cast<int*>(tab + 64);  // position -> column (nx)
  int* xb = col_at + nx;                // Xbar (nx)
  int* pos = xb + nx;                   // own column -> position (w)
  __shared__ IdClCand cand[2];          // this CTA's candidate by step parity (read by every CTA)
  __shared__ IdClCand best_s;
  __shared__ CpqrSmem<NT> csm;
  double* const Mall = work + woff[t];
  double* const Mq = Mall + (int64_t)q * w * ny;
  double* const stage = Mall + (int64_t)CS * w * ny;  // [parity][CTA][ny]
  auto staged = [&](int parity, int cta) { return stage + ((int64_t)parity * CS + cta) * ny; };
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
  for (int b = tid; b < nx; b += NT) col_at[b] = b;
  for (int b = tid; b < w; b += NT) pos[b] = j0 + b;
  __syncthreads();
  // own columns of A^T: Mq[a + ny*jl] = K(Xbar[j0 + jl], Y^*[a])
  const int* yv = ys + (int64_t)i * r;
  for (int64_t e = tid; e < (int64_t)wl * ny; e += NT) {
    const int a = (int)(e % ny), jl = (int)(e / ny);
    Mq[e] = kernel_pts_d(kid, p2, Xf, X, n, d, xb[j0 + jl], yv[a]);
  }
  __syncthreads();
  for (int jl = warp; jl < wl; jl += NW) {
    const double* col = Mq + (int64_t)ny * jl;
    double s = 0.0;
    for (int a = lane; a < ny; a += 32) s += col[a] * col[a];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) nrm2[jl] = s;
  }
  __syncthreads();
  // the candidate among the own live columns (position >= tt), published in shared memory, its
  // column (rows tt..) staged in global memory
  auto publish = [&](int tt) {
    if (warp == 0) {
      double bx = -1.0;
      int bp = INT_MAX, bj = -1;
      for (int jl = lane; jl < wl; jl += 32) {
        const int ps = pos[jl];
        if (ps < tt) continue;
        const double x = sqrt(nrm2[jl]);
        if (x > bx || (x == bx && ps < bp)) {
          bx = x;
          bp = ps;
          bj = j0 + jl;
        }
      }
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
      if (lane == 0) best_s = cand[tt & 1] = IdClCand{bx, bp, bj};
    }
    __syncthreads();
    const int bj = best_s.j;
    if (bj >= 0) {
      const double* col = Mq + (int64_t)ny * (bj - j0);
      double* dst = staged(tt & 1, q);
      for (int a = tt + tid; a < ny; a += NT) dst[a] = col[a];
    }
  };
  publish(0);
  const int kmax = ny < nx ? ny : nx;
  double r11 = 0.0;
  int k = 0;
  int pend_jl = -1, pend_row = 0;  // own pivot column whose diagonal is written after the barrier
  double pend_alpha = 0.0;
  for (int tt = 0; tt < kmax; tt++) {
    cl.sync();
    if (pend_jl >= 0 && tid == 0) Mq[(int64_t)ny * pend_jl + pend_row] = pend_alpha;
    pend_jl = -1;
    if (warp == 0) {  // the pivot: the best of the CTAs' candidates
      IdClCand c{-1.0, INT_MAX, -1};
      if (lane < CS) c = *cl.map_shared_rank(&cand[tt & 1], lane);
      for (int o = 16; o > 0; o >>= 1) {
        const double x2 = __shfl_xor_sync(0xffffffffu, c.x, o);
        const int p2_ = __shfl_xor_sync(0xffffffffu, c.pos, o);
        const int j2 = __shfl_xor_sync(0xffffffffu, c.j, o);
        if (x2 > c.x || (x2 == c.x && p2_ < c.pos)) c = IdClCand{x2, p2_, j2};
      }
      if (lane == 0) best_s = c;
    }
    __syncthreads();
    const IdClCand b = best_s;
    const double nrm = b.x;
    if (tt == 0) {
      r11 = nrm;
      if (r11 == 0.0) break;
    }
    if (nrm < tol * r11) break;
    const int p = b.j, owner = p / w;
    // the Householder vector of column p (rows tt..) from the owner's staged copy
    const double* src = staged(tt & 1, owner);
    const double x0 = src[tt];
    const double alpha = x0 >= 0.0 ? -nrm : nrm;
    double part = 0.0;
    for (int a = tt + tid; a < ny; a += NT) {
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
      if (jt >= j0 && jt < j0 + wl) pos[jt - j0] = b.pos;
      if (p >= j0 && p < j0 + wl) pos[p - j0] = tt;
    }
    __syncthreads();
    // own live columns (positions > tt): reflector, residual norm over rows > tt
    for (int jl = warp; jl < wl; jl += NW) {
      if (pos[jl] <= tt) continue;
      double* col = Mq + (int64_t)ny * jl;
      if (vtv > 0.0) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int a = tt + lane;
        for (; a + 96 < ny; a += 128) {
          const double c0 = col[a], c1 = col[a + 32], c2 = col[a + 64], c3 = col[a + 96];
          s0 += v[a] * c0;
          s1 += v[a + 32] * c1;
          s2 += v[a + 64] * c2;
          s3 += v[a + 96] * c3;
        }
        for (; a < ny; a += 32) s0 += v[a] * col[a];
        double s = (s0 + s1) + (s2 + s3);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const double f = 2.0 * s / vtv;
        double n0 = 0.0, n1 = 0.0, n2 = 0.0, n3 = 0.0;
        a = tt + lane;
        for (; a + 96 < ny; a += 128) {
          const double a0 = col[a] - f * v[a], a1 = col[a + 32] - f * v[a + 32];
          const double a2 = col[a + 64] - f * v[a + 64], a3 = col[a + 96] - f * v[a + 96];
          col[a] = a0;
          col[a + 32] = a1;
          col[a + 64] = a2;
          col[a + 96] = a3;
          if (a > tt) n0 += a0 * a0;
          n1 += a1 * a1;
          n2 += a2 * a2;
          n3 += a3 * a3;
        }
        for (; a < ny; a += 32) {
          const double x = col[a] - f * v[a];
          col[a] = x;
          if (a > tt) n0 += x * x;
        }
        double nn = (n0 + n1) + (n2 + n3);
        for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
        if (lane == 0) nrm2[jl] = nn;
      } else {
        double nn = 0.0;
        for (int a = tt + 1 + lane; a < ny; a += 32) nn += col[a] * col[a];
        for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
        if (lane == 0) nrm2[jl] = nn;
      }
    }
    k = tt + 1;
    __syncthreads();
    publish(tt + 1);
  }
  if (pend_jl >= 0 && tid == 0) Mq[(int64_t)ny * pend_jl + pend_row] = pend_alpha;
  cl.sync();  // every R column final and visible (global memory, cluster scope)
  // T = R11^{-1} R12 on the own live columns (positions >= k), R11 read from its owners' slices
  // through a pointer table (in v's space: k <= ny); four partial sums per row
  const double** rcol = reinterpret_cast<const double**>(v);
  for (int l = tid; l < k; l += NT) {
    const int jj = col_at[l];
    rcol[l] = Mall + (int64_t)ny * jj;  // slice q' starts at q' w ny: column jj is at jj * ny
  }
  __syncthreads();
  for (int jl = tid; jl < wl; jl += NT) {
    if (pos[jl] < k) continue;
    double* col = Mq + (int64_t)ny * jl;
    for (int a = k - 1; a >= 0; a--) {
      double s0 = col[a], s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int l = a + 1;
      for (; l + 3 < k; l += 4) {
        s0 -= rcol[l][a] * col[l];
        s1 -= rcol[l + 1][a] * col[l + 1];
        s2 -= rcol[l + 2][a] * col[l + 2];
        s3 -= rcol[l + 3][a] * col[l + 3];
      }
      for (; l < k; l++) s0 -= rcol[l][a] * col[l];
      col[a] = ((s0 + s1) + (s2 + s3)) / rcol[a][a];
    }
  }
  __syncthreads();
  // outputs: skeleton (pivot order), U (nx x k column-major): identity rows of the skeleton, T for
  // the others
  // every CTA writes the rows of its own columns (coalesced along them): the identity for the
  // skeleton columns, T for the others
  double* Ui = U + uoff[t];
  if (q == 0)
    for (int a = tid; a < k; a += NT) sk[(int64_t)i * r + a] = xb[col_at[a]];
  for (int e = tid; e < wl * k; e += NT) {
    const int jl = e % wl, tt = e / wl;
    const int ps = pos[jl];
    Ui[j0 + jl + (int64_t)nx * tt] = ps < k ? (ps == tt ? 1.0 : 0.0) : Mq[(int64_t)ny * jl + tt];
  }
  if (q == 0 && tid == 0) {
    kout[i] = k;
    atomicAdd(evals, (unsigned long long)nx * ny);
  }
  cl.sync();  // no CTA leaves while another may still read its shared memory
}

// shared-memory path: the whole block and the CPQR live in shared memory (cpqr.cuh, row-major).
// NT = kIdSmemThreads for the staged classes (several CTAs per SM), kIdLeanThreads for the lean
// one-CTA-per-SM class (coordinates read from global memory, no staging).
// PANEL: this instantiation runs the nodes whose blocks take the panel layout (id_panel); the other
// one the rest (its registers stay at the unblocked CPQR's ~64, for occupancy)
template <int D, int NT, bool PANEL>
__global__ void __launch_bounds__(NT, NT >= 512 ? 1 : NT >= 256 ? 2 : (PANEL ? 6 : 8)) id_kernel_smem(
    int base, int kid, double p2, double tol, const double* __restrict__ Xf, const double* __restrict__ X, int64_t n,
    int d_unused, int r,
    const int* __restrict__ is_leaf, const int* __restrict__ nbegin, const int* __restrict__ first_child,
    const int* __restrict__ nchild, const int* __restrict__ ys_cnt, const int* __restrict__ ys,
    const int* __restrict__ xbar_n, const int64_t* __restrict__ uoff, double* U, int* kout, int* sk,
    unsigned long long* evals, int cls, int use_panel, const int* __restrict__ id_path,
    const int* __restrict__ list) {
  extern __shared__ double sh[];
  __shared__ PanelSmem<NT, PANEL ? kIdPanelNb : 1> psm;
  __shared__ CpqrSmem<NT> csm_cm;
  __shared__ CpqrRmSmem<NT> csm;
  constexpr bool kLean = NT >= kIdMidThreads;  // the lean layout (the lean and mid classes)
  const int tn = list[blockIdx.x];  // the launch's node list (id_sizes_kernel: this class and kind)
  const int i = base + tn;
  const int nx = xbar_n[i];
  const int ny = ys_cnt[i];
  const int tid = threadIdx.x;
  if (nx == 0 || id_path[i] == 11) return;  // (id_kernel_warp's nodes)
  {  // cls < 0: every node of the staged classes (merged launch)
    const int nc = id_smem_class(ny, nx, D);
    if (kLean ? nc != (NT == kIdLeanThreads ? kIdLean : kIdMid) : (nc < 0 || nc >= kIdMid || (cls >= 0 && nc != cls)))
      return;
  }
  // the panel-blocked CPQR (cpqr_panel.cuh) when the node's columns fit the thread groups, else
  // the warp-per-column one (cpqr.cuh); both on A^T column-major, leading dimension ld <= ny + 15
  constexpr int kRmax = NT >= 512 ? 4 : 2;
  static_assert(kRmax == (NT >= 512 ? 4 : 2), "id_panel_rmax");
  const int G = panel_group(nx, NT);
  const bool fits_panel = id_panel(ny, nx, NT);  // the block's layout (id_block_doubles)
  if (fits_panel != PANEL) return;  // the other instantiation's node
  const bool panel = PANEL && (use_panel & (kLean ? 2 : 1));
  const int ld = panel ? panel_ld(ny, G) : ny;
  double* M = sh;
  double* Fs = M + (int64_t)(fits_panel ? ny + id_pad_rows(nx, NT) : ny) * nx;
  double* nrm2 = Fs + (fits_panel ? kIdPanelNb * nx : 0);
  double* v = nrm2 + nx;
  double* tab = kLean ? v + ny : v + ny + D * (nx + ny);  // exp table
  int* piv = reinterpret_cast<int*>(tab + 64);
  int* xb = piv + nx;
  // staged coordinates: Xbar [c * nx + b], Y^* [c * ny + a]; before the table in the staged classes,
  // behind xb in the lean one, whose CTAs all get the level's largest request (id_lean_request): a
  // node whose block leaves room stages them too (its block generation then reads no global memory)
  double* cx = kLean ? reinterpret_cast<double*>(xb + nx) : v + ny;
  double* cy = cx + D * nx;
  const bool staged = !kLean || [&] {
    unsigned dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    return id_smem_bytes_lean(ny, nx, NT) + 8LL * D * (nx + ny) <= (int64_t)dyn;
  }();
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
  if (staged) {
    for (int a = tid; a < ny; a += NT)
#pragma unroll
      for (int c = 0; c < D; c++) cy[c * ny + a] = X[c * n + yv[a]];
    __syncthreads();
    for (int b = tid; b < nx; b += NT)
#pragma unroll
      for (int c = 0; c < D; c++) cx[c * nx + b] = Xf[c * n + xb[b]];
  }
  __syncthreads();
  // Xbar is kappa's first argument (coordinates from Xf), Y^* the second
  auto coord_x = [&](int c, int b) { return staged ? cx[c * nx + b] : Xf[c * n + xb[b]]; };
  auto coord_y = [&](int c, int a) { return staged ? cy[c * ny + a] : X[c * n + yv[a]]; };
  // unblocked fallback: wide blocks row-major with a thread per column (cta_cpqr_rm), tall ones
  // column-major with a warp per column (cta_cpqr); the panel CPQR is column-major (ld)
  const bool rm = !panel && !id_tall(ny, nx, NT);
  int k;
  if (rm) {
    // A^T row-major: M[a*nx + b] = K(Xbar[b], Y^*[a]); thread per column b, the column's point in
    // registers, rows' points broadcast from shared memory (or L1)
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
    // A^T column-major: M[a + ld*b] = K(Xbar[b], Y^*[a]), Y^* ascending; a warp per column b (its
    // point broadcast), lanes over the rows a
    for (int b = tid >> 5; b < nx; b += NT / 32) {
      double xb_[D];
#pragma unroll
      for (int c = 0; c < D; c++) xb_[c] = coord_x(c, b);
      for (int a = tid & 31; a < ny; a += 32) {
        double sq = 0.0, dt = 0.0;
#pragma unroll
        for (int c = 0; c < D; c++) {
          const double yc = coord_y(c, a), df = xb_[c] - yc;
          sq = fma(df, df, sq);
          dt = fma(xb_[c], yc, dt);
        }
        M[a + ld * b] = kid == H2_KERNEL_COSDOT ? kernel_cosdot(dt) : kernel_s(kid, p2, sq, tab);
      }
    }
    __syncthreads();
    if constexpr (PANEL) {
      k = panel ? cta_cpqr_panel<NT, kIdPanelNb, kRmax>(M, ld, ny, nx, tol, G, piv, Fs, psm)
                : cta_cpqr<NT>(M, ny, nx, tol, piv, nrm2, v, csm_cm);
    } else {
      k = cta_cpqr<NT>(M, ny, nx, tol, piv, nrm2, v, csm_cm);
    }
  }
  double* Ui = U + uoff[tn];
  for (int a = tid; a < k; a += NT) sk[(int64_t)i * r + a] = xb[piv[a]];
  // T of position c: in physical column piv[c] (panel: columns never move) or c (swapped columns)
  for (int e = tid; e < nx * k; e += NT) {
    const int c = e % nx, tt = e / nx;
    const double val = c < k ? (c == tt ? 1.0 : 0.0)
                             : rm ? M[tt * nx + c] : M[tt + (int64_t)ld * (panel ? piv[c] : c)];
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

// dynamic shared memory of the cluster kernel: v (ny <= r) + nrm2 (w) + exp table doubles; col_at,
// Xbar (nx) + pos (w) ints -- sized for the level's largest |Xbar|
static size_t id_cl_smem(int r, int nx_max) {
  return sizeof(double) * ((size_t)r + (size_t)nx_max + 64) + sizeof(int) * (3 * (size_t)nx_max) + 64;
}

// the largest cluster size the device schedules for the cluster kernel (16 needs the non-portable
// opt-in), queried once; H2_ID_CLUSTER=0 disables the path (diagnostics)
static int id_cluster_probe() {
  const char* env = getenv("H2_ID_CLUSTER");
  if (env && atoi(env) == 0) return 0;
  int best = 0;
  for (int c : {16, 8}) {
    if (c == 16 && cudaFuncSetAttribute(id_kernel_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                       cudaSuccess)
      continue;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(c);
    cfg.blockDim = dim3(kIdClThreads);
    cfg.dynamicSmemBytes = 96 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, id_kernel_cluster, &cfg) == cudaSuccess && nc > 0) {
      best = c;
      break;
    }
  }
  cudaGetLastError();
  return best;
}
static int id_cluster_max() {
  static const int cs = id_cluster_probe();  // thread-safe one-time initialisation
  return cs;
}

// One getBasis sweep (Algorithm 2 lines 10-12) into the handle's row-basis fields, kappa's first
// argument (Xbar) read from Xf.
static void id_sweep_pass(h2_handle* h, const double* Xf, int stat_kmax, int stat_evals) {
  cudaStream_t s = h->stream;
  H2_CUDA_TRY(cudaFuncSetAttribute(id_kernel_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  H2_CUDA_TRY(cudaFuncSetAttribute(id_kernel_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  const int cs = id_cluster_max();
  static const int use_panel = [] {  // H2_ID_PANEL (A/B knob): bit mask of the paths running the
    const char* e = getenv("H2_ID_PANEL");  // panel CPQR: 1 staged, 2 lean, 4 global memory
    return e ? atoi(e) : 3;
  }();
  static const int warp_min = [] {  // H2_ID_WARP_MIN (tuning knob): levels with at least this many
    const char* e = getenv("H2_ID_WARP_MIN");  // nodes use the warp-per-node path (0: never)
    return e ? atoi(e) : 0;
  }();
  static const int64_t cl_min = [] {  // H2_ID_CLMIN (tuning knob): cluster-path threshold, block entries
    const char* e = getenv("H2_ID_CLMIN");
    return e ? (int64_t)atoll(e) : (int64_t)256 * 1024;
  }();
  const int nn = h->nnodes;
  h->k = halloc<int>(h, nn);
  h->sk = halloc<int>(h, (size_t)nn * h->r);
  h->xbar_n = halloc<int>(h, nn);
  h->child_off = halloc<int>(h, nn);
  h->u_off = halloc<int64_t>(h, nn + 1);
  h->id_path = halloc<int>(h, nn);
  H2_CUDA_TRY(cudaMemsetAsync(h->id_path, 0xff, sizeof(int) * nn, s));
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
    constexpr int kSmaxN = 2 * kIdClasses + 3;
    Scratch sz(sizeof(int64_t) * 2 * (count + 1) + 4 * kSmaxN, s), off(sizeof(int64_t) * 2 * (count + 1), s);
    // one max per class (+ lean), the largest |Xbar| of the cluster-path nodes, then the kind
    // flags per class (+ lean)
    int* smax = reinterpret_cast<int*>(sz.as<int64_t>() + 2 * (count + 1));
    H2_CUDA_TRY(cudaMemsetAsync(smax, 0, kSmaxN * sizeof(int), s));
    int64_t *wsz = sz.as<int64_t>(), *usz = wsz + count + 1;
    int64_t *woff = off.as<int64_t>(), *uo = woff + count + 1;
    Scratch clw(sizeof(int) * (1 + (size_t)count), s);  // cluster-path node count + list
    int* cl_cnt = clw.as<int>();
    int* cl_list = cl_cnt + 1;
    H2_CUDA_TRY(cudaMemsetAsync(cl_cnt, 0, sizeof(int), s));
    constexpr int kNLists = 2 * (kIdClasses + 1) + 2;  // (class, kind) lists + merged staged lists
    Scratch lw(sizeof(int) * (kNLists + (size_t)kNLists * count), s);
    int* lcnt = lw.as<int>();
    int* lists = lcnt + kNLists;
    H2_CUDA_TRY(cudaMemsetAsync(lcnt, 0, sizeof(int) * kNLists, s));
    Scratch wpw(sizeof(int) * (2 + (size_t)count), s);  // warp-path node count, slot bytes, list
    int* wp_cnt = wpw.as<int>();
    int* wp_list = wp_cnt + 2;
    H2_CUDA_TRY(cudaMemsetAsync(wp_cnt, 0, 2 * sizeof(int), s));
    const int warp_level = warp_min > 0 && count >= warp_min;
    id_sizes_kernel<<<(count + 1 + 255) / 256, 256, 0, s>>>(base, count, h->d, h->is_leaf, h->nbegin, h->nend,
                                                            h->first_child, h->nchild, h->ys_cnt, h->k, h->xbar_n,
                                                            h->child_off, wsz, usz, smax, cs, cl_min, cl_cnt, cl_list,
                                                            h->id_path, warp_level, wp_cnt, wp_list, lcnt, lists);
    scan_excl_i64(wsz, woff, count + 1, s);
    scan_excl_i64(usz, uo, count + 1, s);
    H2_CHECK_LAUNCH();
    int64_t tot[2];
    int smem_bytes[kSmaxN] = {0};
    H2_CUDA_TRY(cudaMemcpyAsync(&tot[0], woff + count, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaMemcpyAsync(&tot[1], uo + count, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaMemcpyAsync(smem_bytes, smax, kSmaxN * sizeof(int), cudaMemcpyDeviceToHost, s));
    const int* kinds = smem_bytes + kIdClasses + 2;
    int ncl = 0, wph[2] = {0, 0}, lc[kNLists];
    H2_CUDA_TRY(cudaMemcpyAsync(lc, lcnt, sizeof(int) * kNLists, cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaMemcpyAsync(&ncl, cl_cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaMemcpyAsync(wph, wp_cnt, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
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
    cudaEvent_t cl_done = nullptr;
    if (ncl > 0) {  // the largest blocks: one thread-block cluster per node, on its own stream
      cudaStream_t cst = h->aux[2] ? h->aux[2] : s;
      cudaEvent_t fork = nullptr;
      if (cst != s) {
        H2_CUDA_TRY(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        H2_CUDA_TRY(cudaEventCreateWithFlags(&cl_done, cudaEventDisableTiming));
        H2_CUDA_TRY(cudaEventRecord(fork, s));
        H2_CUDA_TRY(cudaStreamWaitEvent(cst, fork, 0));
        cudaEventDestroy(fork);
      }
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3((unsigned)(ncl * cs));
      cfg.blockDim = dim3(kIdClThreads);
      cfg.dynamicSmemBytes = id_cl_smem(h->r, smem_bytes[kIdClasses + 1]);
      cfg.stream = cst;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      H2_CUDA_TRY(cudaLaunchKernelEx(&cfg, id_kernel_cluster, base, (const int*)cl_list, h->kid, p2, h->id_tol,
                                     Xf, (const double*)h->X, h->n, h->d, h->r, (const int*)h->is_leaf,
                                     (const int*)h->nbegin, (const int*)h->first_child, (const int*)h->nchild,
                                     (const int*)h->ys_cnt, (const int*)h->ys, (const int*)h->xbar_n,
                                     (const int64_t*)woff, work.as<double>(), (const int64_t*)(h->u_off + base), U,
                                     h->k, h->sk, ev.as<unsigned long long>()));
      if (cl_done) H2_CUDA_TRY(cudaEventRecord(cl_done, cst));
      h->gpu_launches += 1;
    }
    if (tot[0] > 0) {  // some node's block exceeds the shared-memory path: global-memory CPQR
      // the two thread-count variants run concurrently on auxiliary streams (disjoint nodes)
      cudaStream_t sa = h->aux[0] ? h->aux[0] : s, sb = h->aux[1] ? h->aux[1] : s;
      cudaEvent_t gev[3];
      for (auto& e : gev) H2_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      H2_CUDA_TRY(cudaEventRecord(gev[0], s));
      H2_CUDA_TRY(cudaStreamWaitEvent(sa, gev[0], 0));
      H2_CUDA_TRY(cudaStreamWaitEvent(sb, gev[0], 0));
      // (static + dynamic shared memory above 48 KB needs the opt-in)
      H2_CUDA_TRY(cudaFuncSetAttribute(id_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(double) * kIdGlobalFs));
      H2_CUDA_TRY(cudaFuncSetAttribute(id_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(double) * kIdGlobalFs));
      const size_t gfs = (use_panel & 4) ? sizeof(double) * kIdGlobalFs : 0;  // F only for the panel
      id_kernel<256><<<count, 256, gfs, sa>>>(base, h->kid, p2, h->id_tol, Xf, h->X, h->n, h->d, h->r, h->is_leaf,
                                           h->nbegin, h->first_child, h->nchild, h->ys_cnt, h->ys, h->xbar_n, woff,
                                           work.as<double>(), h->u_off + base, U, h->k, h->sk,
                                           ev.as<unsigned long long>(), 0, kIdBigBlock, cs, cl_min, use_panel, h->id_path);
      id_kernel<1024><<<count, 1024, gfs, sb>>>(base, h->kid, p2, h->id_tol, Xf, h->X, h->n, h->d, h->r, h->is_leaf,
                                             h->nbegin, h->first_child, h->nchild, h->ys_cnt, h->ys, h->xbar_n, woff,
                                             work.as<double>(), h->u_off + base, U, h->k, h->sk,
                                             ev.as<unsigned long long>(), kIdBigBlock, INT64_MAX, cs, cl_min,
                                             use_panel, h->id_path);
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
    for (int cls = 0; cls < kIdMid; cls++) {
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
      for (int cls = 0; cls < kIdMid; cls++)
        if (smem_bytes[cls] > 0) launches[nl++] = cls;
    if (smem_bytes[kIdMid] > 0) launches[nl++] = kIdMid;
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
      int kind = 0;  // instantiations this launch needs
      if (cls >= 0) kind = kinds[cls];
      else
        for (int c2 = 0; c2 < kIdMid; c2++) kind |= kinds[c2];
      for (int pv = 0; pv < 2; pv++) {
        if (!(kind & (1 << pv))) continue;
        const int lid = cls >= 0 ? cls * 2 + pv : 2 * (kIdClasses + 1) + pv;
        const int nlaunch = lc[lid];
        if (nlaunch == 0) continue;
        const int* llist = lists + (int64_t)lid * count;
        cudaStream_t cs = s;
        if (fan) {
          const int a = used % h2_handle::kAux;
          cs = h->aux[a];
          if (used < h2_handle::kAux) H2_CUDA_TRY(cudaStreamWaitEvent(cs, lev_ev[h2_handle::kAux], 0));
          used++;
        }
        const bool lean = cls == kIdLean, mid = cls == kIdMid;
        switch (h->d) {
#define H2_ID_LAUNCH(DD, NTT, PV, MAXS)                                                                          \
  do {                                                                                                          \
    H2_CUDA_TRY(cudaFuncSetAttribute(id_kernel_smem<DD, NTT, PV>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                     MAXS));                                                                    \
    id_kernel_smem<DD, NTT, PV><<<nlaunch, NTT, smem, cs>>>(                                                     \
        base, h->kid, p2, h->id_tol, Xf, h->X, h->n, h->d, h->r, h->is_leaf, h->nbegin, h->first_child,          \
        h->nchild,                                                                                              \
        h->ys_cnt, h->ys, h->xbar_n, h->u_off + base, U, h->k, h->sk, ev.as<unsigned long long>(), cls,         \
        use_panel, h->id_path, llist);                                                                          \
  } while (0)
#define H2_ID_CASE(DD)                                                                                          \
  case DD:                                                                                                      \
    if (lean) {                                                                                                 \
      if (pv) H2_ID_LAUNCH(DD, kIdLeanThreads, true, kIdLeanMax);                                               \
      else H2_ID_LAUNCH(DD, kIdLeanThreads, false, kIdLeanMax);                                                 \
    } else if (mid) {                                                                                           \
      if (pv) H2_ID_LAUNCH(DD, kIdMidThreads, true, kIdMidMax);                                                 \
      else H2_ID_LAUNCH(DD, kIdMidThreads, false, kIdMidMax);                                                   \
    } else {                                                                                                    \
      if (pv) H2_ID_LAUNCH(DD, kIdSmemThreads, true, kIdSmemMax);                                               \
      else H2_ID_LAUNCH(DD, kIdSmemThreads, false, kIdSmemMax);                                                 \
    }                                                                                                           \
    break;
          H2_ID_CASE(1) H2_ID_CASE(2) H2_ID_CASE(3) H2_ID_CASE(4)
          H2_ID_CASE(5) H2_ID_CASE(6) H2_ID_CASE(7) H2_ID_CASE(8)
#undef H2_ID_CASE
#undef H2_ID_LAUNCH
        }
        H2_CHECK_LAUNCH();
        h->gpu_launches += 1;
      }
    }
    if (wph[0] > 0) {  // the warp-per-node path, on the main stream concurrently with the class launches
      const int slot = (wph[1] + 7) / 8;
      const int smem = (int)(sizeof(double) * (size_t)slot * kIdWarpPerCta);
      const unsigned g = (unsigned)((wph[0] + kIdWarpPerCta - 1) / kIdWarpPerCta);
      switch (h->d) {
#define H2_IDW_CASE(DD)                                                                                         \
  case DD:                                                                                                      \
    H2_CUDA_TRY(cudaFuncSetAttribute(id_kernel_warp<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize,          \
                                     kIdWarpPerCta * kIdWarpMaxBytes + 64));                                    \
    id_kernel_warp<DD><<<g, 32 * kIdWarpPerCta, smem, s>>>(                                                    \
        base, wp_list, wph[0], slot, h->kid, p2, h->id_tol, Xf, h->X, h->n, h->r, h->is_leaf, h->nbegin,      \
        h->first_child, h->nchild, h->ys_cnt, h->ys, h->xbar_n, h->u_off + base, U, h->k, h->sk,              \
        ev.as<unsigned long long>());                                                                          \
    break;
        H2_IDW_CASE(1) H2_IDW_CASE(2) H2_IDW_CASE(3) H2_IDW_CASE(4)
        H2_IDW_CASE(5) H2_IDW_CASE(6) H2_IDW_CASE(7) H2_IDW_CASE(8)
#undef H2_IDW_CASE
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
    if (cl_done) {
      H2_CUDA_TRY(cudaStreamWaitEvent(s, cl_done, 0));
      cudaEventDestroy(cl_done);
    }
    h->gpu_launches += 2;
    srrqr_level(h, base, count, Xf, U);  // h2_options.srrqr_f > 0: SRRQR swaps (srrqr.cu)
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
  defer_stat(h, stat_kmax, km.p, sizeof(int));
  defer_stat(h, stat_evals, ev.p, sizeof(unsigned long long));
}

// a8: the row bases (getBasis(K_{Xbar Y*}), first argument X + a for the shifted multiquadric) and,
// on the non-symmetric path, the column bases: getBasis(K_{Y* Xbar}^T) = the same sweep for the
// transposed kernel kappa^T(x, y) = kappa(y, x) (Algorithm 2 line 11), whose first argument is
// X - a; its results move to the *_col fields.  For a symmetric kernel the second sweep repeats the
// first bit for bit (V = U).
void id_sweep(h2_handle* h) {
  id_sweep_pass(h, h->Xf, kStatKmax, kStatIdEvals);
  if (!h->nonsym) {
    h->k_col = h->k;
    h->sk_col = h->sk;
    h->xbar_col_n = h->xbar_n;
    h->child_off_col = h->child_off;
    h->u_off_col = h->u_off;
    h->V = h->U;
    h->v_total = h->u_total;
    h->kmax_col = h->kmax;
    return;
  }
  int *k = h->k, *sk = h->sk, *xb = h->xbar_n, *co = h->child_off, *path = h->id_path, kmax = h->kmax;
  int64_t* uo = h->u_off;
  double* U = h->U;
  const int64_t ut = h->u_total, ev = h->id_kernel_evals;
  id_sweep_pass(h, h->Xfn, kStatKmaxCol, kStatIdEvalsCol);
  h->k_col = h->k;
  h->sk_col = h->sk;
  h->xbar_col_n = h->xbar_n;
  h->child_off_col = h->child_off;
  h->u_off_col = h->u_off;
  h->V = h->U;
  h->v_total = h->u_total;
  h->kmax_col = h->kmax;
  h->id_kernel_evals += ev;
  h->k = k;
  h->sk = sk;
  h->xbar_n = xb;
  h->child_off = co;
  h->id_path = path;
  h->kmax = kmax;
  h->u_off = uo;
  h->U = U;
  h->u_total = ut;
}

}  // namespace h2
