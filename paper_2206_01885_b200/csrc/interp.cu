// interp.cu -- the interpolation-based H^2 of the paper's memory comparison (section 6.3,
// P:1069-1098): bases from Eq. (2.2) instead of HiDR + ID.  Readings Q1-Q4
// (DESIGN.md section 3): p Chebyshev points of the first kind per dimension on every tree cell,
// r = p^d; U_leaf = [L_alpha(x)]_{x in X_i}; a non-leaf node's U stacks the transfers
// L^(i)_alpha(Q_c) of its children in the data-driven layout (Xbar_i = the children's nodes), so
// the coupling fill (fill.cu, on the node coordinates Xq) and the matvec (matvec.cu) are the
// data-driven ones; a node has a basis iff it or an ancestor has an admissible pair.
#include "h2_internal.cuh"

namespace h2 {

struct RloArr {
  double v[kMaxD];
};

// Q4, one level: k_i = r iff node i has an admissible pair or its parent has a basis
__global__ void interp_k_kernel(int base, int count, const int64_t* __restrict__ il_off,
                                const int* __restrict__ parent, int r, int* k) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const int i = base + t;
  const int p = parent[i];
  k[i] = (il_off[i + 1] > il_off[i] || (p >= 0 && k[p] > 0)) ? r : 0;
}

// |Xbar_i| (leaf: its points; else nchild r), the entries of U_i, the row offset of a node inside
// its parent's Xbar (child order)
__global__ void interp_sizes_kernel(int nn, int r, const int* __restrict__ k, const int* __restrict__ is_leaf,
                                    const int* __restrict__ nbegin, const int* __restrict__ nend,
                                    const int* __restrict__ nchild, const int* __restrict__ parent,
                                    const int* __restrict__ first_child, int* xbar_n, int* child_off, int64_t* usz) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > nn) return;
  if (i == nn) {
    usz[nn] = 0;
    return;
  }
  const int nx = k[i] > 0 ? (is_leaf[i] ? nend[i] - nbegin[i] : nchild[i] * r) : 0;
  xbar_n[i] = nx;
  usz[i] = (int64_t)nx * k[i];
  const int p = parent[i];
  child_off[i] = p >= 0 ? (i - first_child[p]) * r : 0;
}

// Q1: z_a = cos((2a + 1) pi / (2p))
__device__ __forceinline__ double cheb_z(int a, int p) {
  return cos(__ddiv_rn(__dmul_rn(__dadd_rn(__dmul_rn(2.0, (double)a), 1.0), 3.141592653589793), __dmul_rn(2.0, (double)p)));
}

// node i's box: width w = W 2^-level, centre (rlo + cell w) + w/2 (the oracle's operation order)
__device__ __forceinline__ void node_box(int i, int c, int nn, const int* __restrict__ level, const int* __restrict__ cell,
                                         double W, const RloArr& rlo, double& center, double& half) {
  const double w = ldexp(W, -level[i]);
  center = __dadd_rn(__dadd_rn(rlo.v[c], __dmul_rn((double)cell[(int64_t)c * nn + i], w)), __dmul_rn(0.5, w));
  half = __dmul_rn(0.5, w);
}

// Q_i: Xq[c nq + i r + alpha] = centre_c + half z_{a_c(alpha)} (alpha = sum_c a_c p^c); sk = its slot
__global__ void interp_nodes_kernel(int nn, int d, int p, int r, const int* __restrict__ level,
                                    const int* __restrict__ cell, double W, RloArr rlo, const int* __restrict__ k,
                                    double* Xq, int64_t nq, int* sk) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)nn * r;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / r), al = (int)(e - (int64_t)i * r);
    sk[e] = (int)e;
    if (k[i] == 0) continue;
    int rem = al;
    for (int c = 0; c < d; c++) {
      const int a = rem % p;
      rem /= p;
      double center, half;
      node_box(i, c, nn, level, cell, W, rlo, center, half);
      Xq[c * nq + e] = __dadd_rn(center, __dmul_rn(half, cheb_z(a, p)));
    }
  }
}

// U_i, one CTA per node with a basis: rows in chunks of kIpRows; per (row, dimension) the p 1-D
// Lagrange values l_a(u), u = (x - centre)/half (Q2, b ascending), into shared memory; then the
// entries L_alpha = prod_c l_{a_c} (c ascending), row index fastest (column-major U, coalesced).
constexpr int kIpRows = 32, kIpThreads = 256;
__global__ void __launch_bounds__(kIpThreads) interp_u_kernel(int nn, int d, int p, int r, const int* __restrict__ k,
                                                              const int* __restrict__ is_leaf,
                                                              const int* __restrict__ nbegin,
                                                              const int* __restrict__ first_child,
                                                              const int* __restrict__ xbar_n,
                                                              const int64_t* __restrict__ u_off,
                                                              const int* __restrict__ level, const int* __restrict__ cell,
                                                              double W, RloArr rlo, const double* __restrict__ X,
                                                              int64_t n, const double* __restrict__ Xq, int64_t nq,
                                                              double* U) {
  extern __shared__ double lsm[];  // [kIpRows][d][p]
  __shared__ double z[kInterpMaxP], cen[kMaxD], hal[kMaxD];
  const int i = blockIdx.x;
  if (k[i] == 0) return;
  if (threadIdx.x < p) z[threadIdx.x] = cheb_z(threadIdx.x, p);
  if (threadIdx.x < d) node_box(i, threadIdx.x, nn, level, cell, W, rlo, cen[threadIdx.x], hal[threadIdx.x]);
  __syncthreads();
  const int nx = xbar_n[i];
  const bool leaf = is_leaf[i];
  double* Ui = U + u_off[i];
  for (int r0 = 0; r0 < nx; r0 += kIpRows) {
    const int rows = nx - r0 < kIpRows ? nx - r0 : kIpRows;
    for (int e = threadIdx.x; e < rows * d * p; e += blockDim.x) {
      const int t = e / (d * p), c = (e / p) % d, a = e % p;
      const int row = r0 + t;
      // the row's coordinate: a point of the leaf, or a Chebyshev node of a child (child order)
      const double x = leaf ? X[c * n + nbegin[i] + row]
                            : Xq[c * nq + (int64_t)(first_child[i] + row / r) * r + row % r];
      const double u = __ddiv_rn(__dsub_rn(x, cen[c]), hal[c]);
      double l = 1.0;
      for (int b = 0; b < p; b++)
        if (b != a) l = __dmul_rn(l, __ddiv_rn(__dsub_rn(u, z[b]), __dsub_rn(z[a], z[b])));
      lsm[e] = l;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * r; e += blockDim.x) {
      const int t = e % rows, al = e / rows;
      double v = 1.0;
      int rem = al;
      for (int c = 0; c < d; c++) {
        v = __dmul_rn(v, lsm[(t * d + c) * p + rem % p]);
        rem /= p;
      }
      Ui[(int64_t)al * nx + r0 + t] = v;
    }
    __syncthreads();
  }
}

void interp_sweep(h2_handle* h, int p) {
  cudaStream_t s = h->stream;
  const int nn = h->nnodes, d = h->d, r = h->r;
  h->k = halloc<int>(h, nn);
  h->sk = halloc<int>(h, (size_t)nn * r);
  h->xbar_n = halloc<int>(h, nn);
  h->child_off = halloc<int>(h, nn);
  h->u_off = halloc<int64_t>(h, nn + 1);
  for (int l = 0; l <= h->depth; l++) {
    const LevelRange lr = level_range(h, l);
    const int cnt = lr.end - lr.begin;
    if (cnt > 0) interp_k_kernel<<<(cnt + 255) / 256, 256, 0, s>>>(lr.begin, cnt, h->il_off, h->parent, r, h->k);
  }
  Scratch usz(sizeof(int64_t) * (nn + 1), s);
  interp_sizes_kernel<<<(nn + 256) / 256, 256, 0, s>>>(nn, r, h->k, h->is_leaf, h->nbegin, h->nend, h->nchild,
                                                       h->parent, h->first_child, h->xbar_n, h->child_off,
                                                       usz.as<int64_t>());
  scan_excl_i64(usz.as<int64_t>(), h->u_off, nn + 1, s);
  H2_CHECK_LAUNCH();
  h->u_total = read1(h->u_off + nn, s);
  h->U = halloc<double>(h, h->u_total);
  h->nq = (int64_t)nn * r;
  h->Xq = halloc<double>(h, (size_t)h->nq * d);
  RloArr rlo{};
  for (int c = 0; c < d; c++) rlo.v[c] = h->rlo[c];
  interp_nodes_kernel<<<grid_for(h->nq, 256), 256, 0, s>>>(nn, d, p, r, h->level, h->cell, h->W, rlo, h->k, h->Xq,
                                                           h->nq, h->sk);
  const size_t smem = sizeof(double) * kIpRows * d * p;
  if (smem > 48 * 1024)
    H2_CUDA_TRY(cudaFuncSetAttribute(interp_u_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  interp_u_kernel<<<nn, kIpThreads, smem, s>>>(nn, d, p, r, h->k, h->is_leaf, h->nbegin, h->first_child, h->xbar_n,
                                               h->u_off, h->level, h->cell, h->W, rlo, h->X, h->n, h->Xq, h->nq, h->U);
  H2_CHECK_LAUNCH();
  h->gpu_launches += h->depth + 4;
  h->kmax = r;
  // symmetric kernels: the column bases are the row bases (the fill and the matvec read both)
  h->k_col = h->k;
  h->sk_col = h->sk;
  h->xbar_col_n = h->xbar_n;
  h->child_off_col = h->child_off;
  h->u_off_col = h->u_off;
  h->V = h->U;
  h->v_total = h->u_total;
  h->kmax_col = r;
}

}  // namespace h2
