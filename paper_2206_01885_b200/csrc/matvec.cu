// matvec.cu -- y = K~ x with the four-pass H^2 product:
//   upward    z^_i = U_i^T x_i at leaves, z^_p = sum_c R_c^T z^_c      (levels deepest -> 1)
//   coupling  y^_i += B_ij z^_j and y^_j += B_ij^T z^_i, i < j            (stored or on the fly)
//   downward  y^_c += R_c y^_p, then y_i += U_i y^_i at leaves          (levels 1 -> deepest)
//   nearfield y_i += D_ij x_j and y_j += D_ij^T x_i, i <= j              (stored or on the fly)
// Accumulation uses fp64 atomics (order-dependent rounding only).  Used for accuracy checks.
#include "h2_internal.cuh"

namespace h2 {

constexpr int kMvThreads = 128;

__global__ void permute_in_kernel(const double* __restrict__ x, const int* __restrict__ perm, int64_t n, double* xt) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    xt[t] = x[perm[t]];
}

__global__ void permute_out_kernel(const double* __restrict__ yt, const int* __restrict__ perm, int64_t n, double* y) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    y[perm[t]] = yt[t];
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
__device__ __forceinline__ double kval(int kid, double p2, const double* __restrict__ X, int64_t n, int a, int b) {
  return kernel_pts<D>(kid, p2, X, n, a, b);
}

template <int D>
__global__ void coupling_kernel(int64_t np, const int2* __restrict__ pairs, const int64_t* __restrict__ voff,
                                const double* __restrict__ B, int kid, double p2, const double* __restrict__ X,
                                int64_t n, const int* __restrict__ k, const int* __restrict__ sk, int r,
                                const double* __restrict__ zh, double* yh) {
  for (int64_t p = blockIdx.x; p < np; p += gridDim.x) {
    const int2 pr = pairs[p];
    const int i = pr.x, j = pr.y, ki = k[i], kj = k[j];
    const double* Bp = B ? B + voff[p] : nullptr;
    const int* si = sk + (int64_t)i * r;
    const int* sj = sk + (int64_t)j * r;
    const double* zi = zh + (int64_t)i * r;
    const double* zj = zh + (int64_t)j * r;
    for (int a = threadIdx.x; a < ki; a += blockDim.x) {  // y^_i += B z^_j
      double s = 0.0;
      for (int b = 0; b < kj; b++) s += (Bp ? Bp[(int64_t)a * kj + b] : kval<D>(kid, p2, X, n, si[a], sj[b])) * zj[b];
      atomicAdd(yh + (int64_t)i * r + a, s);
    }
    for (int b = threadIdx.x; b < kj; b += blockDim.x) {  // y^_j += B^T z^_i
      double s = 0.0;
      for (int a = 0; a < ki; a++) s += (Bp ? Bp[(int64_t)a * kj + b] : kval<D>(kid, p2, X, n, si[a], sj[b])) * zi[a];
      atomicAdd(yh + (int64_t)j * r + b, s);
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
                                 const double* __restrict__ Dv, int kid, double p2, const double* __restrict__ X,
                                 int64_t n, const int* __restrict__ nbegin, const int* __restrict__ nend,
                                 const double* __restrict__ xt, double* yt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t p = blockIdx.x; p < np; p += gridDim.x) {
    const int2 pr = pairs[p];
    const int i = pr.x, j = pr.y;
    const int bi = nbegin[i], bj = nbegin[j], ni = nend[i] - bi, nj = nend[j] - bj;
    const double* Dp = Dv ? Dv + voff[p] : nullptr;
    for (int a = warp; a < ni; a += nw) {  // y_i += D x_j (warp per row, coalesced)
      double s = 0.0;
      for (int b = lane; b < nj; b += 32)
        s += (Dp ? Dp[(int64_t)a * nj + b] : kval<D>(kid, p2, X, n, bi + a, bj + b)) * xt[bj + b];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) atomicAdd(yt + bi + a, s);
    }
    if (i != j)
      for (int b = threadIdx.x; b < nj; b += blockDim.x) {  // y_j += D^T x_i
        double s = 0.0;
        for (int a = 0; a < ni; a++)
          s += (Dp ? Dp[(int64_t)a * nj + b] : kval<D>(kid, p2, X, n, bi + a, bj + b)) * xt[bi + a];
        atomicAdd(yt + bj + b, s);
      }
  }
}

template <int D>
static void launch_far_near(const h2_handle* h, double p2, const double* zh, double* yh, const double* xt, double* yt,
                            int which) {
  cudaStream_t s = h->stream;
  if (which == 0 && h->n_cp > 0) {
    unsigned g = (unsigned)(h->n_cp < 148 * 64 ? h->n_cp : 148 * 64);
    coupling_kernel<D><<<g, kMvThreads, 0, s>>>(h->n_cp, h->cp_pairs, h->cp_off, h->cp_stored ? h->cp_val : nullptr,
                                                h->kid, p2, h->X, h->n, h->k, h->sk, h->r, zh, yh);
  }
  if (which == 1 && h->n_np > 0) {
    unsigned g = (unsigned)(h->n_np < 148 * 64 ? h->n_np : 148 * 64);
    nearfield_kernel<D><<<g, kMvThreads, 0, s>>>(h->n_np, h->np_pairs, h->np_off, h->np_stored ? h->np_val : nullptr,
                                                 h->kid, p2, h->X, h->n, h->nbegin, h->nend, xt, yt);
  }
}

static void far_near(const h2_handle* h, double p2, const double* zh, double* yh, const double* xt, double* yt,
                     int which) {
  switch (h->d) {
#define H2_MV_CASE(DD) \
  case DD:             \
    launch_far_near<DD>(h, p2, zh, yh, xt, yt, which); break;
    H2_MV_CASE(1) H2_MV_CASE(2) H2_MV_CASE(3) H2_MV_CASE(4)
    H2_MV_CASE(5) H2_MV_CASE(6) H2_MV_CASE(7) H2_MV_CASE(8)
#undef H2_MV_CASE
  }
}

// Sharded handles (shard.cu): the upward pass runs on the owned subtrees, the z^ of the levels
// >= cut are summed over the ranks (each node is non-zero on its owner only), and the levels
// above the cut are then computed by every rank; coupling and nearfield apply the rank's own
// (row-owned) blocks in both directions, so y^ and y are partial sums completed by allreduces.
void matvec(const h2_handle* h, const double* x, double* y) {
  cudaStream_t s = h->stream;
  const int64_t n = h->n;
  const int nn = h->nnodes, r = h->r;
  const bool sharded = h->nranks > 1;
  Scratch xt(sizeof(double) * n, s), yt(sizeof(double) * n, s), zh(sizeof(double) * (size_t)nn * r, s),
      yh(sizeof(double) * (size_t)nn * r, s);
  H2_CUDA_TRY(cudaMemsetAsync(yt.p, 0, sizeof(double) * n, s));
  H2_CUDA_TRY(cudaMemsetAsync(yh.p, 0, sizeof(double) * (size_t)nn * r, s));
  H2_CUDA_TRY(cudaMemsetAsync(zh.p, 0, sizeof(double) * (size_t)nn * r, s));
  permute_in_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, h->perm, n, xt.as<double>());
  auto up = [&](int l) {
    const LevelRange lr = level_range(h, l);
    if (lr.end > lr.begin)
      up_kernel<<<lr.end - lr.begin, kMvThreads, 0, s>>>(lr.begin, r, h->is_leaf, h->nbegin, h->first_child,
                                                         h->nchild, h->k, h->xbar_n, h->child_off, h->u_off, h->U,
                                                         xt.as<double>(), zh.as<double>());
  };
  const int cut = sharded ? (h->cut > 1 ? h->cut : 1) : 1;
  for (int l = h->depth; l >= cut; l--) up(l);
  if (sharded) comm_allreduce_sum(h->comm, zh.as<double>(), zh.as<double>(), (int64_t)nn * r, s);
  for (int l = cut - 1; l >= 1; l--) up(l);
  const double p2 = kernel_p2(h->kid, h->kp);
  far_near(h, p2, zh.as<double>(), yh.as<double>(), xt.as<double>(), yt.as<double>(), 0);
  if (sharded) comm_allreduce_sum(h->comm, yh.as<double>(), yh.as<double>(), (int64_t)nn * r, s);
  for (int l = 1; l <= h->depth; l++) {
    const LevelRange lr = level_range(h, l);
    if (lr.end > lr.begin)
      down_kernel<<<lr.end - lr.begin, kMvThreads, 0, s>>>(lr.begin, r, h->is_leaf, h->nbegin, h->parent, h->k,
                                                           h->xbar_n, h->child_off, h->u_off, h->U, h->p_lo, h->p_hi,
                                                           yh.as<double>(), yt.as<double>());
  }
  far_near(h, p2, zh.as<double>(), yh.as<double>(), xt.as<double>(), yt.as<double>(), 1);
  if (sharded) comm_allreduce_sum(h->comm, yt.as<double>(), yt.as<double>(), n, s);
  permute_out_kernel<<<grid_for(n, 256), 256, 0, s>>>(yt.as<double>(), h->perm, n, y);
  H2_CHECK_LAUNCH();
  H2_CUDA_TRY(cudaStreamSynchronize(s));
}

}  // namespace h2
