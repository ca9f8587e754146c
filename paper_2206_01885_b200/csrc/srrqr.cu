// srrqr.cu -- strong rank-revealing refinement of getBasis (Eq.(4.1): "P [I; G]
// ... where ||G||_max is bounded by a prescribed constant"), h2_options.srrqr_f > 0.
//
// After the ID kernels of a level (cpqr.cuh / cpqr_panel.cuh: column-pivoted QR, rank k by the stop
// rule), a node whose U_i = P [I; G] has an entry |G| > f is refined by Gu & Eisenstat's swaps at
// fixed rank: swap the skeleton column t with the non-skeleton column c of the largest |T_tc| (T =
// R11^{-1} R12 = G^T; ties -> lowest Xbar index c, then lowest t), and refactor; every swap
// multiplies |det R11| by |T_tc| > f >= 1, so the loop ends.  The refactorisation is a Householder QR
// WITHOUT pivoting of the k skeleton columns (in skeleton order) of the regenerated block A^T =
// K(Xbar_i, Y_i^*)^T, the reflectors applied to the other columns, T by back substitution -- the
// arithmetic the oracle's orc_srrqr_swaps follows.  Most nodes pass the check (max |G| <= f) and
// cost one scan of U_i; the flagged ones run one CTA each on a global-memory workspace.
#include <climits>

#include "cpqr.cuh"

namespace h2 {

constexpr int kSrThreads = 256;

// flag[t] = node base + t needs swaps (some |U| > f; skeleton rows hold 0 / 1)
__global__ void srrqr_flag_kernel(int base, int count, const int* __restrict__ kout, const int* __restrict__ xbar_n,
                                  const int64_t* __restrict__ u_off, const double* __restrict__ U, double f,
                                  int* cnt, int* list, int* nxmax) {
  const int t = blockIdx.x;
  if (t >= count) return;
  const int i = base + t;
  const int k = kout[i], nx = xbar_n[i];
  if (k == 0 || k >= nx) return;
  const double* Ui = U + u_off[i];
  int bad = 0;
  for (int64_t e = threadIdx.x; e < (int64_t)nx * k; e += blockDim.x) bad |= fabs(Ui[e]) > f;
  bad = __syncthreads_or(bad);
  if (bad && threadIdx.x == 0) {
    list[atomicAdd(cnt, 1)] = t;
    atomicMax(nxmax, nx);
  }
}

// one CTA per flagged node; work: per CTA 2 ny nx doubles (the block, the working copy) + nx ints x 3
__global__ void __launch_bounds__(kSrThreads) srrqr_fix_kernel(
    int base, const int* __restrict__ list, int kid, double p2, const double* __restrict__ Xf,
    const double* __restrict__ X, int64_t n, int d, int r, const int* __restrict__ is_leaf,
    const int* __restrict__ nbegin, const int* __restrict__ first_child, const int* __restrict__ nchild,
    const int* __restrict__ ys_cnt, const int* __restrict__ ys, const int* __restrict__ kout,
    const int* __restrict__ xbar_n, const int64_t* __restrict__ u_off, double* U, int* sk, double f,
    int64_t wstride, double* work, unsigned long long* nswaps) {
  __shared__ CpqrSmem<kSrThreads> csm;
  __shared__ double s_wv[kSrThreads / 32];
  __shared__ int s_wc[kSrThreads / 32], s_wt[kSrThreads / 32];
  __shared__ int s_bc, s_bt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kSrThreads / 32;
  const int i = base + list[blockIdx.x];
  const int k = kout[i], nx = xbar_n[i], ny = ys_cnt[i];
  double* M0 = work + (int64_t)blockIdx.x * wstride;  // A^T, ny x nx column-major
  double* W = M0 + (int64_t)ny * nx;                   // the working factorisation, columns in order
  double* v = W + (int64_t)ny * nx;                    // ny
  int* xb = reinterpret_cast<int*>(v + ny);            // Xbar (nx)
  int* order = xb + nx;                                // working column -> Xbar column (nx)
  int* isk = order + nx;                               // Xbar column -> skeleton position or -1 (nx)
  double* Ui = U + u_off[i];
  // Xbar_i: the leaf's points or the children's skeletons in child order
  if (is_leaf[i]) {
    for (int b = tid; b < nx; b += kSrThreads) xb[b] = nbegin[i] + b;
  } else {
    int o = 0;
    for (int c = 0; c < nchild[i]; c++) {
      const int ch = first_child[i] + c;
      const int kc = kout[ch];
      for (int a = tid; a < kc; a += kSrThreads) xb[o + a] = sk[(int64_t)ch * r + a];
      o += kc;
    }
  }
  __syncthreads();
  const int* yv = ys + (int64_t)i * r;
  for (int64_t e = tid; e < (int64_t)ny * nx; e += kSrThreads) {
    const int a = (int)(e % ny), b = (int)(e / ny);
    M0[e] = kernel_pts_d(kid, p2, Xf, X, n, d, xb[b], yv[a]);
  }
  // skeleton positions of the Xbar columns: U_i restricted to the skeleton rows is the identity
  for (int b = tid; b < nx; b += kSrThreads) {
    int pos = -1;
    for (int t = 0; t < k && pos < 0; t++)
      if (sk[(int64_t)i * r + t] == xb[b]) pos = t;
    isk[b] = pos;
  }
  __syncthreads();
  int swaps = 0;
  for (;;) {
    // the largest |T_tc| > f over the non-skeleton columns c (ties -> lowest c, then lowest t)
    auto better = [](double v1, int c1, int t1, double v2, int c2, int t2) {
      return v1 > v2 || (v1 == v2 && (c1 < c2 || (c1 == c2 && t1 < t2)));
    };
    double best = -1.0;
    int bc = INT_MAX, bt = INT_MAX;
    for (int64_t e = tid; e < (int64_t)nx * k; e += kSrThreads) {
      const int c = (int)(e % nx), t = (int)(e / nx);
      if (isk[c] >= 0) continue;
      const double a = fabs(Ui[c + (int64_t)nx * t]);
      if (a > f && better(a, c, t, best, bc, bt)) {
        best = a;
        bc = c;
        bt = t;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double b2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int c2 = __shfl_xor_sync(0xffffffffu, bc, o), t2 = __shfl_xor_sync(0xffffffffu, bt, o);
      if (better(b2, c2, t2, best, bc, bt)) {
        best = b2;
        bc = c2;
        bt = t2;
      }
    }
    if (lane == 0) {
      s_wv[warp] = best;
      s_wc[warp] = bc;
      s_wt[warp] = bt;
    }
    __syncthreads();
    if (tid == 0) {
      double b = -1.0;
      int c0 = INT_MAX, t0 = INT_MAX;
      for (int w = 0; w < NW; w++)
        if (better(s_wv[w], s_wc[w], s_wt[w], b, c0, t0)) {
          b = s_wv[w];
          c0 = s_wc[w];
          t0 = s_wt[w];
        }
      s_bc = c0;
      s_bt = t0;
    }
    __syncthreads();
    const int c = s_bc, t = s_bt;
    if (c == INT_MAX || swaps >= 64 * k) break;
    swaps++;
    // swap: Xbar column c takes skeleton position t, the old skeleton column becomes a non-skeleton
    if (tid == 0) {
      for (int b = 0; b < nx; b++)
        if (isk[b] == t) isk[b] = -1;
      isk[c] = t;
    }
    __syncthreads();
    // working order: the skeleton columns in position order, then the others in Xbar order
    if (tid == 0) {
      for (int b = 0; b < nx; b++)
        if (isk[b] >= 0) order[isk[b]] = b;
      int o = k;
      for (int b = 0; b < nx; b++)
        if (isk[b] < 0) order[o++] = b;
    }
    __syncthreads();
    for (int64_t e = tid; e < (int64_t)ny * nx; e += kSrThreads) {
      const int a = (int)(e % ny), q = (int)(e / ny);
      W[e] = M0[a + (int64_t)ny * order[q]];
    }
    __syncthreads();
    // Householder QR without pivoting of the first k columns, applied to all columns
    for (int tt = 0; tt < k; tt++) {
      double* ct = W + (int64_t)ny * tt;
      double part = 0.0;
      for (int a = tt + tid; a < ny; a += kSrThreads) part += ct[a] * ct[a];
      const double n2 = cta_sum<kSrThreads>(part, csm);
      const double x0 = ct[tt];
      const double alpha = x0 >= 0.0 ? -sqrt(n2) : sqrt(n2);
      for (int a = tt + tid; a < ny; a += kSrThreads) v[a] = a == tt ? x0 - alpha : ct[a];
      __syncthreads();
      double pv = 0.0;
      for (int a = tt + tid; a < ny; a += kSrThreads) pv += v[a] * v[a];
      const double vtv = cta_sum<kSrThreads>(pv, csm);
      if (vtv > 0.0)
        for (int q = tt + 1 + warp; q < nx; q += NW) {
          double* col = W + (int64_t)ny * q;
          double s = 0.0;
          for (int a = tt + lane; a < ny; a += 32) s += v[a] * col[a];
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          const double fct = 2.0 * s / vtv;
          for (int a = tt + lane; a < ny; a += 32) col[a] -= fct * v[a];
        }
      __syncthreads();
      if (tid == 0) ct[tt] = alpha;
      __syncthreads();
    }
    // T = R11^{-1} R12 (thread per column), written into U_i's non-skeleton rows
    for (int q = k + tid; q < nx; q += kSrThreads) {
      double* col = W + (int64_t)ny * q;
      for (int a = k - 1; a >= 0; a--) {
        double s = col[a];
        for (int l = a + 1; l < k; l++) s -= W[a + (int64_t)ny * l] * col[l];
        col[a] = s / W[a + (int64_t)ny * a];
      }
      const int b = order[q];
      for (int tt = 0; tt < k; tt++) Ui[b + (int64_t)nx * tt] = col[tt];
    }
    for (int tt = tid; tt < k; tt += kSrThreads) {
      const int b = order[tt];
      for (int t2 = 0; t2 < k; t2++) Ui[b + (int64_t)nx * t2] = t2 == tt ? 1.0 : 0.0;
    }
    __syncthreads();
  }
  // the skeleton in position order
  for (int b = tid; b < nx; b += kSrThreads)
    if (isk[b] >= 0) sk[(int64_t)i * r + isk[b]] = xb[b];
  if (tid == 0 && swaps) atomicAdd(nswaps, (unsigned long long)swaps);
}

// one level's refinement (called by the ID sweep after the level's ID kernels, on h->stream)
void srrqr_level(h2_handle* h, int base, int count, const double* Xf, double* U) {
  if (!(h->srrqr_f > 0.0) || count == 0) return;
  cudaStream_t s = h->stream;
  Scratch meta(sizeof(int) * (2 + (size_t)count), s);
  int* cnt = meta.as<int>();
  int* nxmax = cnt + 1;
  int* list = cnt + 2;
  H2_CUDA_TRY(cudaMemsetAsync(cnt, 0, 2 * sizeof(int), s));
  srrqr_flag_kernel<<<count, 128, 0, s>>>(base, count, h->k, h->xbar_n, h->u_off, U, h->srrqr_f, cnt, list, nxmax);
  H2_CHECK_LAUNCH();
  int hv[2];
  H2_CUDA_TRY(cudaMemcpyAsync(hv, cnt, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  H2_CUDA_TRY(cudaStreamSynchronize(s));
  h->gpu_launches += 1;
  const int nflag = hv[0], nxm = hv[1];
  if (nflag == 0) return;
  // per CTA: M0, W (ny nx each, ny <= r), v (r), 3 nx ints
  const int64_t wstride = 2LL * h->r * nxm + h->r + (3LL * nxm + 1) / 2 + 2;
  const int batch = 256;
  for (int b0 = 0; b0 < nflag; b0 += batch) {
    const int nb = nflag - b0 < batch ? nflag - b0 : batch;
    Scratch work(sizeof(double) * (size_t)wstride * nb, s);
    Scratch sw(sizeof(unsigned long long), s);
    H2_CUDA_TRY(cudaMemsetAsync(sw.p, 0, sizeof(unsigned long long), s));
    srrqr_fix_kernel<<<nb, kSrThreads, 0, s>>>(base, list + b0, h->kid, kernel_p2(h->kid, h->kp), Xf, h->X, h->n,
                                               h->d, h->r, h->is_leaf, h->nbegin, h->first_child, h->nchild,
                                               h->ys_cnt, h->ys, h->k, h->xbar_n, h->u_off, U, h->sk, h->srrqr_f,
                                               wstride, work.as<double>(), sw.as<unsigned long long>());
    H2_CHECK_LAUNCH();
    h->srrqr_swaps += (int64_t)read1(sw.as<unsigned long long>(), s);
    h->gpu_launches += 1;
  }
}

}  // namespace h2
