// fill.cu -- a9/a10: coupling blocks B_ij = K(X^_i, X^_j) over the admissible pairs and dense
// nearfield blocks K(X_i, X_j) over the leaf nearfield pairs (Algorithm 2, PAPER.md P:496-503;
// reading G1).  Symmetric kernels: only i < j (coupling) and i <= j (nearfield) are stored, each
// block row-major.
//
// The fill is HBM-write / FP64 bound.  Work is partitioned by a flat ENTRY index space cut into
// tiles of kFillTile entries (a pair owns ceil(size/kFillTile) tiles), so a 60M-entry block and a
// 16-entry block are balanced alike.  A persistent grid (blocks_per_SM x 148) walks the tiles;
// one binary search per tile maps it to its pair; each thread then writes entries e, e+256, ...
// (consecutive threads -> consecutive addresses, streaming stores).
#include "h2_internal.cuh"

namespace h2 {

constexpr int kFillThreads = 256;
constexpr int kFillTile = 4096;

// number of symmetric-once pairs of each row (mode 0 coupling: j > i, both ranks > 0;
// mode 1 nearfield: j >= i)
__global__ void pair_count_kernel(int mode, int nnodes, const int64_t* __restrict__ off, const int* __restrict__ idx,
                                  const int* __restrict__ k, int64_t* cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > nnodes) return;
  if (i == nnodes) {
    cnt[i] = 0;
    return;
  }
  int64_t c = 0;
  if (mode == 1 || k[i] > 0)
    for (int64_t e = off[i]; e < off[i + 1]; e++) {
      int j = idx[e];
      if (mode == 0 ? (j > i && k[j] > 0) : (j >= i)) c++;
    }
  cnt[i] = c;
}

__global__ void pair_emit_kernel(int mode, int nnodes, const int64_t* __restrict__ off, const int* __restrict__ idx,
                                 const int* __restrict__ k, const int* __restrict__ nbegin,
                                 const int* __restrict__ nend, const int64_t* __restrict__ pos, int2* pairs,
                                 int64_t* size) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnodes) return;
  if (mode == 0 && k[i] == 0) return;
  int64_t o = pos[i];
  for (int64_t e = off[i]; e < off[i + 1]; e++) {
    int j = idx[e];
    if (mode == 0 ? (j > i && k[j] > 0) : (j >= i)) {
      pairs[o] = make_int2(i, j);
      size[o] = mode == 0 ? (int64_t)k[i] * k[j] : (int64_t)(nend[i] - nbegin[i]) * (nend[j] - nbegin[j]);
      o++;
    }
  }
}

__global__ void tiles_kernel(int64_t np, const int64_t* __restrict__ size, int64_t* ntiles) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= np; p += (int64_t)gridDim.x * blockDim.x)
    ntiles[p] = p < np ? (size[p] + kFillTile - 1) / kFillTile : 0;
}

template <int D, int KID, int MODE>
__global__ void __launch_bounds__(kFillThreads) fill_kernel(int64_t ntiles, int64_t np, const int64_t* __restrict__ toff,
                                                            const int2* __restrict__ pairs,
                                                            const int64_t* __restrict__ voff,
                                                            const int* __restrict__ nbegin,
                                                            const int* __restrict__ nend, const int* __restrict__ k,
                                                            const int* __restrict__ sk, int r,
                                                            const double* __restrict__ X, int64_t n, double p2,
                                                            double* __restrict__ out) {
  __shared__ int64_t s_pair;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    if (threadIdx.x == 0) {
      int64_t lo = 0, hi = np - 1;  // last p with toff[p] <= tile
      while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (toff[mid] <= tile) lo = mid;
        else hi = mid - 1;
      }
      s_pair = lo;
    }
    __syncthreads();
    const int64_t p = s_pair;
    __syncthreads();
    const int2 pr = pairs[p];
    const int i = pr.x, j = pr.y;
    const int ni = MODE == 0 ? k[i] : nend[i] - nbegin[i];
    const int nj = MODE == 0 ? k[j] : nend[j] - nbegin[j];
    const int64_t size = (int64_t)ni * nj;
    const int64_t e0 = (tile - toff[p]) * kFillTile;
    const int64_t e1 = e0 + kFillTile < size ? e0 + kFillTile : size;
    double* o = out + voff[p];
    const int bi = nbegin[i], bj = nbegin[j];
    const int* si = sk + (int64_t)i * r;
    const int* sj = sk + (int64_t)j * r;
    int64_t e = e0 + threadIdx.x;
    if (e >= e1) continue;
    int row = (int)(e / nj), col = (int)(e - (int64_t)row * nj);
    const int dq = kFillThreads / nj, dr = kFillThreads - dq * nj;
    for (; e < e1; e += kFillThreads) {
      const int a = MODE == 0 ? si[row] : bi + row;
      const int b = MODE == 0 ? sj[col] : bj + col;
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < D; c++) {
        double df = X[c * n + a] - X[c * n + b];
        s = fma(df, df, s);
      }
      __stcs(o + e, kernel_s(KID, p2, s));
      col += dr;
      row += dq;
      if (col >= nj) {
        col -= nj;
        row++;
      }
    }
  }
}

template <int KID, int MODE>
static void launch_fill_k(int d, unsigned grid, cudaStream_t s, int64_t ntiles, int64_t np, const int64_t* toff,
                          const int2* pairs, const int64_t* voff, const h2_handle* h, double p2, double* out) {
  switch (d) {
#define H2_FILL_CASE(DD)                                                                                     \
  case DD:                                                                                                   \
    fill_kernel<DD, KID, MODE><<<grid, kFillThreads, 0, s>>>(ntiles, np, toff, pairs, voff, h->nbegin,       \
                                                             h->nend, h->k, h->sk, h->r, h->X, h->n, p2, out); \
    break;
    H2_FILL_CASE(1) H2_FILL_CASE(2) H2_FILL_CASE(3) H2_FILL_CASE(4)
    H2_FILL_CASE(5) H2_FILL_CASE(6) H2_FILL_CASE(7) H2_FILL_CASE(8)
#undef H2_FILL_CASE
  }
}

template <int MODE>
static void launch_fill(const h2_handle* h, int64_t ntiles, int64_t np, const int64_t* toff, const int2* pairs,
                        const int64_t* voff, double* out) {
  const double p2 = kernel_p2(h->kid, h->kp);
  int64_t g = ntiles < 148 * 8 ? ntiles : 148 * 8;
  if (g < 1) return;
  if (h->kid == H2_KERNEL_COULOMB)
    launch_fill_k<H2_KERNEL_COULOMB, MODE>(h->d, (unsigned)g, h->stream, ntiles, np, toff, pairs, voff, h, p2, out);
  else if (h->kid == H2_KERNEL_GAUSSIAN)
    launch_fill_k<H2_KERNEL_GAUSSIAN, MODE>(h->d, (unsigned)g, h->stream, ntiles, np, toff, pairs, voff, h, p2, out);
  else
    launch_fill_k<H2_KERNEL_MATERN32, MODE>(h->d, (unsigned)g, h->stream, ntiles, np, toff, pairs, voff, h, p2, out);
}

// builds the symmetric-once pair list of one class with entry offsets; returns (pairs, entries)
static void make_pairs(h2_handle* h, int mode, int64_t& np, int2*& pairs, int64_t*& voff, int64_t& entries) {
  cudaStream_t s = h->stream;
  const int nn = h->nnodes;
  const int64_t* off = mode == 0 ? h->il_off : h->nf_off;
  const int* idx = mode == 0 ? h->il_idx : h->nf_idx;
  Scratch cnt(sizeof(int64_t) * (nn + 1), s), pos(sizeof(int64_t) * (nn + 1), s);
  pair_count_kernel<<<(nn + 1 + 255) / 256, 256, 0, s>>>(mode, nn, off, idx, h->k, cnt.as<int64_t>());
  scan_excl_i64(cnt.as<int64_t>(), pos.as<int64_t>(), nn + 1, s);
  H2_CHECK_LAUNCH();
  np = read1(pos.as<int64_t>() + nn, s);
  pairs = halloc<int2>(h, np);
  voff = halloc<int64_t>(h, np + 1);
  Scratch size(sizeof(int64_t) * (np + 1), s);
  H2_CUDA_TRY(cudaMemsetAsync(size.as<int64_t>() + np, 0, sizeof(int64_t), s));
  pair_emit_kernel<<<(nn + 255) / 256, 256, 0, s>>>(mode, nn, off, idx, h->k, h->nbegin, h->nend,
                                                    pos.as<int64_t>(), pairs, size.as<int64_t>());
  scan_excl_i64(size.as<int64_t>(), voff, np + 1, s);
  H2_CHECK_LAUNCH();
  h->gpu_launches += 5;
  entries = read1(voff + np, s);
}

__global__ void adjdiff_kernel(int64_t np, const int64_t* __restrict__ voff, int64_t* size) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np; p += (int64_t)gridDim.x * blockDim.x)
    size[p] = voff[p + 1] - voff[p];
}

static int64_t pool_available(cudaStream_t s) {
  size_t fr = 0, tot = 0;
  H2_CUDA_TRY(cudaMemGetInfo(&fr, &tot));
  int dev = 0;
  H2_CUDA_TRY(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  H2_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t reserved = 0, used = 0;
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
  (void)s;
  return (int64_t)fr + (int64_t)(reserved > used ? reserved - used : 0);
}

void fill_blocks(h2_handle* h, int storage, int64_t budget) {
  cudaStream_t s = h->stream;
  make_pairs(h, 0, h->n_cp, h->cp_pairs, h->cp_off, h->cp_entries);
  make_pairs(h, 1, h->n_np, h->np_pairs, h->np_off, h->np_entries);
  const int64_t cb = h->cp_entries * 8, nb = h->np_entries * 8;
  bool store_cp = false, store_np = false;
  if (storage == H2_STORE_ALL) {
    store_cp = store_np = true;
  } else if (storage == H2_STORE_AUTO) {
    int64_t avail = budget > 0 ? budget : pool_available(s) - ((int64_t)4 << 30);
    // greedy: the smaller class first
    if (cb <= nb) {
      if (cb <= avail) store_cp = true, avail -= cb;
      if (nb <= avail) store_np = true;
    } else {
      if (nb <= avail) store_np = true, avail -= nb;
      if (cb <= avail) store_cp = true;
    }
  }
  cudaEvent_t ev[4];
  if (h->timing)
    for (auto& e : ev) H2_CUDA_TRY(cudaEventCreate(&e));
  if (store_cp) {
    h->cp_val = halloc<double>(h, h->cp_entries);
    h->cp_stored = 1;
  }
  if (store_np) {
    h->np_val = halloc<double>(h, h->np_entries);
    h->np_stored = 1;
  }
  for (int mode = 0; mode < 2; mode++) {
    int64_t np = mode == 0 ? h->n_cp : h->n_np;
    if (h->timing) H2_CUDA_TRY(cudaEventRecord(ev[2 * mode], s));
    if ((mode == 0 ? store_cp : store_np) && np > 0) {
      const int64_t* voff = mode == 0 ? h->cp_off : h->np_off;
      Scratch sizes(sizeof(int64_t) * (np + 1), s), nt(sizeof(int64_t) * (np + 1), s),
          toff(sizeof(int64_t) * (np + 1), s);
      adjdiff_kernel<<<grid_for(np, 256), 256, 0, s>>>(np, voff, sizes.as<int64_t>());
      tiles_kernel<<<grid_for(np + 1, 256), 256, 0, s>>>(np, sizes.as<int64_t>(), nt.as<int64_t>());
      scan_excl_i64(nt.as<int64_t>(), toff.as<int64_t>(), np + 1, s);
      H2_CHECK_LAUNCH();
      int64_t ntiles = read1(toff.as<int64_t>() + np, s);
      if (h->timing) H2_CUDA_TRY(cudaEventRecord(ev[2 * mode], s));
      if (mode == 0) launch_fill<0>(h, ntiles, np, toff.as<int64_t>(), h->cp_pairs, voff, h->cp_val);
      else launch_fill<1>(h, ntiles, np, toff.as<int64_t>(), h->np_pairs, voff, h->np_val);
      H2_CHECK_LAUNCH();
      h->gpu_launches += 4;
    }
    if (h->timing) H2_CUDA_TRY(cudaEventRecord(ev[2 * mode + 1], s));
  }
  if (h->timing) {
    H2_CUDA_TRY(cudaEventSynchronize(ev[3]));
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[2], ev[3]);
    h->stage_ms[6] = a;
    h->stage_ms[7] = b;
    for (auto& e : ev) cudaEventDestroy(e);
  }
}

// ---- sampled reads of stored entries for the parity tests ----------------------------------
__global__ void sample_kernel(int64_t count, const int32_t* kind, const int64_t* pair, const int64_t* entry,
                              const int2* cpp, const int64_t* cpo, const double* cpv, const int2* npp,
                              const int64_t* npo, const double* npv, const int* nbegin, const int* nend,
                              const int* k, const int* sk, int r, double* val, int32_t* rp, int32_t* cp) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < count; s += (int64_t)gridDim.x * blockDim.x) {
    int md = kind[s];
    int64_t p = pair[s], e = entry[s];
    int2 pr = md == 0 ? cpp[p] : npp[p];
    int nj = md == 0 ? k[pr.y] : nend[pr.y] - nbegin[pr.y];
    int row = (int)(e / nj), col = (int)(e % nj);
    val[s] = md == 0 ? cpv[cpo[p] + e] : npv[npo[p] + e];
    rp[s] = md == 0 ? sk[(int64_t)pr.x * r + row] : nbegin[pr.x] + row;
    cp[s] = md == 0 ? sk[(int64_t)pr.y * r + col] : nbegin[pr.y] + col;
  }
}

void sample_blocks(const h2_handle* h, int64_t count, const int32_t* kind, const int64_t* pair, const int64_t* entry,
                   double* value, int32_t* row_pt, int32_t* col_pt) {
  cudaStream_t s = h->stream;
  for (int64_t q = 0; q < count; q++) {
    if (kind[q] == 0 && (!h->cp_stored || pair[q] < 0 || pair[q] >= h->n_cp))
      throw Error{H2_ERR_INVALID_ARG, "coupling sample out of range or not stored"};
    if (kind[q] == 1 && (!h->np_stored || pair[q] < 0 || pair[q] >= h->n_np))
      throw Error{H2_ERR_INVALID_ARG, "nearfield sample out of range or not stored"};
    if (kind[q] != 0 && kind[q] != 1) throw Error{H2_ERR_INVALID_ARG, "sample kind must be 0 or 1"};
  }
  Scratch in(count * (4 + 8 + 8) + 64, s), out(count * (8 + 4 + 4) + 64, s);
  int32_t* dk = in.as<int32_t>();
  int64_t* dp = reinterpret_cast<int64_t*>(in.as<char>() + ((count * 4 + 15) / 16) * 16);
  int64_t* de = dp + count;
  double* dv = out.as<double>();
  int32_t* dr = reinterpret_cast<int32_t*>(dv + count);
  int32_t* dc = dr + count;
  H2_CUDA_TRY(cudaMemcpyAsync(dk, kind, 4 * count, cudaMemcpyHostToDevice, s));
  H2_CUDA_TRY(cudaMemcpyAsync(dp, pair, 8 * count, cudaMemcpyHostToDevice, s));
  H2_CUDA_TRY(cudaMemcpyAsync(de, entry, 8 * count, cudaMemcpyHostToDevice, s));
  sample_kernel<<<grid_for(count, 256), 256, 0, s>>>(count, dk, dp, de, h->cp_pairs, h->cp_off, h->cp_val,
                                                     h->np_pairs, h->np_off, h->np_val, h->nbegin, h->nend, h->k,
                                                     h->sk, h->r, dv, dr, dc);
  H2_CHECK_LAUNCH();
  H2_CUDA_TRY(cudaMemcpyAsync(value, dv, 8 * count, cudaMemcpyDeviceToHost, s));
  H2_CUDA_TRY(cudaMemcpyAsync(row_pt, dr, 4 * count, cudaMemcpyDeviceToHost, s));
  H2_CUDA_TRY(cudaMemcpyAsync(col_pt, dc, 4 * count, cudaMemcpyDeviceToHost, s));
  H2_CUDA_TRY(cudaStreamSynchronize(s));
}

}  // namespace h2
