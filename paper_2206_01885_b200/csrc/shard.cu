// shard.cu -- subtree sharding of the build over ranks (BASELINE north_star: "the
// tree is sharded across the GPUs of one box by subtrees below a cut level; points are
// replicated; each level's skeleton indices and representors are exchanged with NCCL allgather;
// top levels above the cut are computed redundantly").
//
// Plan (identical on every rank: the tree is built redundantly and deterministically; the plan is
// made before the lists, which each rank then builds for its own rows only, lists.cu):
//   * cut level c = the shallowest level with >= 64 nodes per rank (else the most populous level);
//   * the cut-level nodes (Morton order) are split into nranks contiguous runs balanced by an
//     integer work estimate of their subtrees (3^d n_leaf^2 + 64 n_leaf per leaf, 65536 per node);
//     node ids of one level are in Morton order, so the nodes a rank owns at every level >= c form
//     ONE contiguous id range;
//   * HiDR and the ID sweep run, at levels >= c, on the owned range only; levels < c are computed
//     by every rank;
//   * block rows (a9, a10, the matvec's leaf outputs) belong to the rank whose point range
//     [p_lo, p_hi) holds the row node's first point; the ranges tile [0, n) and split it at the
//     cut-level boundaries, so a node at level >= c belongs to its subtree's owner.
// Exchanges (comm.cu): after HiDR up below the cut, the X_i^* slots of every level >= c; after the
// ID sweep below the cut, the skeleton slots X^_i (+ k_i).  One allgather each: a rank's owned
// (count, slots) ranges of all levels >= c are packed into one fixed-size slot.
#include <algorithm>

#include "h2_internal.cuh"

namespace h2 {

// integer work estimate of one node, from the tree alone (the plan precedes the lists, which are
// then built for the rank's own rows only): a leaf's nearfield entries ~ 3^d n_leaf^2 (its
// neighbours hold about as many points as it does) plus 64 per point, and 65536 per node (its
// HiDR search and ID).  int64, so sums are exact and the plan is bit-identical on every rank.
__global__ void shard_weight_kernel(int nnodes, int cut, int d, const int* __restrict__ level,
                                    const int* __restrict__ parent, const int* __restrict__ is_leaf,
                                    const int* __restrict__ nbegin, const int* __restrict__ nend, int cut_base,
                                    int* anc, unsigned long long* wcut) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnodes) return;
  if (level[i] < cut) {
    anc[i] = -1;
    return;
  }
  int a = i;
  while (level[a] > cut) a = parent[a];
  anc[i] = a;
  int64_t w3 = 1;
  for (int c = 0; c < d; c++) w3 *= 3;
  const int64_t ni = nend[i] - nbegin[i];
  int64_t w = 65536;
  if (is_leaf[i]) w += w3 * ni * ni + 64 * ni;
  atomicAdd(wcut + (a - cut_base), (unsigned long long)w);
}

// one CTA per segment: dst[0, words) = src[0, words) (32-bit words)
struct Seg {
  const int* src;
  int* dst;
  int64_t words;
};
__global__ void seg_copy_kernel(const Seg* __restrict__ segs) {
  const Seg sg = segs[blockIdx.x];
  for (int64_t t = threadIdx.x; t < sg.words; t += blockDim.x) sg.dst[t] = sg.src[t];
}

static int64_t slot_words(const h2_handle* h, int q) {  // packed size of rank q's (cnt, slots) ranges
  int64_t w = 0;
  for (int l = h->cut; l <= h->depth; l++) w += (int64_t)(h->rng_hi[q][l] - h->rng_lo[q][l]) * (1 + h->r);
  return w;
}

void shard_plan(h2_handle* h) {
  const int R = h->nranks, nn = h->nnodes;
  cudaStream_t s = h->stream;
  std::vector<int64_t> counts(h->depth + 1);
  for (int l = 0; l <= h->depth; l++) counts[l] = h->lvl_start[l + 1] - h->lvl_start[l];
  h->cut = h2_shard_cut_level(counts.data(), h->depth + 1, R);
  const int c = h->cut, base = h->lvl_start[c], ncut = (int)counts[c];
  Scratch anc(sizeof(int) * nn, s), wc(sizeof(unsigned long long) * ncut, s);
  H2_CUDA_TRY(cudaMemsetAsync(wc.p, 0, sizeof(unsigned long long) * ncut, s));
  shard_weight_kernel<<<(nn + 255) / 256, 256, 0, s>>>(nn, c, h->d, h->level, h->parent, h->is_leaf, h->nbegin,
                                                       h->nend, base, anc.as<int>(), wc.as<unsigned long long>());
  H2_CHECK_LAUNCH();
  std::vector<int64_t> w(ncut);
  std::vector<int> a(nn), nb(ncut);
  H2_CUDA_TRY(cudaMemcpyAsync(w.data(), wc.p, sizeof(int64_t) * ncut, cudaMemcpyDeviceToHost, s));
  H2_CUDA_TRY(cudaMemcpyAsync(a.data(), anc.p, sizeof(int) * nn, cudaMemcpyDeviceToHost, s));
  H2_CUDA_TRY(cudaMemcpyAsync(nb.data(), h->nbegin + base, sizeof(int) * ncut, cudaMemcpyDeviceToHost, s));
  H2_CUDA_TRY(cudaStreamSynchronize(s));
  std::vector<int64_t> first(R + 1);
  if (h2_shard_split(w.data(), ncut, R, first.data()) != H2_OK) throw Error{H2_ERR_INTERNAL, "shard split failed"};
  h->rng_lo.assign(R, std::vector<int>(h->depth + 1));
  h->rng_hi.assign(R, std::vector<int>(h->depth + 1));
  for (int q = 0; q < R; q++)
    for (int l = 0; l <= h->depth; l++) {
      const int b = h->lvl_start[l], e = h->lvl_start[l + 1];
      if (l < c) {  // redundant levels: every rank computes the whole level
        h->rng_lo[q][l] = b;
        h->rng_hi[q][l] = e;
        continue;
      }
      // ancestors are non-decreasing along a level (Morton order): owned nodes are contiguous
      auto lo = std::lower_bound(a.begin() + b, a.begin() + e, base + (int)first[q]);
      auto hi = std::lower_bound(a.begin() + b, a.begin() + e, base + (int)first[q + 1]);
      h->rng_lo[q][l] = (int)(lo - a.begin());
      h->rng_hi[q][l] = (int)(hi - a.begin());
    }
  const int q = h->rank;
  h->p_lo = q == 0 ? 0 : (first[q] < ncut ? nb[first[q]] : h->n);
  h->p_hi = q == R - 1 ? h->n : (first[q + 1] < ncut ? nb[first[q + 1]] : h->n);
  h->gpu_launches += 1;
}

// every rank's (cnt[i], slots[i*r ...]) for its owned nodes of the levels >= cut, made global
void exchange_slots(h2_handle* h, int* cnt, int* slots) {
  if (h->nranks == 1) return;
  cudaStream_t s = h->stream;
  const int R = h->nranks, r = h->r, me = h->rank;
  int64_t sw = 1;  // fixed per-rank slot: the largest packed size over the ranks
  for (int q = 0; q < R; q++) sw = std::max(sw, slot_words(h, q));
  Scratch send(sizeof(int) * sw, s), recv(sizeof(int) * sw * R, s);
  std::vector<Seg> segs;
  // pack: my ranges into the send slot
  int64_t o = 0;
  for (int l = h->cut; l <= h->depth; l++) {
    const int lo = h->rng_lo[me][l], m = h->rng_hi[me][l] - lo;
    if (m == 0) continue;
    segs.push_back({cnt + lo, send.as<int>() + o, m});
    segs.push_back({slots + (int64_t)lo * r, send.as<int>() + o + m, (int64_t)m * r});
    o += (int64_t)m * (1 + r);
  }
  const size_t npack = segs.size();
  // unpack: every other rank's slot into place
  for (int q = 0; q < R; q++) {
    if (q == me) continue;
    const int* src = recv.as<int>() + (int64_t)q * sw;
    int64_t oq = 0;
    for (int l = h->cut; l <= h->depth; l++) {
      const int lo = h->rng_lo[q][l], m = h->rng_hi[q][l] - lo;
      if (m == 0) continue;
      segs.push_back({src + oq, cnt + lo, m});
      segs.push_back({src + oq + m, slots + (int64_t)lo * r, (int64_t)m * r});
      oq += (int64_t)m * (1 + r);
    }
  }
  Scratch table(sizeof(Seg) * std::max<size_t>(segs.size(), 1), s);
  H2_CUDA_TRY(cudaMemcpyAsync(table.p, segs.data(), sizeof(Seg) * segs.size(), cudaMemcpyHostToDevice, s));
  if (npack) seg_copy_kernel<<<(unsigned)npack, 256, 0, s>>>(table.as<Seg>());
  H2_CHECK_LAUNCH();
  comm_allgather(h->comm, send.p, recv.p, sizeof(int) * sw, s);
  if (segs.size() > npack) seg_copy_kernel<<<(unsigned)(segs.size() - npack), 256, 0, s>>>(table.as<Seg>() + npack);
  H2_CHECK_LAUNCH();
  // the table is host-sourced: keep it alive until the copies ran (bounded wait: a dead peer
  // raises H2_ERR_NCCL instead of hanging)
  comm_sync(h->comm, s);
  h->gpu_launches += 2;
}

}  // namespace h2

using namespace h2;

extern "C" {

int32_t h2_shard_cut_level(const int64_t* level_counts, int32_t nlevels, int32_t nranks) {
  if (!level_counts || nlevels < 1 || nranks < 1) return 0;
  int best = 0;
  for (int l = 0; l < nlevels; l++) {
    if (level_counts[l] >= 64LL * nranks) return l;
    if (level_counts[l] > level_counts[best]) best = l;
  }
  return best;
}

int h2_shard_split(const int64_t* weights, int64_t ncut, int32_t nranks, int64_t* first) {
  if (!first || nranks < 1 || ncut < 0 || (ncut > 0 && !weights)) return H2_ERR_INVALID_ARG;
  __int128 total = 0;
  for (int64_t t = 0; t < ncut; t++) {
    if (weights[t] < 0) return H2_ERR_INVALID_ARG;
    total += weights[t];
  }
  // first[q] = the smallest t with prefix(t) * nranks >= q * total (prefix(t) = sum of w[0..t))
  first[0] = 0;
  __int128 pre = 0;
  int64_t t = 0;
  for (int q = 1; q < nranks; q++) {
    while (t < ncut && pre * nranks < (__int128)q * total) pre += weights[t++];
    first[q] = t;
  }
  first[nranks] = ncut;
  return H2_OK;
}

}  // extern "C"
