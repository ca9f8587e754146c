// prims.cu -- device memory pool and the device-wide primitives used by the stages: a two-launch
// prefix sum (per-tile reduction, then a scan of the tile sums fused with the tile scans) and a
// stable LSD radix sort (8-bit digits; one onesweep launch per digit: decoupled look-back over the
// tiles' published digit counts) -- both written here, no library kernels.
#include <cstdlib>
#include <map>
#include <mutex>
#include <unordered_map>

#include "prims.cuh"

namespace h2 {

// Size-matched caching allocator.  Every allocation of the build is served from blocks freed by
// earlier builds when one of a close size exists (the sizes repeat exactly from build to build),
// otherwise from cudaMalloc.  Freed blocks are kept (never cudaFree'd except to recover from an
// out-of-memory), so steady-state builds make no driver allocation calls at all.  A block is
// tagged with the stream that freed it and an event recorded there at the free: another stream
// may take it only once that event has completed (no host or device wait is ever introduced --
// the build runs two streams concurrently, and a wait on the busy one would serialise them);
// otherwise a fresh block is allocated, so steady state keeps per-stream blocks.
struct CachedBlock {
  void* p;
  size_t size;
  cudaStream_t stream;
  int dev;
  cudaEvent_t freed;  // recorded on `stream` when the block was freed (its last use precedes it)
};
static std::mutex g_mu;
static std::multimap<size_t, CachedBlock> g_free;
static std::unordered_map<void*, CachedBlock> g_live;

static size_t round_size(size_t b) {
  if (b < 512) return 512;
  if (b < (1u << 20)) return (b + 511) & ~size_t(511);
  return (b + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
}

static void release_cached(int dev) {  // caller holds g_mu
  H2_CUDA_TRY(cudaDeviceSynchronize());
  for (auto it = g_free.begin(); it != g_free.end();) {
    if (it->second.dev == dev) {
      cudaFree(it->second.p);
      cudaEventDestroy(it->second.freed);
      it = g_free.erase(it);
    } else {
      ++it;
    }
  }
}

void* dev_alloc(size_t bytes, cudaStream_t s) {
  int dev = 0;
  H2_CUDA_TRY(cudaGetDevice(&dev));
  const size_t size = round_size(bytes);
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto it = g_free.lower_bound(size); it != g_free.end() && it->first <= size + size / 4 + (size_t(2) << 20);
       ++it) {
    if (it->second.dev != dev) continue;
    if (it->second.stream != s) {
      const cudaError_t q = cudaEventQuery(it->second.freed);
      if (q == cudaErrorNotReady) {
        cudaGetLastError();
        continue;
      }
      H2_CUDA_TRY(q);
    }
    CachedBlock b = it->second;
    g_free.erase(it);
    b.stream = s;
    g_live[b.p] = b;
    return b.p;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, size);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    release_cached(dev);
    e = cudaMalloc(&p, size);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error{H2_ERR_OOM, "device allocation of " + std::to_string(bytes) + " bytes failed: " +
                                cudaGetErrorString(e)};
  }
  cudaEvent_t ev = nullptr;
  H2_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  g_live[p] = CachedBlock{p, size, s, dev, ev};
  return p;
}

void dev_free(void* p, cudaStream_t s) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_live.find(p);
  if (it == g_live.end()) return;
  CachedBlock b = it->second;
  g_live.erase(it);
  b.stream = s;
  cudaEventRecord(b.freed, s);
  g_free.emplace(b.size, b);
}

// bytes held by the cache and free for reuse on the current device (the AUTO storage budget
// counts them as available)
size_t cached_free_bytes() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  size_t t = 0;
  for (auto& kv : g_free)
    if (kv.second.dev == dev) t += kv.second.size;
  return t;
}

void hfree(h2_handle* h, void* p) {
  for (auto& a : h->allocs)
    if (a == p) {
      dev_free(p, h->stream);
      a = nullptr;
      return;
    }
}

// ==========================================================================================
// Prefix sum in two launches, no inter-CTA waiting: (1) every tile of kScanTile items writes its
// sum; (2) every tile adds up the sums of the tiles before it (a block reduction over at most a
// few thousand values -- cheaper than a serial look-back chain at these sizes) and scans its
// items.  Tiles are read warp-striped: warp w owns 32 kScanIPT consecutive items, read in
// kScanIPT coalesced rounds of 32 and scanned round after round with a carry.
// ==========================================================================================
constexpr int kScanNT = 256, kScanIPT = 16, kScanTile = kScanNT * kScanIPT;

static thread_local int64_t g_prim_launches = 0;  // kernels launched by the primitives (this thread)
int64_t prim_launches() { return g_prim_launches; }

template <typename T>
__global__ void __launch_bounds__(kScanNT) scan_reduce_kernel(const T* __restrict__ in, int64_t n,
                                                              long long* __restrict__ tile_sum) {
  __shared__ long long s_warp[kScanNT / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t base = blockIdx.x * (int64_t)kScanTile;
  long long acc = 0;
#pragma unroll
  for (int k = 0; k < kScanIPT; k++) {
    const int64_t p = base + k * kScanNT + tid;
    if (p < n) acc += (long long)in[p];
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) s_warp[w] = acc;
  __syncthreads();
  if (tid == 0) {
    long long t = 0;
    for (int q = 0; q < kScanNT / 32; q++) t += s_warp[q];
    tile_sum[blockIdx.x] = t;
  }
}

template <typename T, bool INCLUSIVE>
__global__ void __launch_bounds__(kScanNT) scan_apply_kernel(const T* __restrict__ in, T* __restrict__ out,
                                                             int64_t n, const long long* __restrict__ tile_sum) {
  __shared__ long long s_warp[kScanNT / 32];
  __shared__ long long s_red[kScanNT / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t tile = blockIdx.x;
  // prefix of this tile: sum of the tile sums before it
  long long pre_t = 0;
  for (int64_t q = tid; q < tile; q += kScanNT) pre_t += tile_sum[q];
  for (int o = 16; o > 0; o >>= 1) pre_t += __shfl_xor_sync(0xffffffffu, pre_t, o);
  if (lane == 0) s_red[w] = pre_t;
  const int64_t wbase = tile * kScanTile + (int64_t)w * (32 * kScanIPT) + lane;
  long long v[kScanIPT], pre[kScanIPT];
#pragma unroll
  for (int k = 0; k < kScanIPT; k++) {
    const int64_t p = wbase + 32 * k;
    v[k] = p < n ? (long long)in[p] : 0;
  }
  long long carry = 0;
#pragma unroll
  for (int k = 0; k < kScanIPT; k++) {
    long long incl = v[k];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    pre[k] = carry + incl - v[k];
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) s_warp[w] = carry;
  __syncthreads();
  long long off = 0;
#pragma unroll
  for (int q = 0; q < kScanNT / 32; q++) off += s_red[q] + (q < w ? s_warp[q] : 0);
#pragma unroll
  for (int k = 0; k < kScanIPT; k++) {
    const int64_t p = wbase + 32 * k;
    if (p < n) out[p] = (T)(off + pre[k] + (INCLUSIVE ? v[k] : 0));
  }
}

template <typename T, bool INCLUSIVE>
static void device_scan(const T* in, T* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  Scratch ts(sizeof(long long) * tiles, s);
  if (tiles > 1) scan_reduce_kernel<T><<<(unsigned)tiles, kScanNT, 0, s>>>(in, n, ts.as<long long>());
  scan_apply_kernel<T, INCLUSIVE><<<(unsigned)tiles, kScanNT, 0, s>>>(in, out, n, ts.as<long long>());
  H2_CHECK_LAUNCH();
  g_prim_launches += tiles > 1 ? 2 : 1;
}

void scan_incl_i32(const int* in, int* out, int64_t n, cudaStream_t s) { device_scan<int, true>(in, out, n, s); }

void scan_excl_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  device_scan<int64_t, false>(in, out, n, s);
}

// ==========================================================================================
// Stable LSD radix sort of 64-bit keys (optionally carrying 32-bit values), 8-bit digits.
// Per digit: (1) count -- per-tile digit histograms, digit-major [digit][tile]; (2) the prefix
// sum above over that matrix gives every (digit, tile) its output offset; (3) scatter -- each
// tile ranks its keys stably (warps take consecutive 384-key spans in 12 rounds of 32, in-warp
// ranks by __match_any_sync, warp spans combined per digit), reorders them in shared memory and
// writes each digit's run contiguously.
// ==========================================================================================
constexpr int kSortNT = 256, kSortIPT = 12, kSortTile = kSortNT * kSortIPT, kSortWarps = kSortNT / 32;

__global__ void __launch_bounds__(kSortNT) radix_count_kernel(const unsigned long long* __restrict__ keys, int64_t n,
                                                            int shift, int64_t ntiles, int64_t* counts) {
  __shared__ int hist[256];
  hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = blockIdx.x * (int64_t)kSortTile;
#pragma unroll 4
  for (int k = 0; k < kSortIPT; k++) {
    const int64_t p = base + k * kSortNT + threadIdx.x;
    if (p < n) atomicAdd(&hist[(int)((keys[p] >> shift) & 255ULL)], 1);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = hist[threadIdx.x];
}

template <bool VALS>
__global__ void __launch_bounds__(kSortNT) radix_scatter_kernel(const unsigned long long* __restrict__ kin,
                                                              const int* __restrict__ vin, int64_t n, int shift,
                                                              int64_t ntiles, const int64_t* __restrict__ offsets,
                                                              unsigned long long* __restrict__ kout,
                                                              int* __restrict__ vout) {
  __shared__ unsigned long long sk[kSortTile];
  __shared__ int sv[VALS ? kSortTile : 1];
  __shared__ int wcnt[kSortWarps][256];  // per warp digit counts, then per warp digit prefixes
  __shared__ int dstart[256];             // tile-local start of every digit
  __shared__ long long gofs[256];         // this tile's output offset of every digit
  __shared__ BlockScanSmem<kSortNT> scan;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t base = blockIdx.x * (int64_t)kSortTile;
  for (int d = tid; d < kSortWarps * 256; d += kSortNT) (&wcnt[0][0])[d] = 0;
  gofs[tid] = offsets[(int64_t)tid * ntiles + blockIdx.x];
  __syncthreads();
  unsigned long long key[kSortIPT];
  int val[kSortIPT], rank[kSortIPT];
  auto digit_of = [&](int k, int64_t p) { return p < n ? (int)((key[k] >> shift) & 255ULL) : 256; };
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < kSortIPT; k++) {
    // warp w's span is positions [w, w + 1) * 32 kSortIPT of the tile; round k covers 32 of them
    const int64_t p = base + w * (32 * kSortIPT) + k * 32 + lane;
    const bool ok = p < n;
    key[k] = ok ? kin[p] : ~0ULL;
    if (VALS) val[k] = ok ? vin[p] : 0;
    const int dg = digit_of(k, p);  // padding: a 257th digit, never written
    const unsigned peers = __match_any_sync(0xffffffffu, dg);
    const int before = dg < 256 ? wcnt[w][dg] : 0;
    rank[k] = before + __popc(peers & lt);
    __syncwarp();
    if (dg < 256 && (peers & lt) == 0) wcnt[w][dg] = before + __popc(peers);  // group leader
    __syncwarp();
  }
  __syncthreads();
  // per digit (thread = digit): exclusive prefix over the warps, tile count
  int tcount = 0;
  {
    const int d = tid;
    for (int q = 0; q < kSortWarps; q++) {
      const int c = wcnt[q][d];
      wcnt[q][d] = tcount;
      tcount += c;
    }
  }
  int total;
  const int start = block_excl_sum<kSortNT>(tcount, &total, scan);
  dstart[tid] = start;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kSortIPT; k++) {
    const int64_t p = base + w * (32 * kSortIPT) + k * 32 + lane;
    const int dg = digit_of(k, p);
    if (dg < 256) {
      const int pos = dstart[dg] + wcnt[w][dg] + rank[k];
      sk[pos] = key[k];
      if (VALS) sv[pos] = val[k];
    }
  }
  __syncthreads();
  const int valid = (int)(n - base < kSortTile ? n - base : kSortTile);
  for (int pos = tid; pos < valid; pos += kSortNT) {
    const unsigned long long kk = sk[pos];
    const int d = (int)((kk >> shift) & 255ULL);
    const int64_t o = gofs[d] + (pos - dstart[d]);
    kout[o] = kk;
    if (VALS) vout[o] = sv[pos];
  }
}

// Onesweep variant (the default): the digit histograms of ALL passes come from one read of the
// keys (radix_hist_kernel, or fused into the producer of the keys -- tree.cu's quantisation), and
// each pass is ONE launch: a tile takes its id from a counter (launch order, so every earlier tile
// is resident or done), ranks its keys as above, publishes its per-digit count and finds its
// per-digit offset by a decoupled look-back over the earlier tiles' published counts / inclusive
// prefixes (status words: 2 flag bits + a 62-bit value), then scatters.  No count kernel, no
// device scan per pass.
constexpr unsigned long long kStAgg = 1ULL << 62, kStInc = 2ULL << 62, kStVal = (1ULL << 62) - 1;

__global__ void __launch_bounds__(kSortNT) radix_hist_kernel(const unsigned long long* __restrict__ keys, int64_t n,
                                                           int passes, unsigned* __restrict__ hist) {
  __shared__ unsigned sh[8][256];
  for (int t = threadIdx.x; t < 8 * 256; t += kSortNT) (&sh[0][0])[t] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)kSortNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kSortNT) {
    const unsigned long long k = keys[i];
    for (int p = 0; p < passes; p++) atomicAdd(&sh[p][(k >> (8 * p)) & 255ULL], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < passes * 256; t += kSortNT) {
    const unsigned v = (&sh[0][0])[t];
    if (v) atomicAdd(hist + t, v);
  }
}

template <bool VALS>
__global__ void __launch_bounds__(kSortNT) radix_onesweep_kernel(const unsigned long long* __restrict__ kin,
                                                               const int* __restrict__ vin, int64_t n, int shift,
                                                               const unsigned* __restrict__ hist,
                                                               unsigned long long* status, unsigned* ctr,
                                                               unsigned long long* __restrict__ kout,
                                                               int* __restrict__ vout) {
  __shared__ unsigned long long sk[kSortTile];
  __shared__ int sv[VALS ? kSortTile : 1];
  __shared__ int wcnt[kSortWarps][256];
  __shared__ int dstart[256];
  __shared__ long long gofs[256];
  __shared__ BlockScanSmem<kSortNT> scan;
  __shared__ unsigned s_tile;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ctr, 1u);
  for (int d = tid; d < kSortWarps * 256; d += kSortNT) (&wcnt[0][0])[d] = 0;
  // the digit's global start: exclusive prefix of this pass's histogram
  int dtot;
  const int dbase = block_excl_sum<kSortNT>((int)hist[tid], &dtot, scan);  // (its barrier orders s_tile / wcnt)
  const unsigned tile = s_tile;
  const int64_t base = (int64_t)tile * kSortTile;
  unsigned long long key[kSortIPT];
  int val[kSortIPT], rank[kSortIPT];
  auto digit_of = [&](int k, int64_t p) { return p < n ? (int)((key[k] >> shift) & 255ULL) : 256; };
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < kSortIPT; k++) {
    const int64_t p = base + w * (32 * kSortIPT) + k * 32 + lane;
    const bool ok = p < n;
    key[k] = ok ? kin[p] : ~0ULL;
    if (VALS) val[k] = ok ? vin[p] : 0;
    const int dg = digit_of(k, p);
    const unsigned peers = __match_any_sync(0xffffffffu, dg);
    const int before = dg < 256 ? wcnt[w][dg] : 0;
    rank[k] = before + __popc(peers & lt);
    __syncwarp();
    if (dg < 256 && (peers & lt) == 0) wcnt[w][dg] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  int tcount = 0;
  {
    const int d = tid;
    for (int q = 0; q < kSortWarps; q++) {
      const int c = wcnt[q][d];
      wcnt[q][d] = tcount;
      tcount += c;
    }
  }
  // publish this tile's count of digit tid, then look back for its exclusive prefix
  volatile unsigned long long* st = status;
  const int64_t me = (int64_t)tile * 256 + tid;
  if (tile == 0) {
    st[me] = kStInc | (unsigned long long)tcount;
    gofs[tid] = dbase;
  } else {
    st[me] = kStAgg | (unsigned long long)tcount;
    unsigned long long excl = 0;
    for (int64_t t = (int64_t)tile - 1;; t--) {
      unsigned long long v;
      do {
        v = st[t * 256 + tid];
      } while ((v & ~kStVal) == 0);
      excl += v & kStVal;
      if ((v & ~kStVal) == kStInc) break;
    }
    st[me] = kStInc | (excl + (unsigned long long)tcount);
    gofs[tid] = dbase + (long long)excl;
  }
  int total;
  const int start = block_excl_sum<kSortNT>(tcount, &total, scan);
  dstart[tid] = start;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kSortIPT; k++) {
    const int64_t p = base + w * (32 * kSortIPT) + k * 32 + lane;
    const int dg = digit_of(k, p);
    if (dg < 256) {
      const int pos = dstart[dg] + wcnt[w][dg] + rank[k];
      sk[pos] = key[k];
      if (VALS) sv[pos] = val[k];
    }
  }
  __syncthreads();
  const int valid = (int)(n - base < kSortTile ? n - base : kSortTile);
  for (int pos = tid; pos < valid; pos += kSortNT) {
    const unsigned long long kk = sk[pos];
    const int d = (int)((kk >> shift) & 255ULL);
    const int64_t o = gofs[d] + (pos - dstart[d]);
    kout[o] = kk;
    if (VALS) vout[o] = sv[pos];
  }
}

// H2_SORT_ONESWEEP=0 (A/B knob): the count / scan / scatter passes
static bool sort_onesweep() {
  static const bool v = [] {
    const char* e = getenv("H2_SORT_ONESWEEP");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

static void radix_sort(unsigned long long* kin, unsigned long long* kout, int* vin, int* vout, int64_t n, int end_bit,
                       cudaStream_t s, const unsigned* hist_in) {
  if (n <= 0) return;
  const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
  const int passes = (end_bit + 7) / 8;
  Scratch kt(passes > 1 ? sizeof(unsigned long long) * n : 8, s), vt(passes > 1 && vin ? sizeof(int) * n : 8, s);
  if (sort_onesweep()) {
    const size_t st_words = (size_t)passes * ntiles * 256;
    Scratch ws(sizeof(unsigned long long) * st_words + sizeof(unsigned) * (8 * 256 + 8), s);
    unsigned long long* status = ws.as<unsigned long long>();
    unsigned* hist = reinterpret_cast<unsigned*>(status + st_words);
    unsigned* ctr = hist + 8 * 256;
    H2_CUDA_TRY(cudaMemsetAsync(ws.p, 0, sizeof(unsigned long long) * st_words + sizeof(unsigned) * (8 * 256 + 8), s));
    if (!hist_in) {
      radix_hist_kernel<<<(unsigned)grid_for(n, kSortNT, 148 * 4), kSortNT, 0, s>>>(kin, n, passes, hist);
      H2_CHECK_LAUNCH();
      g_prim_launches += 1;
      hist_in = hist;
    }
    const unsigned long long* ksrc = kin;
    const int* vsrc = vin;
    for (int p = 0; p < passes; p++) {
      const bool to_out = ((passes - 1 - p) % 2) == 0;
      unsigned long long* kdst = to_out ? kout : kt.as<unsigned long long>();
      int* vdst = vin ? (to_out ? vout : vt.as<int>()) : nullptr;
      unsigned long long* stp = status + (size_t)p * ntiles * 256;
      if (vin)
        radix_onesweep_kernel<true><<<(unsigned)ntiles, kSortNT, 0, s>>>(ksrc, vsrc, n, 8 * p, hist_in + 256 * p, stp,
                                                                         ctr + p, kdst, vdst);
      else
        radix_onesweep_kernel<false><<<(unsigned)ntiles, kSortNT, 0, s>>>(ksrc, nullptr, n, 8 * p, hist_in + 256 * p,
                                                                          stp, ctr + p, kdst, nullptr);
      H2_CHECK_LAUNCH();
      g_prim_launches += 1;
      ksrc = kdst;
      vsrc = vdst;
    }
    return;
  }
  Scratch counts(sizeof(int64_t) * 256 * ntiles, s), offs(sizeof(int64_t) * 256 * ntiles, s);
  // ping-pong so that the last pass writes kout / vout
  const unsigned long long* ksrc = kin;
  const int* vsrc = vin;
  for (int p = 0; p < passes; p++) {
    const bool to_out = ((passes - 1 - p) % 2) == 0;
    unsigned long long* kdst = to_out ? kout : kt.as<unsigned long long>();
    int* vdst = vin ? (to_out ? vout : vt.as<int>()) : nullptr;
    radix_count_kernel<<<(unsigned)ntiles, kSortNT, 0, s>>>(ksrc, n, 8 * p, ntiles, counts.as<int64_t>());
    H2_CHECK_LAUNCH();
    scan_excl_i64(counts.as<int64_t>(), offs.as<int64_t>(), 256 * ntiles, s);
    if (vin)
      radix_scatter_kernel<true><<<(unsigned)ntiles, kSortNT, 0, s>>>(ksrc, vsrc, n, 8 * p, ntiles,
                                                                      offs.as<int64_t>(), kdst, vdst);
    else
      radix_scatter_kernel<false><<<(unsigned)ntiles, kSortNT, 0, s>>>(ksrc, nullptr, n, 8 * p, ntiles,
                                                                       offs.as<int64_t>(), kdst, nullptr);
    H2_CHECK_LAUNCH();
    g_prim_launches += 2;  // count + scatter (the scan counts itself)
    ksrc = kdst;
    vsrc = vdst;
  }
}

// keys_out / vals_out receive the stable sort of (keys_in, vals_in) by the key's bits [0, end_bit)
void sort_pairs_u64_i32(unsigned long long* kin, unsigned long long* kout, int* vin, int* vout, int64_t n,
                        int end_bit, cudaStream_t s, const unsigned* hist) {
  radix_sort(kin, kout, vin, vout, n, end_bit, s, hist);
}

void sort_keys_u64(unsigned long long* kin, unsigned long long* kout, int64_t n, int end_bit, cudaStream_t s) {
  radix_sort(kin, kout, nullptr, nullptr, n, end_bit, s, nullptr);
}

}  // namespace h2
