// prims.cu -- device memory pool and the CUB primitives (scan, radix sort) used by the stages.
#include <cub/cub.cuh>
#include <map>
#include <mutex>
#include <unordered_map>

#include "h2_internal.cuh"

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

void scan_incl_i32(const int* in, int* out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  H2_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out, n, s));
  Scratch t(tmp, s);
  H2_CUDA_TRY(cub::DeviceScan::InclusiveSum(t.p, tmp, in, out, n, s));
}

void scan_excl_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  H2_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
  Scratch t(tmp, s);
  H2_CUDA_TRY(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, n, s));
}

void sort_pairs_u64_i32(unsigned long long* kin, unsigned long long* kout, int* vin, int* vout, int64_t n,
                        int end_bit, cudaStream_t s) {
  size_t tmp = 0;
  H2_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, n, 0, end_bit, s));
  Scratch t(tmp, s);
  H2_CUDA_TRY(cub::DeviceRadixSort::SortPairs(t.p, tmp, kin, kout, vin, vout, n, 0, end_bit, s));
}

void sort_keys_u64(unsigned long long* kin, unsigned long long* kout, int64_t n, int end_bit, cudaStream_t s) {
  size_t tmp = 0;
  H2_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp, kin, kout, n, 0, end_bit, s));
  Scratch t(tmp, s);
  H2_CUDA_TRY(cub::DeviceRadixSort::SortKeys(t.p, tmp, kin, kout, n, 0, end_bit, s));
}

}  // namespace h2
