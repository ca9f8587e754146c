// prims.cu -- device memory pool and the CUB primitives (scan, radix sort) used by the stages.
#include <cub/cub.cuh>

#include "h2_internal.cuh"

namespace h2 {

static cudaMemPool_t pool_for_current_device() {
  int dev = 0;
  H2_CUDA_TRY(cudaGetDevice(&dev));
  static cudaMemPool_t pools[64] = {nullptr};
  if (!pools[dev]) {
    cudaMemPool_t p;
    H2_CUDA_TRY(cudaDeviceGetDefaultMemPool(&p, dev));
    uint64_t thr = UINT64_MAX;  // keep freed blocks cached: repeated builds reuse HBM
    H2_CUDA_TRY(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr));
    pools[dev] = p;
  }
  return pools[dev];
}

void* dev_alloc(size_t bytes, cudaStream_t s) {
  void* p = nullptr;
  cudaMemPool_t pool = pool_for_current_device();
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, s);
  if (e == cudaErrorMemoryAllocation) {
    // give cached blocks back and retry once
    cudaGetLastError();
    H2_CUDA_TRY(cudaStreamSynchronize(s));
    H2_CUDA_TRY(cudaMemPoolTrimTo(pool, 0));
    e = cudaMallocFromPoolAsync(&p, bytes, pool, s);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error{H2_ERR_OOM, "device allocation of " + std::to_string(bytes) + " bytes failed: " +
                                cudaGetErrorString(e)};
  }
  return p;
}

void dev_free(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
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
