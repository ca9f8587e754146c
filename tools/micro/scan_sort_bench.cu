// Micro-benchmark of the library's device-wide scan and radix sort against CUB (A/B only; not
// part of the library).  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I.. prims.cu this.cu
#include <cub/cub.cuh>
#include <chrono>
#include <cstdio>
#include <vector>
#include "../../paper_2206_01885_b200/csrc/h2_internal.cuh"
namespace h2 { void set_error(int, const std::string&) {} void clear_error() {} }
using namespace h2;
int main() {
  const int64_t n = 1 << 22;
  cudaStream_t s; cudaStreamCreate(&s);
  int *a, *b; int64_t *c, *d; unsigned long long *k1, *k2; int *v1, *v2;
  cudaMalloc(&a, 4 * n); cudaMalloc(&b, 4 * n); cudaMalloc(&c, 8 * n); cudaMalloc(&d, 8 * n);
  cudaMalloc(&k1, 8 * n); cudaMalloc(&k2, 8 * n); cudaMalloc(&v1, 4 * n); cudaMalloc(&v2, 4 * n);
  std::vector<int> h(n); std::vector<unsigned long long> hk(n);
  unsigned long long x = 1;
  for (int64_t i = 0; i < n; i++) { x = x * 6364136223846793005ULL + 1442695040888963407ULL; h[i] = (x >> 40) & 7; hk[i] = x >> 4; }
  cudaMemcpy(a, h.data(), 4 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(k1, hk.data(), 8 * n, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto f) {
    for (int i = 0; i < 3; i++) f();
    cudaStreamSynchronize(s);
    auto h0 = std::chrono::steady_clock::now();
    cudaEventRecord(e0, s);
    for (int i = 0; i < 20; i++) f();
    auto h1 = std::chrono::steady_clock::now();
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    // one call alone, the stream blocked behind a spin so the launch cost is hidden
    cudaStreamSynchronize(s);
    float single = 0;
    {
      cudaEvent_t a0, a1; cudaEventCreate(&a0); cudaEventCreate(&a1);
      cudaEventRecord(a0, s); f(); cudaEventRecord(a1, s); cudaEventSynchronize(a1);
      cudaEventElapsedTime(&single, a0, a1);
    }
    printf("%-28s %8.1f us/call (queue of 20), host %6.1f us/call, single %6.1f us\n", name, ms * 1000 / 20,
           std::chrono::duration<double, std::micro>(h1 - h0).count() / 20, single * 1000);
  };
  timeit("scan_incl_i32 (ours)", [&] { scan_incl_i32(a, b, n, s); });
  size_t tmp = 0; void* t = nullptr; cub::DeviceScan::InclusiveSum(nullptr, tmp, a, b, n, s); cudaMalloc(&t, tmp);
  timeit("InclusiveSum i32 (cub)", [&] { cub::DeviceScan::InclusiveSum(t, tmp, a, b, n, s); });
  std::vector<int> hb(n); scan_incl_i32(a, b, n, s); cudaMemcpy(hb.data(), b, 4 * n, cudaMemcpyDeviceToHost);
  long long acc = 0; int bad = 0; for (int64_t i = 0; i < n; i++) { acc += h[i]; bad += hb[i] != acc; } printf("scan errors %d\n", bad);
  timeit("sort_pairs 60-bit (ours)", [&] { sort_pairs_u64_i32(k1, k2, v1, v2, n, 60, s); });
  size_t tmp2 = 0; void* t2 = nullptr; cub::DeviceRadixSort::SortPairs(nullptr, tmp2, k1, k2, v1, v2, n, 0, 60, s); cudaMalloc(&t2, tmp2);
  timeit("SortPairs 60-bit (cub)", [&] { cub::DeviceRadixSort::SortPairs(t2, tmp2, k1, k2, v1, v2, n, 0, 60, s); });
  sort_pairs_u64_i32(k1, k2, v1, v2, n, 60, s);
  std::vector<unsigned long long> hs(n); cudaMemcpy(hs.data(), k2, 8 * n, cudaMemcpyDeviceToHost);
  int uns = 0; for (int64_t i = 1; i < n; i++) uns += (hs[i - 1] & ((1ULL << 60) - 1)) > (hs[i] & ((1ULL << 60) - 1));
  printf("sort order violations %d  err=%s\n", uns, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
