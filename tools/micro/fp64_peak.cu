// fp64_peak.cu -- measured FP64 pipe peak of this B200 (DFMA / DADD / DMUL per second) at the clocks
// the GPU sustains under load.  Used as the FP64 roofline denominator (BASELINE.md §2 asks for it
// before any FP64 fraction is quoted).
//
// Every thread runs 8 independent dependency chains of one instruction type (enough to cover the
// FP64 pipe latency), CTAs of 256 threads, 8 CTAs per SM over all SMs; each kernel runs ~0.5 s,
// repeated 6 times after a warm-up, and the median is reported.  Flops: DFMA = 2, DADD / DMUL = 1.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_peak fp64_peak.cu
//   ./fp64_peak > profiles/r02_fp64_peak.json
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

template <int OP>
__global__ void __launch_bounds__(256) chains(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; c++) x[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
#pragma unroll
      for (int c = 0; c < 8; c++) {
        if (OP == 0) x[c] = fma(x[c], a, b);
        else if (OP == 1) x[c] = x[c] + b;
        else x[c] = x[c] * a;
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; c++) s += x[c];
  if (s == 1234.5) out[blockIdx.x] = s;  // keeps the chains live
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  const int blocks = sms * 8, threads = 256;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double rate[3];
  for (int op = 0; op < 3; op++) {
    auto launch = [&](int iters) {
      if (op == 0) chains<0><<<blocks, threads>>>(out, iters, 0.9999999, 1e-7);
      else if (op == 1) chains<1><<<blocks, threads>>>(out, iters, 0.9999999, 1e-7);
      else chains<2><<<blocks, threads>>>(out, iters, 0.9999999, 1e-7);
    };
    launch(2000);  // warm-up (clocks ramp)
    cudaDeviceSynchronize();
    // size one launch to ~0.5 s
    int iters = 2000;
    cudaEventRecord(e0);
    launch(iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    iters = std::max(1, (int)(iters * 500.0 / std::max(ms, 0.01f)));
    std::vector<double> r;
    for (int rep = 0; rep < 6; rep++) {
      cudaEventRecord(e0);
      launch(iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double instr = (double)blocks * threads * iters * 16 * 8;
      r.push_back(instr / (ms * 1e-3));
    }
    std::sort(r.begin(), r.end());
    rate[op] = 0.5 * (r[2] + r[3]);
  }
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"dfma_per_s\": %.4e, \"dadd_per_s\": %.4e, \"dmul_per_s\": %.4e, "
         "\"fp64_tflops\": %.3f, \"lanes_per_sm_at_max_clock\": %.2f, \"max_clock_mhz\": %.0f, "
         "\"how\": \"8 independent chains x 256 threads x 8 CTAs per SM, ~0.5 s per launch, median of 6 after "
         "warm-up; TFLOPS = 2 x DFMA/s\"}\n",
         prop.name, sms, rate[0], rate[1], rate[2], 2.0 * rate[0] / 1e12, rate[0] / (sms * clk * 1e3), clk / 1e3);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
