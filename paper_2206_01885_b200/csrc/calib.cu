// calib.cu -- a5: r1 = r2 = r from the tolerance (Algorithm 2 line 2).
//
// Readings (E1-E6): r1 = r2 = r; for every level l holding an admissible pair, box
// width w = W 2^-l; Z1 = 256 SplitMix64 points in [0,w]^d, Z2 = the same construction shifted by
// w/tau in every coordinate (the Eq.(2.1) boundary); for m = 1, 2, ...: Z2* = Vol(Z2, m^d), ID of
// K(Z1, Z2*) at tolerance 1e-3 eps, e = ||K(Z1,Z2) - U K(Z1^,Z2)||_F / ||K(Z1,Z2)||_F; the level's
// budget is the first m^d with e < 1e-2 eps, or m^d >= 256 (pass-through); r = max over levels.
// All (level, m) trials run as one batched launch: one CTA per trial.
#include "cpqr.cuh"
#include "vol.cuh"

namespace h2 {

constexpr int kCalThreads = 256;
constexpr int N = kCalibPoints;

struct CalWork {  // per-trial global workspace
  double Z1[N * kMaxD], Z2[N * kMaxD];
  double M[N * N];
  double Ks[N * N];
  double nrm2[N], v[N];
  int piv[N], sel[N];
};

// k-th SplitMix64 output of the stream seeded with `seed` (counter form of the sequential
// generator: state_k = seed + (k+1) * golden gamma)
__device__ __forceinline__ unsigned long long splitmix_at(unsigned long long seed, unsigned long long k) {
  unsigned long long z = seed + (k + 1ULL) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

struct PtAcc {
  const double* Z;
  int d;
  __device__ __forceinline__ double coord(int pos, int c) const { return Z[pos * d + c]; }
  __device__ __forceinline__ int index(int pos) const { return pos; }
};

template <int D>
__global__ void __launch_bounds__(kCalThreads) calib_kernel(int kid, double p2, double eps, double tau,
                                                            const double* __restrict__ wl, const int* __restrict__ lv,
                                                            const int* __restrict__ mv, CalWork* work, double* err,
                                                            int* pass) {
  __shared__ VolSmem<D, kCalThreads> vsm;
  __shared__ CpqrSmem<kCalThreads> csm;
  __shared__ int s_ns;
  const int tid = threadIdx.x;
  CalWork& W = work[blockIdx.x];
  const double w = wl[blockIdx.x];
  const int level = lv[blockIdx.x], m = mv[blockIdx.x];
  const unsigned long long seed = kCalibSeed + (unsigned long long)level;
  const double shift = __ddiv_rn(w, tau);
  for (int e = tid; e < N * D; e += kCalThreads) {
    double u1 = (double)(splitmix_at(seed, e) >> 11) * 0x1.0p-53;
    double u2 = (double)(splitmix_at(seed, N * D + e) >> 11) * 0x1.0p-53;
    W.Z1[e] = __dmul_rn(u1, w);
    W.Z2[e] = __dadd_rn(__dmul_rn(u2, w), shift);
  }
  __syncthreads();
  long long G = 1;
  for (int c = 0; c < D; c++) G *= m;
  if (G >= N) {
    for (int i = tid; i < N; i += kCalThreads) W.sel[i] = i;
    if (tid == 0) s_ns = N;
  } else {
    PtAcc acc{W.Z2, D};
    int c = cta_vol<D, kCalThreads>(acc, N, (int)G, W.sel, vsm);
    if (tid == 0) s_ns = c;
  }
  __syncthreads();
  const int ns = s_ns;
  // M = K(Z1, Z2*)^T : ns x N column-major (columns = Z1 candidates)
  for (int e = tid; e < ns * N; e += kCalThreads) {
    int a = e % ns, b = e / ns;
    double s = 0.0;
    for (int c = 0; c < D; c++) {
      double df = W.Z1[b * D + c] - W.Z2[W.sel[a] * D + c];
      s = fma(df, df, s);
    }
    W.M[e] = kernel_s(kid, p2, s);
  }
  __syncthreads();
  const int k = cta_cpqr<kCalThreads>(W.M, ns, N, 1e-3 * eps, W.piv, W.nrm2, W.v, csm);
  // Ks[t][e] = K(Z1[piv[t]], Z2[e]) for the k skeleton rows
  for (int x = tid; x < k * N; x += kCalThreads) {
    int t = x / N, e = x % N;
    double s = 0.0;
    for (int c = 0; c < D; c++) {
      double df = W.Z1[W.piv[t] * D + c] - W.Z2[e * D + c];
      s = fma(df, df, s);
    }
    W.Ks[x] = kernel_s(kid, p2, s);
  }
  __syncthreads();
  double num = 0.0, den = 0.0;
  for (int x = tid; x < N * N; x += kCalThreads) {
    int c = x / N, e = x % N;  // c = position in the pivoted order
    int row = W.piv[c];
    double s = 0.0;
    for (int q = 0; q < D; q++) {
      double df = W.Z1[row * D + q] - W.Z2[e * D + q];
      s = fma(df, df, s);
    }
    double kv = kernel_s(kid, p2, s);
    den += kv * kv;
    if (c >= k) {
      double ap = 0.0;
      for (int t = 0; t < k; t++) ap += W.M[t + ns * c] * W.Ks[t * N + e];
      double df = kv - ap;
      num += df * df;
    }
  }
  num = cta_sum<kCalThreads>(num, csm);
  den = cta_sum<kCalThreads>(den, csm);
  if (tid == 0) {
    double e = den > 0.0 ? sqrt(num) / sqrt(den) : 0.0;
    err[blockIdx.x] = e;
    pass[blockIdx.x] = (e < 1e-2 * eps) || G >= N;
  }
}

__global__ void level_has_il_kernel(int nnodes, const int* __restrict__ level, const int64_t* __restrict__ il_off,
                                    int* has) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nnodes && il_off[i + 1] > il_off[i]) has[level[i]] = 1;
}

int calibrate(h2_handle* h) {
  cudaStream_t s = h->stream;
  const int d = h->d;
  Scratch hasd(sizeof(int) * 64, s);
  H2_CUDA_TRY(cudaMemsetAsync(hasd.p, 0, sizeof(int) * 64, s));
  level_has_il_kernel<<<(h->nnodes + 255) / 256, 256, 0, s>>>(h->nnodes, h->level, h->il_off, hasd.as<int>());
  H2_CHECK_LAUNCH();
  h->gpu_launches += 1;
  int has[64];
  H2_CUDA_TRY(cudaMemcpyAsync(has, hasd.p, sizeof(int) * 64, cudaMemcpyDeviceToHost, s));
  H2_CUDA_TRY(cudaStreamSynchronize(s));
  // Trials in two phases: first every m with m^d <= 64 (cheap blocks) for all levels, then the
  // larger m only for levels that have not passed yet.  The chosen m is the first passing one
  // either way (the phases only avoid evaluating trials beyond it).
  std::vector<int> levels;
  for (int l = 0; l <= h->depth; l++)
    if (has[l]) levels.push_back(l);
  int r = 1;
  if (levels.empty()) return r;
  const double p2 = kernel_p2(h->kid, h->kp);
  auto Gof = [&](int m) {
    long long G = 1;
    for (int c = 0; c < d; c++) G *= m;
    return G;
  };
  std::vector<int> chosen_m(levels.size(), 0);
  for (int phase = 0; phase < 2; phase++) {
    std::vector<double> wl;
    std::vector<int> lv, mv, li;
    for (size_t q = 0; q < levels.size(); q++) {
      if (chosen_m[q]) continue;
      for (int m = 1;; m++) {
        const long long G = Gof(m);
        const bool in_phase = phase == 0 ? (G <= 64 || m == 1) : (G > 64 || m == 1);
        if (in_phase && !(phase == 1 && G <= 64)) {
          wl.push_back(ldexp(h->W, -levels[q]));
          lv.push_back(levels[q]);
          mv.push_back(m);
          li.push_back((int)q);
        }
        if (G >= N || (phase == 0 && G > 64)) break;
      }
    }
    const int T = (int)wl.size();
    if (T == 0) break;
    const int batch = 256;
    Scratch work(sizeof(CalWork) * (T < batch ? T : batch), s);
    Scratch params(sizeof(double) * T + sizeof(int) * 2 * T, s), outs(sizeof(double) * T + sizeof(int) * T, s);
    double* dw = params.as<double>();
    int* dl = reinterpret_cast<int*>(dw + T);
    int* dm = dl + T;
    double* derr = outs.as<double>();
    int* dpass = reinterpret_cast<int*>(derr + T);
    H2_CUDA_TRY(cudaMemcpyAsync(dw, wl.data(), sizeof(double) * T, cudaMemcpyHostToDevice, s));
    H2_CUDA_TRY(cudaMemcpyAsync(dl, lv.data(), sizeof(int) * T, cudaMemcpyHostToDevice, s));
    H2_CUDA_TRY(cudaMemcpyAsync(dm, mv.data(), sizeof(int) * T, cudaMemcpyHostToDevice, s));
    for (int b0 = 0; b0 < T; b0 += batch) {
      int nb = T - b0 < batch ? T - b0 : batch;
      switch (d) {
#define H2_CAL_CASE(DD)                                                                                  \
  case DD:                                                                                               \
    calib_kernel<DD><<<nb, kCalThreads, 0, s>>>(h->kid, p2, h->id_tol, h->tau, dw + b0, dl + b0, dm + b0, \
                                                work.as<CalWork>(), derr + b0, dpass + b0);               \
    break;
        H2_CAL_CASE(1) H2_CAL_CASE(2) H2_CAL_CASE(3) H2_CAL_CASE(4)
        H2_CAL_CASE(5) H2_CAL_CASE(6) H2_CAL_CASE(7) H2_CAL_CASE(8)
#undef H2_CAL_CASE
      }
      H2_CHECK_LAUNCH();
      h->gpu_launches += 1;
    }
    std::vector<int> pass(T);
    H2_CUDA_TRY(cudaMemcpyAsync(pass.data(), dpass, sizeof(int) * T, cudaMemcpyDeviceToHost, s));
    H2_CUDA_TRY(cudaStreamSynchronize(s));
    for (int t = 0; t < T; t++)  // trials of a level are in increasing m: keep the first pass
      if (pass[t] && (!chosen_m[li[t]] || mv[t] < chosen_m[li[t]])) chosen_m[li[t]] = mv[t];
  }
  for (size_t q = 0; q < levels.size(); q++) {
    const long long G = Gof(chosen_m[q]);
    if (G > r) r = (int)G;
  }
  return r;
}

}  // namespace h2
