// api.cu -- the C ABI of include/h2.h: argument validation, the Algorithm 2 stage sequence
// (PAPER.md P:459-506), per-stage timing, export hooks and error reporting.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "h2_internal.cuh"

namespace h2 {

static thread_local int g_err = H2_OK;
static thread_local std::string g_msg;

void set_error(int code, const std::string& msg) {
  g_err = code;
  g_msg = msg;
}
void clear_error() {
  g_err = H2_OK;
  g_msg.clear();
}

static void free_handle(h2_handle* h) {
  if (!h) return;
  for (void* p : h->allocs)
    if (p) dev_free(p, h->stream);
  cudaStreamSynchronize(h->stream);
  delete h;
}

// The build's two internal streams on the current device (per host thread, created once, never
// destroyed: cached allocator blocks stay tagged with them).  `main` carries a1-a9 at the
// highest priority; `side` carries the nearfield fill (a10) at the lowest, so the latency-bound
// level kernels take SMs first whenever a fill CTA retires.
struct BuildStreams {
  cudaStream_t main = nullptr, side = nullptr, calib = nullptr, calib2 = nullptr;
  cudaStream_t aux[h2_handle::kAux] = {};
};
static BuildStreams& build_streams() {
  thread_local BuildStreams per_dev[64];
  int dev = 0;
  H2_CUDA_TRY(cudaGetDevice(&dev));
  BuildStreams& b = per_dev[dev & 63];
  if (!b.main) {
    int least = 0, greatest = 0;
    H2_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    H2_CUDA_TRY(cudaStreamCreateWithPriority(&b.main, cudaStreamNonBlocking, greatest));
    // H2_SIDE_PRIORITY=1 (A/B knob): the nearfield fill at the highest priority instead
    const char* sp = getenv("H2_SIDE_PRIORITY");
    H2_CUDA_TRY(cudaStreamCreateWithPriority(&b.side, cudaStreamNonBlocking, sp && atoi(sp) ? greatest : least));
    H2_CUDA_TRY(cudaStreamCreateWithPriority(&b.calib, cudaStreamNonBlocking, greatest));
    H2_CUDA_TRY(cudaStreamCreateWithPriority(&b.calib2, cudaStreamNonBlocking, greatest));
    for (auto& a : b.aux) H2_CUDA_TRY(cudaStreamCreateWithPriority(&a, cudaStreamNonBlocking, greatest));
  }
  return b;
}

// H2_SERIAL=1 (A/B knob, read once) forces h2_options.serial_fill for every build
static bool serial_fill_env() {
  static const bool v = [] {
    const char* e = getenv("H2_SERIAL");
    return e && atoi(e) != 0;
  }();
  return v;
}

template <class T>
static std::vector<T> d2h(const T* d, size_t count, cudaStream_t s) {
  std::vector<T> v(count);
  if (count) H2_CUDA_TRY(cudaMemcpyAsync(v.data(), d, sizeof(T) * count, cudaMemcpyDeviceToHost, s));
  H2_CUDA_TRY(cudaStreamSynchronize(s));
  return v;
}

unsigned long long* build_stats() {
  thread_local unsigned long long* pinned = nullptr;
  if (!pinned) H2_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&pinned), sizeof(unsigned long long) * 64));
  return pinned;
}

// a1-a4 and a6-a7 of `base`, copied into the fresh handle h (device arrays duplicated on
// h->stream; the base keeps its own): the geometry a rebuild for another kernel reuses
static void clone_geometry(h2_handle* h, const h2_handle* b) {
  cudaStream_t s = h->stream;
  auto dup = [&](auto* src, size_t count) {
    using T = std::remove_cv_t<std::remove_pointer_t<decltype(src)>>;
    T* dst = halloc<T>(h, count);
    if (count) H2_CUDA_TRY(cudaMemcpyAsync(dst, src, sizeof(T) * count, cudaMemcpyDeviceToDevice, s));
    return dst;
  };
  const size_t n = b->n, nn = b->nnodes, d = b->d, r = b->r;
  h->W = b->W;
  std::memcpy(h->rlo, b->rlo, sizeof(h->rlo));
  h->L = b->L;
  h->X = dup(b->X, n * d);
  h->perm = dup(b->perm, n);
  h->key = dup(b->key, n);
  h->nnodes = b->nnodes;
  h->depth = b->depth;
  h->nleaves = b->nleaves;
  h->lvl_start = b->lvl_start;
  h->level = dup(b->level, nn);
  h->nbegin = dup(b->nbegin, nn);
  h->nend = dup(b->nend, nn);
  h->parent = dup(b->parent, nn);
  h->first_child = dup(b->first_child, nn);
  h->nchild = dup(b->nchild, nn);
  h->is_leaf = dup(b->is_leaf, nn);
  h->cell = dup(b->cell, nn * d);
  h->n_il = b->n_il;
  h->n_nf = b->n_nf;
  h->il_off = dup(b->il_off, nn + 1);
  h->nf_off = dup(b->nf_off, nn + 1);
  h->il_idx = dup(b->il_idx, (size_t)b->n_il);
  h->nf_idx = dup(b->nf_idx, (size_t)b->n_nf);
  h->csp = b->csp;
  h->r = b->r;
  h->xs_cnt = dup(b->xs_cnt, nn);
  h->xs = dup(b->xs, nn * r);
  h->ys_cnt = dup(b->ys_cnt, nn);
  h->ys = dup(b->ys, nn * r);
  h->hidr_dist_evals = 0;  // nothing of HiDR ran for this handle
  h->hidr_dist_done = 0;
  h->hidr_up_evals = 0;
  h->nranks = b->nranks;
  h->rank = b->rank;
  h->cut = b->cut;
  h->p_lo = b->p_lo;
  h->p_hi = b->p_hi;
  h->rng_lo = b->rng_lo;
  h->rng_hi = b->rng_hi;
  h->gpu_launches += 0;  // copies only
}

// out[k n + t] = X[k n + t] + sign a_k (tree-order SoA coordinates shifted by +-a)
struct ShiftVec {
  double a[kMaxD];
};
__global__ void shift_coords_kernel(int64_t n, int d, const double* __restrict__ X, ShiftVec a, double sign,
                                    double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * d; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = X[e] + sign * a.a[e / n];
}

// kappa's first-argument coordinates (h2_internal.cuh: Xf = X + a, Xfn = X - a for the shifted
// multiquadric; X itself for the other kernels)
static void make_first_arg_coords(h2_handle* h) {
  if (h->kid != H2_KERNEL_MQSHIFT) {
    h->Xf = h->Xfn = h->X;
    return;
  }
  ShiftVec a{};
  for (int c = 0; c < h->d; c++) a.a[c] = h->kpa[c];
  const int64_t m = (int64_t)h->n * h->d;
  h->Xf = halloc<double>(h, m);
  h->Xfn = halloc<double>(h, m);
  shift_coords_kernel<<<grid_for(m, 256), 256, 0, h->stream>>>(h->n, h->d, h->X, a, 1.0, h->Xf);
  shift_coords_kernel<<<grid_for(m, 256), 256, 0, h->stream>>>(h->n, h->d, h->X, a, -1.0, h->Xfn);
  H2_CHECK_LAUNCH();
  h->gpu_launches += 2;
}

}  // namespace h2

using namespace h2;

extern "C" {

int h2_last_error(void) { return g_err; }
const char* h2_last_error_message(void) { return g_msg.c_str(); }

void h2_options_default(h2_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->storage = H2_STORE_AUTO;
}

// The build (h2_build_ex) and the rebuild from a base handle's geometry (h2_rebuild_ex: `base`
// non-null -- a1-a7 are copied from it, only a8-a10 run for the new kernel).
static h2_handle* build_impl(const double* points, int64_t n, int32_t d, int32_t kernel_id,
                             const double* kernel_params, double id_tol, int32_t leaf_size, double admissibility,
                             const h2_options* opt, const h2_handle* base) {
  clear_error();
  h2_options o;
  h2_options_default(&o);
  if (opt) o = *opt;
  if ((!points && !base) || n < 1 || n >= (1LL << 31) - 1 || d < 1 || d > kMaxD || leaf_size < 1 || !(admissibility > 0.0) ||
      !(admissibility <= 0.7) || !(id_tol > 0.0) || !(id_tol < 1.0) || o.r_override < 0 || o.r_override > 4096 ||
      o.storage < 0 || o.storage > 2 || o.reduct < H2_REDUCT_VOLUME || o.reduct > H2_REDUCT_SURFACE ||
      (o.reduct == H2_REDUCT_SURFACE && d != 2 && d != 3) || !(o.srrqr_f == 0.0 || o.srrqr_f >= 1.0) ||
      !std::isfinite(o.srrqr_f) || o.interp_p < 0 || o.interp_p > kInterpMaxP ||
      (o.interp_p > 0 && (std::pow((double)o.interp_p, d) > 4096.0 || base || o.comm || o.nonsymmetric ||
                          kernel_id == H2_KERNEL_MQSHIFT || o.srrqr_f != 0.0))) {
    set_error(H2_ERR_INVALID_ARG, "invalid argument (n, d, leaf_size, admissibility, id_tol or options)");
    return nullptr;
  }
  if (kernel_id < H2_KERNEL_COULOMB || kernel_id > H2_KERNEL_MQSHIFT) {
    set_error(H2_ERR_UNKNOWN_KERNEL, "unknown kernel_id");
    return nullptr;
  }
  double kp = 0.0, kpa[kMaxD] = {0};
  if (kernel_id == H2_KERNEL_MQSHIFT) {  // {c, a_0, ..., a_{d-1}}
    bool ok = kernel_params && kernel_params[0] > 0.0 && std::isfinite(kernel_params[0]);
    for (int c = 0; ok && c < d; c++) {
      ok = std::isfinite(kernel_params[1 + c]);
      kpa[c] = kernel_params[1 + c];
    }
    if (!ok) {
      set_error(H2_ERR_INVALID_ARG, "H2_KERNEL_MQSHIFT needs d + 1 finite parameters {c > 0, a_0..a_{d-1}}");
      return nullptr;
    }
    kp = kernel_params[0];
  } else if (kernel_id != H2_KERNEL_COULOMB && kernel_id != H2_KERNEL_BUMP && kernel_id != H2_KERNEL_COSDOT) {
    if (!kernel_params || !(kernel_params[0] > 0.0) || !std::isfinite(kernel_params[0])) {
      set_error(H2_ERR_INVALID_ARG, "kernel parameter (h or l) must be finite and > 0");
      return nullptr;
    }
    kp = kernel_params[0];
  }
  h2_handle* h = new h2_handle();
  h->n = (int)n;
  h->d = d;
  h->kid = kernel_id;
  h->kp = kp;
  std::memcpy(h->kpa, kpa, sizeof(kpa));
  h->nonsym = o.nonsymmetric || kernel_id == H2_KERNEL_MQSHIFT;
  h->srrqr_f = o.srrqr_f;
  h->interp_p = o.interp_p;
  h->id_tol = id_tol;
  h->q = leaf_size;
  h->tau = admissibility;
  h->stream = static_cast<cudaStream_t>(o.stream);
  h->timing = o.timing;
  h->hidr_prune = o.hidr_brute ? 0 : 1;
  h->reduct = o.reduct;
  h->comm = o.comm;
  h->nranks = h2_comm_size(o.comm);
  h->rank = h2_comm_rank(o.comm);
  h->p_hi = h->n;
  cudaEvent_t ev[8];
  int nev = 0;
  cudaStream_t user = h->stream;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  try {
    BuildStreams& bs = build_streams();
    unsigned long long* stats = build_stats();  // the deferred statistics of this build (h2_internal.cuh)
    for (int q = 0; q < kStatCount; q++) stats[q] = 0;
    H2_CUDA_TRY(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    H2_CUDA_TRY(cudaEventCreateWithFlags(&join_ev, cudaEventDisableTiming));
    // all work runs on the internal streams, ordered after what the caller queued on `user`
    H2_CUDA_TRY(cudaEventRecord(fork_ev, user));
    H2_CUDA_TRY(cudaStreamWaitEvent(bs.main, fork_ev, 0));
    h->stream = bs.main;
    for (int a = 0; a < h2_handle::kAux; a++) h->aux[a] = bs.aux[a];
    h->low = bs.side;
    if (h->timing) {
      for (auto& e : ev) H2_CUDA_TRY(cudaEventCreate(&e));
      nev = 8;
    }
    auto mark = [&](int i) {
      if (h->timing) H2_CUDA_TRY(cudaEventRecord(ev[i], h->stream));
    };
    const double* pts = points;
    Scratch staged;
    if (o.points_on_host && !base) {
      staged = Scratch(sizeof(double) * (size_t)n * d, h->stream);
      H2_CUDA_TRY(cudaMemcpyAsync(staged.p, points, sizeof(double) * (size_t)n * d, cudaMemcpyHostToDevice,
                                  h->stream));
      pts = staged.as<double>();
    }
    const int64_t prims0 = prim_launches();
    NfJob nf;
    CalibJob cal;
    mark(0);
    const bool interp = o.interp_p > 0;  // the interpolation baseline (interp.cu)
    const bool calibrated = o.r_override <= 0 && !base && !interp;
    if (base) {
      clone_geometry(h, base);  // a1-a4, a6-a7 (and the shard plan) of the base handle
      make_first_arg_coords(h);
      mark(1);
    } else {
      build_tree(h, pts);  // a1-a3
      make_first_arg_coords(h);
      mark(1);
      if (calibrated) {  // a5 phase 0 overlaps a4 (calib.cu)
        H2_CUDA_TRY(cudaEventRecord(fork_ev, h->stream));
        H2_CUDA_TRY(cudaStreamWaitEvent(bs.calib, fork_ev, 0));
        H2_CUDA_TRY(cudaStreamWaitEvent(bs.calib2, fork_ev, 0));
        calibrate_begin(h, bs.calib, bs.calib2, cal);
        // H2_CAL_SYNC=1 (probe knob): finish a5 before a4 starts (the trials' own duration then
        // shows up in the lists stage)
        static const bool cal_sync = [] {
          const char* e = getenv("H2_CAL_SYNC");
          return e && atoi(e) != 0;
        }();
        if (cal_sync) {
          H2_CUDA_TRY(cudaStreamSynchronize(bs.calib));
          H2_CUDA_TRY(cudaStreamSynchronize(bs.calib2));
        }
      }
      if (h->nranks > 1) shard_plan(h);  // cut level, owned subtrees and block rows (shard.cu)
      build_lists(h);                    // a4 (sharded: the rank's own rows)
    }
    mark(2);
    // a10 needs only the tree and the nearfield list: it starts now on the side stream and
    // overlaps a5-a9 (serial_fill: after a9 on the main stream instead)
    const bool serial = o.serial_fill || serial_fill_env();
    if (!serial) fill_nearfield_begin(h, bs.side, o.storage, o.mem_budget_bytes, nf);
    if (interp) {
      int r = 1;
      for (int c = 0; c < d; c++) r *= o.interp_p;
      h->r = r;
      mark(3);
      mark(4);
    } else if (!base) {
      h->r = calibrated ? calibrate_end(h, cal) : o.r_override;  // a5
      mark(3);
      hidr_up(h);  // a6
      mark(4);
      hidr_down(h);  // a7
    } else {
      mark(3);
      mark(4);
    }
    mark(5);
    if (interp) interp_sweep(h, o.interp_p);  // Eq. (2.2) bases instead of a8
    else id_sweep(h);                         // a8
    mark(6);
    fill_coupling(h, o.storage, o.mem_budget_bytes, nf);  // a9
    if (serial) fill_nearfield_begin(h, h->stream, o.storage, o.mem_budget_bytes, nf);
    fill_nearfield_join(h, nf);
    mark(7);
    H2_CUDA_TRY(cudaEventRecord(join_ev, h->stream));
    H2_CUDA_TRY(cudaStreamWaitEvent(user, join_ev, 0));
    h->gpu_launches += (int)(prim_launches() - prims0);
    h->stream = user;
    for (auto& a : h->aux) a = nullptr;
    H2_CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (!base) {
      h->hidr_up_evals = (int64_t)stats[kStatHidrUp];
      h->hidr_dist_evals = (int64_t)(stats[kStatHidrUp] + stats[kStatHidrDown]);
      h->hidr_dist_done = (int64_t)stats[kStatHidrDone];
    }
    if (!interp) {
      h->kmax = (int)stats[kStatKmax];
      h->id_kernel_evals = (int64_t)(stats[kStatIdEvals] + stats[kStatIdEvalsCol]);
      h->kmax_col = h->nonsym ? (int)stats[kStatKmaxCol] : h->kmax;
    }
    if (h->timing) {
      nf.finish_timing(h);
      for (int i = 0; i < 6; i++) cudaEventElapsedTime(&h->stage_ms[i], ev[i], ev[i + 1]);
      cudaEventElapsedTime(&h->stage_ms[8], ev[0], ev[7]);
    }
  } catch (const Error& e) {
    set_error(e.code, e.msg);
    comm_abort(o.comm);  // LOCAL transport: release the other ranks' barriers
    cudaGetLastError();
    cudaDeviceSynchronize();  // the internal streams may still use the handle's buffers
    cudaGetLastError();
    h->stream = user;
    for (int i = 0; i < nev; i++) cudaEventDestroy(ev[i]);
    if (fork_ev) cudaEventDestroy(fork_ev);
    if (join_ev) cudaEventDestroy(join_ev);
    free_handle(h);
    return nullptr;
  } catch (const std::exception& e) {
    set_error(H2_ERR_INTERNAL, e.what());
    comm_abort(o.comm);
    cudaDeviceSynchronize();
    cudaGetLastError();
    h->stream = user;
    for (int i = 0; i < nev; i++) cudaEventDestroy(ev[i]);
    if (fork_ev) cudaEventDestroy(fork_ev);
    if (join_ev) cudaEventDestroy(join_ev);
    free_handle(h);
    return nullptr;
  }
  cudaEventDestroy(fork_ev);
  cudaEventDestroy(join_ev);
  for (int i = 0; i < nev; i++) cudaEventDestroy(ev[i]);
  return h;
}

h2_handle* h2_build_ex(const double* points, int64_t n, int32_t d, int32_t kernel_id, const double* kernel_params,
                       double id_tol, int32_t leaf_size, double admissibility, const h2_options* opt) {
  return build_impl(points, n, d, kernel_id, kernel_params, id_tol, leaf_size, admissibility, opt, nullptr);
}

h2_handle* h2_rebuild_ex(const h2_handle* base, int32_t kernel_id, const double* kernel_params, double id_tol,
                         const h2_options* opt) {
  clear_error();
  if (!base || !base->xs || !base->ys) {
    set_error(H2_ERR_INVALID_ARG, "h2_rebuild_ex: null base handle");
    return nullptr;
  }
  h2_options o;
  h2_options_default(&o);
  if (opt) o = *opt;
  if (o.comm != base->comm) {
    set_error(H2_ERR_INVALID_ARG, "h2_rebuild_ex: opt->comm must be the base handle's comm");
    return nullptr;
  }
  o.r_override = 0;  // the base's r and representor sets are reused
  return build_impl(nullptr, base->n, base->d, kernel_id, kernel_params, id_tol, base->q, base->tau, &o, base);
}

h2_handle* h2_build(const double* points, int64_t n, int32_t d, int32_t kernel_id, const double* kernel_params,
                    double id_tol, int32_t leaf_size, double admissibility) {
  return h2_build_ex(points, n, d, kernel_id, kernel_params, id_tol, leaf_size, admissibility, nullptr);
}

int h2_matvec(const h2_handle* h, const double* x, double* y) {
  clear_error();
  if (!h || !x || !y || x == y) {
    set_error(H2_ERR_INVALID_ARG, "h2_matvec: null handle/pointer or aliasing x, y");
    return H2_ERR_INVALID_ARG;
  }
  try {
    matvec(h, x, y);
  } catch (const Error& e) {
    set_error(e.code, e.msg);
    comm_abort(h->comm);
    cudaGetLastError();
    return e.code;
  } catch (const std::exception& e) {
    set_error(H2_ERR_INTERNAL, e.what());
    comm_abort(h->comm);
    cudaGetLastError();
    return H2_ERR_INTERNAL;
  }
  return H2_OK;
}

int h2_matvec_ex(const h2_handle* h, const double* x, double* y, int64_t n) {
  clear_error();
  if (h && n != h->n) {
    set_error(H2_ERR_DIM_MISMATCH, "h2_matvec_ex: vector length " + std::to_string(n) + " != n = " +
                                       std::to_string(h->n));
    return H2_ERR_DIM_MISMATCH;
  }
  return h2_matvec(h, x, y);
}

void h2_free(h2_handle* h) { free_handle(h); }

int h2_info(const h2_handle* h, h2_info_t* out) {
  clear_error();
  if (!h || !out) {
    set_error(H2_ERR_INVALID_ARG, "h2_info: null argument");
    return H2_ERR_INVALID_ARG;
  }
  std::memset(out, 0, sizeof(*out));
  out->n = h->n;
  out->d = h->d;
  out->depth = h->depth;
  out->r = h->r;
  out->nnodes = h->nnodes;
  out->nleaves = h->nleaves;
  out->csp = h->csp;
  out->n_il = h->n_il;
  out->n_nf = h->n_nf;
  out->coupling_entries = h->cp_entries;
  out->nearfield_entries = h->np_entries;
  out->stored_bytes = 8 * ((h->cp_stored ? h->cp_entries : 0) + (h->np_stored ? h->np_entries : 0));
  out->coupling_stored = h->cp_stored;
  out->nearfield_stored = h->np_stored;
  out->hidr_dist_evals = h->hidr_dist_evals;
  out->hidr_dist_done = h->hidr_dist_done;
  out->hidr_up_evals = h->hidr_up_evals;
  out->nonsymmetric = h->nonsym;
  out->kmax_col = h->kmax_col;
  out->srrqr_swaps = h->srrqr_swaps;
  out->id_kernel_evals = h->id_kernel_evals;
  out->kmax = h->kmax;
  out->gpu_launches = h->gpu_launches;
  std::memcpy(out->stage_ms, h->stage_ms, sizeof(out->stage_ms));
  return H2_OK;
}

static std::vector<char> export_bytes(const h2_handle* h, int what) {
  cudaStream_t s = h->stream;
  const int nn = h->nnodes, n = h->n, d = h->d, r = h->r;
  auto bytes = [](const void* p, size_t b) {
    std::vector<char> v(b);
    std::memcpy(v.data(), p, b);
    return v;
  };
  auto pack_slots = [&](const int* cnt_d, const int* slots_d, bool offsets) {
    auto cnt = d2h(cnt_d, nn, s);
    std::vector<int64_t> off(nn + 1, 0);
    for (int i = 0; i < nn; i++) off[i + 1] = off[i] + cnt[i];
    if (offsets) return bytes(off.data(), sizeof(int64_t) * (nn + 1));
    auto sl = d2h(slots_d, (size_t)nn * r, s);
    std::vector<int> out(off[nn]);
    for (int i = 0; i < nn; i++)
      for (int a = 0; a < cnt[i]; a++) out[off[i] + a] = sl[(size_t)i * r + a];
    return bytes(out.data(), sizeof(int) * out.size());
  };
  switch (what) {
    case H2_EXPORT_PERM: {
      auto v = d2h(h->perm, n, s);
      return bytes(v.data(), 4ull * n);
    }
    case H2_EXPORT_NODES: {
      const int* arrs[7] = {h->level, h->nbegin, h->nend, h->parent, h->first_child, h->nchild, h->is_leaf};
      std::vector<int> out((size_t)nn * 7);
      for (int a = 0; a < 7; a++) {
        auto v = d2h(arrs[a], nn, s);
        for (int i = 0; i < nn; i++) out[(size_t)i * 7 + a] = v[i];
      }
      return bytes(out.data(), 4 * out.size());
    }
    case H2_EXPORT_IL_OFF:
    case H2_EXPORT_NF_OFF: {
      auto v = d2h(what == H2_EXPORT_IL_OFF ? h->il_off : h->nf_off, nn + 1, s);
      return bytes(v.data(), 8 * v.size());
    }
    case H2_EXPORT_IL_IDX:
    case H2_EXPORT_NF_IDX: {
      int64_t m = what == H2_EXPORT_IL_IDX ? h->n_il : h->n_nf;
      auto v = d2h(what == H2_EXPORT_IL_IDX ? h->il_idx : h->nf_idx, m, s);
      return bytes(v.data(), 4 * v.size());
    }
    case H2_EXPORT_XS_OFF:
    case H2_EXPORT_XS_IDX:
      if (!h->xs) break;
      return pack_slots(h->xs_cnt, h->xs, what == H2_EXPORT_XS_OFF);
    case H2_EXPORT_YS_OFF:
    case H2_EXPORT_YS_IDX:
      if (!h->ys) break;
      return pack_slots(h->ys_cnt, h->ys, what == H2_EXPORT_YS_OFF);
    case H2_EXPORT_SK_OFF:
    case H2_EXPORT_SK_IDX:
      if (!h->k) break;
      return pack_slots(h->k, h->sk, what == H2_EXPORT_SK_OFF);
    case H2_EXPORT_K:
    case H2_EXPORT_XBAR_N: {
      if (!h->k) break;
      auto v = d2h(what == H2_EXPORT_K ? h->k : h->xbar_n, nn, s);
      return bytes(v.data(), 4 * v.size());
    }
    case H2_EXPORT_K_COL:
    case H2_EXPORT_XBARC_N: {
      if (!h->k_col) break;
      auto v = d2h(what == H2_EXPORT_K_COL ? h->k_col : h->xbar_col_n, nn, s);
      return bytes(v.data(), 4 * v.size());
    }
    case H2_EXPORT_SKC_OFF:
    case H2_EXPORT_SKC_IDX:
      if (!h->k_col) break;
      return pack_slots(h->k_col, h->sk_col, what == H2_EXPORT_SKC_OFF);
    case H2_EXPORT_U_OFF:
    case H2_EXPORT_U:
    case H2_EXPORT_V_OFF:
    case H2_EXPORT_V: {
      const bool col = what == H2_EXPORT_V_OFF || what == H2_EXPORT_V;
      if (!h->k || (col && !h->k_col)) break;
      auto k = d2h(col ? h->k_col : h->k, nn, s);
      auto xb = d2h(col ? h->xbar_col_n : h->xbar_n, nn, s);
      std::vector<int64_t> off(nn + 1, 0);
      for (int i = 0; i < nn; i++) off[i + 1] = off[i] + (int64_t)k[i] * xb[i];
      if (what == H2_EXPORT_U_OFF || what == H2_EXPORT_V_OFF) return bytes(off.data(), 8 * off.size());
      auto uo = d2h(col ? h->u_off_col : h->u_off, nn + 1, s);
      auto U = d2h(col ? h->V : h->U, col ? h->v_total : h->u_total, s);
      std::vector<double> out(off[nn]);
      for (int i = 0; i < nn; i++)
        if (off[i + 1] > off[i]) std::memcpy(&out[off[i]], &U[uo[i]], 8 * (off[i + 1] - off[i]));
      return bytes(out.data(), 8 * out.size());
    }
    case H2_EXPORT_ID_PATH: {
      if (!h->id_path) break;
      auto v = d2h(h->id_path, nn, s);
      return bytes(v.data(), 4 * v.size());
    }
    case H2_EXPORT_SHARD: {
      std::vector<int64_t> v = {h->nranks, h->rank, h->cut, h->p_lo, h->p_hi};
      for (int l = 0; l <= h->depth; l++) {
        const LevelRange lr = level_range(h, l);
        v.push_back(lr.begin);
        v.push_back(lr.end);
      }
      return bytes(v.data(), 8 * v.size());
    }
    case H2_EXPORT_INTERP_Q: {
      if (!h->Xq) break;
      auto v = d2h(h->Xq, (size_t)h->nq * d, s);
      std::vector<double> out((size_t)h->nq * d);
      for (int64_t t = 0; t < h->nq; t++)
        for (int c = 0; c < d; c++) out[(size_t)t * d + c] = v[(size_t)c * h->nq + t];
      return bytes(out.data(), 8 * out.size());
    }
    case H2_EXPORT_TREE_X: {
      auto v = d2h(h->X, (size_t)n * d, s);
      std::vector<double> out((size_t)n * d);
      for (int t = 0; t < n; t++)
        for (int c = 0; c < d; c++) out[(size_t)t * d + c] = v[(size_t)c * n + t];
      return bytes(out.data(), 8 * out.size());
    }
    default:
      break;
  }
  throw Error{H2_ERR_INVALID_ARG, "unknown export id or stage not built"};
}

int h2_export(const h2_handle* h, int what, void* host_buf, size_t cap_bytes, size_t* needed_bytes) {
  clear_error();
  if (!h) {
    set_error(H2_ERR_INVALID_ARG, "h2_export: null handle");
    return H2_ERR_INVALID_ARG;
  }
  try {
    auto v = export_bytes(h, what);
    if (needed_bytes) *needed_bytes = v.size();
    if (!host_buf || cap_bytes < v.size()) {
      set_error(H2_ERR_INVALID_ARG, "h2_export: buffer too small");
      return H2_ERR_INVALID_ARG;
    }
    if (!v.empty()) std::memcpy(host_buf, v.data(), v.size());
  } catch (const Error& e) {
    set_error(e.code, e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(H2_ERR_INTERNAL, e.what());
    return H2_ERR_INTERNAL;
  }
  return H2_OK;
}

int h2_sample_blocks(const h2_handle* h, int64_t count, const int32_t* kind, const int64_t* pair,
                     const int64_t* entry, double* value, int32_t* row_pt, int32_t* col_pt) {
  clear_error();
  if (!h || count < 0 || (count > 0 && (!kind || !pair || !entry || !value || !row_pt || !col_pt))) {
    set_error(H2_ERR_INVALID_ARG, "h2_sample_blocks: invalid argument");
    return H2_ERR_INVALID_ARG;
  }
  if (count == 0) return H2_OK;
  try {
    sample_blocks(h, count, kind, pair, entry, value, row_pt, col_pt);
  } catch (const Error& e) {
    set_error(e.code, e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(H2_ERR_INTERNAL, e.what());
    return H2_ERR_INTERNAL;
  }
  return H2_OK;
}

}  // extern "C"
