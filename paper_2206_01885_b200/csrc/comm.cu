// comm.cu -- the exchange layer of the sharded build (BASELINE north_star: "each
// level's skeleton indices and representors are exchanged with NCCL allgather over NVLink").
//
// Two transports behind one internal interface (allgather of fixed-size per-rank slots, and a
// float64 sum-allreduce used only by the sharded matvec):
//   * NCCL  -- one process per GPU; ncclAllGather / ncclAllReduce enqueued on the build's stream
//              (NVLink 5 / NVSwitch inside a box).  libnccl is resolved at run time (dlopen of the
//              copy PyTorch already loaded, or $H2_NCCL_LIB), so the library has no link-time NCCL
//              dependency.
//   * LOCAL -- R virtual ranks that are host threads of ONE process (tests on a single GPU): the
//              exchange is a host barrier + device-to-device copies, after each rank's stream has
//              been synchronised.  No kernel ever waits on another rank's kernel.
#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>

#include "h2_internal.cuh"

// ---- NCCL entry points (resolved with dlsym; signatures of nccl.h, NCCL 2.x) -----------------
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { kNcclUint8 = 1, kNcclFloat64 = 8, kNcclSum = 0 };

struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("H2_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      if (!nm || !*nm) continue;
      api.so = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.so) break;
    }
    if (!api.so) return;
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.so, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(api.so, "ncclCommInitRank"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(api.so, "ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(api.so, "ncclAllReduce"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.so, "ncclCommDestroy"));
    api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(dlsym(api.so, "ncclCommAbort"));
    api.CommGetAsyncError =
        reinterpret_cast<decltype(api.CommGetAsyncError)>(dlsym(api.so, "ncclCommGetAsyncError"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.so, "ncclGetErrorString"));
  });
  if (!api.so || !api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.AllReduce || !api.CommDestroy)
    throw h2::Error{H2_ERR_NCCL, "libnccl not found (import torch first, or set H2_NCCL_LIB)"};
  return api;
}

#define H2_NCCL_TRY(expr)                                                                              \
  do {                                                                                                 \
    ncclResult_t _r = (expr);                                                                          \
    if (_r != 0)                                                                                       \
      throw ::h2::Error{H2_ERR_NCCL, std::string(#expr) + ": " +                                       \
                                         (nccl().GetErrorString ? nccl().GetErrorString(_r) : "error")}; \
  } while (0)

namespace h2 {

// ---- LOCAL groups: R host threads of one process -----------------------------------------------
struct LocalGroup {
  int nranks = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long generation = 0;
  bool aborted = false;
  std::vector<const void*> send;
  int members = 0;  // live h2_comm objects of the group
};

static std::mutex g_groups_mu;
static std::map<long long, std::shared_ptr<LocalGroup>> g_groups;

}  // namespace h2

struct h2_comm {
  int kind = 0;  // 1 NCCL, 2 LOCAL
  int nranks = 1, rank = 0;
  ncclComm_t nc = nullptr;
  bool aborted = false;  // NCCL: aborted after a failure on this rank; every later call fails
  std::shared_ptr<h2::LocalGroup> group;
  long long key = 0;
};

namespace h2 {

constexpr double kLocalTimeoutSec = 300.0;

// all ranks of the group reach this point (or the call throws on abort / timeout)
static void local_barrier(LocalGroup& g) {
  std::unique_lock<std::mutex> lk(g.mu);
  if (g.aborted) throw Error{H2_ERR_NCCL, "local comm: group aborted by another rank"};
  const unsigned long long gen = g.generation;
  if (++g.arrived == g.nranks) {
    g.arrived = 0;
    g.generation++;
    g.cv.notify_all();
    return;
  }
  const bool ok = g.cv.wait_for(lk, std::chrono::duration<double>(kLocalTimeoutSec),
                                [&] { return g.generation != gen || g.aborted; });
  if (g.aborted || !ok) {
    g.aborted = true;
    g.cv.notify_all();
    throw Error{H2_ERR_NCCL, ok ? "local comm: group aborted by another rank" : "local comm: barrier timeout"};
  }
}

// A rank that fails between collectives would leave its peers blocked inside NCCL kernels: abort
// the communicator (ncclCommAbort makes the peers' pending and later collectives return errors)
// and mark the comm unusable.  LOCAL: release the other threads' barriers.
void comm_abort(h2_comm* c) {
  if (!c) return;
  if (c->kind == 1) {
    if (c->aborted) return;
    c->aborted = true;
    if (c->nc) {
      try {
        NcclApi& api = nccl();
        if (api.CommAbort) api.CommAbort(c->nc);
      } catch (...) {
      }
      c->nc = nullptr;
    }
    return;
  }
  if (c->kind != 2) return;
  std::lock_guard<std::mutex> lk(c->group->mu);
  c->group->aborted = true;
  c->group->cv.notify_all();
}

static void nccl_usable(const h2_comm* c) {
  if (c->aborted || !c->nc) throw Error{H2_ERR_NCCL, "NCCL comm was aborted after an earlier failure"};
}

// Waits for stream s after NCCL collectives were enqueued on it: polls the stream and the
// communicator's asynchronous error, and gives up after $H2_NCCL_TIMEOUT_S seconds (default 300),
// instead of a bare cudaStreamSynchronize that would hang forever when a peer has died.
void comm_sync(h2_comm* c, cudaStream_t s) {
  if (!c || c->kind != 1) {
    H2_CUDA_TRY(cudaStreamSynchronize(s));
    return;
  }
  static const double limit = [] {
    const char* e = getenv("H2_NCCL_TIMEOUT_S");
    return e ? atof(e) : 300.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) H2_CUDA_TRY(q);
    NcclApi& api = nccl();
    if (api.CommGetAsyncError && c->nc) {
      ncclResult_t ae = 0;
      if (api.CommGetAsyncError(c->nc, &ae) == 0 && ae != 0 && ae != 7 /* ncclInProgress */)
        throw Error{H2_ERR_NCCL, std::string("NCCL asynchronous error: ") +
                                     (api.GetErrorString ? api.GetErrorString(ae) : "error")};
    }
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit)
      throw Error{H2_ERR_NCCL, "NCCL collective did not complete within H2_NCCL_TIMEOUT_S"};
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

__global__ void sum_ranks_kernel(int nranks, int64_t count, const double* __restrict__ all, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nranks; q++) s += all[(int64_t)q * count + t];  // rank order: identical on every rank
    out[t] = s;
  }
}

// recv[q * bytes ... (q+1) * bytes) = rank q's send buffer, for every rank q (DEVICE buffers)
void comm_allgather(h2_comm* c, const void* send, void* recv, size_t bytes, cudaStream_t s) {
  if (c->kind == 1) {
    nccl_usable(c);
    H2_NCCL_TRY(nccl().AllGather(send, recv, bytes, kNcclUint8, c->nc, s));
    return;
  }
  LocalGroup& g = *c->group;
  H2_CUDA_TRY(cudaStreamSynchronize(s));
  {
    std::lock_guard<std::mutex> lk(g.mu);
    g.send[c->rank] = send;
  }
  local_barrier(g);
  for (int q = 0; q < c->nranks; q++)
    if (bytes)
      H2_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(recv) + (size_t)q * bytes, g.send[q], bytes,
                                  cudaMemcpyDeviceToDevice, s));
  H2_CUDA_TRY(cudaStreamSynchronize(s));
  local_barrier(g);  // nobody reuses its send buffer before every rank has copied it
}

// out[t] = sum over ranks of in[t] (DEVICE, fp64); the LOCAL transport sums in rank order
void comm_allreduce_sum(h2_comm* c, const double* in, double* out, int64_t count, cudaStream_t s) {
  if (c->kind == 1) {
    nccl_usable(c);
    H2_NCCL_TRY(nccl().AllReduce(in, out, (size_t)count, kNcclFloat64, kNcclSum, c->nc, s));
    return;
  }
  Scratch all(sizeof(double) * (size_t)count * c->nranks, s);
  comm_allgather(c, in, all.p, sizeof(double) * (size_t)count, s);
  sum_ranks_kernel<<<grid_for(count, 256), 256, 0, s>>>(c->nranks, count, all.as<double>(), out);
  H2_CHECK_LAUNCH();
}

}  // namespace h2

using namespace h2;

extern "C" {

int h2_comm_nccl_unique_id(unsigned char id[128]) {
  clear_error();
  if (!id) {
    set_error(H2_ERR_INVALID_ARG, "h2_comm_nccl_unique_id: null id");
    return H2_ERR_INVALID_ARG;
  }
  try {
    ncclUniqueId u;
    H2_NCCL_TRY(nccl().GetUniqueId(&u));
    std::memcpy(id, u.internal, 128);
  } catch (const Error& e) {
    set_error(e.code, e.msg);
    return e.code;
  }
  return H2_OK;
}

h2_comm* h2_comm_init_nccl(int32_t nranks, int32_t rank, const unsigned char id[128]) {
  clear_error();
  if (nranks < 1 || rank < 0 || rank >= nranks || !id) {
    set_error(H2_ERR_INVALID_ARG, "h2_comm_init_nccl: need 0 <= rank < nranks and an id");
    return nullptr;
  }
  try {
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    ncclComm_t nc = nullptr;
    H2_NCCL_TRY(nccl().CommInitRank(&nc, nranks, u, rank));
    h2_comm* c = new h2_comm();
    c->kind = 1;
    c->nranks = nranks;
    c->rank = rank;
    c->nc = nc;
    return c;
  } catch (const Error& e) {
    set_error(e.code, e.msg);
    return nullptr;
  }
}

h2_comm* h2_comm_init_nccl_dev(int32_t nranks, int32_t rank, const unsigned char id[128], int32_t device) {
  clear_error();
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    set_error(H2_ERR_INVALID_ARG, "h2_comm_init_nccl_dev: no such CUDA device");
    return nullptr;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    set_error(H2_ERR_CUDA, "h2_comm_init_nccl_dev: cudaSetDevice failed");
    return nullptr;
  }
  return h2_comm_init_nccl(nranks, rank, id);
}

h2_comm* h2_comm_init_local(int32_t nranks, int32_t rank, int64_t group_key) {
  clear_error();
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    set_error(H2_ERR_INVALID_ARG, "h2_comm_init_local: need 0 <= rank < nranks");
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_groups_mu);
  auto& gp = g_groups[group_key];
  if (!gp) {
    gp = std::make_shared<LocalGroup>();
    gp->nranks = nranks;
    gp->send.assign(nranks, nullptr);
  }
  if (gp->nranks != nranks) {
    set_error(H2_ERR_INVALID_ARG, "h2_comm_init_local: nranks differs from the group's");
    return nullptr;
  }
  gp->members++;
  h2_comm* c = new h2_comm();
  c->kind = 2;
  c->nranks = nranks;
  c->rank = rank;
  c->group = gp;
  c->key = group_key;
  return c;
}

void h2_comm_free(h2_comm* c) {
  if (!c) return;
  if (c->kind == 1 && c->nc && !c->aborted) {
    try {
      nccl().CommDestroy(c->nc);
    } catch (...) {
    }
  }
  if (c->kind == 2) {
    std::lock_guard<std::mutex> lk(g_groups_mu);
    if (--c->group->members == 0) g_groups.erase(c->key);
  }
  delete c;
}

int32_t h2_comm_size(const h2_comm* c) { return c ? c->nranks : 1; }
int32_t h2_comm_rank(const h2_comm* c) { return c ? c->rank : 0; }

}  // extern "C"
