// Library-owned collectives for sample sharding (include/cggm.h, "sample sharding"): an NCCL
// communicator loaded at run time, or caller-provided callbacks.  north_star: "each GPU holds row
// blocks of X and Y, and NCCL allreduce ... combines the partial X^T Y, X^T(X Theta) and R^T R
// sums.  The q x q Cholesky/inverse runs on one GPU and is then broadcast".
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

#include "common.cuh"

namespace cggm {
namespace {

// NCCL entry points, resolved from the libnccl.so.2 already in the process (torch's) or the
// system one: the library has no link-time NCCL dependency and loads without it.
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.CommGetAsyncError = reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(sym("ncclCommAbort"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.Broadcast &&
             api.GetErrorString && api.CommGetAsyncError && api.CommAbort;
    if (!api.ok) api.why = "libnccl.so.2 lacks an expected symbol";
  });
  return api;
}

[[noreturn]] void nccl_fail(const char* what, ncclResult_t r) {
  throw CudaError{CGGM_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r)};
}

ncclDataType_t nccl_type(int dtype) { return dtype == 1 ? ncclFloat32 : ncclFloat64; }

// A collective that never completes (a peer died, a hung rank) would otherwise block the caller's
// next synchronisation forever: after each NCCL call, wait for it on the host while polling the
// communicator's asynchronous error state, with a deadline (CGGM_NCCL_TIMEOUT_S, default 600 s;
// 0 disables the wait).  On an error or the deadline the communicator is aborted (so no later call
// can hang on it) and CGGM_ERR_NCCL is returned.
double nccl_timeout_s() {
  static double t = [] {
    const char* e = std::getenv("CGGM_NCCL_TIMEOUT_S");
    return e ? std::atof(e) : 600.0;
  }();
  return t;
}

void nccl_wait(Ctx* c, const char* what) {
  const double limit = nccl_timeout_s();
  if (limit <= 0) return;
  cudaEvent_t ev;
  CGGM_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CGGM_CUDA_CHECK(cudaEventRecord(ev, c->stream));
  const auto t0 = std::chrono::steady_clock::now();
  ncclComm_t comm = static_cast<ncclComm_t>(c->comm.nccl);
  for (;;) {
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) {
      cudaEventDestroy(ev);
      CGGM_CUDA_CHECK(q);
    }
    ncclResult_t ae = ncclSuccess;
    nccl().CommGetAsyncError(comm, &ae);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if ((ae != ncclSuccess && ae != ncclInProgress) || el > limit) {
      cudaEventDestroy(ev);
      nccl().CommAbort(comm);
      c->comm = CommState{};   // detached: the calls are single-rank again
      throw CudaError{CGGM_ERR_NCCL, std::string(what) + (ae != ncclSuccess && ae != ncclInProgress
                                                              ? std::string(": asynchronous error ") +
                                                                    nccl().GetErrorString(ae)
                                                              : ": not complete after " + std::to_string(limit) +
                                                                    " s (CGGM_NCCL_TIMEOUT_S); communicator aborted")};
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  cudaEventDestroy(ev);
}

}  // namespace

void comm_allreduce(Ctx* c, void* buf, int64_t count, int dtype) {
  if (!comm_attached(c) || count <= 0) return;
  if (c->comm.kind == 1) {
    const ncclResult_t r = nccl().AllReduce(buf, buf, (size_t)count, nccl_type(dtype), ncclSum,
                                            static_cast<ncclComm_t>(c->comm.nccl), c->stream);
    if (r != ncclSuccess) nccl_fail("ncclAllReduce", r);
    nccl_wait(c, "ncclAllReduce");
  } else {
    CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    if (c->comm.ar(c->comm.user, buf, count, dtype) != 0)
      throw CudaError{CGGM_ERR_NCCL, "external all-reduce callback failed"};
  }
}

void comm_bcast(Ctx* c, void* buf, int64_t count, int dtype, int root) {
  if (!comm_attached(c) || count <= 0) return;
  if (c->comm.kind == 1) {
    const ncclResult_t r = nccl().Broadcast(buf, buf, (size_t)count, nccl_type(dtype), root,
                                            static_cast<ncclComm_t>(c->comm.nccl), c->stream);
    if (r != ncclSuccess) nccl_fail("ncclBroadcast", r);
    nccl_wait(c, "ncclBroadcast");
  } else {
    CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    if (c->comm.bc(c->comm.user, buf, count, dtype, root) != 0)
      throw CudaError{CGGM_ERR_NCCL, "external broadcast callback failed"};
  }
}

void comm_unique_id(char id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  const NcclApi& api = nccl();
  if (!api.ok) throw CudaError{CGGM_ERR_NCCL, api.why};
  ncclUniqueId u;
  const ncclResult_t r = api.GetUniqueId(&u);
  if (r != ncclSuccess) nccl_fail("ncclGetUniqueId", r);
  std::memcpy(id, &u, 128);
}

void comm_init_nccl(Ctx* c, const char id[128], int rank, int world) {
  const NcclApi& api = nccl();
  if (!api.ok) throw CudaError{CGGM_ERR_NCCL, api.why};
  comm_release(c);
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t comm = nullptr;
  const ncclResult_t r = api.CommInitRank(&comm, world, u, rank);
  if (r != ncclSuccess) nccl_fail("ncclCommInitRank", r);
  c->comm.kind = 1;
  c->comm.rank = rank;
  c->comm.world = world;
  c->comm.nccl = comm;
}

void comm_release(Ctx* c) {
  if (c->comm.kind == 1 && c->comm.nccl) {
    cudaStreamSynchronize(c->stream);
    nccl().CommDestroy(static_cast<ncclComm_t>(c->comm.nccl));
  }
  c->comm = CommState{};
}

}  // namespace cggm
