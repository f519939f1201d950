// C-ABI of libcggm (include/cggm.h): argument validation, workspace, orchestration of the
// kernels for the five hot-path calls.  No torch types cross this boundary.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>

#include "kernels.cuh"
#include "../../include/cggm_testing.h"

struct cggm_ctx {
  cggm::Ctx impl;
};

namespace cggm {

void* ws_get(Ctx* c, int slot, size_t bytes) {
  if (c->slots.size() < WS_NUM) c->slots.resize(WS_NUM);
  Buffer& b = c->slots[slot];
  if (b.ptr && b.bytes >= bytes) return b.ptr;
  if (b.ptr) {
    CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    cudaFree(b.ptr);
    b.ptr = nullptr;
    b.bytes = 0;
  }
  size_t alloc = bytes < 256 ? 256 : bytes;
  alloc = (alloc + 4095) & ~size_t(4095);
  c->ws_generation++;   // invalidates captured graphs that hold workspace pointers
  cudaError_t e = cudaMalloc(&b.ptr, alloc);
  if (e != cudaSuccess) {
    cudaGetLastError();
    b.ptr = nullptr;
    throw CudaError{CGGM_ERR_OOM, "workspace allocation of " + std::to_string(alloc) + " bytes failed"};
  }
  b.bytes = alloc;
  return b.ptr;
}

namespace {

struct ArgError {
  cggm_status code;
  std::string msg;
};

[[noreturn]] void fail(cggm_status code, const std::string& msg) { throw CudaError{code, msg}; }

void check_ctx_dtype(Ctx* c) {
  if (c->dtype != CGGM_F64) fail(CGGM_ERR_UNSUPPORTED, "only CGGM_F64 is implemented in this build");
}

void check_dense(const char* name, const void* p, int64_t rows, int64_t cols, int64_t ld, bool required = true) {
  if (rows < 0 || cols < 0) fail(CGGM_ERR_INVALID_ARG, std::string(name) + ": negative dimension");
  if (!p) {
    if (required && rows > 0 && cols > 0) fail(CGGM_ERR_INVALID_ARG, std::string(name) + ": null pointer");
    return;
  }
  if (ld < (rows > 1 ? rows : 1)) fail(CGGM_ERR_INVALID_ARG, std::string(name) + ": leading dimension < rows");
}

void check_csc_host(const char* name, const cggm_csc* A, int64_t nrows, int64_t ncols) {
  if (!A) fail(CGGM_ERR_INVALID_ARG, std::string(name) + ": null cggm_csc");
  if (A->nrows != nrows || A->ncols != ncols)
    fail(CGGM_ERR_SHAPE, std::string(name) + ": shape " + std::to_string(A->nrows) + "x" + std::to_string(A->ncols) +
                             " expected " + std::to_string(nrows) + "x" + std::to_string(ncols));
  if (A->nnz < 0) fail(CGGM_ERR_INVALID_ARG, std::string(name) + ": negative nnz");
  if (A->ncols > 0 && !A->colptr) fail(CGGM_ERR_INVALID_ARG, std::string(name) + ": null colptr");
  if (A->nnz > 0 && (!A->rowidx || !A->val)) fail(CGGM_ERR_INVALID_ARG, std::string(name) + ": null rowidx/val");
  if (nrows > INT32_MAX) fail(CGGM_ERR_UNSUPPORTED, std::string(name) + ": more than 2^31 rows");
}

// device scalars block (WS_SCAL): [0] int fail_col, [1] int flag, doubles from byte 64
struct Scal {
  int* fail;
  int* flag;
  double* dbl;  // general doubles
};

Scal scal(Ctx* c, size_t ndoubles) {
  char* base = static_cast<char*>(ws_get(c, WS_SCAL, 64 + ndoubles * 8));
  return Scal{reinterpret_cast<int*>(base), reinterpret_cast<int*>(base + 4), reinterpret_cast<double*>(base + 64)};
}

void validate_csc_dev(Ctx* c, const cggm_csc* A, bool symmetric, const char* name) {
  if (c->validate < 1 || A->ncols == 0) return;
  Scal s = scal(c, 0);
  init_scalars(c, s.fail, s.flag);
  if (c->dtype == CGGM_F64) check_csc<double>(c, A, symmetric, s.flag);
  else check_csc<float>(c, A, symmetric, s.flag);
  int* h = static_cast<int*>(c->host_scratch);
  CGGM_CUDA_CHECK(cudaMemcpyAsync(h, s.flag, 4, cudaMemcpyDeviceToHost, c->stream));
  CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  if (h[0] & 3) fail(CGGM_ERR_BAD_SPARSE, std::string(name) + ": invalid CSC structure");
  if (h[0] & 4) fail(CGGM_ERR_NOT_SYMMETRIC, std::string(name) + ": not exactly symmetric");
}

inline int64_t even(int64_t x) { return x + (x & 1); }

// leading dimension padded to a 16-byte multiple (TMA global strides)
template <typename T>
inline int64_t pad_ld(int64_t x) {
  constexpr int64_t m = 16 / sizeof(T);
  return (x + m - 1) / m * m;
}

// run f(T{}) with T the ctx element type (CGGM_F64 -> double, CGGM_F32 -> float)
template <class F>
void dispatch(Ctx* c, F&& f) {
  if (c->dtype == CGGM_F64) f(double{});
  else f(float{});
}

template <class F>
cggm_status guard(cggm_ctx* ctx, F f) {
  if (!ctx) return CGGM_ERR_INVALID_ARG;
  Ctx* c = &ctx->impl;
  c->last_error.clear();
  try {
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) fail(CGGM_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    f(c);
    return CGGM_OK;
  } catch (const CudaError& e) {
    c->last_error = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    c->last_error = e.what();
    return CGGM_ERR_CUDA;
  }
}

// column indices of a block's S_Theta entries, local -> global (cggm_active_theta_block)
__global__ void k_col_offset(int32_t* col, const ActTotals* tot, long long cap, int32_t off) {
  const long long m = min((long long)tot->m_T, cap);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
    col[i] += off;
}
}  // namespace
}  // namespace cggm

using namespace cggm;
static_assert(CGGM_PROF_NTAGS == TAG_NUM, "profile tags out of sync");

extern "C" {

const char* cggm_version(void) { return "libcggm 0.1 (sm_100a, FP64 DMMA)"; }

cggm_status cggm_ctx_create(cggm_ctx** out, int device, cggm_dtype dtype, void* cuda_stream) {
  if (!out) return CGGM_ERR_INVALID_ARG;
  *out = nullptr;
  if (dtype != CGGM_F64 && dtype != CGGM_F32) return CGGM_ERR_INVALID_ARG;
  cudaDeviceProp prop;
  if (cudaSetDevice(device) != cudaSuccess || cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    cudaGetLastError();
    return CGGM_ERR_CUDA;
  }
  if (prop.major != 10) return CGGM_ERR_CUDA;  // built for sm_100a only
  cggm_ctx* ctx = new cggm_ctx();
  Ctx* c = &ctx->impl;
  c->device = device;
  c->dtype = dtype;
  c->stream = static_cast<cudaStream_t>(cuda_stream);
  c->num_sms = prop.multiProcessorCount;
  c->slots.resize(WS_NUM);
  if (const char* e = std::getenv("CGGM_PRIO")) c->prio_mode = std::atoi(e);
  if (const char* e = std::getenv("CGGM_LA_MIN")) c->la_min = std::atoi(e);
  if (const char* e = std::getenv("CGGM_K01")) c->k01 = std::atoi(e);
  if (const char* e = std::getenv("CGGM_PDL")) c->pdl = std::atoi(e);
  if (const char* e = std::getenv("CGGM_OBJ_GATE")) c->gate_cols = std::atoll(e);
  if (const char* e = std::getenv("CGGM_GL_OVERLAP")) c->gl_overlap = std::atoi(e);
  if (const char* e = std::getenv("CGGM_SIGMA_REC")) c->sig_min = std::atoi(e) > 0 ? std::max(128, std::atoi(e)) : 0;
  if (const char* e = std::getenv("CGGM_SIGMA_REC_F32"))
    c->sig_min_f32 = std::atoi(e) > 0 ? std::max(128, std::atoi(e)) : 0;
  if (const char* e = std::getenv("CGGM_NO_SMALL_ASYNC")) c->no_small_async = std::atoi(e);
  if (const char* e = std::getenv("CGGM_GRAPH")) c->use_graphs = std::atoi(e);
  if (const char* e = std::getenv("CGGM_SMALL_KMAX")) c->small_kmax = std::atoi(e);
  if (const char* e = std::getenv("CGGM_NO_ACTIVE_VEC")) c->no_active_vec = std::atoi(e);
  if (const char* e = std::getenv("CGGM_ACT_ONEPASS")) c->act_onepass = std::atoi(e);
  if (const char* e = std::getenv("CGGM_NO_SPLIT_K")) c->no_split_k = std::atoi(e);
  if (const char* e = std::getenv("CGGM_NO_VEC_EPI")) c->no_vec_epi = std::atoi(e);
  if (const char* e = std::getenv("CGGM_PERSIST_TPC")) c->persist_tpc = std::atoi(e);
  if (const char* e = std::getenv("CGGM_MID_TILE")) c->mid_tile = std::atoi(e);
  if (const char* e = std::getenv("CGGM_MID_MIN_WAVES")) c->mid_min_waves = std::atoi(e);
  if (const char* e = std::getenv("CGGM_LEAF_SWEEP")) c->leaf_sweep = std::atoi(e);
  if (const char* e = std::getenv("CGGM_CD_COOP")) c->cd_coop = std::atoi(e);
  if (const char* e = std::getenv("CGGM_CD_PREFETCH")) c->cd_prefetch = std::atoi(e);
  if (const char* e = std::getenv("CGGM_CD_BLOCK")) c->cd_block = std::atoi(e);
  if (const char* e = std::getenv("CGGM_CD_PANEL")) c->cd_panel = std::atoi(e);
  if (const char* e = std::getenv("CGGM_GRAPH_PROF")) c->graph_prof = std::atoi(e);
  if (const char* e = std::getenv("CGGM_TF32_CHUNK")) c->tf32_chunk = std::atoi(e);
  if (const char* e = std::getenv("CGGM_SYNC_CHECK")) c->sync_check = std::atoi(e);
  if (const char* e = std::getenv("CGGM_TF32_CFREL")) c->tf32_cfrel = std::atoi(e);
  if (const char* e = std::getenv("CGGM_TF32_TS_CHUNK")) c->tf32_ts_chunk = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("CGGM_TF32_MIN_TILES")) c->tf32_min_tiles = std::atoi(e);
  if (const char* e = std::getenv("CGGM_TF32_MIN_K")) c->tf32_min_k = std::atoi(e);
  if (const char* e = std::getenv("CGGM_TF32_PRODUCER"))
    c->tf32_producer = std::string(e) == "ldg" ? 1 : std::string(e) == "tma" ? 0 : 2;
  if (const char* e = std::getenv("CGGM_FUSE_GRADL")) c->fuse_gradl = std::atoi(e);
  if (const char* e = std::getenv("CGGM_TF32_DEBUG")) c->tf32_dbg = std::atoi(e);
  if (const char* e = std::getenv("CGGM_F32_ENGINE")) c->f32_engine = std::string(e) == "ffma" ? 1 : 0;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    delete ctx;
    return CGGM_ERR_CUDA;
  }
  c->encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  if (cudaMallocHost(&c->host_scratch, 4096) != cudaSuccess) {
    delete ctx;
    return CGGM_ERR_OOM;
  }
  *out = ctx;
  return CGGM_OK;
}

cggm_status cggm_ctx_destroy(cggm_ctx* ctx) {
  if (!ctx) return CGGM_ERR_INVALID_ARG;
  Ctx* c = &ctx->impl;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& b : c->slots)
    if (b.ptr) cudaFree(b.ptr);
  if (c->host_scratch) cudaFreeHost(c->host_scratch);
  if (c->aux) {
    cudaStreamSynchronize(c->aux);
    cudaStreamDestroy(c->aux);
    cudaEventDestroy(c->ev_fork);
    cudaEventDestroy(c->ev_join);
  }
  for (int l = 0; l < 2; ++l)
    for (cudaStream_t st : {c->la_chain[l], c->la_upd[l], c->la_bg[l]})
      if (st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
      }
  if (c->la_sig) {
    cudaStreamSynchronize(c->la_sig);
    cudaStreamDestroy(c->la_sig);
  }
  if (c->gate_ev) cudaEventDestroy(c->gate_ev);
  if (c->gl_side) {
    cudaStreamSynchronize(c->gl_side);
    cudaStreamDestroy(c->gl_side);
    cudaEventDestroy(c->ev_gl0);
    cudaEventDestroy(c->ev_gl1);
  }
  for (auto e : c->la_events) cudaEventDestroy(e);
  if (c->copy) {
    cudaStreamSynchronize(c->copy);
    cudaStreamDestroy(c->copy);
    cudaStreamSynchronize(c->syys);
    cudaStreamDestroy(c->syys);
    cudaEventDestroy(c->ev_h_lam);
    cudaEventDestroy(c->ev_h_xt);
    cudaEventDestroy(c->ev_h_y);
  }
  if (c->ev_w) cudaEventDestroy(c->ev_w);
  if (c->ev_syy) cudaEventDestroy(c->ev_syy);
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
  if (c->gorigin) {
    cudaStreamSynchronize(c->gorigin);
    cudaStreamDestroy(c->gorigin);
    cudaEventDestroy(c->ev_gpre);
    cudaEventDestroy(c->ev_gpost);
  }
  if (c->hi) {
    cudaStreamSynchronize(c->hi);
    cudaStreamDestroy(c->hi);
    cudaEventDestroy(c->ev_join_hi);
  }
  for (auto e : c->evpool) cudaEventDestroy(e);
  if (c->ts_buf) cudaFree(c->ts_buf);
  comm_release(c);
  delete ctx;
  return CGGM_OK;
}

cggm_status cggm_ctx_set_stream(cggm_ctx* ctx, void* s) {
  if (!ctx) return CGGM_ERR_INVALID_ARG;
  ctx->impl.stream = static_cast<cudaStream_t>(s);
  return CGGM_OK;
}

cggm_status cggm_ctx_set_option(cggm_ctx* ctx, int option, int64_t value) {
  if (!ctx) return CGGM_ERR_INVALID_ARG;
  Ctx* c = &ctx->impl;
  switch (option) {
    case CGGM_OPT_LOOKAHEAD_MIN:
      if (value < 0) return CGGM_ERR_INVALID_ARG;
      c->la_min = (int)std::min<int64_t>(value, 1 << 30);
      return CGGM_OK;
    case CGGM_OPT_GRAPHS:
      if (value != 0 && value != 1) return CGGM_ERR_INVALID_ARG;
      c->use_graphs = (int)value;
      return CGGM_OK;
    case CGGM_OPT_FACTOR_REUSE:
      if (value != 0 && value != 1) return CGGM_ERR_INVALID_ARG;
      c->factor_reuse = (int)value;
      c->reuse_valid = 0;
      return CGGM_OK;
    case CGGM_OPT_SIGMA_BLOCK:
      if (value != 0 && (value < 128 || value > (1 << 30))) return CGGM_ERR_INVALID_ARG;
      c->sig_min = c->sig_min_f32 = (int)value;
      return CGGM_OK;
    default:
      return CGGM_ERR_INVALID_ARG;
  }
}

cggm_status cggm_ctx_set_validate(cggm_ctx* ctx, int level) {
  if (!ctx || level < 0) return CGGM_ERR_INVALID_ARG;
  ctx->impl.validate = level;
  return CGGM_OK;
}

cggm_status cggm_ctx_launch_count(cggm_ctx* ctx, int64_t* count) {
  if (!ctx || !count) return CGGM_ERR_INVALID_ARG;
  *count = ctx->impl.launches;
  return CGGM_OK;
}

cggm_status cggm_ctx_release_workspace(cggm_ctx* ctx) {
  return guard(ctx, [&](Ctx* c) {
    CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    for (auto& b : c->slots) {
      if (b.ptr) cudaFree(b.ptr);
      b.ptr = nullptr;
      b.bytes = 0;
    }
  });
}

cggm_status cggm_ctx_profile(cggm_ctx* ctx, int enable) {
  if (!ctx) return CGGM_ERR_INVALID_ARG;
  Ctx* c = &ctx->impl;
  c->prof = enable != 0;
  if (c->prof) {
    c->prof_recs.clear();
    c->evnext = 0;
    const char* e = std::getenv("CGGM_PROF_TS");
    if (e && std::atoi(e) && !c->ts_buf) {
      c->ts_cap = 1 << 20;
      if (cudaMalloc(&c->ts_buf, c->ts_cap * 8) != cudaSuccess) {
        cudaGetLastError();
        c->ts_buf = nullptr;
        c->ts_cap = 0;
      }
    }
  }
  return CGGM_OK;
}

cggm_status cggm_ctx_profile_read(cggm_ctx* ctx, double* ms, int64_t* launches, int32_t ntags) {
  return guard(ctx, [&](Ctx* c) {
    if (!ms || !launches || ntags < CGGM_PROF_NTAGS) fail(CGGM_ERR_INVALID_ARG, "profile arrays too small");
    CGGM_CUDA_CHECK(cudaDeviceSynchronize());
    for (int t = 0; t < CGGM_PROF_NTAGS; ++t) {
      ms[t] = 0.0;
      launches[t] = 0;
    }
    std::vector<unsigned long long> ts;
    if (c->ts_buf) {
      ts.resize(c->evnext);
      CGGM_CUDA_CHECK(cudaMemcpy(ts.data(), c->ts_buf, c->evnext * 8, cudaMemcpyDeviceToHost));
    }
    for (const auto& r : c->prof_recs) {
      float e = 0.f;
      if (c->ts_buf) e = (float)((ts[r.b] - ts[r.a]) * 1e-6);
      else CGGM_CUDA_CHECK(cudaEventElapsedTime(&e, c->evpool[r.a], c->evpool[r.b]));
      ms[r.tag] += e;
      launches[r.tag] += 1;
    }
    c->prof_recs.clear();
    c->evnext = 0;
  });
}

const char* cggm_profile_tag_name(int32_t tag) {
  static const char* names[CGGM_PROF_NTAGS] = {"misc", "covariances", "densify", "chol_gemm", "chol_leaf",
                                               "lauum", "spmm", "w_sigma", "psi_gradL", "grad_theta",
                                               "obj_trsm", "active_set", "obj_reduce", "grad_lambda"};
  return (tag >= 0 && tag < CGGM_PROF_NTAGS) ? names[tag] : "?";
}

const char* cggm_last_error(cggm_ctx* ctx) { return ctx ? ctx->impl.last_error.c_str() : "null ctx"; }

}  // extern "C"  (the definitions below keep the C linkage declared in cggm.h)

// ------------------------------------------------------------------ a1
// ================================================================== sample sharding: communicator
cggm_status cggm_comm_unique_id(char id[128]) {
  if (!id) return CGGM_ERR_INVALID_ARG;
  try {
    comm_unique_id(id);
    return CGGM_OK;
  } catch (const CudaError& e) {
    return e.code;
  }
}

cggm_status cggm_comm_init(cggm_ctx* ctx, const char id[128], int32_t rank, int32_t world) {
  return guard(ctx, [&](Ctx* c) {
    if (!id) fail(CGGM_ERR_INVALID_ARG, "null unique id");
    if (world < 1 || rank < 0 || rank >= world) fail(CGGM_ERR_INVALID_ARG, "need 0 <= rank < world");
    comm_init_nccl(c, id, rank, world);
  });
}

cggm_status cggm_comm_init_external(cggm_ctx* ctx, int32_t rank, int32_t world, cggm_allreduce_fn allreduce,
                                    cggm_broadcast_fn broadcast, void* user) {
  return guard(ctx, [&](Ctx* c) {
    if (!allreduce || !broadcast) fail(CGGM_ERR_INVALID_ARG, "null collective callback");
    if (world < 1 || rank < 0 || rank >= world) fail(CGGM_ERR_INVALID_ARG, "need 0 <= rank < world");
    comm_release(c);
    c->comm.kind = 2;
    c->comm.rank = rank;
    c->comm.world = world;
    c->comm.ar = allreduce;
    c->comm.bc = broadcast;
    c->comm.user = user;
  });
}

cggm_status cggm_device_alloc(cggm_ctx* ctx, int64_t bytes, void** dev_ptr) {
  return guard(ctx, [&](Ctx* c) {
    if (!dev_ptr || bytes <= 0) fail(CGGM_ERR_INVALID_ARG, "need bytes > 0 and an output pointer");
    if (cudaMalloc(dev_ptr, (size_t)bytes) != cudaSuccess) {
      cudaGetLastError();
      *dev_ptr = nullptr;
      fail(CGGM_ERR_OOM, "cggm_device_alloc failed");
    }
    (void)c;
  });
}

cggm_status cggm_device_free(cggm_ctx* ctx, void* dev_ptr) {
  return guard(ctx, [&](Ctx* c) {
    if (dev_ptr) CGGM_CUDA_CHECK(cudaFree(dev_ptr));
    (void)c;
  });
}

cggm_status cggm_ipc_get_handle(cggm_ctx* ctx, const void* dev_ptr, char handle[64]) {
  return guard(ctx, [&](Ctx* c) {
    if (!dev_ptr || !handle) fail(CGGM_ERR_INVALID_ARG, "null pointer");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    cudaIpcMemHandle_t h;
    CGGM_CUDA_CHECK(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
    std::memcpy(handle, &h, 64);
    (void)c;
  });
}

cggm_status cggm_ipc_open_handle(cggm_ctx* ctx, const char handle[64], void** dev_ptr) {
  return guard(ctx, [&](Ctx* c) {
    if (!dev_ptr || !handle) fail(CGGM_ERR_INVALID_ARG, "null pointer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    CGGM_CUDA_CHECK(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    (void)c;
  });
}

cggm_status cggm_ipc_close_handle(cggm_ctx* ctx, void* dev_ptr) {
  return guard(ctx, [&](Ctx* c) {
    if (!dev_ptr) fail(CGGM_ERR_INVALID_ARG, "null pointer");
    CGGM_CUDA_CHECK(cudaIpcCloseMemHandle(dev_ptr));
    (void)c;
  });
}

cggm_status cggm_peer_allreduce(cggm_ctx* ctx, int32_t world, int32_t rank, void* const* bufs, int64_t count) {
  return guard(ctx, [&](Ctx* c) {
    if (world < 1 || world > 8 || rank < 0 || rank >= world) fail(CGGM_ERR_INVALID_ARG, "need 0 <= rank < world <= 8");
    if (count < 0) fail(CGGM_ERR_INVALID_ARG, "negative count");
    if (!bufs) fail(CGGM_ERR_INVALID_ARG, "null buffer array");
    for (int k = 0; k < world; ++k)
      if (!bufs[k] && count > 0) fail(CGGM_ERR_INVALID_ARG, "null peer buffer");
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      peer_allreduce<T>(c, world, rank, bufs, count);
    });
  });
}

cggm_status cggm_comm_destroy(cggm_ctx* ctx) {
  return guard(ctx, [&](Ctx* c) { comm_release(c); });
}

cggm_status cggm_comm_info(cggm_ctx* ctx, int32_t* rank, int32_t* world) {
  return guard(ctx, [&](Ctx* c) {
    if (!rank || !world) fail(CGGM_ERR_INVALID_ARG, "null output pointer");
    *rank = c->comm.rank;
    *world = c->comm.world;
  });
}

// ld-padded column-major matrix as one flat buffer for a collective (padding included)
static int64_t flat_count(int64_t rows, int64_t cols, int64_t ld) { return cols > 0 ? ld * (cols - 1) + rows : 0; }
static int dt_code(Ctx* c) { return c->dtype == CGGM_F32 ? 1 : 0; }

cggm_status cggm_covariances(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, int64_t q, const void* X,
                             int64_t ldx, const void* Y, int64_t ldy, void* Syy, int64_t ldsyy, void* Sxy,
                             int64_t ldsxy) {
  return guard(ctx, [&](Ctx* c) {
    if (n_local < 0 || p < 0 || q < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    if (n_total < 1 || n_total < n_local) fail(CGGM_ERR_INVALID_ARG, "n_total must be >= max(1, n_local)");
    check_dense("Y", Y, n_local, q, ldy);
    check_dense("Syy", Syy, q, q, ldsyy, false);
    if (Sxy) {
      check_dense("X", X, n_local, p, ldx);
      check_dense("Sxy", Sxy, p, q, ldsxy);
    }
    const double inv_n = 1.0 / (double)n_total;
    Phase ph(c, TAG_COV);
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      if (Syy) {
        EpilogueT<T> e; e.out1 = static_cast<T*>(Syy); e.ld1 = ldsyy; e.a1 = inv_n;
        gemm(c, true, false, q, q, n_local, static_cast<const T*>(Y), ldy, static_cast<const T*>(Y), ldy, e,
             SYM_LOWER | SYM_MIRROR);
      }
      if (Sxy) {
        EpilogueT<T> e; e.out1 = static_cast<T*>(Sxy); e.ld1 = ldsxy; e.a1 = inv_n;
        gemm(c, true, false, p, q, n_local, static_cast<const T*>(X), ldx, static_cast<const T*>(Y), ldy, e, 0);
      }
    });
    if (Syy) comm_allreduce(c, Syy, flat_count(q, q, ldsyy), dt_code(c));   // sum of the shards' partials
    if (Sxy) comm_allreduce(c, Sxy, flat_count(p, q, ldsxy), dt_code(c));
  });
}

// ================================================================== NEXT-1 / NEXT-2 (cd.cu)
cggm_status cggm_gram(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, const void* X, int64_t ldx,
                      void* Sxx, int64_t ldsxx) {
  return guard(ctx, [&](Ctx* c) {
    if (n_local < 0 || p < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    if (n_total < 1 || n_total < n_local) fail(CGGM_ERR_INVALID_ARG, "n_total must be >= max(1, n_local)");
    check_dense("X", X, n_local, p, ldx);
    check_dense("Sxx", Sxx, p, p, ldsxx);
    Phase ph(c, TAG_COV);
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      EpilogueT<T> e; e.out1 = static_cast<T*>(Sxx); e.ld1 = ldsxx; e.a1 = 1.0 / (double)n_total;
      gemm(c, true, false, p, p, n_local, static_cast<const T*>(X), ldx, static_cast<const T*>(X), ldx, e,
           SYM_LOWER | SYM_MIRROR);
    });
    comm_allreduce(c, Sxx, flat_count(p, p, ldsxx), dt_code(c));
  });
}

static void check_list(const char* name, const int32_t* r, const int32_t* cidx, int64_t m) {
  if (m < 0) fail(CGGM_ERR_INVALID_ARG, std::string(name) + ": negative list length");
  if (m > 0 && (!r || !cidx)) fail(CGGM_ERR_INVALID_ARG, std::string(name) + ": null list");
}

cggm_status cggm_lambda_direction(cggm_ctx* ctx, int64_t q, const void* Sigma, int64_t ldsigma, const void* Psi,
                                  int64_t ldpsi, const void* GradL, int64_t ldgl, const cggm_csc* Lambda,
                                  const int32_t* L_row, const int32_t* L_col, int64_t m_L, double lam_L,
                                  int penalize_diag, int passes, void* D, double* delta, double* l1_lambda) {
  return guard(ctx, [&](Ctx* c) {
    check_ctx_dtype(c);
    if (q < 1 || passes < 0) fail(CGGM_ERR_INVALID_ARG, "need q >= 1, passes >= 0");
    if (!(lam_L >= 0.0)) fail(CGGM_ERR_INVALID_ARG, "lam_L must be >= 0");
    check_dense("Sigma", Sigma, q, q, ldsigma);
    check_dense("Psi", Psi, q, q, ldpsi);
    check_dense("GradL", GradL, q, q, ldgl);
    check_csc_host("Lambda", Lambda, q, q);
    check_list("L", L_row, L_col, m_L);
    if (m_L > 0 && !D) fail(CGGM_ERR_INVALID_ARG, "null D");
    const int64_t ldu = pad_ld<double>(q);
    double* U = static_cast<double*>(ws_get(c, WS_CD_U, (size_t)ldu * q * 8));
    double* out = static_cast<double*>(ws_get(c, WS_CD_OUT, 64));
    // a fresh direction: D = 0 (zeroed by the kernel), so U = D Sigma = 0
    CGGM_CUDA_CHECK(cudaMemsetAsync(U, 0, (size_t)ldu * q * 8, c->stream));
    double* coef = static_cast<double*>(ws_get(c, WS_CD_COEF, (size_t)std::max<int64_t>(m_L, 1) * 4 * 8));
    if (coop_ok(c)) {
      double* Z = static_cast<double*>(ws_get(c, WS_CD_Z, (size_t)ldu * q * 8));
      CGGM_CUDA_CHECK(cudaMemsetAsync(Z, 0, (size_t)ldu * q * 8, c->stream));
      const size_t aux = (size_t)q * 4 + 2 * (size_t)(q + 1) * 8 + (size_t)std::max<int64_t>(m_L, 1) * 8 +
                         (size_t)2 * q * 8 + 4 * 64;
      char* w = static_cast<char*>(ws_get(c, WS_CD_AUX, aux));
      int* cnt = reinterpret_cast<int*>(w);
      int64_t* scr = reinterpret_cast<int64_t*>(w + ((size_t)q * 4 + 63) / 64 * 64);
      int64_t* lp = scr + (q + 1);
      double* dmu = reinterpret_cast<double*>(lp + (q + 1));
      double* colbuf = dmu + std::max<int64_t>(m_L, 1);
      lambda_cd_coop(c, (int)q, static_cast<const double*>(Sigma), ldsigma, static_cast<const double*>(Psi), ldpsi,
                     static_cast<const double*>(GradL), ldgl, Lambda, L_row, L_col, m_L, lam_L, penalize_diag, passes,
                     static_cast<double*>(D), U, Z, ldu, coef, cnt, scr, lp, dmu, colbuf, out);
    } else {
      lambda_cd(c, (int)q, static_cast<const double*>(Sigma), ldsigma, static_cast<const double*>(Psi), ldpsi,
                static_cast<const double*>(GradL), ldgl, Lambda, L_row, L_col, m_L, lam_L, penalize_diag, passes,
                static_cast<double*>(D), U, ldu, coef, out);
    }
    if (delta || l1_lambda) {
      double h[3];
      CGGM_CUDA_CHECK(cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
      CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
      if (delta) {
        delta[0] = h[0];
        delta[1] = h[1];
      }
      if (l1_lambda) *l1_lambda = h[2];
    }
  });
}

cggm_status cggm_lambda_step(cggm_ctx* ctx, int64_t q, const cggm_csc* Lambda, const int32_t* L_row,
                             const int32_t* L_col, int64_t m_L, const void* D, double alpha, cggm_csc* out) {
  return guard(ctx, [&](Ctx* c) {
    check_ctx_dtype(c);
    if (q < 1) fail(CGGM_ERR_INVALID_ARG, "need q >= 1");
    check_csc_host("Lambda", Lambda, q, q);
    check_list("L", L_row, L_col, m_L);
    if (!out || out->nrows != q || out->ncols != q || !out->colptr) fail(CGGM_ERR_INVALID_ARG, "bad out CSC");
    if (m_L > 0 && (!D || !out->rowidx || !out->val)) fail(CGGM_ERR_INVALID_ARG, "null D / out arrays");
    if (out->nnz < 2 * m_L) {
      out->nnz = 2 * m_L;
      fail(CGGM_ERR_CAPACITY, "out capacity < 2 m_L (required size written to out->nnz)");
    }
    int* cnt = static_cast<int*>(ws_get(c, WS_CD_IDX, (size_t)3 * q * 4 + (size_t)2 * (q + 1) * 8 + 64));
    int64_t* scan = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(cnt) + ((size_t)3 * q * 4 + 63) / 64 * 64);
    list_to_csc(c, (int)q, L_row, L_col, m_L, true, Lambda, static_cast<const double*>(D), alpha, nullptr,
                const_cast<int64_t*>(out->colptr), const_cast<int32_t*>(out->rowidx),
                static_cast<double*>(const_cast<void*>(out->val)), cnt, scan);
    int64_t nnz = 0;
    CGGM_CUDA_CHECK(cudaMemcpyAsync(&nnz, out->colptr + q, 8, cudaMemcpyDeviceToHost, c->stream));
    CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    out->nnz = nnz;
  });
}

// the Theta sweep on S_xx columns Sxx (p x ncx, ldsxx): the full matrix (xmap null) or the compact
// columns of the active rows (xmap device, p entries)
static void theta_cd_run(Ctx* c, int64_t p, int64_t q, const void* Sigma, int64_t ldsigma, const void* Sxx,
                         int64_t ldsxx, const int32_t* xmap, const void* Sxy, int64_t ldsxy, const cggm_csc* Theta,
                         const int32_t* T_row, const int32_t* T_col, int64_t m_T, double lam_T, int passes,
                         cggm_csc* out, double* l1_theta) {
    if (!out || out->nrows != p || out->ncols != q || !out->colptr) fail(CGGM_ERR_INVALID_ARG, "bad out CSC");
    if (m_T > 0 && (!out->rowidx || !out->val)) fail(CGGM_ERR_INVALID_ARG, "null out arrays");
    if (out->nnz < m_T) {
      out->nnz = m_T;
      fail(CGGM_ERR_CAPACITY, "out capacity < m_T (required size written to out->nnz)");
    }
    const int64_t ldv = pad_ld<double>(p);
    double* V = static_cast<double*>(ws_get(c, WS_CD_V, (size_t)ldv * q * 8));
    double* sc = static_cast<double*>(ws_get(c, WS_CD_OUT, 64));
    int* cnt = static_cast<int*>(ws_get(c, WS_CD_IDX, (size_t)3 * q * 4 + (size_t)2 * (q + 1) * 8 + 64));
    int64_t* scan = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(cnt) + ((size_t)3 * q * 4 + 63) / 64 * 64);
    double* T = static_cast<double*>(const_cast<void*>(out->val));   // the sweep runs on the output values
    double* coef = static_cast<double*>(ws_get(c, WS_CD_COEF, (size_t)std::max<int64_t>(m_T, 1) * 2 * 8));
    if (coop_ok(c)) {
      const int64_t ldvr = pad_ld<double>(q);   // row-major V: p rows of stride ldvr
      V = static_cast<double*>(ws_get(c, WS_CD_V, (size_t)ldvr * p * 8));
      CGGM_CUDA_CHECK(cudaMemsetAsync(V, 0, (size_t)ldvr * p * 8, c->stream));
      const size_t aux = (size_t)q * 4 + 2 * (size_t)(q + 1) * 8 + (size_t)std::max<int64_t>(m_T, 1) * 8 +
                         (size_t)p * 8 + 4 * 64;
      char* w = static_cast<char*>(ws_get(c, WS_CD_AUX, aux));
      int* cnt2 = reinterpret_cast<int*>(w);
      int64_t* scr = reinterpret_cast<int64_t*>(w + ((size_t)q * 4 + 63) / 64 * 64);
      int64_t* lp = scr + (q + 1);
      double* dmu = reinterpret_cast<double*>(lp + (q + 1));
      double* colbuf = dmu + std::max<int64_t>(m_T, 1);
      theta_cd_coop(c, (int)p, (int)q, static_cast<const double*>(Sigma), ldsigma, static_cast<const double*>(Sxx),
                    ldsxx, xmap, static_cast<const double*>(Sxy), ldsxy, Theta, T_row, T_col, m_T, lam_T, passes, T,
                    V, ldvr, coef, cnt2, scr, lp, dmu, colbuf, sc);
    } else {
      CGGM_CUDA_CHECK(cudaMemsetAsync(V, 0, (size_t)ldv * q * 8, c->stream));
      theta_sigma(c, (int)q, Theta, static_cast<const double*>(Sigma), ldsigma, V, ldv);
      theta_cd(c, (int)p, (int)q, static_cast<const double*>(Sigma), ldsigma, static_cast<const double*>(Sxx), ldsxx,
               xmap, static_cast<const double*>(Sxy), ldsxy, Theta, T_row, T_col, m_T, lam_T, passes, T, V, ldv, coef,
               sc);
    }
    list_to_csc(c, (int)q, T_row, T_col, m_T, false, nullptr, nullptr, 0.0, T, const_cast<int64_t*>(out->colptr),
                const_cast<int32_t*>(out->rowidx), T, cnt, scan);
    double h = 0.0;
    CGGM_CUDA_CHECK(cudaMemcpyAsync(&h, sc, 8, cudaMemcpyDeviceToHost, c->stream));
    CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    out->nnz = m_T;
    if (l1_theta) *l1_theta = h;
}

cggm_status cggm_theta_cd(cggm_ctx* ctx, int64_t p, int64_t q, const void* Sigma, int64_t ldsigma, const void* Sxx,
                          int64_t ldsxx, const void* Sxy, int64_t ldsxy, const cggm_csc* Theta, const int32_t* T_row,
                          const int32_t* T_col, int64_t m_T, double lam_T, int passes, cggm_csc* out,
                          double* l1_theta) {
  return guard(ctx, [&](Ctx* c) {
    check_ctx_dtype(c);
    if (q < 1 || p < 1 || passes < 0) fail(CGGM_ERR_INVALID_ARG, "need p, q >= 1, passes >= 0");
    if (!(lam_T >= 0.0)) fail(CGGM_ERR_INVALID_ARG, "lam_T must be >= 0");
    check_dense("Sigma", Sigma, q, q, ldsigma);
    check_dense("Sxx", Sxx, p, p, ldsxx);
    check_dense("Sxy", Sxy, p, q, ldsxy);
    check_csc_host("Theta", Theta, p, q);
    check_list("T", T_row, T_col, m_T);
    theta_cd_run(c, p, q, Sigma, ldsigma, Sxx, ldsxx, nullptr, Sxy, ldsxy, Theta, T_row, T_col, m_T, lam_T, passes,
                 out, l1_theta);
  });
}

cggm_status cggm_gram_rows(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, const void* X, int64_t ldx,
                           const int32_t* T_row, int64_t m_T, void* Sxx_cols, int64_t ldsxx, int64_t cap,
                           int32_t* xmap, int64_t* n_cols) {
  return guard(ctx, [&](Ctx* c) {
    check_ctx_dtype(c);
    if (n_local < 0 || p < 1 || m_T < 0 || cap < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    if (n_total < 1 || n_total < n_local) fail(CGGM_ERR_INVALID_ARG, "n_total must be >= max(1, n_local)");
    check_dense("X", X, n_local, p, ldx);
    if (m_T > 0 && !T_row) fail(CGGM_ERR_INVALID_ARG, "null T_row");
    if (!xmap || !n_cols) fail(CGGM_ERR_INVALID_ARG, "null xmap / n_cols");
    if (cap > 0) check_dense("Sxx_cols", Sxx_cols, p, cap, ldsxx);
    int32_t* rows = static_cast<int32_t*>(ws_get(c, WS_CD_IDX, (size_t)p * 4 + 64));
    long long* cnt = reinterpret_cast<long long*>(static_cast<char*>(ws_get(c, WS_CD_OUT, 64)) + 32);
    row_map(c, (int)p, T_row, m_T, xmap, rows, cnt);
    long long k = 0;
    CGGM_CUDA_CHECK(cudaMemcpyAsync(c->host_scratch, cnt, 8, cudaMemcpyDeviceToHost, c->stream));
    CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    std::memcpy(&k, c->host_scratch, 8);
    *n_cols = k;
    if (k > cap) fail(CGGM_ERR_CAPACITY, "more active rows than Sxx_cols columns (required count in n_cols)");
    if (k == 0) return;
    const int64_t ldg = pad_ld<double>(n_local > 0 ? n_local : 1);
    double* G = static_cast<double*>(ws_get(c, WS_CD_U, (size_t)ldg * k * 8));
    gather_cols(c, n_local, k, static_cast<const double*>(X), ldx, rows, G, ldg);
    Epilogue e; e.out1 = static_cast<double*>(Sxx_cols); e.ld1 = ldsxx; e.a1 = 1.0 / (double)n_total;
    gemm(c, true, false, p, k, n_local, static_cast<const double*>(X), ldx, G, ldg, e, 0);
    if (comm_attached(c)) comm_allreduce(c, Sxx_cols, (k - 1) * ldsxx + p, 0);
  });
}

cggm_status cggm_theta_cd_rows(cggm_ctx* ctx, int64_t p, int64_t q, const void* Sigma, int64_t ldsigma,
                               const void* Sxx_cols, int64_t ldsxx, const int32_t* xmap, int64_t n_cols,
                               const void* Sxy, int64_t ldsxy, const cggm_csc* Theta, const int32_t* T_row,
                               const int32_t* T_col, int64_t m_T, double lam_T, int passes, cggm_csc* out,
                               double* l1_theta) {
  return guard(ctx, [&](Ctx* c) {
    check_ctx_dtype(c);
    if (q < 1 || p < 1 || passes < 0 || n_cols < 0) fail(CGGM_ERR_INVALID_ARG, "need p, q >= 1, passes >= 0");
    if (!(lam_T >= 0.0)) fail(CGGM_ERR_INVALID_ARG, "lam_T must be >= 0");
    if (!xmap) fail(CGGM_ERR_INVALID_ARG, "null xmap");
    check_dense("Sigma", Sigma, q, q, ldsigma);
    if (n_cols > 0) check_dense("Sxx_cols", Sxx_cols, p, n_cols, ldsxx);
    check_dense("Sxy", Sxy, p, q, ldsxy);
    check_csc_host("Theta", Theta, p, q);
    check_list("T", T_row, T_col, m_T);
    theta_cd_run(c, p, q, Sigma, ldsigma, n_cols > 0 ? Sxx_cols : Sigma, n_cols > 0 ? ldsxx : ldsigma, xmap, Sxy,
                 ldsxy, Theta, T_row, T_col, m_T, lam_T, passes, out, l1_theta);
  });
}

int cggm::stream_priority(int which) {
  // which: 0 chain tail (Sigma product, W Sigma, Psi, grad_Theta), 1 objective origin, 2-4 inverse
  // recursion (critical chain, deferred updates, background products), 5-7 the objective's
  // recursion, 8 the Sigma blocks formed inside the inverse recursion, 9 the host-input S_yy.  The recursions' critical chains outrank the big throughput GEMMs, so
  // their latency-bound kernels start as soon as SMs free up (measured 429.7 -> 426.1 ms at large
  // against {0, 5, 0, 1, 2, 3, 4, 5}).
  static int off[10] = {4, 5, 1, 2, 3, 0, 4, 5, 3, 2};
  static bool init = false;
  if (!init) {
    if (const char* e = std::getenv("CGGM_PRIO_SCHEME")) {
      int k = 0;
      for (const char* q = e; *q && k < 10; ++k) {
        off[k] = std::atoi(q);
        while (*q && *q != ',') ++q;
        if (*q == ',') ++q;
      }
    }
    init = true;
  }
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  return std::min(least, greatest + off[which]);
}

// ================================================================== enqueue-only cores
// Each core only enqueues work on c->stream (no host synchronisation); results stay on the
// device in a per-lane scalar block until the matching readback.  Lanes (0 = caller's stream,
// 1 = auxiliary stream) own disjoint workspace slots so the composite call can overlap them.

struct Lane {
  int dense, scal, pack;  // workspace slots
};
static const Lane kLane[2] = {{WS_DENSE_A, WS_SCAL, WS_PACK0}, {WS_DENSE_B, WS_SCAL2, WS_PACK2}};

static Scal scal_lane(Ctx* c, int lane, size_t ndoubles) {
  char* base = static_cast<char*>(ws_get(c, kLane[lane].scal, 64 + ndoubles * 8));
  return Scal{reinterpret_cast<int*>(base), reinterpret_cast<int*>(base + 4), reinterpret_cast<double*>(base + 64)};
}

static int64_t n_leaves(int64_t q) { return (q + leaf_nb() - 1) / leaf_nb(); }

// ------------------------------------------------------------------ a3
// Scal layout: dbl[0] = logdet sum, dbl[8..] leaf slots
template <typename T>
static void invert_enqueue(Ctx* c, int lane, const cggm_csc* Lambda, T* Sigma, int64_t ldsigma,
                           int xslot = WS_LINV) {
  const int64_t q = Lambda->nrows;
  const int64_t lda = pad_ld<T>(q);
  const int nb = leaf_nb();
  const int64_t nleaves = n_leaves(q);
  T* A = static_cast<T*>(ws_get(c, kLane[lane].dense, (size_t)lda * q * sizeof(T)));
  Scal s = scal_lane(c, lane, 8 + nleaves);
  double* slots = s.dbl + 8;
  ViewT<T> Av{A, lda, q, q};
  densify_csc(c, Lambda, Av);
  init_scalars(c, s.fail, s.flag);
  if (Sigma) {
    T* X = static_cast<T*>(ws_get(c, xslot, (size_t)lda * q * sizeof(T)));
    CGGM_CUDA_CHECK(cudaMemsetAsync(X, 0, (size_t)lda * q * sizeof(T), c->stream));
    const size_t tmp_elems = chol_tmp_elems(q);
    T* tmp = static_cast<T*>(ws_get(c, WS_TMP, tmp_elems * sizeof(T)));
    const int smin = sizeof(T) == 8 ? c->sig_min : c->sig_min_f32;
    if (smin > 0 && q >= smin) {   // Sigma assembled inside the recursion
      potrf_recursive<T>(c, Av, ViewT<T>{X, lda, q, q}, true, nullptr, slots, s.fail, tmp, tmp_elems, nullptr, 0,
                         nullptr, 0, Sigma, ldsigma);
    } else {
      potrf_recursive<T>(c, Av, ViewT<T>{X, lda, q, q}, true, nullptr, slots, s.fail, tmp, tmp_elems);
      lauum<T>(c, ViewT<T>{X, lda, q, q}, ViewT<T>{Sigma, ldsigma, q, q});
    }
  } else {
    T* leafinv = static_cast<T*>(ws_get(c, WS_LEAFINV, (size_t)nleaves * nb * nb * sizeof(T)));
    potrf_recursive<T>(c, Av, ViewT<T>{nullptr, lda, q, q}, false, leafinv, slots, s.fail, nullptr, 0);
  }
  sum_arrays_1(c, slots, nleaves, s.dbl);
}

// factor reuse: Sigma from the kept L^{-1} (one symmetric product), the kept trial's (fail_col,
// log-det) into this lane's scalar block
template <typename T>
static void invert_from_kept(Ctx* c, int lane, int64_t q, T* Sigma, int64_t ldsigma, int xslot) {
  const int64_t lda = pad_ld<T>(q);
  T* X = static_cast<T*>(ws_get(c, xslot, (size_t)lda * q * sizeof(T)));
  Scal s = scal_lane(c, lane, 8 + n_leaves(q));
  const char* kept = static_cast<const char*>(ws_get(c, WS_REUSE_SCAL, 64 + 8));
  CGGM_CUDA_CHECK(cudaMemcpyAsync(s.fail, kept, 4, cudaMemcpyDeviceToDevice, c->stream));
  CGGM_CUDA_CHECK(cudaMemcpyAsync(s.dbl, kept + 64, 8, cudaMemcpyDeviceToDevice, c->stream));
  lauum<T>(c, ViewT<T>{X, lda, q, q}, ViewT<T>{Sigma, ldsigma, q, q});
}

// D2H of (fail_col, logdet) from a lane's scalar block; caller synchronises
static void chol_readback_async(Ctx* c, int lane, char* h) {
  Scal s = scal_lane(c, lane, 0);
  CGGM_CUDA_CHECK(cudaMemcpyAsync(h, s.fail, 4, cudaMemcpyDeviceToHost, c->stream));
  CGGM_CUDA_CHECK(cudaMemcpyAsync(h + 8, s.dbl, 8, cudaMemcpyDeviceToHost, c->stream));
}

static CholResult chol_decode(const char* h) {
  int fc;
  double ld;
  std::memcpy(&fc, h, 4);
  std::memcpy(&ld, h + 8, 8);
  CholResult r;
  r.is_pd = (fc == INT_MAX);
  r.fail_col = r.is_pd ? -1 : fc;
  r.logdet = r.is_pd ? ld : std::numeric_limits<double>::quiet_NaN();
  return r;
}

cggm_status cggm_invert_logdet(cggm_ctx* ctx, const cggm_csc* Lambda, void* Sigma, int64_t ldsigma, double* logdet,
                               int32_t* is_pd, int64_t* fail_col) {
  return guard(ctx, [&](Ctx* c) {
    if (!Lambda) fail(CGGM_ERR_INVALID_ARG, "Lambda is null");
    const int64_t q = Lambda->nrows;
    check_csc_host("Lambda", Lambda, q, q);
    check_dense("Sigma", Sigma, q, q, ldsigma, false);
    if (!logdet || !is_pd || !fail_col) fail(CGGM_ERR_INVALID_ARG, "null host output pointer");
    if (q == 0) {
      *logdet = 0.0; *is_pd = 1; *fail_col = -1;
      return;
    }
    validate_csc_dev(c, Lambda, true, "Lambda");
    char* h = static_cast<char*>(c->host_scratch);
    CholResult r{};
    if (c->comm.rank == 0) {   // with a communicator only rank 0 factors (north_star)
      dispatch(c, [&](auto tag) {
        using T = decltype(tag);
        invert_enqueue<T>(c, 0, Lambda, static_cast<T*>(Sigma), ldsigma);
      });
      chol_readback_async(c, 0, h);
      CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
      r = chol_decode(h);
    }
    if (comm_attached(c)) {   // Sigma and (logdet, is_pd, fail_col) from rank 0
      if (Sigma) comm_bcast(c, Sigma, flat_count(q, q, ldsigma), dt_code(c), 0);
      double* sc = static_cast<double*>(ws_get(c, WS_COMM, 64));
      double* hs = reinterpret_cast<double*>(h + 512);
      hs[0] = r.logdet;
      hs[1] = (double)r.is_pd;
      hs[2] = (double)r.fail_col;
      CGGM_CUDA_CHECK(cudaMemcpyAsync(sc, hs, 3 * 8, cudaMemcpyHostToDevice, c->stream));
      comm_bcast(c, sc, 3, 0, 0);
      CGGM_CUDA_CHECK(cudaMemcpyAsync(hs, sc, 3 * 8, cudaMemcpyDeviceToHost, c->stream));
      CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
      r.logdet = hs[0];
      r.is_pd = hs[1] > 0.5 ? 1 : 0;
      r.fail_col = (int64_t)hs[2];
    }
    *logdet = r.logdet;
    *is_pd = r.is_pd;
    *fail_col = r.fail_col;
  });
}

// ================================================================== dense building blocks (NEXT-3)
cggm_status cggm_gemm(cggm_ctx* ctx, int32_t transA, int32_t transB, int64_t M, int64_t N, int64_t K, double alpha,
                      const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc,
                      int32_t flags) {
  return guard(ctx, [&](Ctx* c) {
    if (M < 0 || N < 0 || K < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    if (flags & ~63) fail(CGGM_ERR_INVALID_ARG, "unknown gemm flag");
    if (M == 0 || N == 0) return;
    check_dense("C", C, M, N, ldc);
    if (K > 0) {
      check_dense("A", A, transA ? K : M, transA ? M : K, lda);
      check_dense("B", B, transB ? N : K, transB ? K : N, ldb);
      if (C == A || C == B) fail(CGGM_ERR_INVALID_ARG, "C aliases an operand");
    }
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      EpilogueT<T> e; e.out1 = static_cast<T*>(C); e.ld1 = ldc; e.a1 = alpha;
      if (beta != 0.0) { e.in1a = static_cast<const T*>(C); e.ld1a = ldc; e.b1 = beta; }
      gemm(c, transA != 0, transB != 0, M, N, K, static_cast<const T*>(A), lda, static_cast<const T*>(B), ldb, e,
           flags);
    });
  });
}

cggm_status cggm_chol_inverse_dense(cggm_ctx* ctx, int64_t q, void* A, int64_t lda, void* X, int64_t ldx,
                                    double* logdet, int32_t* is_pd, int64_t* fail_col) {
  return guard(ctx, [&](Ctx* c) {
    if (q < 1) fail(CGGM_ERR_INVALID_ARG, "need q >= 1");
    check_dense("A", A, q, q, lda);
    check_dense("X", X, q, q, ldx);
    if (lda % 2 || ldx % 2) fail(CGGM_ERR_INVALID_ARG, "leading dimensions must be even");
    if (!logdet || !is_pd || !fail_col) fail(CGGM_ERR_INVALID_ARG, "null host output pointer");
    const int64_t nleaves = n_leaves(q);
    Scal s = scal_lane(c, 0, 8 + nleaves);
    double* slots = s.dbl + 8;
    init_scalars(c, s.fail, s.flag);
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      CGGM_CUDA_CHECK(cudaMemsetAsync(X, 0, (size_t)ldx * q * sizeof(T), c->stream));
      const size_t tmp_elems = chol_tmp_elems(q);
      T* tmp = static_cast<T*>(ws_get(c, WS_TMP, tmp_elems * sizeof(T)));
      potrf_recursive<T>(c, ViewT<T>{static_cast<T*>(A), lda, q, q}, ViewT<T>{static_cast<T*>(X), ldx, q, q}, true,
                         nullptr, slots, s.fail, tmp, tmp_elems);
    });
    sum_arrays_1(c, slots, nleaves, s.dbl);
    char* h = static_cast<char*>(c->host_scratch);
    chol_readback_async(c, 0, h);
    CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    const CholResult r = chol_decode(h);
    *logdet = r.logdet;
    *is_pd = r.is_pd;
    *fail_col = r.fail_col;
  });
}

cggm_status cggm_symmetrize(cggm_ctx* ctx, int64_t n, void* S, int64_t lds) {
  return guard(ctx, [&](Ctx* c) {
    if (n < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    if (n == 0) return;
    check_dense("S", S, n, n, lds);
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      symmetrize<T>(c, n, static_cast<T*>(S), lds);
    });
  });
}

cggm_status cggm_densify(cggm_ctx* ctx, const cggm_csc* A, void* D, int64_t ldd) {
  return guard(ctx, [&](Ctx* c) {
    if (!A) fail(CGGM_ERR_INVALID_ARG, "null CSC");
    check_csc_host("A", A, A->nrows, A->ncols);
    if (A->nrows == 0 || A->ncols == 0) return;
    check_dense("D", D, A->nrows, A->ncols, ldd);
    validate_csc_dev(c, A, false, "A");
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      densify_csc<T>(c, A, ViewT<T>{static_cast<T*>(D), ldd, A->nrows, A->ncols});
    });
  });
}

// ------------------------------------------------------------------ a6
template <typename T>
static ActTotals* active_enqueue(Ctx* c, int64_t p, int64_t q, const T* GradL, int64_t ldgl, const T* GradT,
                                 int64_t ldgt, const cggm_csc* Lambda, const cggm_csc* Theta,
                                 const cggm_active_out* o) {
  ActWs ws = active_ws(c, q);
  Phase ph(c, TAG_ACTIVE);
  active_compact<T>(c, p, q, GradL, ldgl, GradT, ldgt, Lambda, Theta, o->lam_L, o->lam_T, o->penalize_diag, o->tie_eps, ws,
                 o->L_row, o->L_col, o->T_row, o->T_col, o->cap_L, o->cap_T);
  return ws.tot;
}

static void active_decode(const ActTotals& h, cggm_active_out* o) {
  o->m_L = h.m_L;
  o->m_T = h.m_T;
  o->ties_L = h.ties_L;
  o->ties_T = h.ties_T;
  o->subgrad_l1 = h.sub_L + h.sub_T;
  if (o->m_L > o->cap_L || o->m_T > o->cap_T)
    fail(CGGM_ERR_CAPACITY, "active set larger than capacity (m_L=" + std::to_string(o->m_L) +
                                ", m_T=" + std::to_string(o->m_T) + ")");
}

static void check_active_args(const cggm_active_out* o) {
  if (!o) fail(CGGM_ERR_INVALID_ARG, "null cggm_active_out");
  if (!(o->lam_L >= 0.0) || !(o->lam_T >= 0.0)) fail(CGGM_ERR_INVALID_ARG, "negative lambda");
  if (!(o->tie_eps >= 0.0)) fail(CGGM_ERR_INVALID_ARG, "negative tie_eps");
  if (o->cap_L < 0 || o->cap_T < 0) fail(CGGM_ERR_INVALID_ARG, "negative capacity");
  if ((o->cap_L > 0 && (!o->L_row || !o->L_col)) || (o->cap_T > 0 && (!o->T_row || !o->T_col)))
    fail(CGGM_ERR_INVALID_ARG, "null active-set output list with positive capacity");
}

static void active_sync(Ctx* c, ActTotals* T, cggm_active_out* o) {
  ActTotals h;
  CGGM_CUDA_CHECK(cudaMemcpyAsync(c->host_scratch, T, sizeof(ActTotals), cudaMemcpyDeviceToHost, c->stream));
  CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  std::memcpy(&h, c->host_scratch, sizeof(ActTotals));
  active_decode(h, o);
}

cggm_status cggm_active_set(cggm_ctx* ctx, int64_t p, int64_t q, const void* GradL, int64_t ldgl, const void* GradT,
                            int64_t ldgt, const cggm_csc* Lambda, const cggm_csc* Theta, cggm_active_out* out) {
  return guard(ctx, [&](Ctx* c) {
    if (p < 0 || q < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    check_active_args(out);
    check_dense("GradL", GradL, q, q, ldgl);
    check_dense("GradT", GradT, p, q, ldgt);
    check_csc_host("Lambda", Lambda, q, q);
    check_csc_host("Theta", Theta, p, q);
    out->m_L = out->m_T = out->ties_L = out->ties_T = 0;
    out->subgrad_l1 = 0.0;
    if (q == 0) return;
    validate_csc_dev(c, Lambda, true, "Lambda");
    validate_csc_dev(c, Theta, false, "Theta");
    ActTotals* tot = nullptr;
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      tot = active_enqueue<T>(c, p, q, static_cast<const T*>(GradL), ldgl, static_cast<const T*>(GradT), ldgt, Lambda,
                              Theta, out);
    });
    active_sync(c, tot, out);
  });
}

// ------------------------------------------------------------------ a2/a4/a5
// W (n_local x q, ldw) must already hold X Theta.
// Active sets built inside psi_enqueue (fused).  With GradT == NULL the p x q grad_Theta is streamed:
// computed in column chunks into a workspace buffer and compacted immediately (never stored).
struct Fuse {
  const cggm_csc* Lambda;
  const cggm_csc* Theta;
  const cggm_active_out* o;
  ActWs ws;
};
constexpr int64_t GT_CHUNK = 2048;

// split-k for W Sigma when the 128x128 grid fills its last wave poorly and K is long (the halves
// keep 2500+ k-steps each): wave efficiency of tiles vs 2 x tiles on num_sms SMs
static bool split_wsigma(Ctx* c, int64_t n, int64_t q) {
  if (c->no_split_k || q < 4096) return false;
  const int64_t tiles = ((n + 127) / 128) * ((q + 127) / 128), S = c->num_sms;
  if (tiles < S || tiles >= 16 * S) return false;
  auto eff = [&](int64_t t) { return (double)t / (double)(((t + S - 1) / S) * S); };
  return eff(2 * tiles) > eff(tiles) + 0.02;
}

template <typename T>
static void psi_enqueue(Ctx* c, int64_t n_local, int64_t n_total, int64_t p, int64_t q, const T* Xd, int64_t ldx,
                        const T* Yd, int64_t ldy, const T* W, int64_t ldw, const T* Sg, int64_t ldsigma, const T* Syy,
                        int64_t ldsyy, const T* Sxy, int64_t ldsxy, T* Psi, int64_t ldpsi, T* GradL, int64_t ldgl,
                        T* GradT, int64_t ldgt, const Fuse* fz, bool collective = false, T* E_out = nullptr,
                        int64_t lde_out = 0) {
  const int64_t ldn = pad_ld<T>(n_local > 0 ? n_local : 1);
  const int dt = sizeof(T) == 4 ? 1 : 0;
  T* R = static_cast<T*>(ws_get(c, WS_R, (size_t)ldn * q * sizeof(T)));
  // E = Y + W Sigma: library workspace, or the caller's buffer (cggm_psi_residual)
  T* E = E_out ? E_out : static_cast<T*>(ws_get(c, WS_E, (size_t)ldn * q * sizeof(T)));
  const int64_t lde = E_out ? lde_out : ldn;
  {  // a4: acc = W Sigma -> R = acc / sqrt(n), E = Y + acc
    Phase ph(c, TAG_WSIGMA);
    const bool want_e = ((GradT || fz) && !Sxy) || E_out;
    if (sizeof(T) == 8 && split_wsigma(c, n_local, q)) {
      // too few 128x128 tiles for whole waves (n = 1000, q = 20000: 8.5 waves): both k-halves of
      // each tile as separate CTAs, partials added into a zeroed accumulator, then R and E
      T* Acc = static_cast<T*>(ws_get(c, WS_ACC, (size_t)ldn * q * sizeof(T)));
      CGGM_CUDA_CHECK(cudaMemsetAsync(Acc, 0, (size_t)ldn * q * sizeof(T), c->stream));
      EpilogueT<T> e; e.out1 = Acc; e.ld1 = ldn; e.a1 = 1.0;
      gemm(c, false, false, n_local, q, q, W, ldw, Sg, ldsigma, e, SPLIT_K2);
      r_e_from_acc(c, n_local, q, Acc, ldn, Yd, ldy, R, ldn, want_e ? E : nullptr, lde,
                   1.0 / std::sqrt((double)n_total));
    } else {
      EpilogueT<T> e; e.out1 = R; e.ld1 = ldn; e.a1 = 1.0 / std::sqrt((double)n_total);
      if (want_e) { e.out2 = E; e.ld2 = lde; e.a2 = 1.0; e.in2a = Yd; e.ld2a = ldy; e.b2 = 1.0; }
      gemm(c, false, false, n_local, q, q, W, ldw, Sg, ldsigma, e, 0);
    }
  }
  {  // a4/a5: Psi = R^T R (mirrored), then grad_Lambda = (S_yy - Sigma) - Psi as one streaming pass;
     // with CGGM_FUSE_GRADL=1 the same GEMM's second epilogue output instead (-Psi + S_yy -
     // Sigma per element, both triangles from one value), unless Psi must first be all-reduced.  Measured
     // at `large`: the fused epilogue adds 2.6 ms to the Psi GEMM and saves the 1.8 ms pass -> off
    Phase ph(c, TAG_PSI);
    EpilogueT<T> e; e.out1 = Psi; e.ld1 = ldpsi; e.a1 = 1.0;
    const bool fuse_gl = GradL && !collective && c->fuse_gradl;
    if (fuse_gl) {
      e.out2 = GradL; e.ld2 = ldgl; e.a2 = -1.0;
      e.in2a = Syy; e.ld2a = ldsyy; e.b2 = 1.0;
      e.in2b = Sg; e.ld2b = ldsigma; e.c2 = -1.0;
    }
    gemm(c, true, false, q, q, n_local, R, ldn, R, ldn, e, SYM_LOWER | SYM_MIRROR);
    if (collective) comm_allreduce(c, Psi, flat_count(q, q, ldpsi), dt);   // Psi = sum_r R_r^T R_r
  }
  const cggm_active_out* o = fz ? fz->o : nullptr;
  // grad_Lambda and the S_Lambda compaction (HBM-bound) depend only on Psi: with CGGM_GL_OVERLAP they
  // run on a side stream beside the DMMA-bound X^T E GEMM, joined before the S_Theta part (measured
  // neutral at `large`: 409.2-409.8 ms either way; off by default)
  cudaStream_t chain = c->stream, side = nullptr;
  struct StreamBack {
    Ctx* c;
    cudaStream_t s;
    ~StreamBack() { c->stream = s; }
  } stream_back{c, chain};
  if (c->gl_overlap && fz && GradL && !collective && !c->fuse_gradl && GradT) {
    if (!c->gl_side) {
      int least = 0, greatest = 0;
      CGGM_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      CGGM_CUDA_CHECK(cudaStreamCreateWithPriority(&c->gl_side, cudaStreamNonBlocking,
                                                   c->gl_overlap == 2 ? least : greatest));
      CGGM_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_gl0, cudaEventDisableTiming));
      CGGM_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_gl1, cudaEventDisableTiming));
    }
    side = c->gl_side;
    CGGM_CUDA_CHECK(cudaEventRecord(c->ev_gl0, chain));
    CGGM_CUDA_CHECK(cudaStreamWaitEvent(side, c->ev_gl0, 0));
    c->stream = side;
  }
  if (GradL && !(c->fuse_gradl && !collective)) {   // (fused: the Psi GEMM's second output above)
    Phase pg(c, TAG_GRADL);
    grad_lambda(c, q, Syy, ldsyy, Sg, ldsigma, Psi, ldpsi, GradL, ldgl);
  }
  if (fz) {
    Phase ph(c, TAG_ACTIVE);
    active_begin(c, q, fz->ws);
    active_lambda<T>(c, q, GradL, ldgl, fz->Lambda, o->lam_L, o->penalize_diag, o->tie_eps, fz->ws, o->L_row,
                     o->L_col, o->cap_L);
  }
  if (side) {
    CGGM_CUDA_CHECK(cudaEventRecord(c->ev_gl1, side));
    c->stream = chain;
  }
  // a5: GradT = (2/n) X^T E   (or 2 S_xy + (2/sqrt n) X^T R), columns [j0, j0 + nc) into `out`
  auto grad_theta = [&](int64_t j0, int64_t nc, T* out, int64_t ldo) {
    Phase ph(c, TAG_GRADT);
    EpilogueT<T> e; e.out1 = out; e.ld1 = ldo;
    if (!Sxy) {
      e.a1 = 2.0 / (double)n_total;
      gemm(c, true, false, p, nc, n_local, Xd, ldx, E + j0 * lde, lde, e, 0);
    } else {
      e.a1 = 2.0 / std::sqrt((double)n_total);
      e.in1a = Sxy + j0 * ldsxy; e.ld1a = ldsxy; e.b1 = 2.0;
      gemm(c, true, false, p, nc, n_local, Xd, ldx, R + j0 * ldn, ldn, e, 0);
    }
    if (collective) comm_allreduce(c, out, flat_count(p, nc, ldo), dt);   // sum_r (2/n) X_r^T E_r
  };
  if (GradT) {
    grad_theta(0, q, GradT, ldgt);
    if (side) CGGM_CUDA_CHECK(cudaStreamWaitEvent(chain, c->ev_gl1, 0));
    if (fz) {
      Phase ph(c, TAG_ACTIVE);
      active_theta_chunk<T>(c, p, 0, q, GradT, ldgt, fz->Theta, o->lam_T, o->tie_eps, fz->ws, o->T_row, o->T_col,
                            o->cap_T);
    }
  } else if (fz && sizeof(T) == 8 && !collective && !Sxy && c->k01 && p > 0) {
    // K01: grad_Theta never stored -- S_Theta, its ties and the subgradient taken in the X^T E
    // epilogue while each tile is in shared memory (one GEMM over all q columns, no chunks)
    const SelWs sw = sel_ws(c, p, q);
    EpilogueT<T> e;
    e.a1 = 2.0 / (double)n_total;
    {
      Phase ph(c, TAG_ACTIVE);
      e.sel = select_begin(c, p, q, fz->ws, sw, fz->Theta, o->lam_T, o->tie_eps);
    }
    {
      Phase ph(c, TAG_GRADT);
      gemm(c, true, false, p, q, n_local, Xd, ldx, E, lde, e, 0);
    }
    if (side) CGGM_CUDA_CHECK(cudaStreamWaitEvent(chain, c->ev_gl1, 0));
    Phase ph(c, TAG_ACTIVE);
    select_end(c, p, q, fz->ws, sw, o->T_row, o->T_col, o->cap_T);
  } else if (fz) {
    const int64_t ldc = pad_ld<T>(p);
    T* chunk = static_cast<T*>(ws_get(c, WS_GTCHUNK, (size_t)ldc * std::min<int64_t>(GT_CHUNK, q) * sizeof(T)));
    for (int64_t j0 = 0; j0 < q; j0 += GT_CHUNK) {
      const int64_t nc = std::min<int64_t>(GT_CHUNK, q - j0);
      grad_theta(j0, nc, chunk, ldc);
      Phase ph(c, TAG_ACTIVE);
      active_theta_chunk<T>(c, p, j0, nc, chunk, ldc, fz->Theta, o->lam_T, o->tie_eps, fz->ws, o->T_row, o->T_col,
                            o->cap_T);
    }
  }
  if (fz) {
    Phase ph(c, TAG_ACTIVE);
    active_end(c, q, fz->ws);
  }
}

cggm_status cggm_psi_grad(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, int64_t q, const void* X,
                          int64_t ldx, const void* Y, int64_t ldy, const cggm_csc* Theta, const void* Sigma,
                          int64_t ldsigma, const void* Syy, int64_t ldsyy, const void* Sxy, int64_t ldsxy, void* Psi,
                          int64_t ldpsi, void* GradL, int64_t ldgl, void* GradT, int64_t ldgt, const cggm_csc* Lambda,
                          cggm_active_out* fused) {
  return guard(ctx, [&](Ctx* c) {
    if (n_local < 0 || p < 0 || q < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    if (n_total < 1 || n_total < n_local) fail(CGGM_ERR_INVALID_ARG, "n_total must be >= max(1, n_local)");
    check_dense("X", X, n_local, p, ldx);
    check_dense("Y", Y, n_local, q, ldy);
    check_csc_host("Theta", Theta, p, q);
    check_dense("Sigma", Sigma, q, q, ldsigma);
    check_dense("Psi", Psi, q, q, ldpsi);
    check_dense("GradL", GradL, q, q, ldgl, false);
    check_dense("GradT", GradT, p, q, ldgt, false);
    check_dense("Sxy", Sxy, p, q, ldsxy, false);
    if (GradL) {
      check_dense("Syy", Syy, q, q, ldsyy);
      if (n_local != n_total && !comm_attached(c))
        fail(CGGM_ERR_INVALID_ARG, "GradL needs the all-reduced Psi: pass GradL=NULL when sharded without a comm");
    }
    if (Sxy && n_local != n_total) fail(CGGM_ERR_INVALID_ARG, "the S_xy route is not a per-shard partial sum");
    if (fused) {
      check_active_args(fused);
      if (!GradL) fail(CGGM_ERR_INVALID_ARG, "fused active sets need GradL");
      check_csc_host("Lambda", Lambda, q, q);
    }
    if (q == 0) return;
    validate_csc_dev(c, Theta, false, "Theta");
    if (fused) validate_csc_dev(c, Lambda, true, "Lambda");
    ActTotals* tot = nullptr;
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      const int64_t ldn = pad_ld<T>(n_local > 0 ? n_local : 1);
      T* W = static_cast<T*>(ws_get(c, WS_W, (size_t)ldn * q * sizeof(T)));
      spmm_x_theta<T>(c, static_cast<const T*>(X), ldx, n_local, Theta, ViewT<T>{W, ldn, n_local, q});
      Fuse fz{Lambda, Theta, fused, fused ? active_ws(c, q) : ActWs{}};
      psi_enqueue<T>(c, n_local, n_total, p, q, static_cast<const T*>(X), ldx, static_cast<const T*>(Y), ldy, W, ldn,
                     static_cast<const T*>(Sigma), ldsigma, static_cast<const T*>(Syy), ldsyy,
                     static_cast<const T*>(Sxy), ldsxy, static_cast<T*>(Psi), ldpsi, static_cast<T*>(GradL), ldgl,
                     static_cast<T*>(GradT), ldgt, fused ? &fz : nullptr, comm_attached(c));
      if (fused) tot = fz.ws.tot;
    });
    if (fused) active_sync(c, tot, fused);
  });
}

cggm_status cggm_grad_lambda(cggm_ctx* ctx, int64_t q, const void* Syy, int64_t ldsyy, const void* Sigma,
                             int64_t ldsigma, const void* Psi, int64_t ldpsi, void* GradL, int64_t ldgl) {
  return guard(ctx, [&](Ctx* c) {
    if (q < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    check_dense("Syy", Syy, q, q, ldsyy);
    check_dense("Sigma", Sigma, q, q, ldsigma);
    check_dense("Psi", Psi, q, q, ldpsi);
    check_dense("GradL", GradL, q, q, ldgl);
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      grad_lambda<T>(c, q, static_cast<const T*>(Syy), ldsyy, static_cast<const T*>(Sigma), ldsigma,
                     static_cast<const T*>(Psi), ldpsi, static_cast<T*>(GradL), ldgl);
    });
  });
}

// Psi partial (all-reduced with a communicator) and the residual E = Y + X Theta Sigma of this
// shard's rows into the caller's buffer: the sharded evaluation's grad_Theta is then formed column
// block by column block ((2/n) X_r^T E_r, cggm_gemm) and reduce-scattered by the caller.
cggm_status cggm_psi_residual(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, int64_t q, const void* X,
                              int64_t ldx, const void* Y, int64_t ldy, const cggm_csc* Theta, const void* Sigma,
                              int64_t ldsigma, void* Psi, int64_t ldpsi, void* E, int64_t lde) {
  return guard(ctx, [&](Ctx* c) {
    if (n_local < 0 || p < 0 || q < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    if (n_total < 1 || n_total < n_local) fail(CGGM_ERR_INVALID_ARG, "n_total must be >= max(1, n_local)");
    check_dense("X", X, n_local, p, ldx);
    check_dense("Y", Y, n_local, q, ldy);
    check_csc_host("Theta", Theta, p, q);
    check_dense("Sigma", Sigma, q, q, ldsigma);
    check_dense("Psi", Psi, q, q, ldpsi);
    check_dense("E", E, n_local, q, lde);
    if (q == 0) return;
    validate_csc_dev(c, Theta, false, "Theta");
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      const int64_t ldn = pad_ld<T>(n_local > 0 ? n_local : 1);
      T* W = static_cast<T*>(ws_get(c, WS_W, (size_t)ldn * q * sizeof(T)));
      spmm_x_theta<T>(c, static_cast<const T*>(X), ldx, n_local, Theta, ViewT<T>{W, ldn, n_local, q});
      psi_enqueue<T>(c, n_local, n_total, p, q, static_cast<const T*>(X), ldx, static_cast<const T*>(Y), ldy, W, ldn,
                     static_cast<const T*>(Sigma), ldsigma, nullptr, 0, nullptr, 0, static_cast<T*>(Psi), ldpsi,
                     nullptr, 0, nullptr, 0, nullptr, comm_attached(c), static_cast<T*>(E), lde);
    });
  });
}

// S_Theta entries of columns [col0, col0 + ncols) from a gradient block (P:296-303 for that block,
// reading A5-A7), with global column indices, in column-major order; host totals.  The block of a
// column-range owner in the sharded evaluation (its reduce-scattered grad_Theta columns).
cggm_status cggm_active_theta_block(cggm_ctx* ctx, int64_t p, int64_t col0, int64_t ncols, const void* GradT,
                                   int64_t ldgt, const cggm_csc* Theta, double lam_T, double tie_eps, int32_t* T_row,
                                   int32_t* T_col, int64_t cap, int64_t* m, int64_t* ties, double* subgrad) {
  return guard(ctx, [&](Ctx* c) {
    if (p < 0 || ncols < 0 || col0 < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension or column");
    if (!Theta) fail(CGGM_ERR_INVALID_ARG, "null Theta");
    if (col0 + ncols > Theta->ncols) fail(CGGM_ERR_SHAPE, "column block beyond Theta's columns");
    check_csc_host("Theta", Theta, p, Theta->ncols);
    check_dense("GradT", GradT, p, ncols, ldgt);
    if (!(lam_T >= 0.0) || !(tie_eps >= 0.0)) fail(CGGM_ERR_INVALID_ARG, "negative lambda or tie_eps");
    if (cap < 0 || (cap > 0 && (!T_row || !T_col))) fail(CGGM_ERR_INVALID_ARG, "bad output list");
    if (!m) fail(CGGM_ERR_INVALID_ARG, "null m");
    *m = 0;
    if (ties) *ties = 0;
    if (subgrad) *subgrad = 0.0;
    if (ncols == 0) return;
    validate_csc_dev(c, Theta, false, "Theta");
    // the block as a CSC of its own: the column pointers of columns col0.. (absolute offsets into the
    // same row / value arrays)
    cggm_csc sub = *Theta;
    sub.ncols = ncols;
    sub.colptr = Theta->colptr + col0;
    ActTotals* tot = nullptr;
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      ActWs ws = active_ws(c, ncols);
      Phase ph(c, TAG_ACTIVE);
      active_begin(c, ncols, ws);
      active_theta_chunk<T>(c, p, 0, ncols, static_cast<const T*>(GradT), ldgt, &sub, lam_T, tie_eps, ws, T_row, T_col,
                            cap);
      active_end(c, ncols, ws);
      if (col0 > 0 && cap > 0) {
        k_col_offset<<<c->num_sms, 256, 0, c->stream>>>(T_col, ws.tot, cap, (int32_t)col0);
        post_launch(c, "k_col_offset");
      }
      tot = ws.tot;
    });
    ActTotals h;
    CGGM_CUDA_CHECK(cudaMemcpyAsync(c->host_scratch, tot, sizeof(ActTotals), cudaMemcpyDeviceToHost, c->stream));
    CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    std::memcpy(&h, c->host_scratch, sizeof(ActTotals));
    *m = h.m_T;
    if (ties) *ties = h.ties_T;
    if (subgrad) *subgrad = h.sub_T;
    if (h.m_T > cap) fail(CGGM_ERR_CAPACITY, "S_Theta block larger than capacity (m=" + std::to_string(h.m_T) + ")");
  });
}

// ------------------------------------------------------------------ a7
// Augmented dense [Lambda; W] ((q + n_local) x q): the Cholesky of the trial Lambda (the PD test)
// leaves Z = W L^{-T} in the bottom rows, ||Z||_F^2 = tr(Lambda^{-1} W^T W) (reading A14).
// Scal layout: dbl[0] logdet sum, dbl[1..5] sums (<Y,Y Lambda>, <W,Y>, ||Z||^2, |Lambda|, |Theta|),
// dbl[16..] per-column partials, then leaf slots.
template <typename T>
static void objective_enqueue(Ctx* c, int lane, int64_t n_local, int64_t q, const T* Yd, int64_t ldy, const T* Wd,
                              int64_t ldwd, const cggm_csc* Lambda, const cggm_csc* Theta,
                              int32_t penalize_diag) {
  const int nb = leaf_nb();
  const int64_t nleaves = n_leaves(q);
  const int64_t ldaug = pad_ld<T>(q + n_local);
  T* A = static_cast<T*>(ws_get(c, kLane[lane].dense, (size_t)ldaug * q * sizeof(T)));
  T* leafinv = static_cast<T*>(ws_get(c, WS_LEAFINV, (size_t)nleaves * nb * nb * sizeof(T)));
  Scal s = scal_lane(c, lane, 16 + 5 * q + nleaves);
  double* res = s.dbl;
  double* partY = s.dbl + 16;
  double* partWY = partY + q;
  double* partZ = partWY + q;
  double* penLp = partZ + q;
  double* penTp = penLp + q;
  double* slots = penTp + q;
  // inverses of the <= BINV diagonal blocks + temporaries (full-inverse subtrees, block products)
  const int64_t binv = block_inverse_size();
  const int64_t ldxd = pad_ld<T>(q);
  const size_t tmp_elems = (size_t)(binv + 4) * (binv + 4);
  const size_t tmp2_elems = (size_t)pad_ld<T>(q + n_local) * binv;
  T* xdiag = static_cast<T*>(ws_get(c, WS_XDIAG, (size_t)ldxd * binv * sizeof(T)));
  T* tmpo = static_cast<T*>(ws_get(c, WS_TMP_OBJ, (tmp_elems + tmp2_elems) * sizeof(T)));
  CGGM_CUDA_CHECK(cudaMemsetAsync(xdiag, 0, (size_t)ldxd * binv * sizeof(T), c->stream));
  densify_csc(c, Lambda, ViewT<T>{A, ldaug, q, q});
  copy2d(c, ViewT<T>{A + q, ldaug, n_local, q}, Wd, ldwd);
  init_scalars(c, s.fail, s.flag);
  potrf_recursive<T>(c, ViewT<T>{A, ldaug, q + n_local, q}, ViewT<T>{nullptr, ldaug, q, q}, false, leafinv, slots, s.fail,
                  tmpo, tmp_elems, xdiag, ldxd, tmpo + tmp_elems, tmp2_elems);
  Phase ph(c, TAG_OBJRED);
  col_partials<T>(c, 0, n_local, q, Yd, ldy, nullptr, 0, Lambda, partY);
  col_partials<T>(c, 1, n_local, q, Wd, ldwd, Yd, ldy, nullptr, partWY);
  col_partials<T>(c, 2, n_local, q, A + q, ldaug, nullptr, 0, nullptr, partZ);
  csc_abs_partials<T>(c, Lambda, penalize_diag == 0, penLp);
  csc_abs_partials<T>(c, Theta, false, penTp);
  sum_arrays_1(c, slots, nleaves, res + 0);
  sum_arrays_1(c, partY, q, res + 1);
  sum_arrays_1(c, partWY, q, res + 2);
  sum_arrays_1(c, partZ, q, res + 3);
  sum_arrays_1(c, penLp, q, res + 4);
  sum_arrays_1(c, penTp, q, res + 5);
}

// factor reuse: the objective with its trial factorisation in full-inverse mode, keeping
// X = L^{-1} in `xslot`; tr(Sigma M) = ||W X^T||^2 / n by one triangular GEMM.  Same scalar block
// layout as objective_enqueue.
template <typename T>
static void objective_fullinv_enqueue(Ctx* c, int lane, int64_t n_local, int64_t q, const T* Yd, int64_t ldy,
                                      const T* Wd, int64_t ldwd, const cggm_csc* Lambda, const cggm_csc* Theta,
                                      int32_t penalize_diag, int xslot) {
  const int64_t nleaves = n_leaves(q);
  const int64_t lda = pad_ld<T>(q);
  T* A = static_cast<T*>(ws_get(c, kLane[lane].dense, (size_t)lda * q * sizeof(T)));
  T* X = static_cast<T*>(ws_get(c, xslot, (size_t)lda * q * sizeof(T)));
  const size_t tmp_elems = chol_tmp_elems(q);
  T* tmp = static_cast<T*>(ws_get(c, WS_TMP2, tmp_elems * sizeof(T)));
  const int64_t ldz = pad_ld<T>(n_local);
  T* Z = static_cast<T*>(ws_get(c, WS_Z, (size_t)ldz * q * sizeof(T)));
  Scal s = scal_lane(c, lane, 16 + 5 * q + nleaves);
  double* res = s.dbl;
  double* partY = s.dbl + 16;
  double* partWY = partY + q;
  double* partZ = partWY + q;
  double* penLp = partZ + q;
  double* penTp = penLp + q;
  double* slots = penTp + q;
  CGGM_CUDA_CHECK(cudaMemsetAsync(X, 0, (size_t)lda * q * sizeof(T), c->stream));
  densify_csc(c, Lambda, ViewT<T>{A, lda, q, q});
  init_scalars(c, s.fail, s.flag);
  potrf_recursive<T>(c, ViewT<T>{A, lda, q, q}, ViewT<T>{X, lda, q, q}, true, nullptr, slots, s.fail, tmp, tmp_elems);
  {  // Z = W X^T (X lower triangular: op(B)[k][j] = X[j][k] vanishes for k > j)
    Phase ph(c, TAG_TRSM);
    EpilogueT<T> e; e.out1 = Z; e.ld1 = ldz;
    gemm(c, false, true, n_local, q, q, Wd, ldwd, X, lda, e, B_KLE_N);
  }
  Phase ph(c, TAG_OBJRED);
  col_partials<T>(c, 0, n_local, q, Yd, ldy, nullptr, 0, Lambda, partY);
  col_partials<T>(c, 1, n_local, q, Wd, ldwd, Yd, ldy, nullptr, partWY);
  col_partials<T>(c, 2, n_local, q, Z, ldz, nullptr, 0, nullptr, partZ);
  csc_abs_partials<T>(c, Lambda, penalize_diag == 0, penLp);
  csc_abs_partials<T>(c, Theta, false, penTp);
  sum_arrays_1(c, slots, nleaves, res + 0);
  sum_arrays_1(c, partY, q, res + 1);
  sum_arrays_1(c, partWY, q, res + 2);
  sum_arrays_1(c, partZ, q, res + 3);
  sum_arrays_1(c, penLp, q, res + 4);
  sum_arrays_1(c, penTp, q, res + 5);
}

static void objective_readback_async(Ctx* c, int lane, char* h) {
  Scal s = scal_lane(c, lane, 0);
  CGGM_CUDA_CHECK(cudaMemcpyAsync(h, s.fail, 4, cudaMemcpyDeviceToHost, c->stream));
  CGGM_CUDA_CHECK(cudaMemcpyAsync(h + 8, s.dbl, 6 * 8, cudaMemcpyDeviceToHost, c->stream));
}

static void objective_decode(const char* h, int64_t n_total, double lam_L, double lam_T, cggm_objective_out* out) {
  CholResult cr = chol_decode(h);
  double v[6];
  std::memcpy(v, h + 8, 6 * 8);
  const double nt = (double)n_total;
  out->pen_L = lam_L * v[4];
  out->pen_T = lam_T * v[5];
  out->is_pd = cr.is_pd;
  out->fail_col = cr.fail_col;
  out->tr_syy_lam = v[1] / nt;
  out->tr_sxy_theta = v[2] / nt;
  if (cr.is_pd) {
    out->logdet = cr.logdet;
    out->tr_sigma_m = v[3] / nt;
    out->g = -out->logdet + out->tr_syy_lam + 2.0 * out->tr_sxy_theta + out->tr_sigma_m;
    out->f = out->g + out->pen_L + out->pen_T;
  } else {
    const double nan = std::numeric_limits<double>::quiet_NaN();
    out->logdet = nan;
    out->tr_sigma_m = nan;
    out->g = INFINITY;
    out->f = INFINITY;
  }
}

cggm_status cggm_objective(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, int64_t q, const void* X,
                           int64_t ldx, const void* Y, int64_t ldy, const cggm_csc* Lambda, const cggm_csc* Theta,
                           double lam_L, double lam_T, int32_t penalize_diag, const void* W, int64_t ldw,
                           cggm_objective_out* out) {
  return guard(ctx, [&](Ctx* c) {
    if (!out) fail(CGGM_ERR_INVALID_ARG, "null cggm_objective_out");
    if (n_local < 0 || p < 0 || q < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    if (n_total < 1 || n_total < n_local) fail(CGGM_ERR_INVALID_ARG, "n_total must be >= max(1, n_local)");
    if (!(lam_L >= 0.0) || !(lam_T >= 0.0)) fail(CGGM_ERR_INVALID_ARG, "negative lambda");
    check_dense("Y", Y, n_local, q, ldy);
    check_csc_host("Lambda", Lambda, q, q);
    check_csc_host("Theta", Theta, p, q);
    if (W) check_dense("W", W, n_local, q, ldw);
    else check_dense("X", X, n_local, p, ldx);
    std::memset(out, 0, sizeof(*out));
    if (q == 0) {
      out->is_pd = 1; out->fail_col = -1;
      return;
    }
    validate_csc_dev(c, Lambda, true, "Lambda");
    validate_csc_dev(c, Theta, false, "Theta");
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      const int64_t ldn = pad_ld<T>(n_local > 0 ? n_local : 1);
      const T* Wd;
      int64_t ldwd;
      if (W) {
        Wd = static_cast<const T*>(W);
        ldwd = ldw;
      } else {
        T* Wb = static_cast<T*>(ws_get(c, WS_W, (size_t)ldn * q * sizeof(T)));
        spmm_x_theta<T>(c, static_cast<const T*>(X), ldx, n_local, Theta, ViewT<T>{Wb, ldn, n_local, q});
        Wd = Wb;
        ldwd = ldn;
      }
      objective_enqueue<T>(c, 0, n_local, q, static_cast<const T*>(Y), ldy, Wd, ldwd, Lambda, Theta, penalize_diag);
    });
    // the three data traces are sums over samples; logdet and penalties are the same on every rank
    comm_allreduce(c, scal_lane(c, 0, 0).dbl + 1, 3, 0);
    char* h = static_cast<char*>(c->host_scratch);
    objective_readback_async(c, 0, h);
    CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    objective_decode(h, n_total, lam_L, lam_T, out);
  });
}

cggm_status cggm_objective_given_inverse(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, int64_t q,
                                         const void* X, int64_t ldx, const void* Y, int64_t ldy,
                                         const cggm_csc* Lambda, const cggm_csc* Theta, double lam_L, double lam_T,
                                         int32_t penalize_diag, const void* W, int64_t ldw, const void* Linv,
                                         int64_t ldlinv, double logdet, cggm_objective_out* out) {
  return guard(ctx, [&](Ctx* c) {
    if (!out) fail(CGGM_ERR_INVALID_ARG, "null cggm_objective_out");
    if (n_local < 0 || p < 0 || q < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    if (n_total < 1 || n_total < n_local) fail(CGGM_ERR_INVALID_ARG, "n_total must be >= max(1, n_local)");
    if (!(lam_L >= 0.0) || !(lam_T >= 0.0)) fail(CGGM_ERR_INVALID_ARG, "negative lambda");
    check_dense("Y", Y, n_local, q, ldy);
    check_csc_host("Lambda", Lambda, q, q);
    check_csc_host("Theta", Theta, p, q);
    check_dense("Linv", Linv, q, q, ldlinv);
    if (W) check_dense("W", W, n_local, q, ldw);
    else check_dense("X", X, n_local, p, ldx);
    std::memset(out, 0, sizeof(*out));
    if (q == 0) {
      out->is_pd = 1; out->fail_col = -1;
      return;
    }
    validate_csc_dev(c, Lambda, true, "Lambda");
    validate_csc_dev(c, Theta, false, "Theta");
    Scal s = scal_lane(c, 0, 16 + 5 * q);
    double* res = s.dbl;
    double* partY = s.dbl + 16;
    double* partWY = partY + q;
    double* partZ = partWY + q;
    double* penLp = partZ + q;
    double* penTp = penLp + q;
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      const int64_t ldn = pad_ld<T>(n_local > 0 ? n_local : 1);
      const T* Wd;
      int64_t ldwd;
      if (W) {
        Wd = static_cast<const T*>(W);
        ldwd = ldw;
      } else {
        T* Wb = static_cast<T*>(ws_get(c, WS_W, (size_t)ldn * q * sizeof(T)));
        spmm_x_theta<T>(c, static_cast<const T*>(X), ldx, n_local, Theta, ViewT<T>{Wb, ldn, n_local, q});
        Wd = Wb;
        ldwd = ldn;
      }
      T* Z = static_cast<T*>(ws_get(c, WS_Z, (size_t)ldn * q * sizeof(T)));
      {  // Z = W Linv^T (Linv lower: op(B)[k][j] = Linv[j][k] vanishes for k > j)
        Phase ph(c, TAG_TRSM);
        EpilogueT<T> e; e.out1 = Z; e.ld1 = ldn;
        if (n_local > 0) gemm(c, false, true, n_local, q, q, Wd, ldwd, static_cast<const T*>(Linv), ldlinv, e, B_KLE_N);
      }
      Phase ph(c, TAG_OBJRED);
      const T* Yd = static_cast<const T*>(Y);
      col_partials<T>(c, 0, n_local, q, Yd, ldy, nullptr, 0, Lambda, partY);
      col_partials<T>(c, 1, n_local, q, Wd, ldwd, Yd, ldy, nullptr, partWY);
      col_partials<T>(c, 2, n_local, q, Z, ldn, nullptr, 0, nullptr, partZ);
      csc_abs_partials<T>(c, Lambda, penalize_diag == 0, penLp);
      csc_abs_partials<T>(c, Theta, false, penTp);
      sum_arrays_1(c, partY, q, res + 1);
      sum_arrays_1(c, partWY, q, res + 2);
      sum_arrays_1(c, partZ, q, res + 3);
      sum_arrays_1(c, penLp, q, res + 4);
      sum_arrays_1(c, penTp, q, res + 5);
    });
    comm_allreduce(c, res + 1, 3, 0);
    double v[6];
    CGGM_CUDA_CHECK(cudaMemcpyAsync(v, res, 6 * 8, cudaMemcpyDeviceToHost, c->stream));
    CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    const double nt = (double)n_total;
    out->pen_L = lam_L * v[4];
    out->pen_T = lam_T * v[5];
    out->is_pd = 1;
    out->fail_col = -1;
    out->logdet = logdet;
    out->tr_syy_lam = v[1] / nt;
    out->tr_sxy_theta = v[2] / nt;
    out->tr_sigma_m = v[3] / nt;
    out->g = -logdet + out->tr_syy_lam + 2.0 * out->tr_sxy_theta + out->tr_sigma_m;
    out->f = out->g + out->pen_L + out->pen_T;
  });
}

// ------------------------------------------------------------------ composite evaluation
// One Newton-iteration evaluation (the bench's unit): the objective's fresh trial Cholesky runs on
// the auxiliary stream, overlapped with Sigma = Lambda^{-1} and the Psi / gradient / active-set
// work on the caller's stream; one host synchronisation at the end.
// Inputs uploaded from host memory by cggm_newton_eval_host: events after each upload
struct HostIn {
  cudaEvent_t ev_lam, ev_xt, ev_y;   // Lambda; X and Theta; Y (S_yy is formed from it here)
};

static void newton_eval_core(Ctx* c, int64_t n, int64_t p, int64_t q, const void* X, int64_t ldx, const void* Y,
                             int64_t ldy, const void* Syy, int64_t ldsyy, const cggm_csc* Lambda, const cggm_csc* Theta,
                             void* Sigma, int64_t ldsigma, void* Psi, int64_t ldpsi, void* GradL, int64_t ldgl,
                             void* GradT, int64_t ldgt, cggm_active_out* active, cggm_eval_out* out,
                             const HostIn* hin) {
  if (!out) fail(CGGM_ERR_INVALID_ARG, "null cggm_eval_out");
  if (c->comm.world > 1)
    fail(CGGM_ERR_UNSUPPORTED, "cggm_newton_eval is single-GPU; with a communicator use the collective calls");
  if (n < 1 || p < 0 || q < 1) fail(CGGM_ERR_INVALID_ARG, "need n >= 1, q >= 1, p >= 0");
  check_dense("X", X, n, p, ldx);
  check_dense("Y", Y, n, q, ldy);
  check_dense("Syy", Syy, q, q, ldsyy);
  check_dense("Sigma", Sigma, q, q, ldsigma);
  check_dense("Psi", Psi, q, q, ldpsi);
  check_dense("GradL", GradL, q, q, ldgl);
  check_dense("GradT", GradT, p, q, ldgt, false);
  check_csc_host("Lambda", Lambda, q, q);
  check_csc_host("Theta", Theta, p, q);
  check_active_args(active);
  std::memset(out, 0, sizeof(*out));
  if (!hin) {
    validate_csc_dev(c, Lambda, true, "Lambda");
    validate_csc_dev(c, Theta, false, "Theta");
  }
  if (!c->aux) {
    // the objective's trial factorisation is filler work: least priority, so its CTAs take the SMs
    // the critical chain (a3 -> a4/a5 -> a6, greatest priority) leaves idle in its latency-bound
    // recursion levels
    int least = 0, greatest = 0;
    CGGM_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CGGM_CUDA_CHECK(cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, stream_priority(1)));
    CGGM_CUDA_CHECK(cudaStreamCreateWithPriority(&c->hi, cudaStreamNonBlocking, stream_priority(0)));
    CGGM_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CGGM_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    CGGM_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_join_hi, cudaEventDisableTiming));
    CGGM_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_w, cudaEventDisableTiming));
    CGGM_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_syy, cudaEventDisableTiming));
  }
  cudaStream_t s_caller = c->stream;
  struct Restore {
    Ctx* c;
    cudaStream_t s;
    ~Restore() { c->stream = s; c->lane = 0; }
  } restore{c, s_caller};
  // allocate every workspace slot up front (allocation may synchronise the device; nothing in the
  // enqueue below may, so that it can be captured into a CUDA graph)
  dispatch(c, [&](auto tag) {
    using T = decltype(tag);
    const size_t es = sizeof(T);
    const int64_t ldn = pad_ld<T>(n);
    const int64_t nleaves = n_leaves(q);
    ws_get(c, WS_DENSE_A, (size_t)pad_ld<T>(q) * q * es);
    ws_get(c, WS_DENSE_B, (size_t)pad_ld<T>(q + n) * q * es);
    ws_get(c, WS_LINV, (size_t)pad_ld<T>(q) * q * es);
    ws_get(c, WS_TMP, chol_tmp_elems(q) * es);
    ws_get(c, WS_LEAFINV, (size_t)nleaves * leaf_nb() * leaf_nb() * es);
    ws_get(c, WS_XDIAG, (size_t)pad_ld<T>(q) * block_inverse_size() * es);
    ws_get(c, WS_TMP_OBJ, ((size_t)(block_inverse_size() + 4) * (block_inverse_size() + 4) +
                           (size_t)pad_ld<T>(q + n) * block_inverse_size()) * es);
    ws_get(c, WS_SCAL, 64 + (8 + nleaves) * 8);
    ws_get(c, WS_SCAL2, 64 + (16 + 5 * q + nleaves) * 8);
    active_ws(c, q);
    ws_get(c, WS_R, (size_t)ldn * q * es);
    ws_get(c, WS_E, (size_t)ldn * q * es);
    if (!GradT && es == 8 && c->k01 && p > 0) sel_ws(c, p, q);
    else if (!GradT) ws_get(c, WS_GTCHUNK, (size_t)pad_ld<T>(p) * std::min<int64_t>(GT_CHUNK, q) * es);
    ws_get(c, WS_W, (size_t)ldn * q * es);
    if (es == 8 && split_wsigma(c, n, q)) ws_get(c, WS_ACC, (size_t)ldn * q * es);
    if (c->factor_reuse) {
      ws_get(c, WS_LINV2, (size_t)pad_ld<T>(q) * q * es);
      ws_get(c, WS_TMP2, chol_tmp_elems(q) * es);
      ws_get(c, WS_Z, (size_t)ldn * q * es);
      ws_get(c, WS_REUSE_SCAL, 64 + 8);
    }
  });
  // factor reuse: Sigma from the kept trial inverse of the previous call (buffer xs_prev); this
  // call's trial inverse goes to the other buffer
  const bool reuse_now = c->factor_reuse && c->reuse_valid && c->reuse_q == q;
  const int xs_prev = c->reuse_buf ? WS_LINV2 : WS_LINV, xs_next = c->reuse_buf ? WS_LINV : WS_LINV2;
  ActTotals* tot = nullptr;
  char* h = static_cast<char*>(c->host_scratch);
  // the whole evaluation, enqueue only: fork onto the chain / objective streams, join back into
  // the caller's stream, D2H of the scalars into pinned host memory
  unsigned hin_wait = 0;   // cudaEventWaitExternal while capturing (events recorded outside the graph)
  const bool gated = c->gate_cols > 0 && !reuse_now;
  if (gated && !c->gate_ev) CGGM_CUDA_CHECK(cudaEventCreateWithFlags(&c->gate_ev, cudaEventDisableTiming));
  auto enqueue = [&](cudaStream_t so) {
    c->stream = so;
    c->gate_done = false;
    if (c->prio_mode) {
      CGGM_CUDA_CHECK(cudaEventRecord(c->ev_fork, so));
      CGGM_CUDA_CHECK(cudaStreamWaitEvent(c->hi, c->ev_fork, 0));
      c->stream = c->hi;
    }
    cudaStream_t s0 = c->stream;
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      const size_t es = sizeof(T);
      const int64_t ldn = pad_ld<T>(n);
      T* W = static_cast<T*>(ws_get(c, WS_W, (size_t)ldn * q * es));
      const T* Xd = static_cast<const T*>(X);
      const T* Yd = static_cast<const T*>(Y);
      // fork; a2 (W = X Theta) and a7 on the auxiliary stream (lane 1), the chain a3 -> a4/a5 -> a6
      // on s0 waits for W only when a4 needs it.  Host inputs (cggm_newton_eval_host): each step
      // waits for the upload of what it reads, so the factorisation starts while X, Y stream in.
      CGGM_CUDA_CHECK(cudaEventRecord(c->ev_fork, s0));
      CGGM_CUDA_CHECK(cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
      try {
        c->stream = c->aux;
        c->lane = 1;
        if (hin) CGGM_CUDA_CHECK(cudaStreamWaitEvent(c->aux, hin->ev_xt, hin_wait));
        spmm_x_theta<T>(c, Xd, ldx, n, Theta, ViewT<T>{W, ldn, n, q});
        CGGM_CUDA_CHECK(cudaEventRecord(c->ev_w, c->aux));
        if (hin) {   // S_yy on its own stream, above the objective's priority: off the chain's critical path
          CGGM_CUDA_CHECK(cudaStreamWaitEvent(c->syys, c->ev_fork, 0));   // joins the capture, if any
          CGGM_CUDA_CHECK(cudaStreamWaitEvent(c->syys, hin->ev_y, hin_wait));
          c->stream = c->syys;
          Phase ph(c, TAG_COV);
          EpilogueT<T> e; e.out1 = static_cast<T*>(const_cast<void*>(Syy)); e.ld1 = ldsyy; e.a1 = 1.0 / (double)n;
          gemm(c, true, false, q, q, n, Yd, ldy, Yd, ldy, e, SYM_LOWER | SYM_MIRROR);
          CGGM_CUDA_CHECK(cudaEventRecord(c->ev_syy, c->syys));
          c->stream = c->aux;
        }
        c->stream = s0;
        c->lane = 0;
      } catch (...) {
        c->stream = s0;
        c->lane = 0;
        throw;
      }
      auto objective_part = [&]() {
        c->stream = c->aux;
        c->lane = 1;
        try {
          if (gated) CGGM_CUDA_CHECK(cudaStreamWaitEvent(c->aux, c->gate_ev, 0));
          if (c->factor_reuse)
            objective_fullinv_enqueue<T>(c, 1, n, q, Yd, ldy, W, ldn, Lambda, Theta, active->penalize_diag, xs_next);
          else
            objective_enqueue<T>(c, 1, n, q, Yd, ldy, W, ldn, Lambda, Theta, active->penalize_diag);
          CGGM_CUDA_CHECK(cudaEventRecord(c->ev_join, c->aux));
        } catch (...) {
          c->stream = s0;
          c->lane = 0;
          throw;
        }
        c->stream = s0;
        c->lane = 0;
      };
      if (!gated) objective_part();
      // a3, a4/a5, a6 on the chain stream (lane 0)
      if (hin) CGGM_CUDA_CHECK(cudaStreamWaitEvent(s0, hin->ev_lam, hin_wait));
      if (reuse_now)
        invert_from_kept<T>(c, 0, q, static_cast<T*>(Sigma), ldsigma, xs_prev);
      else
        invert_enqueue<T>(c, 0, Lambda, static_cast<T*>(Sigma), ldsigma, c->factor_reuse ? xs_prev : (int)WS_LINV);
      if (gated) {
        if (!c->gate_done) CGGM_CUDA_CHECK(cudaEventRecord(c->gate_ev, s0));   // (q below the gate column)
        c->gate_done = false;
        objective_part();
      }
      CGGM_CUDA_CHECK(cudaStreamWaitEvent(s0, c->ev_w, 0));
      if (hin) CGGM_CUDA_CHECK(cudaStreamWaitEvent(s0, c->ev_syy, 0));
      Fuse fz{Lambda, Theta, active, active_ws(c, q)};
      psi_enqueue<T>(c, n, n, p, q, Xd, ldx, Yd, ldy, W, ldn, static_cast<const T*>(Sigma), ldsigma,
                     static_cast<const T*>(Syy), ldsyy, nullptr, 0, static_cast<T*>(Psi), ldpsi,
                     static_cast<T*>(GradL), ldgl, static_cast<T*>(GradT), ldgt, &fz);
      tot = fz.ws.tot;
    });
    c->stream = so;
    if (c->prio_mode) {
      CGGM_CUDA_CHECK(cudaEventRecord(c->ev_join_hi, s0));
      CGGM_CUDA_CHECK(cudaStreamWaitEvent(so, c->ev_join_hi, 0));
    }
    CGGM_CUDA_CHECK(cudaStreamWaitEvent(so, c->ev_join, 0));
    if (c->factor_reuse) {   // keep the trial's (fail_col, log-det) with its inverse
      Scal s1 = scal_lane(c, 1, 0);
      char* kept = static_cast<char*>(ws_get(c, WS_REUSE_SCAL, 64 + 8));
      CGGM_CUDA_CHECK(cudaMemcpyAsync(kept, s1.fail, 4, cudaMemcpyDeviceToDevice, so));
      CGGM_CUDA_CHECK(cudaMemcpyAsync(kept + 64, s1.dbl, 8, cudaMemcpyDeviceToDevice, so));
    }
    chol_readback_async(c, 0, h);
    objective_readback_async(c, 1, h + 64);
    CGGM_CUDA_CHECK(cudaMemcpyAsync(h + 256, tot, sizeof(ActTotals), cudaMemcpyDeviceToHost, so));
  };
  // CUDA graph of the evaluation: the ~3000 launches of the two recursive factorisations would
  // otherwise be throttled by the launch queue (the host blocks enqueueing the first one while the
  // GPU works through it, so the second could not start alongside).  A new argument set runs
  // eagerly once (allocating anything missing), the second call with the same arguments captures.
  std::vector<int64_t> key = {n, p, q, ldx, ldy, ldsyy, ldsigma, ldpsi, ldgl, ldgt, (int64_t)c->ws_generation,
                              (int64_t)c->dtype, c->prio_mode, c->la_min, (int64_t)s_caller, c->sig_min, c->sig_min_f32};
  for (const void* ptr : {X, Y, Syy, (const void*)Sigma, (const void*)Psi, (const void*)GradL, (const void*)GradT})
    key.push_back((int64_t)ptr);
  for (const cggm_csc* m : {Lambda, Theta}) {
    key.insert(key.end(), {m->nrows, m->ncols, m->nnz, (int64_t)m->colptr, (int64_t)m->rowidx, (int64_t)m->val});
  }
  {
    const cggm_active_out* a = active;
    int64_t lb, tb;
    std::memcpy(&lb, &a->lam_L, 8);
    std::memcpy(&tb, &a->lam_T, 8);
    int64_t eb;
    std::memcpy(&eb, &a->tie_eps, 8);
    key.insert(key.end(), {lb, tb, eb, a->penalize_diag, a->cap_L, a->cap_T, (int64_t)a->L_row, (int64_t)a->L_col,
                           (int64_t)a->T_row, (int64_t)a->T_col});
  }
  // host inputs: the uploads run eagerly on the copy stream before the (captured) evaluation, which
  // waits for them through external event-wait nodes
  const bool graphs = c->use_graphs && !c->factor_reuse && (!c->prof || c->graph_prof);
  key.push_back(hin ? 1 : 0);
  key.push_back(c->prof ? 1 : 0);
  if (graphs && !c->gorigin) {
    // capture origin: an internal stream (the caller's may be the legacy default stream, which
    // cannot be captured); ordered after / before the caller's stream by events outside the graph
    int least = 0, greatest = 0;
    CGGM_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CGGM_CUDA_CHECK(cudaStreamCreateWithPriority(&c->gorigin, cudaStreamNonBlocking, greatest));
    CGGM_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_gpre, cudaEventDisableTiming));
    CGGM_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_gpost, cudaEventDisableTiming));
  }
  auto launch_graph = [&]() {
    CGGM_CUDA_CHECK(cudaEventRecord(c->ev_gpre, s_caller));
    CGGM_CUDA_CHECK(cudaStreamWaitEvent(c->gorigin, c->ev_gpre, 0));
    CGGM_CUDA_CHECK(cudaGraphLaunch(c->graph_exec, c->gorigin));
    CGGM_CUDA_CHECK(cudaEventRecord(c->ev_gpost, c->gorigin));
    CGGM_CUDA_CHECK(cudaStreamWaitEvent(s_caller, c->ev_gpost, 0));
  };
  if (graphs && c->graph_exec && key == c->graph_key) {
    launch_graph();
    c->launches += c->graph_launches;
    tot = c->graph_tot;
  } else if (graphs && key == c->graph_key_seen) {
    if (c->graph_exec) {
      cudaGraphExecDestroy(c->graph_exec);
      c->graph_exec = nullptr;
    }
    const int64_t l0 = c->launches;
    CGGM_CUDA_CHECK(cudaStreamBeginCapture(c->gorigin, cudaStreamCaptureModeRelaxed));
    cudaGraph_t g = nullptr;
    bool captured = true;
    try {
      hin_wait = cudaEventWaitExternal;
      enqueue(c->gorigin);
      hin_wait = 0;
    } catch (const CudaError& e) {
      captured = false;
      if (std::getenv("CGGM_GRAPH_DEBUG")) std::fprintf(stderr, "cggm: capture enqueue threw: %s\n", e.msg.c_str());
    } catch (...) {
      captured = false;
    }
    hin_wait = 0;
    c->stream = s_caller;
    c->lane = 0;
    cudaError_t ce = cudaStreamEndCapture(c->gorigin, &g);
    cudaError_t ie = cudaErrorUnknown;
    // node priorities: the chain / objective / side streams' priorities carry into the graph
    if (captured && ce == cudaSuccess && g)
      ie = cudaGraphInstantiateWithFlags(&c->graph_exec, g, cudaGraphInstantiateFlagUseNodePriority);
    if (g) cudaGraphDestroy(g);
    if (ie != cudaSuccess) {
      // something in the enqueue is not capturable here: run this and later calls eagerly
      if (std::getenv("CGGM_GRAPH_DEBUG"))
        std::fprintf(stderr, "cggm: graph capture failed (captured=%d end=%s instantiate=%s); eager from now on\n",
                     (int)captured, cudaGetErrorString(ce), cudaGetErrorString(ie));
      cudaGetLastError();
      c->graph_exec = nullptr;
      c->use_graphs = 0;
      c->launches = l0;
      enqueue(s_caller);
    } else {
      c->graph_launches = c->launches - l0;
      c->graph_key = key;
      c->graph_tot = tot;
      launch_graph();
    }
  } else {
    enqueue(s_caller);
    c->graph_key_seen = key;
  }
  CGGM_CUDA_CHECK(cudaStreamSynchronize(s_caller));
  if (c->factor_reuse) {
    c->reuse_buf ^= 1;   // this call's trial inverse is the next call's Sigma source
    c->reuse_valid = 1;
    c->reuse_q = q;
  }
  CholResult cr = chol_decode(h);
  out->logdet = cr.logdet;
  out->is_pd = cr.is_pd;
  out->fail_col = cr.fail_col;
  objective_decode(h + 64, n, active->lam_L, active->lam_T, &out->obj);
  ActTotals at;
  std::memcpy(&at, h + 256, sizeof(ActTotals));
  active_decode(at, active);
}

// ------------------------------------------------------------------ NEXT-4: memory-bounded evaluation
// The evaluation without any q x q matrix besides the factorisation's (the
// paper's block mode P:555-595, with triangular products of the GPU factor in place of
// CG): L^{-1} from the recursive full-inverse factorisation, then column blocks C of width b --
// pass 1: Sigma_C = L^{-T} L^{-1}_C (two GEMMs: the rows above C dense, the rows from C with the
// triangular k-range), R_C = W Sigma_C / sqrt n and E_C = Y_C + W Sigma_C (one GEMM, two
// epilogues), grad_Theta_C = (2/n) X^T E_C into its active-set chunk; pass 2 (R complete):
// grad_Lambda rows 0..j of each column j of C = Y^T Y_C / n - R^T R_C - Sigma[0:j1, C] into its
// active-set chunk.  The objective reuses L^{-1}: tr(Sigma M) = ||W L^{-T}||^2 / n.  The passes'
// buffers live in the dense-Lambda workspace the factorisation has finished with.
template <typename T>
static void newton_eval_blocked_impl(Ctx* c, int64_t n, int64_t p, int64_t q, const T* Xd, int64_t ldx, const T* Yd,
                                     int64_t ldy, const cggm_csc* Lambda, const cggm_csc* Theta, int64_t b,
                                     cggm_active_out* active, cggm_eval_out* out) {
  const int64_t ldq = pad_ld<T>(q), ldn = pad_ld<T>(n), ldp = pad_ld<T>(std::max<int64_t>(p, 1));
  const int64_t nleaves = n_leaves(q);
  // 1. L^{-1}, log-det, PD
  T* Xl = static_cast<T*>(ws_get(c, WS_LINV, (size_t)ldq * q * sizeof(T)));
  {
    T* A = static_cast<T*>(ws_get(c, WS_DENSE_A, (size_t)ldq * q * sizeof(T)));
    Scal s = scal_lane(c, 0, 8 + nleaves);
    double* slots = s.dbl + 8;
    densify_csc(c, Lambda, ViewT<T>{A, ldq, q, q});
    init_scalars(c, s.fail, s.flag);
    CGGM_CUDA_CHECK(cudaMemsetAsync(Xl, 0, (size_t)ldq * q * sizeof(T), c->stream));
    const size_t tmp_elems = chol_tmp_elems(q);
    T* tmp = static_cast<T*>(ws_get(c, WS_TMP, tmp_elems * sizeof(T)));
    potrf_recursive<T>(c, ViewT<T>{A, ldq, q, q}, ViewT<T>{Xl, ldq, q, q}, true, nullptr, slots, s.fail, tmp,
                       tmp_elems);
    sum_arrays_1(c, slots, nleaves, s.dbl);
  }
  char* h = static_cast<char*>(c->host_scratch);
  chol_readback_async(c, 0, h);
  CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  const CholResult cr = chol_decode(h);
  out->logdet = cr.logdet;
  out->is_pd = cr.is_pd;
  out->fail_col = cr.fail_col;
  if (!cr.is_pd) {
    out->obj.is_pd = 0;
    out->obj.fail_col = cr.fail_col;
    out->obj.f = out->obj.g = INFINITY;
    active->m_L = active->m_T = active->ties_L = active->ties_T = 0;
    active->subgrad_l1 = 0.0;
    return;
  }
  // 2. the block passes' buffers, carved out of the dense copy of Lambda (free after the
  // factorisation: the passes add no memory beyond the factorisation's peak, and nothing is
  // allocated per call); separate workspace slots only if they do not fit
  T *W, *R, *E, *SigC, *GLC, *GTC, *Z;
  {
    const size_t nq = (size_t)ldn * q, qb = (size_t)ldq * b, pb = (size_t)ldp * b;
    auto up = [](size_t e) { return (e + 31) & ~size_t(31); };   // 256-byte aligned carving
    const size_t need = 4 * up(nq) + 2 * up(qb) + up(pb);
    if (need <= (size_t)ldq * q) {
      T* pool = static_cast<T*>(ws_get(c, WS_DENSE_A, (size_t)ldq * q * sizeof(T)));
      W = pool;
      R = W + up(nq);
      E = R + up(nq);
      Z = E + up(nq);
      SigC = Z + up(nq);
      GLC = SigC + up(qb);
      GTC = GLC + up(qb);
    } else {
      W = static_cast<T*>(ws_get(c, WS_W, nq * sizeof(T)));
      R = static_cast<T*>(ws_get(c, WS_R, nq * sizeof(T)));
      E = static_cast<T*>(ws_get(c, WS_E, nq * sizeof(T)));
      Z = static_cast<T*>(ws_get(c, WS_Z, nq * sizeof(T)));
      SigC = static_cast<T*>(ws_get(c, WS_BLK_S, qb * sizeof(T)));
      GLC = static_cast<T*>(ws_get(c, WS_BLK_G, qb * sizeof(T)));
      GTC = static_cast<T*>(ws_get(c, WS_GTCHUNK, pb * sizeof(T)));
    }
  }
  spmm_x_theta<T>(c, Xd, ldx, n, Theta, ViewT<T>{W, ldn, n, q});
  ActWs aws = active_ws(c, q);
  active_begin(c, q, aws);
  const double rs = 1.0 / std::sqrt((double)n);
  // pass 1
  for (int64_t j0 = 0; j0 < q; j0 += b) {
    const int64_t bc = std::min<int64_t>(b, q - j0);
    {  // Sigma_C: rows [0, j0) dense, rows [j0, q) with the k-range starting at the row block
      Phase ph(c, TAG_LAUUM);
      EpilogueT<T> e; e.out1 = SigC; e.ld1 = ldq;
      if (j0 > 0) gemm(c, true, false, j0, bc, q - j0, Xl + j0, ldq, Xl + j0 + j0 * ldq, ldq, e, 0);
      EpilogueT<T> e2; e2.out1 = SigC + j0; e2.ld1 = ldq;
      gemm(c, true, false, q - j0, bc, q - j0, Xl + j0 + j0 * ldq, ldq, Xl + j0 + j0 * ldq, ldq, e2, A_KGE_M);
    }
    {  // R_C = W Sigma_C / sqrt n, E_C = Y_C + W Sigma_C
      Phase ph(c, TAG_WSIGMA);
      EpilogueT<T> e; e.out1 = R + j0 * ldn; e.ld1 = ldn; e.a1 = rs;
      e.out2 = E + j0 * ldn; e.ld2 = ldn; e.a2 = 1.0; e.in2a = Yd + j0 * ldy; e.ld2a = ldy; e.b2 = 1.0;
      gemm(c, false, false, n, bc, q, W, ldn, SigC, ldq, e, 0);
    }
    if (p > 0) {  // grad_Theta_C = (2/n) X^T E_C and its active-set chunk
      Phase ph(c, TAG_GRADT);
      EpilogueT<T> e; e.out1 = GTC; e.ld1 = ldp; e.a1 = 2.0 / (double)n;
      gemm(c, true, false, p, bc, n, Xd, ldx, E + j0 * ldn, ldn, e, 0);
      active_theta_chunk<T>(c, p, j0, bc, GTC, ldp, Theta, active->lam_T, active->tie_eps, aws, active->T_row,
                            active->T_col, active->cap_T);
    }
  }
  // pass 2: grad_Lambda rows 0..j1 of block C = S_yy - Sigma - Psi, its active-set chunk
  for (int64_t j0 = 0; j0 < q; j0 += b) {
    const int64_t bc = std::min<int64_t>(b, q - j0), j1 = j0 + bc;
    Phase ph(c, TAG_GRADL);
    {
      EpilogueT<T> e; e.out1 = GLC; e.ld1 = ldq; e.a1 = 1.0 / (double)n;
      gemm(c, true, false, j1, bc, n, Yd, ldy, Yd + j0 * ldy, ldy, e, 0);                 // S_yy[0:j1, C]
    }
    {
      EpilogueT<T> e; e.out1 = GLC; e.ld1 = ldq; e.a1 = -1.0; e.in1a = GLC; e.ld1a = ldq; e.b1 = 1.0;
      gemm(c, true, false, j1, bc, q - j0, Xl + j0, ldq, Xl + j0 + j0 * ldq, ldq, e, 0);  // - Sigma[0:j1, C]
    }
    {
      EpilogueT<T> e; e.out1 = GLC; e.ld1 = ldq; e.a1 = -1.0; e.in1a = GLC; e.ld1a = ldq; e.b1 = 1.0;
      gemm(c, true, false, j1, bc, n, R, ldn, R + j0 * ldn, ldn, e, 0);                     // - Psi[0:j1, C]
    }
    active_lambda_chunk<T>(c, q, j0, bc, GLC, ldq, Lambda, active->lam_L, active->penalize_diag, active->tie_eps,
                           aws, active->L_row, active->L_col, active->cap_L);
  }
  active_end(c, q, aws);
  // 4. objective at Lambda with the same factor: tr(Sigma M) = ||W L^{-T}||^2 / n
  {
    Phase ph(c, TAG_TRSM);
    EpilogueT<T> e; e.out1 = Z; e.ld1 = ldn;
    gemm(c, false, true, n, q, q, W, ldn, Xl, ldq, e, B_KLE_N);
  }
  Scal s2 = scal_lane(c, 1, 16 + 5 * q);
  double* res = s2.dbl;
  double* partY = res + 16;
  double* partWY = partY + q;
  double* partZ = partWY + q;
  double* penLp = partZ + q;
  double* penTp = penLp + q;
  {
    Phase ph(c, TAG_OBJRED);
    col_partials<T>(c, 0, n, q, Yd, ldy, nullptr, 0, Lambda, partY);
    col_partials<T>(c, 1, n, q, W, ldn, Yd, ldy, nullptr, partWY);
    col_partials<T>(c, 2, n, q, Z, ldn, nullptr, 0, nullptr, partZ);
    csc_abs_partials<T>(c, Lambda, active->penalize_diag == 0, penLp);
    csc_abs_partials<T>(c, Theta, false, penTp);
    sum_arrays_1(c, partY, q, res + 1);
    sum_arrays_1(c, partWY, q, res + 2);
    sum_arrays_1(c, partZ, q, res + 3);
    sum_arrays_1(c, penLp, q, res + 4);
    sum_arrays_1(c, penTp, q, res + 5);
  }
  CGGM_CUDA_CHECK(cudaMemcpyAsync(h + 256, aws.tot, sizeof(ActTotals), cudaMemcpyDeviceToHost, c->stream));
  CGGM_CUDA_CHECK(cudaMemcpyAsync(h + 512, res, 6 * 8, cudaMemcpyDeviceToHost, c->stream));
  CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  double v[6];
  std::memcpy(v, h + 512, 6 * 8);
  const double nt = (double)n;
  cggm_objective_out& o = out->obj;
  o.is_pd = 1;
  o.fail_col = -1;
  o.logdet = cr.logdet;
  o.pen_L = active->lam_L * v[4];
  o.pen_T = active->lam_T * v[5];
  o.tr_syy_lam = v[1] / nt;
  o.tr_sxy_theta = v[2] / nt;
  o.tr_sigma_m = v[3] / nt;
  o.g = -o.logdet + o.tr_syy_lam + 2.0 * o.tr_sxy_theta + o.tr_sigma_m;
  o.f = o.g + o.pen_L + o.pen_T;
  ActTotals at;
  std::memcpy(&at, h + 256, sizeof(ActTotals));
  active_decode(at, active);
}

cggm_status cggm_newton_eval_blocked(cggm_ctx* ctx, int64_t n, int64_t p, int64_t q, const void* X, int64_t ldx,
                                     const void* Y, int64_t ldy, const cggm_csc* Lambda, const cggm_csc* Theta,
                                     int64_t block, cggm_active_out* active, cggm_eval_out* out) {
  return guard(ctx, [&](Ctx* c) {
    if (!out) fail(CGGM_ERR_INVALID_ARG, "null cggm_eval_out");
    if (c->comm.world > 1) fail(CGGM_ERR_UNSUPPORTED, "the memory-bounded evaluation is single-GPU");
    if (n < 1 || p < 0 || q < 1) fail(CGGM_ERR_INVALID_ARG, "need n >= 1, q >= 1, p >= 0");
    if (block < 0) fail(CGGM_ERR_INVALID_ARG, "negative block width");
    check_dense("X", X, n, p, ldx);
    check_dense("Y", Y, n, q, ldy);
    check_csc_host("Lambda", Lambda, q, q);
    check_csc_host("Theta", Theta, p, q);
    check_active_args(active);
    std::memset(out, 0, sizeof(*out));
    validate_csc_dev(c, Lambda, true, "Lambda");
    validate_csc_dev(c, Theta, false, "Theta");
    int64_t b = block > 0 ? block : 1024;   // measured best at large (1024: 544 ms, 2048: 558, 4096: 577)
    b = std::min<int64_t>((b + 1) & ~int64_t(1), q);
    dispatch(c, [&](auto tag) {
      using T = decltype(tag);
      newton_eval_blocked_impl<T>(c, n, p, q, static_cast<const T*>(X), ldx, static_cast<const T*>(Y), ldy, Lambda,
                                  Theta, b, active, out);
    });
  });
}

cggm_status cggm_newton_eval(cggm_ctx* ctx, int64_t n, int64_t p, int64_t q, const void* X, int64_t ldx,
                             const void* Y, int64_t ldy, const void* Syy, int64_t ldsyy, const cggm_csc* Lambda,
                             const cggm_csc* Theta, void* Sigma, int64_t ldsigma, void* Psi, int64_t ldpsi,
                             void* GradL, int64_t ldgl, void* GradT, int64_t ldgt, cggm_active_out* active,
                             cggm_eval_out* out) {
  return guard(ctx, [&](Ctx* c) {
    newton_eval_core(c, n, p, q, X, ldx, Y, ldy, Syy, ldsyy, Lambda, Theta, Sigma, ldsigma, Psi, ldpsi, GradL, ldgl,
                     GradT, ldgt, active, out, nullptr);
  });
}

cggm_status cggm_newton_eval_host(cggm_ctx* ctx, int64_t n, int64_t p, int64_t q, const double* X, int64_t ldx,
                                  const double* Y, int64_t ldy, const cggm_csc* Lambda, const cggm_csc* Theta,
                                  void* Syy, int64_t ldsyy, void* Sigma, int64_t ldsigma, void* Psi, int64_t ldpsi,
                                  void* GradL, int64_t ldgl, void* GradT, int64_t ldgt, cggm_active_out* active,
                                  cggm_eval_out* out) {
  return guard(ctx, [&](Ctx* c) {
    check_ctx_dtype(c);
    if (n < 1 || p < 0 || q < 1) fail(CGGM_ERR_INVALID_ARG, "need n >= 1, q >= 1, p >= 0");
    if (!X && p > 0) fail(CGGM_ERR_INVALID_ARG, "null X");
    if (!Y) fail(CGGM_ERR_INVALID_ARG, "null Y");
    if (ldx < n || ldy < n) fail(CGGM_ERR_INVALID_ARG, "leading dimension < n");
    check_csc_host("Lambda", Lambda, q, q);
    check_csc_host("Theta", Theta, p, q);
    if (!c->copy) {
      CGGM_CUDA_CHECK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
      CGGM_CUDA_CHECK(cudaStreamCreateWithPriority(&c->syys, cudaStreamNonBlocking, stream_priority(9)));
      for (cudaEvent_t* e : {&c->ev_h_lam, &c->ev_h_xt, &c->ev_h_y})
        CGGM_CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    // device copies (workspace), ordered Lambda, Theta + X, Y so that the factorisation can start first
    const int64_t ldxd = pad_ld<double>(n);
    auto up = [&](int slot, const void* src, size_t bytes) -> void* {
      void* d = ws_get(c, slot, std::max<size_t>(bytes, 16));
      if (bytes) CGGM_CUDA_CHECK(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, c->copy));
      return d;
    };
    CGGM_CUDA_CHECK(cudaEventRecord(c->ev_h_lam, c->stream));   // after the caller's prior work
    CGGM_CUDA_CHECK(cudaStreamWaitEvent(c->copy, c->ev_h_lam, 0));
    cggm_csc Ld = *Lambda, Td = *Theta;
    Ld.colptr = static_cast<const int64_t*>(up(WS_H_LCP, Lambda->colptr, (size_t)(q + 1) * 8));
    Ld.rowidx = static_cast<const int32_t*>(up(WS_H_LRI, Lambda->rowidx, (size_t)Lambda->nnz * 4));
    Ld.val = up(WS_H_LVA, Lambda->val, (size_t)Lambda->nnz * 8);
    CGGM_CUDA_CHECK(cudaEventRecord(c->ev_h_lam, c->copy));
    Td.colptr = static_cast<const int64_t*>(up(WS_H_TCP, Theta->colptr, (size_t)(q + 1) * 8));
    Td.rowidx = static_cast<const int32_t*>(up(WS_H_TRI, Theta->rowidx, (size_t)Theta->nnz * 4));
    Td.val = up(WS_H_TVA, Theta->val, (size_t)Theta->nnz * 8);
    double* Xd = static_cast<double*>(ws_get(c, WS_H_X, (size_t)ldxd * std::max<int64_t>(p, 1) * 8));
    double* Yd = static_cast<double*>(ws_get(c, WS_H_Y, (size_t)ldxd * q * 8));
    // structure checks of the uploaded CSCs on the copy stream (they synchronise it: before the large
    // X, Y uploads are enqueued, so only the small CSC copies are waited for)
    {
      struct S {
        Ctx* c;
        cudaStream_t prev;
        ~S() { c->stream = prev; }
      } s_{c, c->stream};
      c->stream = c->copy;
      validate_csc_dev(c, &Ld, true, "Lambda");
      validate_csc_dev(c, &Td, false, "Theta");
    }
    if (p > 0)
      CGGM_CUDA_CHECK(cudaMemcpy2DAsync(Xd, ldxd * 8, X, ldx * 8, n * 8, p, cudaMemcpyHostToDevice, c->copy));
    CGGM_CUDA_CHECK(cudaEventRecord(c->ev_h_xt, c->copy));
    CGGM_CUDA_CHECK(cudaMemcpy2DAsync(Yd, ldxd * 8, Y, ldy * 8, n * 8, q, cudaMemcpyHostToDevice, c->copy));
    CGGM_CUDA_CHECK(cudaEventRecord(c->ev_h_y, c->copy));
    HostIn hin{c->ev_h_lam, c->ev_h_xt, c->ev_h_y};
    newton_eval_core(c, n, p, q, Xd, ldxd, Yd, ldxd, Syy, ldsyy, &Ld, &Td, Sigma, ldsigma, Psi, ldpsi, GradL, ldgl,
                     GradT, ldgt, active, out, &hin);
  });
}

extern "C" cggm_status cggm_test_gemm(cggm_ctx* ctx, int transA, int transB, int64_t M, int64_t N, int64_t K,
                                      const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                                      int64_t ldc, double alpha, double beta, int flags) {
  return guard(ctx, [&](Ctx* c) {
    if (M < 0 || N < 0 || K < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    Epilogue e;
    e.out1 = C; e.ld1 = ldc; e.a1 = alpha;
    if (beta != 0.0) { e.in1a = C; e.ld1a = ldc; e.b1 = beta; }
    gemm(c, transA != 0, transB != 0, M, N, K, A, lda, B, ldb, e, flags);
  });
}

extern "C" cggm_status cggm_test_gemm_mir(cggm_ctx* ctx, int transA, int transB, int64_t M, int64_t N, int64_t K,
                                          const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                                          int64_t ldc, double* Cmir, double alpha, int flags) {
  return guard(ctx, [&](Ctx* c) {
    if (M < 0 || N < 0 || K < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    Epilogue e;
    e.out1 = C; e.ld1 = ldc; e.a1 = alpha; e.mir1 = Cmir;
    gemm(c, transA != 0, transB != 0, M, N, K, A, lda, B, ldb, e, flags | SYM_MIRROR);
  });
}

extern "C" cggm_status cggm_test_gemm_f32(cggm_ctx* ctx, int transA, int transB, int64_t M, int64_t N, int64_t K,
                                          const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                                          int64_t ldc, double alpha, double beta, int flags) {
  return guard(ctx, [&](Ctx* c) {
    if (M < 0 || N < 0 || K < 0) fail(CGGM_ERR_INVALID_ARG, "negative dimension");
    EpilogueT<float> e;
    e.out1 = C; e.ld1 = ldc; e.a1 = alpha;
    if (beta != 0.0) { e.in1a = C; e.ld1a = ldc; e.b1 = beta; }
    gemm(c, transA != 0, transB != 0, M, N, K, A, lda, B, ldb, e, flags);
  });
}

extern "C" cggm_status cggm_test_chol_dense(cggm_ctx* ctx, double* A, int64_t lda, int64_t q, double* X, int64_t ldx,
                                            int full_inverse, double* logdet, int64_t* fail_col) {
  return guard(ctx, [&](Ctx* c) {
    if (c->dtype != CGGM_F64) fail(CGGM_ERR_UNSUPPORTED, "cggm_test_chol_dense is fp64");
    if (!A || q < 1 || lda < q || lda % 2) fail(CGGM_ERR_INVALID_ARG, "need q >= 1 and an even lda >= q");
    if (full_inverse && (!X || ldx < q || ldx % 2)) fail(CGGM_ERR_INVALID_ARG, "need X with an even ldx >= q");
    const int nb = leaf_nb();
    const int64_t nleaves = n_leaves(q);
    Scal s = scal_lane(c, 0, 8 + nleaves);
    double* slots = s.dbl + 8;
    init_scalars(c, s.fail, s.flag);
    ViewT<double> Av{A, lda, q, q};
    if (full_inverse) {
      CGGM_CUDA_CHECK(cudaMemsetAsync(X, 0, (size_t)ldx * q * 8, c->stream));
      const size_t tmp_elems = chol_tmp_elems(q);
      double* tmp = static_cast<double*>(ws_get(c, WS_TMP, tmp_elems * 8));
      potrf_recursive<double>(c, Av, ViewT<double>{X, ldx, q, q}, true, nullptr, slots, s.fail, tmp, tmp_elems);
    } else {
      double* leafinv = static_cast<double*>(ws_get(c, WS_LEAFINV, (size_t)nleaves * nb * nb * 8));
      potrf_recursive<double>(c, Av, ViewT<double>{nullptr, lda, q, q}, false, leafinv, slots, s.fail, nullptr, 0);
    }
    sum_arrays_1(c, slots, nleaves, s.dbl);
    if (logdet || fail_col) {
      char* h = static_cast<char*>(c->host_scratch);
      chol_readback_async(c, 0, h);
      CGGM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
      CholResult r = chol_decode(h);
      if (logdet) *logdet = r.logdet;
      if (fail_col) *fail_col = r.fail_col;
    }
  });
}

extern "C" cggm_status cggm_test_profile_dump(cggm_ctx* ctx, const char* path) {
  return guard(ctx, [&](Ctx* c) {
    if (!path) fail(CGGM_ERR_INVALID_ARG, "null path");
    CGGM_CUDA_CHECK(cudaDeviceSynchronize());
    FILE* f = std::fopen(path, "w");
    if (!f) fail(CGGM_ERR_INVALID_ARG, "cannot open profile dump path");
    std::fprintf(f, "tag,stream,start_ms,end_ms\n");
    std::vector<cudaStream_t> seen;
    if (!c->prof_recs.empty()) {
      std::vector<unsigned long long> ts;
      if (c->ts_buf) {
        ts.resize(c->evnext);
        CGGM_CUDA_CHECK(cudaMemcpy(ts.data(), c->ts_buf, c->evnext * 8, cudaMemcpyDeviceToHost));
      }
      unsigned long long t0 = ~0ull;
      for (const auto& r : c->prof_recs)
        if (c->ts_buf) t0 = std::min(t0, ts[r.a]);
      cudaEvent_t ref = c->ts_buf ? nullptr : c->evpool[c->prof_recs.front().a];
      for (const auto& r : c->prof_recs) {
        size_t si = 0;
        while (si < seen.size() && seen[si] != r.stream) ++si;
        if (si == seen.size()) seen.push_back(r.stream);
        float a = 0.f, b = 0.f;
        if (c->ts_buf) {
          a = (float)((ts[r.a] - t0) * 1e-6);
          b = (float)((ts[r.b] - t0) * 1e-6);
        } else {
          CGGM_CUDA_CHECK(cudaEventElapsedTime(&a, ref, c->evpool[r.a]));
          CGGM_CUDA_CHECK(cudaEventElapsedTime(&b, ref, c->evpool[r.b]));
        }
        std::fprintf(f, "%s,%zu,%.4f,%.4f\n", cggm_profile_tag_name(r.tag), si, a, b);
      }
    }
    std::fclose(f);
  });
}

extern "C" cggm_status cggm_test_set_tile(cggm_ctx* ctx, int mode) {
  if (!ctx || mode < 0 || mode > 6) return CGGM_ERR_INVALID_ARG;
  ctx->impl.force_tile = mode & 3;
  ctx->impl.no_tma3d = (mode & 4) ? 1 : 0;
  return CGGM_OK;
}

extern "C" cggm_status cggm_test_set_f32_engine(cggm_ctx* ctx, int engine) {
  if (!ctx || engine < 0 || engine > 4) return CGGM_ERR_INVALID_ARG;
  ctx->impl.f32_engine = engine == 1 ? 1 : 0;
  if (engine >= 2) ctx->impl.tf32_producer = engine - 2;   // 2: TMA, 3: register-staged, 4: TS form
  return CGGM_OK;
}
