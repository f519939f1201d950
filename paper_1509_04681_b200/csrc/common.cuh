// Shared internals of libcggm: context, workspace, launch accounting, PTX helpers
// (mbarrier, TMA, DMMA) for sm_100a.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/cggm.h"

namespace cggm {

// ------------------------------------------------------------------ context
struct Buffer {
  void* ptr = nullptr;
  size_t bytes = 0;
};

enum ProfTag {
  TAG_MISC = 0,    // validation, init, copies
  TAG_COV,         // S_yy / S_xy GEMMs
  TAG_DENSIFY,     // CSC -> dense
  TAG_CHOL_GEMM,   // Cholesky / triangular-inverse / trsm GEMMs inside the recursion
  TAG_CHOL_LEAF,   // leaf potrf + trtri kernels
  TAG_LAUUM,       // Sigma = L^{-T} L^{-1}
  TAG_SPMM,        // W = X Theta
  TAG_WSIGMA,      // acc = W Sigma (R, E)
  TAG_PSI,         // Psi = R^T R (+ grad_Lambda epilogue)
  TAG_GRADT,       // grad_Theta = (2/n) X^T E
  TAG_TRSM,        // objective triangular solve W L^{-T}
  TAG_ACTIVE,      // active-set count / scan / write
  TAG_OBJRED,      // objective reductions
  TAG_GRADL,       // grad_Lambda = (S_yy - Sigma) - Psi streaming pass
  TAG_NUM
};

struct ActTotals;

// attached communicator (sample sharding; cggm_comm_init / _external)
struct CommState {
  int kind = 0;   // 0 none, 1 NCCL, 2 external callbacks
  int rank = 0, world = 1;
  void* nccl = nullptr;   // ncclComm_t
  cggm_allreduce_fn ar = nullptr;
  cggm_broadcast_fn bc = nullptr;
  void* user = nullptr;
};

struct Ctx {
  int device = 0;
  cggm_dtype dtype = CGGM_F64;
  cudaStream_t stream = nullptr;
  int validate = 1;
  int64_t launches = 0;
  std::string last_error;
  // named workspace slots (grown on demand, never shrunk until release)
  std::vector<Buffer> slots;
  // pinned host scratch for scalar read-back
  void* host_scratch = nullptr;
  PFN_cuTensorMapEncodeTiled_v12000 encode_tiled = nullptr;
  int num_sms = 148;
  int lane = 0;                  // 0: caller's stream, 1: auxiliary stream (separate workspace)
  cudaStream_t aux = nullptr;    // auxiliary stream of the composite evaluation
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t hi = nullptr;     // high-priority stream of the composite evaluation's critical chain
  cudaEvent_t ev_join_hi = nullptr;
  cudaEvent_t ev_w = nullptr, ev_syy = nullptr;      // composite: W ready (lane 1 -> chain); S_yy ready (host inputs)
  cudaStream_t copy = nullptr;                         // host-input uploads (cggm_newton_eval_host)
  cudaStream_t syys = nullptr;                         // host-input S_yy (priority between chain and objective)
  cudaEvent_t ev_h_lam = nullptr, ev_h_xt = nullptr, ev_h_y = nullptr;
  // recursive-factorisation lookahead (chol.cu): per lane a critical-chain stream and two side
  // streams (deferred trailing updates, deferred block products) at decreasing priorities, and a
  // pool of dependency events (reused across calls: every wait is enqueued before a re-record)
  cudaStream_t la_chain[2] = {nullptr, nullptr}, la_upd[2] = {nullptr, nullptr}, la_bg[2] = {nullptr, nullptr};
  cudaStream_t la_sig = nullptr;   // interleaved Sigma assembly (chol.cu), priority slot 8
  // composite: the objective's trial factorisation starts once the inverse recursion reaches column
  // gate_cols (CGGM_OBJ_GATE; 0 = both start together)
  int64_t gate_cols = 0;
  cudaEvent_t gate_ev = nullptr;
  bool gate_done = false;
  cudaStream_t gl_side = nullptr;  // composite: grad_Lambda + the S_Lambda compaction beside the X^T E GEMM
  int pdl = 0;                     // CGGM_PDL=1: programmatic dependent launch for the recursion's kernels (leaves, FP64
                                   // GEMMs): recursion latency -9..-13% alone, the `large` steps (FP64, FP32) unchanged
  int k01 = 0;                     // CGGM_K01=1: grad_Theta = NULL selects S_Theta in the X^T E epilogue (K01) instead of
                                   // streaming column chunks through the scan (measured slower: see DESIGN §6)
  int gl_overlap = 0;              // CGGM_GL_OVERLAP: 1 = side stream at the greatest priority, 2 = at the least, 0 = in line
  cudaEvent_t ev_gl0 = nullptr, ev_gl1 = nullptr;
  int sig_min = 4096;              // CGGM_SIGMA_REC: nodes >= this split their Sigma block (0 = one lauum after the recursion)
  int sig_min_f32 = 0;             // the same for the FP32 variant (CGGM_SIGMA_REC_F32; measured slower at `large`: off)
  std::vector<cudaEvent_t> la_events;
  size_t la_next = 0;
  int la_min = 256;              // defer only when the deferred block is at least this wide (CGGM_LA_MIN; 0 = off)
  int prio_mode = 1;             // composite: 1 = chain on `hi` (greatest priority), objective on `aux`
                                 // (least priority); 0 = chain on the caller's stream (CGGM_PRIO=0)
  // factor reuse (CGGM_OPT_FACTOR_REUSE): the objective's trial factorisation runs in full-inverse
  // mode and keeps L^{-1} (buffer reuse_buf ^ 1 of {WS_LINV, WS_LINV2}); the next evaluation's
  // Sigma is lauum of it.  The caller guarantees the next Lambda is that trial Lambda.
  int factor_reuse = 0;
  int reuse_valid = 0;
  int reuse_buf = 0;
  int64_t reuse_q = -1;
  // CUDA graph of the composite evaluation (cggm_newton_eval), keyed by its full argument set
  int use_graphs = 1;            // CGGM_GRAPH=0 disables
  int graph_prof = 0;            // CGGM_GRAPH_PROF=1: capture the profiling events too (timelines)
  uint64_t ws_generation = 0;    // bumped by every workspace (re)allocation
  cudaGraphExec_t graph_exec = nullptr;
  cudaStream_t gorigin = nullptr;   // capture / launch stream of the graph
  cudaEvent_t ev_gpre = nullptr, ev_gpost = nullptr;
  std::vector<int64_t> graph_key, graph_key_seen;
  int64_t graph_launches = 0;
  ActTotals* graph_tot = nullptr;
  int force_tile = 0;
  int small_kmax = 1024;    // mid-size GEMMs (64-tile grid < #SMs) with K <= this use the 32x32 cp.async kernel (CGGM_SMALL_KMAX)
  int leaf_sweep = 0;       // CGGM_LEAF_SWEEP=1: full-inverse leaves by the panel/sweep kernel (A/B)
  int cd_prefetch = 1;      // CGGM_CD_PREFETCH=0: cooperative Theta sweep without the register/prefetch variant
  int cd_coop = 1;          // CGGM_CD_COOP=0: single-CTA coordinate sweeps (no column batching)
  int cd_panel = -1;        // CGGM_CD_PANEL: panel width of the left-looking blocked Lambda sweep (-1: 512 above the register limit, 0: off)
  int cd_block = -1;        // CGGM_CD_BLOCK: entry-blocked sweeps (-1: when the vector exceeds the register variant, 0: never, 1: always)
  int mid_min_waves = 0;    // CGGM_MID_MIN_WAVES: mid-size products on the 128x64 tiles from this many quarter waves (0 = off)
  int mid_tile = 3;         // CGGM_MID_TILE (3): 128x64 warp-specialised tiles, 2 CTAs/SM, for the large GEMMs (gemm.cu)
  int no_small_async = 0;
  int no_active_vec = 0;
  int act_onepass = 0;
  int no_split_k = 0;   // CGGM_NO_SPLIT_K=1: W Sigma without the split-k grid (A/B)
  int no_vec_epi = 0;
  int persist_tpc = 0;   // CGGM_PERSIST_TPC: tiles per CTA of the persistent warp-specialised GEMM (0: off)   // CGGM_NO_VEC_EPI=1: scalar GEMM epilogue everywhere (A/B)      // CGGM_ACT_ONEPASS=1: Lambda list by the single-pass look-back kernel (not the split one)    // test hook (CGGM_NO_ACTIVE_VEC=1): scalar active-set kernel only   // test hook (CGGM_NO_SMALL_ASYNC=1): direct-load small kernel only
  int fuse_gradl = 0;   // CGGM_FUSE_GRADL=1: grad_Lambda as the Psi GEMM's second epilogue output (measured: the
                        // two-input mirrored epilogue costs the K = n GEMM more than the 1.8 ms pass it saves)
  int sync_check = 0;   // CGGM_SYNC_CHECK=1: synchronise after every launch (fault localisation, see post_launch)
  int tf32_dbg = 0;     // CGGM_TF32_DEBUG (gemm_tf32.cu measurement aid)
  int tf32_producer = 2;   // 3xTF32 form (CGGM_TF32_PRODUCER): 2 = TS (A hi / lo in TMEM, B in shared memory; default),
                           // 0 = SS with the TMA raw ring + converters ("tma"), 1 = SS with register-staged loads ("ldg")
  int tf32_min_tiles = 0;  // FP32 products with fewer 128x128 tiles than this run on FFMA (CGGM_TF32_MIN_TILES)
  int tf32_min_k = 256;    // ... or with K below this (CGGM_TF32_MIN_K; 256 measured best: FP32 medium 9.5 ms, large 146 ms)
  int tf32_cfrel = 0;      // CGGM_TF32_CFREL=1: TS split stages released by the chunk commits (measured neutral)
  int tf32_ts_chunk = 2;   // TS form: k-tiles per drained chunk (CGGM_TF32_TS_CHUNK)
  int tf32_chunk = 4;   // 3xTF32: k-tiles per drained TMEM partial (gemm_tf32.cu; CGGM_TF32_CHUNK, 0 = none)
  int f32_engine = 0;   // FP32 contractions: 0 = 3xTF32 on tcgen05 (gemm_tf32.cu), 1 = SIMT FFMA (CGGM_F32_ENGINE=ffma)
  int no_tma3d = 0;   // test hook: 1 = always use 16-wide 2-D boxes for MN-inner operands  // test hook: 0 auto, 1 = 128x128 tiles, 2 = 64x64 tiles
  // phase profiling (CUDA events around every launch while enabled)
  int cur_tag = TAG_MISC;
  bool prof = false;
  std::vector<cudaEvent_t> evpool;
  unsigned long long* ts_buf = nullptr;   // CGGM_PROF_TS=1: device timestamps instead of events (graph-safe)
  size_t ts_cap = 0;
  size_t evnext = 0;
  struct ProfRec {
    int tag, a, b;
    cudaStream_t stream;
  };
  std::vector<ProfRec> prof_recs;
  CommState comm;
};

// RAII event pair around one launch (no-op unless profiling is enabled)
void prof_stamp(Ctx* c, int idx);
// stream priority of internal stream `which` (0 hi, 1 aux, 2..4 lane-0 chain/upd/bg, 5..7 lane-1):
// offsets from the greatest priority, CGGM_PRIO_SCHEME="h,a,c0,u0,b0,c1,u1,b1" overrides
int stream_priority(int which);   // stream.cu: one-thread kernel writing %globaltimer to ts_buf[idx]

struct Prof {
  Ctx* c;
  int tag;
  int ia = -1;
  Prof(Ctx* c_, int tag_) : c(c_), tag(tag_) {
    if (!c->prof) return;
    ia = take();
    if (c->ts_buf) prof_stamp(c, ia);
    else cudaEventRecord(c->evpool[ia], c->stream);
  }
  ~Prof() {
    if (ia < 0) return;
    int ib = take();
    if (c->ts_buf) prof_stamp(c, ib);
    else cudaEventRecord(c->evpool[ib], c->stream);
    c->prof_recs.push_back(Ctx::ProfRec{tag, ia, ib, c->stream});
  }
  int take() {
    if (c->ts_buf) return (int)(c->evnext < c->ts_cap ? c->evnext++ : c->ts_cap - 1);
    if (c->evnext == c->evpool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      c->evpool.push_back(e);
    }
    return (int)c->evnext++;
  }
};

// scoped phase tag
// a phase of the hot path: the tag the profiler attributes launches to, and an NVTX range of the
// same name (visible in nsys / ncu --nvtx; a no-op without an attached tool)
struct Phase {
  Ctx* c;
  int prev;
  Phase(Ctx* c_, int tag) : c(c_), prev(c_->cur_tag) {
    c->cur_tag = tag;
    nvtxRangePushA(cggm_profile_tag_name(tag));
  }
  ~Phase() {
    nvtxRangePop();
    c->cur_tag = prev;
  }
};

enum Slot {
  WS_DENSE_A = 0,   // dense Lambda -> Cholesky factor (q x q)
  WS_LINV,          // L^{-1} (q x q)
  WS_TMP,           // recursion temporaries
  WS_LEAFINV,       // compact leaf inverses (potrf-only mode)
  WS_W,             // W = X Theta (n x q)
  WS_R,             // R (n x q)
  WS_E,             // E (n x q)
  WS_Z,             // trsm result (n x q)
  WS_SCAL,          // small device scalars / partial-sum arrays
  WS_ACT,           // active-set per-column arrays
  WS_ACC,           // split-k W Sigma accumulator (n x q)
  WS_BLK_S,         // memory-bounded evaluation: a Sigma column block (q x b)
  WS_BLK_G,         // memory-bounded evaluation: a grad_Lambda column block (q x b)
  WS_COMM,          // broadcast scalars (sample sharding)
  WS_PACK0,         // packing for TMA-incompatible operands (lane 0: 0/1, lane 1: 2/3)
  WS_PACK1,
  WS_PACK2,
  WS_PACK3,
  WS_DENSE_B,       // augmented [Lambda; W] of the objective on the auxiliary lane
  WS_XDIAG,         // objective: inverses of the <= 512-column diagonal blocks (q x 512)
  WS_TMP_OBJ,       // objective: recursion temporaries (full-inverse subtrees + block products)
  WS_GTCHUNK,       // streamed grad_Theta column chunk (fused active sets without a stored p x q gradient)
  WS_SEL,           // K01: S_Theta selected in the X^T E epilogue (flag words, column bases, subgradient partials)
  WS_SCAL2,         // scalar block of the auxiliary lane
  WS_CD_U,          // Lambda sweep: U = D Sigma (q x q)
  WS_CD_V,          // Theta sweep: V = Theta Sigma (p x q)
  WS_CD_IDX,        // list -> CSC counts / scans
  WS_CD_OUT,        // sweep scalars
  WS_CD_COEF,       // per-entry sweep constants
  WS_CD_Z,          // Lambda sweep: Z = D Psi (q x q, row-major)
  WS_LINV2,         // factor reuse: the second L^{-1} buffer (the objective's, kept for the next call)
  WS_TMP2,          // factor reuse: the objective lane's full-inverse recursion temporaries
  WS_REUSE_SCAL,    // factor reuse: the kept factor's (fail_col, log-det) scalars
  WS_H_X, WS_H_Y,   // host-input evaluation: device copies of X, Y and of the CSC arrays
  WS_H_LCP, WS_H_LRI, WS_H_LVA, WS_H_TCP, WS_H_TRI, WS_H_TVA,
  WS_CD_AUX,        // cooperative sweeps: list column pointers, per-entry changes, column buffer
  WS_CD_BLK,        // entry-blocked sweeps: chunk partials, the block's coupling matrix, Sigma_j / Psi_j gathers
  WS_CD_PANEL,      // left-looking Lambda sweep: chunk partials of the panel-row recompute
  WS_NUM
};

void* ws_get(Ctx* c, int slot, size_t bytes);  // throws CudaError on OOM
// collectives on the ctx stream over the attached communicator (comm.cu); no-ops without one.
// dtype 0 = double, 1 = float; buffers in device memory, in place.
inline bool comm_attached(const Ctx* c) { return c->comm.kind != 0; }
void comm_allreduce(Ctx* c, void* buf, int64_t count, int dtype);
void comm_bcast(Ctx* c, void* buf, int64_t count, int dtype, int root);
void comm_release(Ctx* c);
void comm_unique_id(char id[128]);
void comm_init_nccl(Ctx* c, const char id[128], int rank, int world);

struct CudaError {
  cggm_status code;
  std::string msg;
};

#define CGGM_CUDA_CHECK(expr)                                                                  \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess)                                                                     \
      throw ::cggm::CudaError{CGGM_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
  } while (0)

// Kernel attributes (cudaFuncSetAttribute) apply to the CURRENT device only: run the setup once per
// device (one bit per ordinal), so contexts on several GPUs in one process each get them.
#define CGGM_ONCE_PER_DEVICE(...)                                       \
  do {                                                                  \
    static std::atomic<uint64_t> _done{0};                              \
    int _dev = 0;                                                       \
    CGGM_CUDA_CHECK(cudaGetDevice(&_dev));                              \
    const uint64_t _bit = uint64_t(1) << (_dev & 63);                   \
    if (!(_done.load(std::memory_order_acquire) & _bit)) {              \
      __VA_ARGS__;                                                      \
      _done.fetch_or(_bit, std::memory_order_acq_rel);                  \
    }                                                                   \
  } while (0)

// After every launch: count it and surface launch errors.
// CGGM_SYNC_CHECK=1 (read at context creation; the stand-in for compute-sanitizer, which this pool
// does not run): synchronise the stream after every launch outside graph capture, so an asynchronous
// fault is reported by the call and kernel that caused it.
inline void post_launch(Ctx* c, const char* what) {
  c->launches++;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && c->sync_check) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(c->stream, &cs);
    if (cs == cudaStreamCaptureStatusNone) e = cudaStreamSynchronize(c->stream);
  }
  if (e != cudaSuccess) throw CudaError{CGGM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

// Device-side checks of a debug build (build.py --debug: -DCGGM_DEBUG): a violated invariant traps
// (the launch then fails with an illegal-instruction error naming the kernel under CGGM_SYNC_CHECK).
#ifdef CGGM_DEBUG
#define CGGM_DASSERT(cond) \
  do {                     \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define CGGM_DASSERT(cond) \
  do {                     \
  } while (0)
#endif

// ------------------------------------------------------------------ dense views
template <typename T>
struct ViewT {
  T* p;
  int64_t ld;
  int64_t rows, cols;
  __host__ __device__ T* at(int64_t i, int64_t j) const { return p + i + j * ld; }
  ViewT sub(int64_t r0, int64_t c0, int64_t nr, int64_t nc) const { return ViewT{p + r0 + c0 * ld, ld, nr, nc}; }
};
using View = ViewT<double>;

// ------------------------------------------------------------------ GEMM interface (gemm.cu)
enum GemmFlags : int {
  A_KLE_M = 1,          // op(A)[m][k] == 0 for k > m  -> k range ends at the tile's last m
  A_KGE_M = 2,          // op(A)[m][k] == 0 for k < m  -> k range starts at the tile's first m
  B_KLE_N = 4,          // op(B)[k][n] == 0 for k > n
  B_KGE_N = 8,          // op(B)[k][n] == 0 for k < n
  SYM_LOWER = 16,       // M == N: compute only tiles I >= J; diagonal tiles write m >= n only
  SYM_MIRROR = 32,      // with SYM_LOWER: also write every value at its transposed position; without
                        // SYM_LOWER (epilogue mir1 set): every value also at its transposed position in mir1
  SPLIT_K2 = 64,        // two CTAs per tile, each half of the k-range, out1 += a1 * partial by atomic
                        // add (out1 must hold zeros; out2 / inputs unsupported).  Two partials added
                        // to zero give a + b in either order: the result is deterministic
};

// K01: the S_Theta selection of P:296-303 taken in the X^T E GEMM epilogue on the
// tile of grad_Theta = a1 * acc while it is in shared memory, instead of storing the p x q gradient
// and scanning it again (FP64 TMA kernels only).  Per output element g: flag = |g| - lam > 0 or
// Theta_ij != 0; tie = not stored and ||g| - lam| <= tie_eps; subgradient = |g + lam sign
// Theta_ij| for a stored nonzero, else max(|g| - lam, 0).
struct SelectT {
  int on = 0;
  double lam = 0.0, tie_eps = 0.0;
  const int64_t* colptr = nullptr;   // Theta (rows = output rows, columns = output columns), device
  const int32_t* rowidx = nullptr;
  const double* val = nullptr;
  uint32_t* flags = nullptr;          // column j's words at flags + j * wpc: 2 per 64-row chunk
  int64_t wpc = 0;                    //   (word 2c: rows 64c + 2l, word 2c + 1: rows 64c + 2l + 1, bit l)
  unsigned long long* cnt = nullptr;  // per column: flagged count (atomic adds onto zero)
  long long* ties = nullptr;          // per column: tie count (atomic adds onto zero)
  double* subpart = nullptr;          // [64-row chunk][column]: subgradient partials (ld ldsub)
  int64_t ldsub = 0;
};

template <typename T>
struct EpilogueT {
  // out1 = a1*acc + b1*in1a + c1*in1b ; out2 = a2*acc + b2*in2a + c2*in2b (null pointers skip terms)
  T* out1 = nullptr; int64_t ld1 = 0; double a1 = 1.0;
  const T* in1a = nullptr; int64_t ld1a = 0; double b1 = 0.0;
  const T* in1b = nullptr; int64_t ld1b = 0; double c1 = 0.0;
  T* out2 = nullptr; int64_t ld2 = 0; double a2 = 1.0;
  const T* in2a = nullptr; int64_t ld2a = 0; double b2 = 0.0;
  const T* in2b = nullptr; int64_t ld2b = 0; double c2 = 0.0;
  // SYM_MIRROR without SYM_LOWER on a rectangular block: the transposed copy a1*acc goes to mir1
  // (ld1) instead of out1 -- the off-diagonal block of a symmetric result (no inputs, no out2)
  T* mir1 = nullptr;
  SelectT sel;   // K01 selection instead of the stores (FP64 TMA kernels; out1 ignored)
};
using Epilogue = EpilogueT<double>;

// C(M x N) epilogue(op(A) op(B)), op(A) = A (transA=false, A is M x K) or A^T (A is K x M).
// op(B) = B (transB=false, B is K x N) or B^T (B is N x K).  Column-major, FP64 DMMA.
void gemm(Ctx* c, bool transA, bool transB, int64_t M, int64_t N, int64_t K,
          const double* A, int64_t lda, const double* B, int64_t ldb, const Epilogue& epi, int flags);
// FP32 variant (gemm_f32.cu): same contract, fp32 accumulation (reading A18): 3xTF32 on the
// tcgen05 tensor cores (gemm_tf32.cu) or the SIMT FFMA engine (Ctx::f32_engine).
void gemm(Ctx* c, bool transA, bool transB, int64_t M, int64_t N, int64_t K,
          const float* A, int64_t lda, const float* B, int64_t ldb, const EpilogueT<float>& epi, int flags);
void gemm_tf32x3(Ctx* c, bool transA, bool transB, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                 const float* B, int64_t ldb, const EpilogueT<float>& epi, int flags, const CUtensorMap& ma,
                 const CUtensorMap& mb, int a3d, int b3d);

// ------------------------------------------------------------------ Cholesky family (chol.cu)
// In-place blocked recursive Cholesky of the lower triangle of A (q x q).
//  full_inverse = true : Linv (q x q, lower, zero upper) receives L^{-1}; A's L21 blocks are not kept.
//  full_inverse = false: A's lower triangle receives L; leaf inverses go to the compact buffer.
// logdet/fail are accumulated on the device (see chol.cu).
struct CholResult {
  double logdet;
  int is_pd;
  int64_t fail_col;
};
//  potrf-only mode with xdiag != null: diagonal subtrees of <= block_inverse_size() columns are
//  factored in full-inverse mode, their inverses kept at xdiag + col0 (ld ldxd, zeroed upper
//  triangles required) and used for the panel solves (tmp2: out-of-place product buffer).
template <typename T>
void potrf_recursive(Ctx* c, ViewT<T> A, ViewT<T> Linv, bool full_inverse, T* leafinv, double* logdet_slots,
                     int* fail_col_dev, T* tmp, size_t tmp_elems, T* xdiag = nullptr, int64_t ldxd = 0,
                     T* tmp2 = nullptr, size_t tmp2_elems = 0, T* sigma = nullptr, int64_t ldsigma = 0);
//  full_inverse with sigma != null (q >= Ctx::sig_min): Sigma = L^{-T} L^{-1} (both triangles)
//  assembled block by block inside the recursion (chol.cu, sig_node_pieces) -- no separate lauum.
int block_inverse_size();
// Sigma = Linv^T Linv (full symmetric).
template <typename T>
void lauum(Ctx* c, ViewT<T> Linv, ViewT<T> Sigma);
size_t chol_tmp_elems(int64_t q);   // full-inverse recursion temporaries (elements)
int leaf_nb();

// ------------------------------------------------------------------ streaming kernels (stream.cu)
template <typename T>
void densify_csc(Ctx* c, const cggm_csc* A, ViewT<T> D);
template <typename T>
void spmm_x_theta(Ctx* c, const T* X, int64_t ldx, int64_t n, const cggm_csc* Theta, ViewT<T> W);
template <typename T>
void check_csc(Ctx* c, const cggm_csc* A, bool symmetric, int* flag_dev);
template <typename T>
void grad_lambda(Ctx* c, int64_t q, const T* Syy, int64_t l1, const T* Sigma, int64_t l2, const T* Psi, int64_t l3,
                 T* G, int64_t l4);
template <typename T>
void copy2d(Ctx* c, ViewT<T> dst, const T* src, int64_t lds);

}  // namespace cggm

// ------------------------------------------------------------------ PTX helpers (device)
namespace cggm {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// orders this thread's generic-proxy shared-memory accesses before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// Ampere-style asynchronous 16-byte global -> shared copy; bytes < 16 zero-fill the tail
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// D(8x8) += A(8x4, row) * B(4x8, col), FP64 tensor pipe (SASS DMMA.8x8x4 on sm_100a).
// Lane (g = lane>>2, t = lane&3) holds A[g][t], B[t][g], C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// programmatic dependent launch: a kernel launched with the PDL attribute may start while its
// same-stream predecessor drains; pdl_wait() blocks until the predecessor has completed and its
// memory is visible (a no-op without the attribute), pdl_trigger() lets the successor's CTAs be
// scheduled once every CTA of this grid has issued it or exited
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

__device__ __forceinline__ void lds128(double& x, double& y, uint32_t addr) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(addr));
}

}  // namespace ptx
// kernel launch on c->stream, with the programmatic-dependent-launch attribute when Ctx::pdl (the
// kernel must call ptx::pdl_wait() before reading anything a predecessor writes)
template <typename... KArgs, typename... Args>
inline void launch_pdl(Ctx* c, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = c->pdl ? 1 : 0;
  CGGM_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace cggm
