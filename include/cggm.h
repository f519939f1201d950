/*
 * libcggm — B200-native (sm_100a) hot path of the alternating Newton coordinate descent
 * solver for l1-regularised sparse conditional Gaussian graphical models
 * (McCarter & Kim, arXiv:1509.04681).  PAPER.md is cited as P:<line>.
 *
 * Problem (§2.1, Eq. 1):  X in R^{n x p}, Y in R^{n x q},
 *   S_yy = Y^T Y / n,  S_xy = X^T Y / n,  S_xx = X^T X / n (never formed),
 *   f(Lambda, Theta) = -log|Lambda| + tr(S_yy Lambda + 2 S_xy^T Theta + Lambda^{-1} Theta^T S_xx Theta)
 *                      + lam_L ||Lambda||_1 + lam_T ||Theta||_1 ,  Lambda SPD.
 *
 * CONVENTIONS (all entry points)
 *  - Every array argument is a DEVICE pointer, caller-allocated and caller-owned; the library
 *    never frees or retains it.  Dense matrices are COLUMN-MAJOR with a leading dimension
 *    ld >= rows (element (i,j) at ptr[i + j*ld]).  Element type is the ctx dtype
 *    (CGGM_F64 = double: FP64 tensor-pipe DMMA engine; CGGM_F32 = float: the FP32 variant, fp32
 *    inputs and fp32 arithmetic/accumulation in every kernel, SIMT FFMA engine; reading A18).
 *    Host scalar outputs are double in both cases.
 *  - Symmetric outputs (S_yy, Sigma, Psi, grad_Lambda) are written as FULL matrices whose two
 *    triangles are bit-identical.
 *  - Sparse Lambda / Theta are passed as cggm_csc (device arrays): int64 colptr[ncols+1],
 *    int32 rowidx[nnz] strictly increasing within each column, values[nnz].  Lambda stores both
 *    triangles and must be exactly symmetric.  Stored zeros count as zero.
 *  - Scalar outputs are HOST pointers; a call that writes host scalars synchronises the ctx
 *    stream.  All device work is enqueued on the ctx stream, in order.
 *  - n_total is the GLOBAL sample count used in every 1/n and 1/sqrt(n) (sample sharding);
 *    n_local is the number of rows of X and Y held by this caller (n_local == n_total on 1 GPU).
 *  - Arguments are validated before any launch (null pointers, negative sizes, ld < rows,
 *    shapes).  With validation level >= 1 (default) the CSC structure (colptr monotone, rows in
 *    range and strictly increasing) and the symmetry of Lambda are checked on the device before
 *    any compute launch (costs one stream sync).
 *  - On error no output is valid, except CGGM_ERR_CAPACITY (two-call pattern, see
 *    cggm_active_set).  cggm_last_error(ctx) returns a message.  A non-PD Lambda is NOT an
 *    error: is_pd = 0 and fail_col = first failing Cholesky column.
 *  - A ctx is not thread-safe; separate ctx objects may be used concurrently (the calls are
 *    pure functions of their inputs).  Internal workspace is library-owned and cached per ctx.
 */
#ifndef CGGM_H
#define CGGM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum cggm_status {
  CGGM_OK = 0,
  CGGM_ERR_INVALID_ARG = 1,   /* null pointer, negative dimension, ld < rows */
  CGGM_ERR_SHAPE = 2,         /* inconsistent shapes between arguments */
  CGGM_ERR_NOT_SYMMETRIC = 3, /* Lambda CSC not exactly symmetric */
  CGGM_ERR_BAD_SPARSE = 4,    /* colptr not monotone / rows out of range or unsorted */
  CGGM_ERR_NONFINITE = 5,     /* reserved: optional input scan */
  CGGM_ERR_CAPACITY = 6,      /* active-set lists larger than the given capacity */
  CGGM_ERR_OOM = 7,           /* workspace allocation failed */
  CGGM_ERR_CUDA = 8,          /* CUDA runtime / launch error */
  CGGM_ERR_NCCL = 9,          /* NCCL (or external collective callback) failure, see cggm_comm_init */
  CGGM_ERR_UNSUPPORTED = 10   /* dtype or mode not implemented */
} cggm_status;

typedef enum cggm_dtype { CGGM_F64 = 0, CGGM_F32 = 1 } cggm_dtype;

typedef struct cggm_ctx cggm_ctx;

/* Sparse matrix, compressed sparse column, device arrays. */
typedef struct cggm_csc {
  int64_t nrows, ncols, nnz;
  const int64_t* colptr; /* device, ncols+1 entries, colptr[0] = 0, colptr[ncols] = nnz */
  const int32_t* rowidx; /* device, nnz entries, strictly increasing within a column */
  const void* val;       /* device, nnz entries of the ctx dtype */
} cggm_csc;

/* Active sets S_Lambda, S_Theta (§2.2) and the minimum-norm-subgradient stopping
 * statistic (§5.1).  Inputs marked (in), device outputs (dev out), host outputs
 * (host out). */
typedef struct cggm_active_out {
  double lam_L, lam_T;     /* (in) thresholds lambda_Lambda, lambda_Theta */
  int32_t penalize_diag;   /* (in) 1: diagonal of Lambda penalised (Eq. 1 literally); 0: lambda_ii = 0 */
  double tie_eps;          /* (in) tie band: entries with ||grad|-lam| <= tie_eps are counted in ties_* */
  int64_t cap_L, cap_T;    /* (in) capacity (entries) of the device lists below */
  int32_t* L_row;          /* (dev out) S_Lambda rows, i <= j, ascending column-major order */
  int32_t* L_col;          /* (dev out) S_Lambda columns */
  int32_t* T_row;          /* (dev out) S_Theta rows, ascending column-major order */
  int32_t* T_col;          /* (dev out) S_Theta columns */
  int64_t m_L, m_T;        /* (host out) |S_Lambda| (upper triangle incl. diagonal), |S_Theta| */
  int64_t ties_L, ties_T;  /* (host out) non-forced entries inside the tie band */
  double subgrad_l1;       /* (host out) ||grad^S(Lambda,Theta)||_1 over all Lambda (both triangles) and Theta entries */
} cggm_active_out;

/* Line-search objective (Eq. 1): f = g + h at an arbitrary Lambda. */
typedef struct cggm_objective_out {
  double f;            /* g + pen_L + pen_T; +INF when Lambda is not PD */
  double g;            /* smooth part; +INF when not PD */
  double logdet;       /* log|Lambda| = 2 sum ln L_jj (NaN when not PD) */
  double tr_syy_lam;   /* tr(S_yy Lambda)        = (1/n_total) <Y, Y Lambda>          (this shard's rows) */
  double tr_sxy_theta; /* tr(S_xy^T Theta)       = (1/n_total) <X Theta, Y>           (this shard's rows) */
  double tr_sigma_m;   /* tr(Sigma Theta^T S_xx Theta) = ||L^{-1} (X Theta)^T||_F^2 / n_total (this shard's rows) */
  double pen_L;        /* lam_L * ||Lambda||_1 (elementwise, diagonal per penalize_diag) */
  double pen_T;        /* lam_T * ||Theta||_1 */
  int32_t is_pd;       /* Cholesky of Lambda succeeded (the line search's PD test) */
  int64_t fail_col;    /* first failing Cholesky column, -1 when PD */
} cggm_objective_out;

/* ---- context ------------------------------------------------------------------------ */
/* Create a context bound to `device`, element type `dtype`, enqueuing on `cuda_stream`
 * (a cudaStream_t; NULL = legacy default stream).  Fails with CGGM_ERR_CUDA when the device
 * is not an sm_100 part. */
cggm_status cggm_ctx_create(cggm_ctx** out, int device, cggm_dtype dtype, void* cuda_stream);
cggm_status cggm_ctx_destroy(cggm_ctx* ctx);
/* Change the stream work is enqueued on. */
cggm_status cggm_ctx_set_stream(cggm_ctx* ctx, void* cuda_stream);
/* Validation level: 0 = host-side argument checks only, 1 = also device CSC checks (default). */
cggm_status cggm_ctx_set_validate(cggm_ctx* ctx, int level);
/* Scheduling options (performance only; results are identical up to summation order, which no
 * option changes for a given argument set):
 *   CGGM_OPT_LOOKAHEAD_MIN: recursive Cholesky lookahead -- trailing updates / block products of at
 *     least this width run on lower-priority side streams while the recursion proceeds (default
 *     256; 0 = everything on one stream, each kernel's duration its own);
 *   CGGM_OPT_GRAPHS: 1 = cggm_newton_eval captures its launches into a CUDA graph on the second
 *     call with the same arguments and replays it afterwards (default), 0 = plain stream launches.
 *   CGGM_OPT_FACTOR_REUSE: 1 = cggm_newton_eval runs the objective's trial factorisation in
 *     full-inverse mode and keeps L_trial^{-1}; the NEXT cggm_newton_eval on this ctx takes
 *     Sigma = L^{-T} L^{-1} from it (one symmetric product, no factorisation) and the log-det / PD
 *     flag from the kept trial -- the secondary "factor-reuse" evaluation of SURVEY.md §8(d),
 *     (4/3) q^3 -> q^3 flop.  The CALLER guarantees that the next Lambda equals the previous call's
 *     Lambda (the accepted line-search trial); q must match, else the call falls back to a full
 *     inverse.  Setting the option (either value) forgets the kept factor.
 *   CGGM_OPT_SIGMA_BLOCK: Sigma = L^{-T} L^{-1} of cggm_invert_logdet / cggm_newton_eval
 *     is assembled inside the recursive inverse: a recursion node at least this wide forms its
 *     off-diagonal block X22^T X21 and the update X21^T X21 of its leading block as soon as its
 *     own L^{-1} block is final, its children likewise; narrower nodes form their whole block in one
 *     product (default 4096 for FP64, 0 for the FP32 variant -- measured slower there; setting the
 *     option sets both; 0 = one symmetric product after the recursion; values below 128 are refused).
 *     Sums of the same products in a different split of the k-range only.
 * Unknown option -> CGGM_ERR_INVALID_ARG. */
typedef enum cggm_option {
  CGGM_OPT_LOOKAHEAD_MIN = 0, CGGM_OPT_GRAPHS = 1, CGGM_OPT_FACTOR_REUSE = 2, CGGM_OPT_SIGMA_BLOCK = 3
} cggm_option;
cggm_status cggm_ctx_set_option(cggm_ctx* ctx, int option, int64_t value);
/* Number of library kernels launched on this ctx so far (for launch accounting). */
cggm_status cggm_ctx_launch_count(cggm_ctx* ctx, int64_t* count);
/* Release the cached internal workspace. */
cggm_status cggm_ctx_release_workspace(cggm_ctx* ctx);
/* Phase profiling: while enabled, every library kernel launch is bracketed by CUDA events on the
 * ctx stream and attributed to a phase tag (0..CGGM_PROF_NTAGS-1, names by cggm_profile_tag_name).
 * enable=1 clears previous records.  _read synchronises the stream and writes per-tag summed
 * kernel milliseconds and launch counts (arrays of >= CGGM_PROF_NTAGS entries), then clears. */
#define CGGM_PROF_NTAGS 14
cggm_status cggm_ctx_profile(cggm_ctx* ctx, int enable);
cggm_status cggm_ctx_profile_read(cggm_ctx* ctx, double* ms, int64_t* launches, int32_t ntags);
const char* cggm_profile_tag_name(int32_t tag);
/* Message of the last error on this ctx ("" if none).  Valid until the next call. */
const char* cggm_last_error(cggm_ctx* ctx);
/* Library version string. */
const char* cggm_version(void);

/* ---- sample sharding: library-owned collectives (north_star) --------------
 * Rank r of a group of `world` holds rows X_r, Y_r of the data (n_local of the n_total samples;
 * every 1/n uses n_total, reading A21).  Once a communicator is attached to a ctx, the calls below
 * become COLLECTIVE (every rank calls them, in the same order, with the same Lambda / Theta / lambda
 * arguments) and return the unsharded results on every rank:
 *   cggm_covariances   S_yy and S_xy partials all-reduced (sum);
 *   cggm_gram          S_xx partial all-reduced;
 *   cggm_invert_logdet rank 0 factors and inverts; Sigma and (logdet, is_pd, fail_col) are
 *                      broadcast from rank 0 (other ranks do no compute; "the q x q
 *                      Cholesky/inverse runs on one GPU and is then broadcast", north_star);
 *   cggm_psi_grad      Psi = sum_r R_r^T R_r and grad_Theta = sum_r (2/n) X_r^T E_r all-reduced
 *                      before grad_Lambda and the active sets, which every rank then forms
 *                      identically (GradL with n_local < n_total is allowed only with a comm);
 *                      with GradT = NULL and fused active sets, each grad_Theta column chunk is
 *                      all-reduced before its scan (bounded buffer);
 *   cggm_objective     every rank factors the trial Lambda (augmented with its own W_r rows); the
 *                      three data traces are all-reduced, logdet and penalties are replicated.
 * cggm_newton_eval / _host with world > 1 return CGGM_ERR_UNSUPPORTED (the composite overlaps
 * its steps on one GPU; sharded callers compose the collective calls above).
 * Collectives are enqueued on the ctx stream.  Failures return CGGM_ERR_NCCL.  After each NCCL
 * collective the call waits for it on the host while polling ncclCommGetAsyncError, with a deadline
 * of CGGM_NCCL_TIMEOUT_S seconds (environment, default 600; 0 = no wait): a peer failure or a hung
 * rank then returns CGGM_ERR_NCCL (the communicator is aborted and detached) instead of blocking
 * the caller forever. */
/* All-reduce over peer memory (CUDA IPC; NVLink peer loads / stores between the GPUs of a node),
 * the alternative to NCCL for the partial sums: every rank registers one symmetric buffer of the
 * same size (cggm_ipc_get_handle on its own, cggm_ipc_open_handle on the others' handles, exchanged
 * by the caller), its GEMM writes its partial straight into it, and after a barrier rank r sums
 * slice r of all ranks' buffers in rank order and writes the sum into slice r of every rank's
 * buffer (cggm_peer_allreduce; in place: each slice is read and written by its owner only); after
 * a second barrier every buffer holds the bit-identical total.  bufs: host array of `world`
 * device pointers (rank k's buffer at bufs[k]), count elements of the ctx dtype.  The same exchange
 * north_star assigns to an NCCL all-reduce (the partial X^T(X Theta) and R^T R sums).  Errors:
 * CGGM_ERR_INVALID_ARG (world outside 1..8, rank out of range, null pointers), CGGM_ERR_CUDA (an
 * IPC call failed, e.g. no peer access between the devices), CGGM_ERR_OOM (cggm_device_alloc). */
/* A device allocation of its own (cudaMalloc on the ctx device), so that its IPC handle covers
 * exactly the buffer (pool sub-allocations would need an offset); freed by cggm_device_free. */
cggm_status cggm_device_alloc(cggm_ctx* ctx, int64_t bytes, void** dev_ptr);
cggm_status cggm_device_free(cggm_ctx* ctx, void* dev_ptr);
cggm_status cggm_ipc_get_handle(cggm_ctx* ctx, const void* dev_ptr, char handle[64]);
cggm_status cggm_ipc_open_handle(cggm_ctx* ctx, const char handle[64], void** dev_ptr);
cggm_status cggm_ipc_close_handle(cggm_ctx* ctx, void* dev_ptr);
cggm_status cggm_peer_allreduce(cggm_ctx* ctx, int32_t world, int32_t rank, void* const* bufs, int64_t count);
/* 128-byte NCCL unique id, created on rank 0 (cggm_comm_unique_id) and sent to the other ranks by
 * the caller (e.g. a torch.distributed broadcast). */
cggm_status cggm_comm_unique_id(char id[128]);
/* Attach an NCCL communicator (rank `rank` of `world`, on the ctx device).  NCCL is loaded at
 * run time (the libnccl.so.2 already in the process, else the system one); CGGM_ERR_NCCL if it
 * cannot be loaded or the init fails.  Replaces any communicator attached before. */
cggm_status cggm_comm_init(cggm_ctx* ctx, const char id[128], int32_t rank, int32_t world);
/* Attach caller-provided collectives instead of NCCL (another transport, or tests that run several
 * ranks on one GPU where NCCL refuses duplicate devices).  The library synchronises the ctx stream
 * before each callback; the callback must complete the operation before returning (result in
 * `buf`, device memory, `count` elements of `dtype`: 0 = double, 1 = float) and return 0 on
 * success. */
typedef int (*cggm_allreduce_fn)(void* user, void* buf, int64_t count, int32_t dtype);
typedef int (*cggm_broadcast_fn)(void* user, void* buf, int64_t count, int32_t dtype, int32_t root);
cggm_status cggm_comm_init_external(cggm_ctx* ctx, int32_t rank, int32_t world, cggm_allreduce_fn allreduce,
                                    cggm_broadcast_fn broadcast, void* user);
/* Detach (and destroy an NCCL) communicator; the calls become single-rank again. */
cggm_status cggm_comm_destroy(cggm_ctx* ctx);
/* rank / world of the attached communicator (0 / 1 when none). */
cggm_status cggm_comm_info(cggm_ctx* ctx, int32_t* rank, int32_t* world);

/* ---- dense building blocks (NEXT-3: the distributed factorisation composes them) -----------
 * The paper parallelises exactly these precomputations across cores; sharded.py's
 * DistributedInverse runs a block-cyclic factorisation and inverse of Lambda over the ranks of a
 * process group out of these calls (every FLOP in this library's kernels, the exchanges by the
 * caller's collectives). */
/* C (M x N, ldc) = alpha * op(A) op(B) + beta * C in the ctx dtype (fp64: DMMA engine; fp32: FFMA
 * engine).  op(A) = A (M x K, lda) or A^T (A is K x M); op(B) = B (K x N) or B^T (B is N x K).
 * flags (cggm_gemm_flags): structural zeros the engine may skip -- bit0 op(A)[m][k] = 0 for k > m,
 * bit1 op(A)[m][k] = 0 for k < m, bit2 op(B)[k][n] = 0 for k > n, bit3 op(B)[k][n] = 0 for k < n --
 * and symmetric outputs: bit4 (M == N) lower tiles only, diagonal tiles m >= n; bit5 with bit4 also
 * write the transposed values.  beta == 0 never reads C.  C must not alias A or B except as an
 * exact in-place operand the engine supports (not guaranteed: treat as an error). */
typedef enum cggm_gemm_flags {
  CGGM_A_KLE_M = 1, CGGM_A_KGE_M = 2, CGGM_B_KLE_N = 4, CGGM_B_KGE_N = 8, CGGM_SYM_LOWER = 16, CGGM_SYM_MIRROR = 32
} cggm_gemm_flags;
cggm_status cggm_gemm(cggm_ctx* ctx, int32_t transA, int32_t transB, int64_t M, int64_t N, int64_t K, double alpha,
                      const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc,
                      int32_t flags);
/* Dense SPD block (q x q, lda even, lower triangle read; A is overwritten with scratch): the
 * recursive Cholesky in full-inverse mode, X (q x q, ldx even) = L^{-1} (lower; zeros above the
 * diagonal), logdet = 2 sum ln L_jj, is_pd / fail_col as cggm_invert_logdet (host outputs). */
cggm_status cggm_chol_inverse_dense(cggm_ctx* ctx, int64_t q, void* A, int64_t lda, void* X, int64_t ldx,
                                    double* logdet, int32_t* is_pd, int64_t* fail_col);
/* S (n x n, lds): copy the strict lower triangle onto the upper (S becomes exactly symmetric). */
cggm_status cggm_symmetrize(cggm_ctx* ctx, int64_t n, void* S, int64_t lds);
/* Dense D (nrows x ncols, ldd) = the CSC matrix (zeros elsewhere). */
cggm_status cggm_densify(cggm_ctx* ctx, const cggm_csc* A, void* D, int64_t ldd);

/* The line-search objective (as cggm_objective) at a Lambda whose inverse Cholesky factor the caller
 * already holds: Linv (q x q, lower) = L^{-1} with Lambda = L L^T and logdet = log|Lambda| (e.g. from
 * DistributedInverse's factorisation of the trial Lambda).  tr(Sigma Theta^T S_xx Theta) is
 * ||W Linv^T||_F^2 / n_total (one triangular GEMM), the other terms as cggm_objective; is_pd = 1,
 * fail_col = -1 (the caller's factorisation is the PD test).  With n_local < n_total the three data
 * traces are this shard's partial sums (all-reduced when a communicator is attached). */
cggm_status cggm_objective_given_inverse(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, int64_t q,
                                         const void* X, int64_t ldx, const void* Y, int64_t ldy,
                                         const cggm_csc* Lambda, const cggm_csc* Theta, double lam_L, double lam_T,
                                         int32_t penalize_diag, const void* W, int64_t ldw, const void* Linv,
                                         int64_t ldlinv, double logdet, cggm_objective_out* out);

/* ---- a1: sample covariances (§2.1) ----------------------------------------- */
/* Syy (q x q, ldsyy) = Y^T Y / n_total (full symmetric), Sxy (p x q, ldsxy) = X^T Y / n_total.
 * Either output may be NULL (skipped).  X: n_local x p (ldx), Y: n_local x q (ldy).
 * With n_local < n_total the outputs are this shard's partial sums (sum over shards = S). */
cggm_status cggm_covariances(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, int64_t q,
                             const void* X, int64_t ldx, const void* Y, int64_t ldy,
                             void* Syy, int64_t ldsyy, void* Sxy, int64_t ldsxy);

/* ---- a3: Sigma = Lambda^{-1}, log-determinant, PD test (§2.3) --------- */
/* Dense blocked Cholesky of the CSC Lambda (q x q).  If Sigma != NULL (q x q, ldsigma) writes
 * Sigma = L^{-T} L^{-1} (full symmetric).  Host outputs: logdet (NaN if not PD), is_pd,
 * fail_col (-1 if PD).  Sigma is unspecified when is_pd == 0. */
cggm_status cggm_invert_logdet(cggm_ctx* ctx, const cggm_csc* Lambda, void* Sigma, int64_t ldsigma,
                               double* logdet, int32_t* is_pd, int64_t* fail_col);

/* ---- a2, a4, a5: W = X Theta, R, Psi, gradients (Eq. 3) --
 *  W = X Theta (SpMM, n_local x q),  acc = W Sigma,  R = acc / sqrt(n_total),
 *  Psi (q x q, ldpsi)    = R^T R                                   (full symmetric)
 *  GradL (q x q, ldgl)   = S_yy - Sigma - Psi                      (nullable; needs Syy)
 *  GradT (p x q, ldgt)   = (2/n_total) X^T (Y + acc)               if Sxy == NULL (identity I3)
 *                        = 2 Sxy + (2/sqrt(n_total)) X^T R         if Sxy != NULL
 * S_xx Theta Sigma is X^T R / sqrt(n): S_xx is never formed (north_star (1)).  With
 * n_local < n_total, Psi and GradT (Sxy == NULL) are this shard's partial sums and GradL must be
 * NULL (form it after the all-reduce with cggm_grad_lambda).  If `fused` != NULL the active
 * sets are also built (same semantics as cggm_active_set; requires GradL).  With fused != NULL
 * and GradT == NULL, grad_Theta is STREAMED: computed in column chunks into library workspace
 * and compacted into S_Theta immediately, never stored (the p x q gradient is 64 GB at the
 * `sharded` size). */
cggm_status cggm_psi_grad(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, int64_t q,
                          const void* X, int64_t ldx, const void* Y, int64_t ldy, const cggm_csc* Theta,
                          const void* Sigma, int64_t ldsigma, const void* Syy, int64_t ldsyy,
                          const void* Sxy, int64_t ldsxy,
                          void* Psi, int64_t ldpsi, void* GradL, int64_t ldgl, void* GradT, int64_t ldgt,
                          const cggm_csc* Lambda, cggm_active_out* fused);

/* grad_Lambda = S_yy - Sigma - Psi, elementwise (Eq. 3), for the sharded path. */
cggm_status cggm_grad_lambda(cggm_ctx* ctx, int64_t q, const void* Syy, int64_t ldsyy,
                             const void* Sigma, int64_t ldsigma, const void* Psi, int64_t ldpsi,
                             void* GradL, int64_t ldgl);

/* ---- sample-sharded grad_Theta by column ranges (SURVEY.md §8(e) "Better": reduce-scatter over
 * column blocks, local compaction, all-gather of the compact lists; sharded.ShardedEvaluator with
 * grad_theta="reduce_scatter").  No rank ever holds a p x q buffer. */
/* Psi (q x q, ldpsi; this shard's partial R_r^T R_r, all-reduced when a communicator is attached) and
 * E (n_local x q, lde) = Y_r + X_r Theta Sigma, the residual whose (2/n_total) X_r^T E_r is the
 * shard's grad_Theta partial (identity I3); W = X Theta as in cggm_psi_grad. */
cggm_status cggm_psi_residual(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, int64_t q, const void* X,
                              int64_t ldx, const void* Y, int64_t ldy, const cggm_csc* Theta, const void* Sigma,
                              int64_t ldsigma, void* Psi, int64_t ldpsi, void* E, int64_t lde);
/* S_Theta = {(i,j) : |GradT_ij| > lam_T or Theta_ij != 0} restricted to the columns
 * [col0, col0 + ncols): GradT is that column block (p x ncols, ldgt; device), Theta the full p x q
 * CSC.  Entries are written in column-major order with GLOBAL column indices into T_row / T_col
 * (device, capacity cap).  Host outputs: m = the block's |S_Theta| (CGGM_ERR_CAPACITY when m > cap;
 * m then holds the required size), ties (nullable) = entries within tie_eps of lam_T not forced by the
 * support, subgrad (nullable) = the block's Theta part of ||grad^S||_1. */
cggm_status cggm_active_theta_block(cggm_ctx* ctx, int64_t p, int64_t col0, int64_t ncols, const void* GradT,
                                   int64_t ldgt, const cggm_csc* Theta, double lam_T, double tie_eps, int32_t* T_row,
                                   int32_t* T_col, int64_t cap, int64_t* m, int64_t* ties, double* subgrad);

/* ---- a6: active sets + stopping statistic (§2.2, §5.1) -------------
 * S_Lambda = {(i,j), i <= j : |GradL_ij| > lam_ij or Lambda_ij != 0}, lam_ii = 0 if !penalize_diag
 * S_Theta  = {(i,j)         : |GradT_ij| > lam_T  or Theta_ij  != 0}
 * Lists are written in ascending column-major order (deterministic).  If m_L > cap_L or
 * m_T > cap_T, m_L/m_T hold the required sizes, CGGM_ERR_CAPACITY is returned and the list
 * contents are unspecified (only the first cap entries may have been written; two-call pattern).  subgrad_l1 = sum over all Lambda entries (both triangles) and
 * Theta entries of |g + lam sign(x)| if x != 0 else max(|g| - lam, 0). */
cggm_status cggm_active_set(cggm_ctx* ctx, int64_t p, int64_t q, const void* GradL, int64_t ldgl,
                            const void* GradT, int64_t ldgt, const cggm_csc* Lambda, const cggm_csc* Theta,
                            cggm_active_out* out);

/* ---- a7: line-search objective with the Cholesky PD test --------
 * Fresh Cholesky of the (trial) Lambda; tr(Sigma Theta^T S_xx Theta) = ||L^{-1} W^T||_F^2 / n
 * with W = X Theta (or the caller's W, n_local x q, ldw, when W != NULL: W is fixed while Theta
 * is, so line-search trials can reuse it).  With n_local < n_total the three trace terms are this
 * shard's partial sums; logdet and the penalties are global. */
cggm_status cggm_objective(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, int64_t q,
                           const void* X, int64_t ldx, const void* Y, int64_t ldy,
                           const cggm_csc* Lambda, const cggm_csc* Theta,
                           double lam_L, double lam_T, int32_t penalize_diag,
                           const void* W, int64_t ldw, cggm_objective_out* out);

/* ---- NEXT-1 / NEXT-2: the coordinate-descent consumers of Algorithm 1 ------- */
/* S_xx = X^T X / n_total (p x p, full symmetric, both triangles written; ldsxx >= p).  Used only by
 * the Theta sweep (the hot path itself never forms S_xx). */
cggm_status cggm_gram(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, const void* X, int64_t ldx,
                      void* Sxx, int64_t ldsxx);
/* Newton direction D_Lambda of Eq. (6) by `passes` coordinate-descent sweeps over the
 * active list (L_row[k] <= L_col[k], column-major, as cggm_active_set writes it), maintaining
 * U = D Sigma (library workspace).  Update of entry k = (i, j):
 *   a = S_ij^2 + S_ii S_jj + S_ii P_jj + S_jj P_ii + 2 S_ij P_ij  (i != j),  S_ii^2 + 2 S_ii P_ii (i == j)
 *   b = GradL_ij + (S D S)_ij + (P D S)_ij + (P D S)_ji,  c = Lambda_ij + D_k,
 *   D_k += -c + S_{lam/a}(c - b/a)          (appendix P:1184-1195 with reading A15)
 * with S = Sigma, P = Psi (q x q device, symmetric), lam = 0 for an unpenalised diagonal.
 * D: m_L device doubles, written (the sweep starts from D = 0).  Host outputs (nullable):
 * delta[0] = tr(GradL^T D), delta[1] = lam-weighted ||Lambda + D||_1 - ||Lambda||_1 (their sum is the
 * Armijo decrease measure, reading A16); l1_lambda = ||Lambda||_1 over all entries.  fp64 ctx only. */
cggm_status cggm_lambda_direction(cggm_ctx* ctx, int64_t q, const void* Sigma, int64_t ldsigma, const void* Psi,
                                  int64_t ldpsi, const void* GradL, int64_t ldgl, const cggm_csc* Lambda,
                                  const int32_t* L_row, const int32_t* L_col, int64_t m_L, double lam_L,
                                  int penalize_diag, int passes, void* D, double* delta, double* l1_lambda);
/* The line-search candidate Lambda + alpha D as a symmetric CSC over the active list
 * and its mirror.  out: nrows = ncols = q, colptr (q+1 device int64), rowidx/val device arrays of
 * capacity out->nnz on entry (>= 2 m_L); on return out->nnz = stored entries (rows sorted per
 * column; entries that became 0 stay stored).  Lambda's nonzeros must all be on the list (they are,
 * by the definition of S_Lambda).  CGGM_ERR_CAPACITY if the arrays are too small. */
cggm_status cggm_lambda_step(cggm_ctx* ctx, int64_t q, const cggm_csc* Lambda, const int32_t* L_row,
                             const int32_t* L_col, int64_t m_L, const void* D, double alpha, cggm_csc* out);
/* Eq. (7) by `passes` coordinate-descent sweeps over the Theta active list (column-
 * major), maintaining V = Theta Sigma (library workspace):
 *   a = 2 Sigma_jj (S_xx)_ii,  b = 2 (S_xy)_ij + 2 (S_xx Theta Sigma)_ij,  c = Theta_ij,
 *   Theta_ij += -c + S_{lam/a}(c - b/a)      (appendix P:1196-1207 with reading A15).
 * Sigma (q x q), Sxx (p x p, cggm_gram), Sxy (p x q, cggm_covariances) device; Theta = the current
 * iterate (its nonzeros are on the list).  out: the new Theta as a CSC over the list (colptr q+1,
 * rowidx/val capacity out->nnz >= m_T on entry, out->nnz = m_T on return).  l1_theta (host,
 * nullable) = ||Theta_new||_1.  The out arrays must not alias Theta's.  fp64 ctx only. */
cggm_status cggm_theta_cd(cggm_ctx* ctx, int64_t p, int64_t q, const void* Sigma, int64_t ldsigma, const void* Sxx,
                          int64_t ldsxx, const void* Sxy, int64_t ldsxy, const cggm_csc* Theta, const int32_t* T_row,
                          const int32_t* T_col, int64_t m_T, double lam_T, int passes, cggm_csc* out,
                          double* l1_theta);

/* On-demand S_xx for the Theta sweep (the paper's (S_xx)_i rows): only
 * the rows of S_xx the active list touches are formed, as columns (S_xx symmetric) of a p x n_cols
 * block.  cggm_gram_rows: xmap (device, p int32, written) = position of row i among the distinct
 * rows of T_row[0..m_T) in ascending order, -1 when absent; Sxx_cols (device, p x cap, ldsxx) column
 * c = X^T X_{rows[c]} / n_total (all-reduced with a communicator); host n_cols = the number of
 * distinct rows (CGGM_ERR_CAPACITY when > cap, n_cols then holds the required count).
 * cggm_theta_cd_rows: cggm_theta_cd with S_xx given as those columns (xmap, n_cols).  fp64 ctx. */
cggm_status cggm_gram_rows(cggm_ctx* ctx, int64_t n_local, int64_t n_total, int64_t p, const void* X, int64_t ldx,
                           const int32_t* T_row, int64_t m_T, void* Sxx_cols, int64_t ldsxx, int64_t cap,
                           int32_t* xmap, int64_t* n_cols);
cggm_status cggm_theta_cd_rows(cggm_ctx* ctx, int64_t p, int64_t q, const void* Sigma, int64_t ldsigma,
                               const void* Sxx_cols, int64_t ldsxx, const int32_t* xmap, int64_t n_cols,
                               const void* Sxy, int64_t ldsxy, const cggm_csc* Theta, const int32_t* T_row,
                               const int32_t* T_col, int64_t m_T, double lam_T, int passes, cggm_csc* out,
                               double* l1_theta);

/* ---- composite: one Newton-iteration evaluation -------------------
 * Same results as cggm_invert_logdet(Lambda) + cggm_psi_grad(residual route, fused active sets)
 * + cggm_objective(Lambda_trial = Lambda, Theta) on one GPU (n samples, no sharding), with the
 * objective's fresh trial Cholesky (the line-search PD test) executed on a library
 * auxiliary stream concurrently with Sigma = Lambda^{-1} and the Psi / gradient / active-set work
 * on the ctx stream.  Inputs as in those calls (Syy from cggm_covariances); active->lam_L, lam_T,
 * penalize_diag are also the objective's.  GradT may be NULL: grad_Theta is then streamed into
 * the active-set compaction and not stored (see cggm_psi_grad).  One host synchronisation at the end; on
 * CGGM_ERR_CAPACITY all other outputs are valid and the list contents are unspecified. */
typedef struct cggm_eval_out {
  double logdet;            /* log|Lambda| from the inverse's factorisation (NaN if not PD) */
  int32_t is_pd;
  int64_t fail_col;
  cggm_objective_out obj;   /* the line-search objective at Lambda */
} cggm_eval_out;

cggm_status cggm_newton_eval(cggm_ctx* ctx, int64_t n, int64_t p, int64_t q,
                             const void* X, int64_t ldx, const void* Y, int64_t ldy, const void* Syy, int64_t ldsyy,
                             const cggm_csc* Lambda, const cggm_csc* Theta,
                             void* Sigma, int64_t ldsigma, void* Psi, int64_t ldpsi, void* GradL, int64_t ldgl,
                             void* GradT, int64_t ldgt, cggm_active_out* active, cggm_eval_out* out);

/* One Newton-iteration evaluation from HOST buffers (the end-to-end form of cggm_newton_eval):
 * X (n x p, ldx >= n) and Y (n x q, ldy >= n) column-major fp64 host arrays, Lambda and Theta CSCs
 * whose colptr / rowidx / val point to HOST memory (page-locked memory makes the uploads
 * asynchronous).  The library uploads into its workspace on an internal copy stream -- Lambda
 * first, so the factorisation starts while X and Y are still in flight -- forms S_yy = Y^T Y / n
 * into Syy (device, q x q, written), and evaluates exactly as cggm_newton_eval; the other
 * outputs (device) and the host scalars are those of cggm_newton_eval (GradT may be NULL: grad_Theta
 * streamed into the active-set compaction, never stored).  fp64 ctx only. */
cggm_status cggm_newton_eval_host(cggm_ctx* ctx, int64_t n, int64_t p, int64_t q, const double* X, int64_t ldx,
                                  const double* Y, int64_t ldy, const cggm_csc* Lambda, const cggm_csc* Theta,
                                  void* Syy, int64_t ldsyy, void* Sigma, int64_t ldsigma, void* Psi, int64_t ldpsi,
                                  void* GradL, int64_t ldgl, void* GradT, int64_t ldgt, cggm_active_out* active,
                                  cggm_eval_out* out);

/* ---- NEXT-4: memory-bounded evaluation ------------------------------------------------------
 * One Newton-iteration evaluation at (Lambda, Theta) without storing Sigma, Psi or grad_Lambda
 * (the paper's block mode, P:555-595 / P:671-825, with triangular products of the GPU factor in
 * place of CG): the q x q memory is the factorisation's (dense Lambda, freed after, and L^{-1});
 * Sigma, Psi and the gradients exist only as b-wide column blocks (block = 0: 1024) consumed by the
 * active-set compaction.  Outputs as cggm_newton_eval without the dense matrices: log-det / PD,
 * the active lists and counts (active, two-call CGGM_ERR_CAPACITY pattern), the subgradient
 * statistic, and the objective at the same Lambda from the same factor (out->obj; a line-search
 * trial is a separate cggm_objective).  X (n x p), Y (n x q) device, n_total = n.  Flops:
 * factorisation (2/3) q^3 + Sigma blocks q^3 (two passes) + 3 n q^2 + 2 n p q. */
cggm_status cggm_newton_eval_blocked(cggm_ctx* ctx, int64_t n, int64_t p, int64_t q, const void* X, int64_t ldx,
                                     const void* Y, int64_t ldy, const cggm_csc* Lambda, const cggm_csc* Theta,
                                     int64_t block, cggm_active_out* active, cggm_eval_out* out);


#ifdef __cplusplus
}
#endif

#endif /* CGGM_H */
