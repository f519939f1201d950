/*
 * Test-only entry points of libcggm (not part of the product API).  Used by tests/ to check the
 * FP64 DMMA GEMM engine in isolation against a plain product on the host.
 */
#ifndef CGGM_TESTING_H
#define CGGM_TESTING_H
#include "cggm.h"
#ifdef __cplusplus
extern "C" {
#endif
/* C (M x N, ldc) = alpha * op(A) op(B) + beta * C, column-major device doubles.
 * flags: bit0 A_KLE_M, bit1 A_KGE_M, bit2 B_KLE_N, bit3 B_KGE_N (triangular k-range, the skipped
 * entries must be zero), bit4 SYM_LOWER (M == N, lower tiles only; diagonal tiles m >= n),
 * bit5 SYM_MIRROR (also write transposed).  beta == 0 never reads C. */
cggm_status cggm_test_gemm(cggm_ctx* ctx, int transA, int transB, int64_t M, int64_t N, int64_t K,
                           const double* A, int64_t lda, const double* B, int64_t ldb,
                           double* C, int64_t ldc, double alpha, double beta, int flags);
/* C (M x N, ldc) = alpha * op(A) op(B) and Cmir (N x M, ldc) = its transpose, written by the same
 * epilogue (SYM_MIRROR without SYM_LOWER: the off-diagonal block of a symmetric result, as the
 * Sigma assembly of the recursive inverse writes it).  flags: the triangular k-range bits only. */
cggm_status cggm_test_gemm_mir(cggm_ctx* ctx, int transA, int transB, int64_t M, int64_t N, int64_t K,
                               const double* A, int64_t lda, const double* B, int64_t ldb,
                               double* C, int64_t ldc, double* Cmir, double alpha, int flags);
/* FP32 variant of cggm_test_gemm (the ctx's FP32 engine, fp32 accumulation). */
cggm_status cggm_test_gemm_f32(cggm_ctx* ctx, int transA, int transB, int64_t M, int64_t N, int64_t K,
                               const float* A, int64_t lda, const float* B, int64_t ldb,
                               float* C, int64_t ldc, double alpha, double beta, int flags);
/* FP32 contraction engine of an F32 ctx: 0 = 3xTF32 on the tcgen05 tensor cores (the ctx's producer:
 * CGGM_TF32_PRODUCER at creation), 1 = SIMT FFMA (also CGGM_F32_ENGINE=ffma), 2 / 3 / 4 = 3xTF32 with
 * the TMA raw-tile producer (SS MMA) / the register-staged producer (SS MMA) / the TS form (A from
 * TMEM). */
cggm_status cggm_test_set_f32_engine(cggm_ctx* ctx, int engine);
/* Force the GEMM CTA tile: bits 0-1: 0 = automatic (small shapes use the 32x32 direct-load kernel),
 * 1 = 128x128 TMA (8 warps), 2 = 64x64 TMA (4 warps), 3 = automatic but K <= 256 small kernel only;
 * bit 2: never use the single 3-D TMA box for MN-inner operands (16-wide 2-D boxes instead). */
cggm_status cggm_test_set_tile(cggm_ctx* ctx, int mode);
/* FP64 tensor-pipe peak: independent DMMA.8x8x4 chains on 2 CTAs/SM for ~`seconds`; returns the
 * achieved TFLOP/s and the timed milliseconds (the roofline denominator bench.py reports). */
cggm_status cggm_test_fp64_peak(cggm_ctx* ctx, double seconds, double* tflops, double* elapsed_ms);
/* L2 -> SM read bandwidth: every SM streams 16-byte loads over a 24 MB L2-resident buffer for
 * ~`seconds`; returns GB/s and the timed milliseconds (the SpMM's L2 roofline denominator). */
cggm_status cggm_test_l2_peak(cggm_ctx* ctx, double seconds, double* gbs, double* elapsed_ms);
/* The recursive Cholesky of a dense q x q SPD matrix A (lower triangle read; overwritten with
 * scratch), on the ctx stream: full_inverse = 1 writes X = L^{-1} (lower, ldx), 0 = potrf only.
 * logdet / fail_col (host, nullable; reading them synchronises) as cggm_invert_logdet.  For
 * latency measurements of the recursion levels and dense parity tests. */
cggm_status cggm_test_chol_dense(cggm_ctx* ctx, double* A, int64_t lda, int64_t q, double* X, int64_t ldx,
                                 int full_inverse, double* logdet, int64_t* fail_col);
/* Timeline of the launches recorded since cggm_ctx_profile(ctx, 1): one CSV line per launch
 * (tag, stream index, start and end milliseconds relative to the first recorded launch).
 * Synchronises the device; call before cggm_ctx_profile_read (which clears the records). */
cggm_status cggm_test_profile_dump(cggm_ctx* ctx, const char* path);
#ifdef __cplusplus
}
#endif
#endif
