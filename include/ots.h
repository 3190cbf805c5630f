/*
 * ots.h -- C-ABI of the B200-native two-stage Householder orthogonalization
 * (arXiv 2602.14449, Algorithm 1 and its B-inner extension).
 *
 * Drop-in boundary for the reference package `orthoqr` 0.1.0 (pure Python,
 * /root/reference/pkg/src/orthoqr).  Every entry point below replaces one
 * reference function on the hot path named by BASELINE.json's north_star;
 * the reference interface each one replaces is cited beside it.  The Python
 * facade `paper_2602_14449_b200` (same names/signatures as orthoqr) binds
 * these with ctypes; INTEGRATION.md shows the binding a maintainer adds.
 *
 * Conventions
 *  - All matrices are ROW-MAJOR (numpy C order, as orthoqr's as_matrix,
 *    core.py:25-32) in DEVICE memory owned by the caller; ld = row stride in
 *    elements, must be even and rows 16-byte aligned.
 *  - Real f64 entry points take `double*`; complex128 entry points take
 *    interleaved (re, im) `double*` with ld counted in complex elements.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    stream-ordered; the only host synchronisation is the status/diagnostic
 *    readback at the end of a call.
 *  - Return value: OTS_OK (0) or a negative code, one per exception class of
 *    orthoqr/errors.py:4-65; ots_last_error() returns the message.
 */
#ifndef OTS_H_
#define OTS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OTS_OK 0
#define OTS_E_DIMENSION -1        /* DimensionError        errors.py:8  */
#define OTS_E_NOT_HERMITIAN -2    /* NotHermitian          errors.py:12 */
#define OTS_E_NOT_PD -3           /* NotPositiveDefinite   errors.py:16 */
#define OTS_E_CONVERGENCE -4      /* ConvergenceError      errors.py:20 */
#define OTS_E_SINGULAR -5         /* SingularError         errors.py:24 */
#define OTS_E_NORM_BOUND -6       /* NormBoundError        errors.py:28 */
#define OTS_E_SINGULAR_T -7       /* SingularTError        errors.py:32 */
#define OTS_E_ORTHONORMALITY -8   /* OrthonormalityError   errors.py:36 */
#define OTS_E_INTRA_FAILURE -9    /* IntraFailure          errors.py:40 */
#define OTS_E_BREAKDOWN -10       /* BreakdownError        errors.py:52 */
#define OTS_E_PARAMETER -12       /* ParameterError        errors.py:60 */
#define OTS_E_VALUE -20           /* ValueError (non-finite / layout) core.py:72 */
#define OTS_E_CUDA -30            /* CUDA runtime failure */
#define OTS_E_UNSUPPORTED -31     /* shape outside this build's kernels */

/* seed choices (reflector.py:41 CHOICES) */
#define OTS_CHOICE_MLU 0
#define OTS_CHOICE_QR 1
#define OTS_CHOICE_POLAR 2
#define OTS_CHOICE_EXPLICIT 3
/* intra methods (twostage.py:25 INTRA_METHODS) */
#define OTS_INTRA_HOUSEHOLDER 0
#define OTS_INTRA_CHOLSHIFT 1

typedef struct ots_ctx ots_ctx;

/* One context per (device, host thread).  Owns the device workspace (grown on
 * demand, never shrunk) and a side stream for the diagnostics. */
int ots_ctx_create(int device, ots_ctx** out);
void ots_ctx_destroy(ots_ctx* ctx);
const char* ots_last_error(const ots_ctx* ctx);
int ots_sm_count(const ots_ctx* ctx);
/* 1 when the last ots_two_stage_f64 call on ctx ran the direct-Q pipeline
 * (tile Grams of [V | A], no materialised X), 0 when it ran the
 * materialised-X pipeline (ineligible shape, or the cancellation test sent
 * it there); both compute twostage.py:57-97. */
int ots_last_fast(const ots_ctx* ctx);
int ots_version(void);

/* two_stage_qr(v, a, choice, intra, p)          -- twostage.py:57-97
 * Q (n x k), R (k x k, upper, exact zeros below), S (k0 x k) written to
 * caller buffers.  diag_host (host, 3 doubles) <- [kappa_t, wt_inv_norm,
 * orthonormality defect]  (ReflectorDiagnostics, reflector.py:168-171,241-247;
 * the defect is what reflector.py:220-223 checks against orth_tol).
 * P (k0 x k0) only for choice EXPLICIT (reflector.py:194-203), else NULL. */
int ots_two_stage_f64(ots_ctx* ctx, int64_t n, int64_t k0, int64_t k,
                      const double* V, int64_t ldv, const double* A, int64_t lda,
                      int choice, int intra, const double* P, int64_t ldp,
                      double orth_tol, int allow_defect,
                      double* Q, int64_t ldq, double* R, int64_t ldr,
                      double* S, int64_t lds, double* diag_host, void* stream);

/* two_stage_qr with the Gram V^T V supplied by the caller (device, k0 x k0,
 * ld ldg, full symmetric): the defect check, seed and diagnostics use it and
 * only V_b^T A_b streams over V.  For the Alg. 3 / Krylov driver
 * (twostage.py:100-151), which assembles the Gram of its growing basis
 * block by block (block_householder_qr(..., incremental_gram=True)). */
int ots_two_stage_gram_f64(ots_ctx* ctx, int64_t n, int64_t k0, int64_t k,
                           const double* V, int64_t ldv, const double* A, int64_t lda,
                           int choice, int intra, const double* P, int64_t ldp,
                           double orth_tol, int allow_defect, const double* gram, int64_t ldg,
                           double* Q, int64_t ldq, double* R, int64_t ldr,
                           double* S, int64_t lds, double* diag_host, void* stream);

/* InnerProduct.weighted(b) for a dense SPD b      -- oblique.py:48-56
 * the reference's chol_b = cholesky(b) (core.py:87-105): lower L (strict
 * upper stored as zeros); OTS_E_NOT_PD when a pivot is not positive. */
int ots_dense_cholesky_f64(ots_ctx* ctx, int64_t n, const double* B, int64_t ldb,
                           double* L, int64_t ldl, void* stream);
/* X <- L^{-T} X (n x m); with X = [I_m; 0] this is initial_b_basis(b, m)
 * (oblique.py:93-108: the top block L_m^{-T} over zero rows) */
int ots_dense_trsm_lt_f64(ots_ctx* ctx, int64_t n, int64_t m, const double* L, int64_t ldl,
                          double* X, int64_t ldx, void* stream);
/* Y = L^T X (n x m): the map under which the b-inner product is Euclidean */
int ots_dense_trmm_lt_f64(ots_ctx* ctx, int64_t n, int64_t m, const double* L, int64_t ldl,
                          const double* X, int64_t ldx, double* Y, int64_t ldy, void* stream);
/* b_two_stage_qr(v, a, u, inner, choice)          -- oblique.py:279-315
 * for a dense SPD b = L L^T (L from ots_dense_cholesky_f64) with the
 * canonical u = initial_b_basis(inner, k0+k): the Euclidean path on
 * (L^T V, L^T A), Q = L^{-T} Q' sgn, R = sgn R', S unchanged. */
int ots_b_two_stage_dense_f64(ots_ctx* ctx, int64_t n, int64_t k0, int64_t k,
                              const double* V, int64_t ldv, const double* A, int64_t lda,
                              const double* L, int64_t ldl, int choice,
                              const double* P, int64_t ldp, double orth_tol,
                              double* Q, int64_t ldq, double* R, int64_t ldr,
                              double* S, int64_t lds, double* diag_host, void* stream);

/* b_two_stage_qr(v, a, u, inner, choice)          -- oblique.py:279-315
 * for the weighted inner product M = diag(d) (d > 0, device, n values) with
 * u = initial_b_basis(inner, k0+k) (oblique.py:93-108): computed as the
 * Euclidean path on (D^1/2 V, D^1/2 A), Q = D^-1/2 Q' sgn, R = sgn R'
 * (positive diagonal as oblique.py:232), S unchanged.
 * orth_tol: the B-path default is 1e-6 (oblique.py:125). */
int ots_b_two_stage_diag_f64(ots_ctx* ctx, int64_t n, int64_t k0, int64_t k,
                             const double* V, int64_t ldv, const double* A, int64_t lda,
                             const double* d, int choice, const double* P, int64_t ldp,
                             double orth_tol, double* Q, int64_t ldq, double* R, int64_t ldr,
                             double* S, int64_t lds, double* diag_host, void* stream);

/* householder_qr(a, nonneg_diag)                 -- core.py:61-84
 * LAPACK dgeqrf+dorgqr semantics (R diagonal signs as dlarfg); with
 * nonneg_diag the phase fix of core.py:75-83. */
int ots_householder_qr_f64(ots_ctx* ctx, int64_t m, int64_t k,
                           const double* A, int64_t lda, double* Q, int64_t ldq,
                           double* R, int64_t ldr, int nonneg_diag, void* stream);

/* complex128 variants (configs[3] of BASELINE.json).  Complex arrays are
 * interleaved (re, im) double pairs, row-major, leading dimensions in complex
 * elements, 16-byte aligned.
 *
 * two_stage_qr(v, a, choice, intra="householder", p) -- twostage.py:57-97
 * on c128 data (zgeqrf/zungqr semantics for the intra QR, LAPACK zlarfg
 * signs: R real diagonal).  k <= 64, k0 <= 256. */
int ots_two_stage_c128(ots_ctx* ctx, int64_t n, int64_t k0, int64_t k,
                       const void* V, int64_t ldv, const void* A, int64_t lda,
                       int choice, int intra, const void* P, int64_t ldp,
                       double orth_tol, int allow_defect,
                       void* Q, int64_t ldq, void* R, int64_t ldr,
                       void* S, int64_t lds, double* diag_host, void* stream);

/* b_two_stage_qr for M = diag(d) on c128 data     -- oblique.py:279-315
 * (d real > 0, device; scaled Euclidean path) */
int ots_b_two_stage_diag_c128(ots_ctx* ctx, int64_t n, int64_t k0, int64_t k,
                              const void* V, int64_t ldv, const void* A, int64_t lda,
                              const double* d, int choice, const void* P, int64_t ldp,
                              double orth_tol, void* Q, int64_t ldq, void* R, int64_t ldr,
                              void* S, int64_t lds, double* diag_host, void* stream);

/* shifted_cholesky_qr(a)                          -- core.py:177-202, c128 */
int ots_shifted_cholesky_qr_c128(ots_ctx* ctx, int64_t m, int64_t k,
                                 const void* A, int64_t lda, void* Q, int64_t ldq,
                                 void* R, int64_t ldr, void* stream);

/* modified_lu(z)                                  -- reflector.py:53-77, c128
 * LU packed complex (ld n), p real (n). */
int ots_modified_lu_c128(ots_ctx* ctx, int64_t n, const void* Z, int64_t ldz,
                         void* LU, double* p, void* stream);

/* householder_qr(a, nonneg_diag)                  -- core.py:61-84, c128 */
int ots_householder_qr_c128(ots_ctx* ctx, int64_t m, int64_t k,
                            const void* A, int64_t lda, void* Q, int64_t ldq,
                            void* R, int64_t ldr, int nonneg_diag, void* stream);

/* compute_metrics(v, a, result, augmented) / orthogonality_loss(q, v)
 *                                                  -- metrics.py:25-73
 * Gram-based on the device: out3 (host) = {loss_orth,
 * cross_orth, rel_residual}.  V may be null (k0 = 0), A null (no residual);
 * E: n x k device scratch for a - v s - q r.  1 <= k <= 64, k0 <= 512. */
int ots_stability_f64(ots_ctx* ctx, int64_t n, int64_t k0, int64_t k,
                      const double* V, int64_t ldv, const double* A, int64_t lda,
                      const double* Q, int64_t ldq, const double* R, int64_t ldr,
                      const double* S, int64_t lds, int augmented,
                      double* E, int64_t lde, double* out3, void* stream);

/* shifted_cholesky_qr(a)                          -- core.py:177-202
 * shifted CholeskyQR + 2 refinements; NotPositiveDefinite on breakdown. */
int ots_shifted_cholesky_qr_f64(ots_ctx* ctx, int64_t m, int64_t k,
                                const double* A, int64_t lda, double* Q, int64_t ldq,
                                double* R, int64_t ldr, void* stream);

/* shifted_cholesky_qr(a, refine_passes)          -- core.py:177-202
 * 1 shifted pass + max(0, refine_passes) unshifted ones (real / c128). */
int ots_shifted_cholesky_qr_ex_f64(ots_ctx* ctx, int64_t m, int64_t k,
                                   const double* A, int64_t lda, double* Q, int64_t ldq,
                                   double* R, int64_t ldr, int refine_passes, void* stream);
int ots_shifted_cholesky_qr_ex_c128(ots_ctx* ctx, int64_t m, int64_t k,
                                    const void* A, int64_t lda, void* Q, int64_t ldq,
                                    void* R, int64_t ldr, int refine_passes, void* stream);

/* compute_metrics / orthogonality_loss for complex128 (metrics.py:25-73):
 * as ots_stability_f64 on interleaved data (ld in complex elements);
 * 1 <= k <= 64, k0 <= 256. */
int ots_stability_c128(ots_ctx* ctx, int64_t n, int64_t k0, int64_t k,
                       const void* V, int64_t ldv, const void* A, int64_t lda,
                       const void* Q, int64_t ldq, const void* R, int64_t ldr,
                       const void* S, int64_t lds, int augmented,
                       void* E, int64_t lde, double* out3, void* stream);

/* orthonormality_defect(v) = ||v^* v - I||_2      -- core.py:43-49
 * (the check build_reflector makes at reflector.py:220-223); *out on the
 * host.  k0 <= 1024 (c128: 512). */
int ots_orthonormality_defect_f64(ots_ctx* ctx, int64_t n, int64_t k0,
                                  const double* V, int64_t ldv, double* out, void* stream);
int ots_orthonormality_defect_c128(ots_ctx* ctx, int64_t n, int64_t k0,
                                   const void* V, int64_t ldv, double* out, void* stream);
/* LAPACK sign vector of a positive-diagonal QR from its Q's
 * top k x k block: svec (device, k entries +-1).  Column-blocked intra QR
 * for k > 64 (householder_qr core.py:61-84 semantics).  k <= 512 (c128 256). */
int ots_qr_signs_f64(ots_ctx* ctx, int64_t k, const double* Qtop, int64_t ldq, double* svec, void* stream);
int ots_qr_signs_c128(ots_ctx* ctx, int64_t k, const void* Qtop, int64_t ldq, double* svec, void* stream);

/* {lambda_min, lambda_max} of v^* v (host out2): spectral_norm (core.py:35-40)
 * = sqrt(lambda_max); InnerProduct.norm/defect (oblique.py:75-90) on L^* x. */
int ots_gram_extremes_f64(ots_ctx* ctx, int64_t n, int64_t k0,
                          const double* V, int64_t ldv, double* out2, void* stream);
int ots_gram_extremes_c128(ots_ctx* ctx, int64_t n, int64_t k0,
                           const void* V, int64_t ldv, double* out2, void* stream);

/* Streaming block products of the classical comparators (BCGS / BCGS2 /
 * CholQR, baselines.py:34-175): the inner-product block c = v^* x
 * (baselines.py:66,113,117,169) and the projector update x - v c
 * (:67,114,118,173).  Device pointers; DMMA kernels of the two-stage path.
 *   ots_gram_*   out (p x q, ld ldo) = P^* B over n rows; B null: P^* P
 *                (full Hermitian).  p, q <= 1024 (c128: 512).
 *   ots_update_* X (n x m) = B + V Z, Z p x m; B null: X = V Z; B may
 *                alias X.  p <= 512 (c128: 256). */
int ots_gram_f64(ots_ctx* ctx, int64_t n, int64_t p, const double* P, int64_t ldp,
                 int64_t q, const double* B, int64_t ldb, double* out, int64_t ldo, void* stream);
int ots_gram_c128(ots_ctx* ctx, int64_t n, int64_t p, const void* P, int64_t ldp,
                  int64_t q, const void* B, int64_t ldb, void* out, int64_t ldo, void* stream);
int ots_update_f64(ots_ctx* ctx, int64_t n, int64_t p, const double* V, int64_t ldv,
                   int64_t m, const double* Z, int64_t ldz, const double* B, int64_t ldb,
                   double* X, int64_t ldx, void* stream);
int ots_update_c128(ots_ctx* ctx, int64_t n, int64_t p, const void* V, int64_t ldv,
                    int64_t m, const void* Z, int64_t ldz, const void* B, int64_t ldb,
                    void* X, int64_t ldx, void* stream);

/* modified_lu(z)                                  -- reflector.py:53-77
 * LU (n x n, L strict-lower unit + U upper, packed, ld n) and p (n). */
int ots_modified_lu_f64(ots_ctx* ctx, int64_t n, const double* Z, int64_t ldz,
                        double* LU, double* p, void* stream);

/* Generalized Householder reflector H = I - W T^{-1} W^*, W = [P;0] - V
 * (GenHouseholder, reflector.py:156-165).  The object keeps a pointer to V
 * (caller keeps V alive) and the k0 x k0 seed state on the device. */
typedef struct ots_refl ots_refl;
/* build_reflector(v, choice, p, orth_tol, allow_defect) -- reflector.py:207-228 */
int ots_build_reflector_f64(ots_ctx* ctx, int64_t n, int64_t k0, const double* V, int64_t ldv,
                            int choice, const double* P, int64_t ldp, double orth_tol,
                            int allow_defect, ots_refl** out, double* defect_host, void* stream);
void ots_reflector_destroy(ots_refl* r);
/* apply_reflector(h, x, adjoint)                   -- reflector.py:231-238 (m <= 64) */
int ots_apply_reflector_f64(ots_ctx* ctx, const ots_refl* r, int64_t m, const double* X, int64_t ldx,
                            double* Y, int64_t ldy, int adjoint, void* stream);
/* reflector_diagnostics(h) -> [kappa_t, wt_inv_norm] -- reflector.py:241-247 */
int ots_reflector_diagnostics_f64(ots_ctx* ctx, const ots_refl* r, double* diag_host, void* stream);
/* t_solver.solve(b, adjoint) on a device k0 x m block  -- reflector.py:80-153 */
int ots_reflector_tsolve_f64(ots_ctx* ctx, const ots_refl* r, int64_t m, double* B, int64_t ldb,
                             int adjoint, void* stream);
/* which = 0: seed P; which = 1: dense T (t_solver.reconstruct()) */
int ots_reflector_get_f64(ots_ctx* ctx, const ots_refl* r, int which, double* out, int64_t ldo,
                          void* stream);

/* complex128 reflector objects (same semantics, interleaved data, ld in
 * complex elements; k0 <= 256, m <= 64 per apply) -- reflector.py:156-247 */
typedef struct ots_zrefl ots_zrefl;
int ots_build_reflector_c128(ots_ctx* ctx, int64_t n, int64_t k0, const void* V, int64_t ldv,
                             int choice, const void* P, int64_t ldp, double orth_tol,
                             int allow_defect, ots_zrefl** out, double* defect_host, void* stream);
void ots_zreflector_destroy(ots_zrefl* r);
int ots_apply_reflector_c128(ots_ctx* ctx, ots_zrefl* r, int64_t m, const void* X, int64_t ldx,
                             void* Y, int64_t ldy, int adjoint, void* stream);
int ots_reflector_diagnostics_c128(ots_ctx* ctx, ots_zrefl* r, double* diag_host, void* stream);
int ots_reflector_tsolve_c128(ots_ctx* ctx, ots_zrefl* r, int64_t m, void* B, int64_t ldb,
                              int adjoint, void* stream);
int ots_reflector_get_c128(ots_ctx* ctx, ots_zrefl* r, int which, void* out, int64_t ldo, void* stream);

/* Per-phase device timings of the last call (CUDA events on the launching
 * stream), enabled with ots_set_profiling(ctx, 1).  names: '\n'-separated. */
int ots_set_profiling(ots_ctx* ctx, int enable);
/* Number of this library's kernels launched by the last full call. */
int ots_last_launch_count(const ots_ctx* ctx);
/* Measured FP64 DMMA peak of this device (TFLOP/s), the FP64 roofline
 * denominator (MEASURED_PEAKS.json has no FP64 figure). */
int ots_fp64_peak(ots_ctx* ctx, double* tflops);
/* Kernel-section cycle counters (only in an -DOTS_TIMING build; else zeros). */
int ots_debug_counters(unsigned long long* out16, int reset);
int ots_last_profile(const ots_ctx* ctx, char* names, int names_cap, float* ms, int cap);

/* ---- phase-split entry points for row-sharded multi-GPU execution ------
 * Each rank owns rows [row0, row0 + n_local) of V, A, Q (rank 0: row0 = 0,
 * n_local >= k0 + k).  Host-side NCCL collectives run between phases
 * (SURVEY.md §8(e)); paper_2602_14449_b200/dist.py is the orchestrator.
 *
 *  1  ots_dist_gram      local [V^T V | V_b^T A_b] partial  -> allreduce(sum)
 *  2  ots_dist_seed      redundant seed / T / Z1 from the summed Gram and the
 *                        rank-0 top rows (broadcast)
 *  3  ots_dist_factor    X = A_b + V_b Z1, local TSQR -> rank R (KT x KT)
 *                        -> allgather
 *  4  ots_dist_tree      redundant top QR of the gathered R's; this rank's C
 *  5  ots_dist_qform     local Q_, partial Y2 = -V_b^T Q_ -> allreduce(sum);
 *                        rank 0 also the sign vector -> broadcast
 *  6  ots_dist_finish    Z2 = T^{-1} Y2, Q = (Q_ + V_b Z2) diag(s), rank 0 top
 */
int ots_dist_begin(ots_ctx* ctx, int64_t n_local, int64_t row0, int64_t k0, int64_t k,
                   const double* V, int64_t ldv, const double* A, int64_t lda,
                   double* Q, int64_t ldq, int choice, const double* P, int64_t ldp,
                   double orth_tol, void* stream);
/* element counts of the exchanged device buffers: [gram, top rows, KT, y2] */
int ots_dist_sizes(ots_ctx* ctx, int64_t* out4);
int ots_dist_gram(ots_ctx* ctx, double* gram_out);
int ots_dist_top_rows(ots_ctx* ctx, double* top_rows_out);   /* rank 0 writes */
/* optional, between ots_dist_top_rows (+ broadcast) and ots_dist_gram: start
 * the V_t-only part of the seed beside this rank's Gram */
int ots_dist_seed_early(ots_ctx* ctx, const double* top_rows);
int ots_dist_seed(ots_ctx* ctx, const double* gram_sum, const double* top_rows);
int ots_dist_factor(ots_ctx* ctx, double* r_local_out);      /* KT x KT */
int ots_dist_tree(ots_ctx* ctx, const double* r_all, int nranks, int rank);
int ots_dist_qform(ots_ctx* ctx, double* y2_out, double* sign_out);  /* sign: rank 0 */
int ots_dist_finish(ots_ctx* ctx, const double* y2_sum, const double* sign,
                    double* R, int64_t ldr, double* S, int64_t lds, double* diag_host);

#ifdef __cplusplus
}
#endif
#endif /* OTS_H_ */
