// Small-matrix state shared by the single-CTA kernels of small.cu.
#pragma once
#include <cuda_runtime.h>

namespace ots {

enum { CHOICE_MLU = 0, CHOICE_QR = 1, CHOICE_POLAR = 2, CHOICE_EXPLICIT = 3 };
constexpr int SMALL_NT = 512;

struct SmallState {
  int k0, k, ld;             // ld = padded leading dim of every small matrix
  int choice;
  int allow_defect;
  double orth_tol;
  // inputs
  const double* V; long ldv;   // top k0 rows are V_t
  const double* A; long lda;   // top k0 rows are A_t
  const double* Gfull; long ldgf; int gf_acol;  // reduced [V^T V | V_b^T A_b]
  const double* Pexp; int ldpe;                  // explicit seed (device) or null
  // small matrices (k0 x k0 or k0 x k, all with leading dim ld)
  double *G, *Vt, *At, *VbA, *P, *Tf, *Tdense, *Wt, *Z1, *Z2, *X1, *X2, *D1, *D2, *Sd;
  double *pvec, *tau, *sig, *sig2, *svec;
  int* piv;
  // outputs
  double* Sout; int lds_out;   // S (k0 x k)
  // B-inner (M = diag(d)) diagnostics: W = D^{-1/2} W' is unweighted, so
  // W^T W = W_t'^T D_t^{-1} W_t' + V^T V (unweighted Gram Gu) - V_t'^T D_t^{-1} V_t'
  const double* Gu; int ldgu;  // null for the Euclidean path
  const double* dinv_top;      // 1/d on the k0 top rows
  // dense B = L L^T: W_top = L_m^{-T} P - V_t (unweighted), W^T W = W_top^T
  // W_top + Gu - V_t^T V_t with V_t the ORIGINAL top rows (dinv_top unused)
  const double* Ltinv; int ldlt;     // L_m^{-T} (k0 x k0, upper), or null
  const double* Vorig; long ldvo;    // original V (top k0 rows read)
  double* dg[6];               // diagnostics scratch (k0 x k0 each, ld)
  double* dlam;                // [3] per-CTA eigenvalues of the diagnostics kernel
  int* dcount;                 // CTA completion counter of the diagnostics kernel
  double* diag;                // [kappa_t, wt_inv_norm, defect]
  int* status;                 // [0] = status code
};

// complex128 k0 x k0 state (zsmall.inc).  Complex matrices are interleaved
// double2 arrays (ld in complex units); `r` is the stacked real embedding
// (k0' = 2 k0, choice EXPLICIT = pivoted LU of phi(T)) used for the T-solves
// and the diagnostics kernel.
struct ZState {
  int k0, k, ldc;
  int choice, allow_defect;
  double orth_tol;
  const double2* V; long ldv;       // top k0 rows of V, A (device)
  const double2* A; long lda;
  const double* Gr; long ldgr;      // real Gram of the interleaved V view (lower valid)
  const double* VbAr; long ldvba;   // real V_b'^T A_b' (2k0 x 2k)
  const double2* Pexp; int ldpe;
  double2 *G, *Vt, *At, *VbA, *P, *T, *Wt, *Z1, *Z2, *W1, *W2, *tau;
  double *Z1x, *Z2x; int ldzx;      // interleaved real expansions (2k0 x 2k)
  double *svec, *svec2;             // sign recovery (k), per real column (2k)
  double2* Sout; int lds_out;
  // B-inner (M = diag(d)): real Gram of the unscaled V view -> phi(V^H V)
  // into GuE for the diagnostics (r.Gu = GuE), 1/d on the top rows -> dinvE
  const double* Gur; long ldgur;
  const double* dB;
  double *GuE, *dinvE;
  SmallState r;
};

cudaError_t launch_seed(const SmallState& s, cudaStream_t st);
bool seed_uses_cluster(const SmallState& s);   // polar seed on a 2-CTA cluster
// part 0: V_t-only seed construction (status[1]); part 1: Gram checks + Z1, S
cudaError_t launch_seed_split(const SmallState& s, int part, cudaStream_t st);
cudaError_t launch_stability(const double* Gvv, long ldvv, const double* Gvq, long ldvq, const double* Gqq,
                             long ldqq, const double* Gee, long ldee, const double* Gaa, long ldaa, int k0, int k,
                             int augmented, double* work, double* out3, cudaStream_t st);
cudaError_t launch_qr_signs(const double* Qtop, long ldq, int k, double* work, double* svec, cudaStream_t st);
cudaError_t launch_zqr_signs(const void* Qtop, long ldq, int k, void* work, double* svec, cudaStream_t st);
cudaError_t launch_sym_extremes(const double* G, long ldg, int m, double* work, double* out2, cudaStream_t st);
cudaError_t launch_neg_copy(const double* X, long ldx, int r, int c, double* Y, long ldy, cudaStream_t st);
cudaError_t launch_zseed(const ZState& z, cudaStream_t st, int part = 0);
cudaError_t launch_zcholqr_step(const double* Gr, long ldg, int k, long m, int shift, void* W, int ld,
                                double* Zx, int ldzx, void* R, int* status, cudaStream_t st);
cudaError_t launch_zmlu(const void* Z, int ldz, int n, void* LU, double* p, double* work, int* status,
                        cudaStream_t st);
cudaError_t launch_zidentity(void* D, int n, int ld, cudaStream_t st);
cudaError_t launch_zrefl_apply(const ZState& z, const double* VhXr, long ldy, int m, int adjoint, const void* X,
                               long ldx, void* Ytop, long ldyt, cudaStream_t st);
cudaError_t launch_ztsolve(const ZState& z, void* B, long ldb, int m, int adjoint, cudaStream_t st);
cudaError_t launch_zz2(const ZState& z, const double* Y2r, long ldy, void* Qtop, long ldq, cudaStream_t st);
cudaError_t launch_zsign(const ZState& z, const void* Qtop, long ldq, const void* Rfin, int ldr, void* Rout,
                         long ldro, cudaStream_t st);
cudaError_t launch_diag(const SmallState& s, cudaStream_t st);
cudaError_t launch_z2(const SmallState& s, cudaStream_t st);
cudaError_t launch_refl_apply(const SmallState& s, int adjoint, cudaStream_t st);
cudaError_t launch_tsolve(const SmallState& s, double* B, int ldb, int m, int adjoint, cudaStream_t st);
cudaError_t launch_sign(const SmallState& s, const double* Qtop, long ldq, const double* Rfin, int ldr,
                        double* Rout, int ldro, cudaStream_t st);
cudaError_t launch_qtop(const SmallState& s, double* Q, long ldq, cudaStream_t st);
cudaError_t launch_cholqr_step(const double* Gf, int ldg, int k, long m, int shift, double* W, int ld,
                               double* Z, double* R, int* status, cudaStream_t st);
cudaError_t launch_mlu(const double* Z, int ldz, int n, double* LU, double* p, double* work, int* status,
                       cudaStream_t st);

}  // namespace ots
