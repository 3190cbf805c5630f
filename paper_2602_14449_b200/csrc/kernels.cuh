// Argument structs and launchers of the streaming / chain kernels (shared by
// tsgemm.cu, chainqr.cu and ots_api.cu).
#pragma once
#include <cuda_runtime.h>

namespace ots {

struct TnArgs {
  const double* P; long ldp; int pc0; int pcols;   // P columns [pc0, pc0+pcols)
  const double* B; long ldb; int bc0; int bcols;   // B2 columns
  long row_begin, row_end;                          // rows reduced over
  long b_row_begin;                                 // B2 rows < this are zero
  long p_row_begin;                                 // P rows < this are zero
  long rows_per_cta;                                // set by the launcher
  double* partial;                                  // [grid][PW][NTOT]
};

struct NnArgs {
  const double* P; long ldp; int kdim;        // P rows x kdim
  const double* Z; long ldz;                  // kdim x ncols
  const double* B; long ldb;                  // may be null (treated as 0)
  double* X; long ldx;
  int ncols;
  long row_begin, row_end;
  const double* colscale;                     // device, ncols entries of +-1, or null
  int* tile_counter;                          // device ticket counter (dynamic tiles) or null
};

struct ChainGeom {
  long nrows;            // rows of the level matrix
  int b;                 // structured tile rows
  int L;                 // structured tiles per chain (max)
  long rpc;              // rows per chain = KT + L*b
  int nchains;
};

struct FactorArgs {
  double* D; long ldd; int ncols;
  ChainGeom G;
  double* U;             // per tile KT*KT, tile id = chain*(L+1) + t
  double* Rout;          // stacked chain R's: chain*KT rows, ld KT
  int head_tri;          // input rows are stacked upper-triangular R's (tree levels);
                         // 2 at launch: level-0 redo of the chains the Gram-form
                         // factor flagged (chain_factor_kernel<KT, true>)
};

// Gram-form tile factorization of level 0 (KT = 64; gsweep.inc).  Pass 1
// reads X (never writes it) and per tall tile (G.b rows, a multiple of 128)
// produces T, the coefficient matrix Cc with Y = X_tile Cc, and the running
// chain R; a chain whose tiles fail the cancellation bound is flagged
// (flags[chain] = 1 and Rout[chain][KT-1][0] = 1) and redone by the exact
// register-tile kernel on 128-row tiles of the same chain rows
// (FactorArgs::head_tri = 2).  Y is never formed: the Q formation of an
// accepted chain computes Q_tile = -X_tile (Cc T C) directly.
struct GsweepArgs {
  double* D; long ldd; int ncols;   // level-0 rows (X in, untouched)
  ChainGeom G;           // tall-tile geometry
  double* U;             // T per tile: chain * tslots + t
  double* Rout;          // chain R's
  double* Cc;            // per tile KT*KT (chain * (G.L+1) + t; tile 0 unused)
  double* Hs;            // head rows per chain (KT x KT): R upper, V strictly lower
  int* flags;            // per chain: 1 = redo exactly (128-row tiles)
  long tslots;           // T slots per chain (the 128-row geometry's L + 1)
  const int* abort_flag = nullptr;   // nonzero at kernel start: do nothing
};

struct QformArgs {
  double* D; long ldd; int ncols;
  ChainGeom G;
  const double* T;       // per tile KT*KT
  const double* Cin;     // stacked chain C's (chain*KT rows, ld KT)
  int grid_max = 0;      // CTAs at most (0: one per SM)
  // level 0 of the Gram-form factor (GsweepArgs): mode 1 forms only the
  // flagged chains (128-row geometry G, Y in D), mode 2 only the accepted
  // ones (tall geometry G, X in D, Cc / Hs); mode 0 every chain
  int mode = 0;
  const double* Cc = nullptr;
  const double* Hs = nullptr;
  const int* flags = nullptr;
  long tslots = 0;       // T slots per chain (0: G.L + 1)
  // gs_coef (direct-Q pipeline): K_t of tall tile (chain, t) goes to
  // Kout + (chain * G.L + t - 1) * kstride + koff instead of being applied
  double* Kout = nullptr;
  long kstride = 0, koff = 0;
};

// Direct-Q pipeline (fastpath.cu): every pointer is offset to the first chain
// row (the QR rows), geometry G = the Gram-form factor's tall tiles.
struct FastArgs {
  const double* V; long ldv;
  const double* A; long lda;
  double* D; long ldd;       // Q rows (heads only: X, then Q_, then Q)
  int k0, k, PW;             // PW = k0 padded to 32
  ChainGeom G;
  double* TG; long tg_stride;   // per tall tile (chain * L + t - 1): [VV | VA] PW x (PW + 64), then AA 64 x 64
  double* part;              // per-CTA totals of [VV | VA]
  const double* Z1; int ldz;
  double* M;                 // the factor's Cc slots (tile Gram of X in, Cc out)
  double* Coef;              // per tall tile: (PW + 64) x 64 = [Z1 K + Z2; K]
  int* flags;                // [0]: bit 0 cancellation, bit 1 a chain flagged by the sweep
  int* ticket;               // dynamic tile counter
};
cudaError_t launch_tgram(const FastArgs& a, int grid, cudaStream_t st);
cudaError_t launch_tgram_reduce(const FastArgs& a, int nparts, const double* Vtop, int ntop, double* out, int ldg,
                                cudaStream_t st);
cudaError_t launch_head_rows(const FastArgs& a, int mode, const double* Z, int ldz, const double* colscale,
                             double* part, int grid, cudaStream_t st);
cudaError_t launch_tile_alg(const FastArgs& a, cudaStream_t st);
cudaError_t launch_coef_b(const FastArgs& a, double* ypart, int grid, cudaStream_t st);
cudaError_t launch_coef_add_z2(const FastArgs& a, const double* Z2, int ldz, cudaStream_t st);
cudaError_t launch_final_nn(const FastArgs& a, const double* colscale, double* X, long ldx, cudaStream_t st);
cudaError_t launch_final_nn128(const FastArgs& a, double* X, long ldx, int ncols_out, cudaStream_t st);
cudaError_t launch_fast_flags(const int* chain_flags, int nch, int* flags, cudaStream_t st);

cudaError_t launch_tsgemm_tn(const TnArgs& a, int PW, int BW, bool alias, bool sym, int grid, cudaStream_t st);
cudaError_t launch_reduce(const double* partial, int nparts, long count, double* out, double alpha, cudaStream_t st);
cudaError_t launch_reduce_strided(const double* partial, int nparts, int rows, int cols, int ldp, double* out,
                                  long ldo, double alpha, cudaStream_t st);
cudaError_t launch_tsgemm_nn(const NnArgs& a, int KT, int nsm, cudaStream_t st);
cudaError_t launch_chain_factor(const FactorArgs& a, int KT, cudaStream_t st);
cudaError_t launch_chain_qform(const QformArgs& a, int KT, cudaStream_t st);
cudaError_t launch_gs_gram(const GsweepArgs& a, cudaStream_t st);
cudaError_t launch_chain_gsweep(const GsweepArgs& a, cudaStream_t st);
cudaError_t launch_gs_qform(const QformArgs& a, cudaStream_t st);
cudaError_t launch_gs_coef(const QformArgs& a, cudaStream_t st);
// complex128 TSQR (zchain.cu): same argument records, pointers to interleaved
// (re, im) data, leading dimensions in complex units
using ZFactorArgs = FactorArgs;
using ZQformArgs = QformArgs;
cudaError_t launch_zchain_factor(const ZFactorArgs& a, int KT, cudaStream_t st);
cudaError_t launch_zchain_qform(const ZQformArgs& a, int KT, cudaStream_t st);
// Gram-form complex level 0 on tall tiles (zchain.cu, zpath.inc): geometry G =
// chains of a 64-row head + L tall tiles; all matrices complex (re, im) 64 x 64
// row-major unless noted.
struct ZgsArgs {
  ChainGeom G;
  const double* TG; long tg_stride;   // per tile (chain * L + t - 1): real Gram of the interleaved view, ld 192
  const double* Rh;                   // head R per chain
  double* T;                          // T per tile: chain * (L + 1) + t
  double* Cc;                         // Cc per tile: chain * (L + 1) + t
  double* Rout;                       // chain R's
  int* flags;                         // per chain: 1 = cancellation, take the exact path
  int ncols;                          // complex columns
  const double* Cin = nullptr;        // coef: stacked chain C's
  double* Kexp = nullptr;             // coef: per tile 128 x 128 real right-multiplier
  double* Chead = nullptr;            // coef: per chain C for the head rows
  double* Hsave = nullptr;            // heads: per chain 64 x 64 side buffer
};
cudaError_t launch_zgs_sweep(const ZgsArgs& a, cudaStream_t st);
cudaError_t launch_zgs_coef(const ZgsArgs& a, cudaStream_t st);
cudaError_t launch_zgs_heads(const ZgsArgs& a, double* D, long ldd, int mode, cudaStream_t st);
int zchain_bmax();
int chain_bmax(int KT);
int debug_counters(unsigned long long* out, int reset);
// dense SPD weights (dense.cu): in-place lower Cholesky, Y = L^T X, X <- L^{-T} X
cudaError_t launch_dense_cholesky(double* A, long ld, int n, int* status, cudaStream_t st);
cudaError_t launch_trmm_lt(const double* L, long ldl, const double* X, long ldx, double* Y, long ldy, int n, int m,
                           cudaStream_t st);
cudaError_t launch_trsm_lt(const double* L, long ldl, double* X, long ldx, int n, int m, cudaStream_t st);
cudaError_t launch_colsign(double* Q, long ldq, long n, int k, const double* R, long ldr, cudaStream_t st);

}  // namespace ots
