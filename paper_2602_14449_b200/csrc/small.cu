// k0 x k0 / k0 x k dense work on one CTA (FP64): seed construction of the
// generalized Householder reflector (reflector.py:174-204), the T-solvers
// (reflector.py:80-153), the orthonormality check (core.py:43-49 via
// reflector.py:220-223), diagnostics from k0 x k0 data only (reflector.py:
// 241-247), LAPACK sign recovery for the intra QR
// (SURVEY Appendix A.1), and the small tails of Algorithm 1 (twostage.py:92,96).
//
// All routines are block-cooperative: every thread of the CTA calls them.
// Matrices are row-major with an explicit leading dimension and may live in
// shared or global (L2-resident) memory (generic addressing).
#include "common.cuh"
#include "small.cuh"
#include <cstdlib>

namespace ots {

#ifdef OTS_TIMING
__device__ unsigned long long g_dbg_small[16];
#define SMARK(slot, t0) if (threadIdx.x == 0) { long long _t = clock64(); atomicAdd(&g_dbg_small[slot], (unsigned long long)(_t - t0)); t0 = _t; }
#else
#define SMARK(slot, t0)
#endif

#define BLK_FOR(i, n) for (int i = threadIdx.x; i < (n); i += blockDim.x)

__device__ __forceinline__ double block_sum(double v, double* red) {
  // red: >= 32 doubles of smem scratch
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];
  __syncthreads();
  return s;
}

__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = red[0];
  for (int i = 1; i < nw; ++i) s = fmax(s, red[i]);
  __syncthreads();
  return s;
}

__device__ void blk_copy(double* D, int ldd, const double* Sr, int lds, int m, int n) {
  BLK_FOR(e, m * n) { int i = e / n, j = e - i * n; D[i * ldd + j] = Sr[(long)i * lds + j]; }
}

__device__ void blk_identity(double* D, int ldd, int n) {
  BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; D[i * ldd + j] = (i == j) ? 1.0 : 0.0; }
}

// C = alpha * op(A) op(B) + beta * C.  Register-tiled: a warp owns 4-row x
// 128-column strips of C, lane l the columns l + 32c (coalesced B rows,
// broadcast A entries).  Summation order per entry is p = 0..k-1 (fma), as
// in a plain dot product.  C must not alias A or B.
__device__ void blk_gemm(double* Cm, int ldc, const double* A, int lda, bool ta, const double* B,
                         int ldb, bool tb, int m, int n, int k, double alpha, double beta) {
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int rs = (m + 3) >> 2, cs = (n + 127) >> 7;
  for (int t = w; t < rs * cs; t += nw) {
    const int i0 = (t / cs) * 4, j0 = (t % cs) * 128;
    int jj[4];
    bool jv[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) { jj[c] = j0 + l + 32 * c; jv[c] = jj[c] < n; }
    bool iv[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) iv[r] = i0 + r < m;
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
    for (int p0 = 0; p0 < k; p0 += 4) {  // 4-deep batches keep loads in flight
      double a[4][4], b[4][4];
#pragma unroll
      for (int pp = 0; pp < 4; ++pp) {
        const int p = p0 + pp;
        const bool pv = p < k;
#pragma unroll
        for (int r = 0; r < 4; ++r)
          a[pp][r] = (pv && iv[r]) ? (ta ? A[p * lda + i0 + r] : A[(i0 + r) * lda + p]) : 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          b[pp][c] = (pv && jv[c]) ? (tb ? B[jj[c] * ldb + p] : B[p * ldb + jj[c]]) : 0.0;
      }
#pragma unroll
      for (int pp = 0; pp < 4; ++pp)
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = fma(a[pp][r], b[pp][c], acc[r][c]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (iv[r] && jv[c]) {
          double* cp = Cm + (i0 + r) * ldc + jj[c];
          *cp = alpha * acc[r][c] + (beta == 0.0 ? 0.0 : beta * *cp);
        }
  }
  __syncthreads();
}

// Solve op(A) X = B in place (B: n x nrhs).  A triangular (lower/upper as
// stored); trans solves with A^T.  Substitution order as trtrs.
// Register-resident substitution: a group of G lanes (same warp) owns one
// right-hand side at a time, lane gl holding rows gl + G q (q < RPT) in
// registers; x_i is broadcast by its owner with a width-G shuffle.  The
// arithmetic per entry (x_i = b_i / a_ii, b_r -= e_ri x_i in order of i) is
// that of the plain column sweep.
template <int RPT, bool TRANS, bool ELOWER>
__device__ __noinline__ void trsm_reg(const double* A, int lda, bool unit, double* B, int ldb, int n,
                                      int nrhs, int G) {
  constexpr bool trans = TRANS, elower = ELOWER;
  const int gl = threadIdx.x % G, grp = threadIdx.x / G, ngrp = blockDim.x / G;
  const unsigned mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  const int nq = (n + G - 1) / G;
  for (int j = grp; j < nrhs; j += ngrp) {
    double b[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) { const int r = gl + G * q; b[q] = (r < n) ? B[r * ldb + j] : 0.0; }
    for (int s = 0; s < nq * G; ++s) {
      const int q = elower ? (s / G) : (nq - 1 - s / G);
      const int g = elower ? (s % G) : (G - 1 - s % G);
      const int i = g + G * q;
      if (i >= n) continue;
      double bq = 0.0;
#pragma unroll
      for (int qq = 0; qq < RPT; ++qq) if (qq == q) bq = b[qq];
      const double dii = unit ? 1.0 : A[i * lda + i];
      const double x = __shfl_sync(mask, bq, g, G) / dii;
#pragma unroll
      for (int q2 = 0; q2 < RPT; ++q2) {
        const int r = gl + G * q2;
        if (r == i) b[q2] = x;
        else if (elower ? (r > i && r < n) : (r < i))
          b[q2] = fma(-(trans ? A[i * lda + r] : A[r * lda + i]), x, b[q2]);
      }
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) { const int r = gl + G * q; if (r < n) B[r * ldb + j] = b[q]; }
  }
}

__device__ void blk_trsm(const double* A, int lda, bool lower, bool trans, bool unit, double* B,
                         int ldb, int n, int nrhs) {
  // effective matrix E = op(A); E is lower iff (lower xor trans)
  const bool elower = lower != trans;
  __syncthreads();
  if (n <= 0 || nrhs <= 0) return;
  int G = 1;
  while (G < 32 && G * 2 * nrhs <= (int)blockDim.x) G *= 2;
  while (G < 32 && (n + G - 1) / G > 16) G *= 2;
  const int rpt = (n + G - 1) / G;
#define OTS_TRSM(R)                                                                   \
  if (trans) { if (elower) trsm_reg<R, true, true>(A, lda, unit, B, ldb, n, nrhs, G);   \
               else trsm_reg<R, true, false>(A, lda, unit, B, ldb, n, nrhs, G); }       \
  else { if (elower) trsm_reg<R, false, true>(A, lda, unit, B, ldb, n, nrhs, G);        \
         else trsm_reg<R, false, false>(A, lda, unit, B, ldb, n, nrhs, G); }
  if (rpt <= 8) { OTS_TRSM(8) }
  else if (rpt <= 16) { OTS_TRSM(16) }
#undef OTS_TRSM
  else {
    for (int s = 0; s < n; ++s) {  // n > 512: plain column sweep
      const int i = elower ? s : (n - 1 - s);
      const double dii = unit ? 1.0 : A[i * lda + i];
      BLK_FOR(j, nrhs) B[i * ldb + j] /= dii;
      __syncthreads();
      const int rem = elower ? (n - 1 - i) : i;
      BLK_FOR(e, rem * nrhs) {
        int rr = e / nrhs, j = e - rr * nrhs;
        int r = elower ? (i + 1 + rr) : rr;
        double eri = trans ? A[i * lda + r] : A[r * lda + i];
        B[r * ldb + j] = fma(-eri, B[i * ldb + j], B[r * ldb + j]);
      }
      __syncthreads();
    }
  }
  __syncthreads();
}

// dgeqr2 on an m x n block (m >= n), LAPACK dlarfg conventions; v below the
// diagonal, R on/above, tau[n].
__device__ void blk_geqr2(double* A, int lda, int m, int n, double* tau, double* red) {
  for (int j = 0; j < n; ++j) {
    double s2 = 0.0;
    for (int r = j + 1 + (int)threadIdx.x; r < m; r += blockDim.x) { double x = A[r * lda + j]; s2 = fma(x, x, s2); }
    s2 = block_sum(s2, red);
    const double alpha = A[j * lda + j];
    double beta = alpha, tj = 0.0, scal = 0.0;
    if (s2 != 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, s2)), alpha);
      tj = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    __syncthreads();
    if (s2 != 0.0)
      for (int r = j + 1 + (int)threadIdx.x; r < m; r += blockDim.x) A[r * lda + j] *= scal;
    if (threadIdx.x == 0) { A[j * lda + j] = beta; tau[j] = tj; }
    __syncthreads();
    if (tj != 0.0) {
      // trailing columns c > j: w = v^T A[:, c]; A[:,c] -= tau w v   (one warp per column)
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int c = j + 1 + w; c < n; c += nw) {
        double d = 0.0;
        for (int r = j + 1 + l; r < m; r += 32) d = fma(A[r * lda + j], A[r * lda + c], d);
        d = warp_sum(d) + A[j * lda + c];
        const double wc = tj * d;
        if (l == 0) A[j * lda + c] -= wc;
        for (int r = j + 1 + l; r < m; r += 32) A[r * lda + c] = fma(-wc, A[r * lda + j], A[r * lda + c]);
      }
    }
    __syncthreads();
  }
}

// dorg2r: Q (m x n) from the reflectors stored in A (in place -> Q); W scratch n*... unused
__device__ void blk_org2r(double* A, int lda, int m, int n, const double* tau, double* red) {
  // Q = H_0 ... H_{n-1} [I; 0], accumulated backwards in place like dorg2r.
  for (int j = n - 1; j >= 0; --j) {
    const double tj = tau[j];
    // apply H_j to Q[j:m, j+1:n]  (columns right of j already hold Q columns)
    if (j < n - 1 && tj != 0.0) {
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int c = j + 1 + w; c < n; c += nw) {
        double d = 0.0;
        for (int r = j + 1 + l; r < m; r += 32) d = fma(A[r * lda + j], A[r * lda + c], d);
        d = warp_sum(d) + A[j * lda + c];
        const double wc = tj * d;
        if (l == 0) A[j * lda + c] -= wc;
        for (int r = j + 1 + l; r < m; r += 32) A[r * lda + c] = fma(-wc, A[r * lda + j], A[r * lda + c]);
      }
    } else if (j < n - 1) {
      // tau == 0: H_j = I, nothing to do for the trailing columns
    }
    __syncthreads();
    // column j: Q[j:, j] = e_j - tau v ; Q[0:j, j] = 0
    for (int r = (int)threadIdx.x; r < m; r += blockDim.x) {
      if (r < j) A[r * lda + j] = 0.0;
      else if (r == j) A[r * lda + j] = 1.0 - tj;
      else A[r * lda + j] = -tj * A[r * lda + j];
    }
    __syncthreads();
  }
}

// Column-major twins (A[c * lda + r] holds entry (r, c)): the same
// Householder sweep with every column contiguous, so the one-warp-per-column
// dots and updates are coalesced when the matrix lives in global memory
// (k0 x k0 seeds too large for shared memory).
__device__ void blk_geqr2_cm(double* A, int lda, int m, int n, double* tau, double* red) {
  for (int j = 0; j < n; ++j) {
    double s2 = 0.0;
    for (int r = j + 1 + (int)threadIdx.x; r < m; r += blockDim.x) { double x = A[(j) * lda + (r)]; s2 = fma(x, x, s2); }
    s2 = block_sum(s2, red);
    const double alpha = A[(j) * lda + (j)];
    double beta = alpha, tj = 0.0, scal = 0.0;
    if (s2 != 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, s2)), alpha);
      tj = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    __syncthreads();
    if (s2 != 0.0)
      for (int r = j + 1 + (int)threadIdx.x; r < m; r += blockDim.x) A[(j) * lda + (r)] *= scal;
    if (threadIdx.x == 0) { A[(j) * lda + (j)] = beta; tau[j] = tj; }
    __syncthreads();
    if (tj != 0.0) {
      // trailing columns c > j: w = v^T A[:, c]; A[:,c] -= tau w v   (one warp per column)
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int c = j + 1 + w; c < n; c += nw) {
        double d = 0.0;
        for (int r = j + 1 + l; r < m; r += 32) d = fma(A[(j) * lda + (r)], A[(c) * lda + (r)], d);
        d = warp_sum(d) + A[(c) * lda + (j)];
        const double wc = tj * d;
        if (l == 0) A[(c) * lda + (j)] -= wc;
        for (int r = j + 1 + l; r < m; r += 32) A[(c) * lda + (r)] = fma(-wc, A[(j) * lda + (r)], A[(c) * lda + (r)]);
      }
    }
    __syncthreads();
  }
}

// dorg2r: Q (m x n) from the reflectors stored in A (in place -> Q); W scratch n*... unused
__device__ void blk_org2r_cm(double* A, int lda, int m, int n, const double* tau, double* red) {
  // Q = H_0 ... H_{n-1} [I; 0], accumulated backwards in place like dorg2r.
  for (int j = n - 1; j >= 0; --j) {
    const double tj = tau[j];
    // apply H_j to Q[j:m, j+1:n]  (columns right of j already hold Q columns)
    if (j < n - 1 && tj != 0.0) {
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int c = j + 1 + w; c < n; c += nw) {
        double d = 0.0;
        for (int r = j + 1 + l; r < m; r += 32) d = fma(A[(j) * lda + (r)], A[(c) * lda + (r)], d);
        d = warp_sum(d) + A[(c) * lda + (j)];
        const double wc = tj * d;
        if (l == 0) A[(c) * lda + (j)] -= wc;
        for (int r = j + 1 + l; r < m; r += 32) A[(c) * lda + (r)] = fma(-wc, A[(j) * lda + (r)], A[(c) * lda + (r)]);
      }
    } else if (j < n - 1) {
      // tau == 0: H_j = I, nothing to do for the trailing columns
    }
    __syncthreads();
    // column j: Q[j:, j] = e_j - tau v ; Q[0:j, j] = 0
    for (int r = (int)threadIdx.x; r < m; r += blockDim.x) {
      if (r < j) A[(j) * lda + (r)] = 0.0;
      else if (r == j) A[(j) * lda + (r)] = 1.0 - tj;
      else A[(j) * lda + (r)] = -tj * A[(j) * lda + (r)];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Blocked Householder QR / Q formation of a square n x n column-major matrix
// in global memory (k0 x k0 seeds too large for shared memory, k0 > ~158):
// QNB-column panels factored by the unblocked sweep above, compact-WY T per
// panel (dlarft, forward), and the trailing columns updated a - V T^T V^T a
// (geqrf) / a - V T V^T a (orgqr, backward) one column per warp with the
// panel's V staged in shared memory -- one pass over the trailing matrix per
// panel instead of one per column.  Same reflectors (v, tau) as the
// unblocked sweep, so R and Q match it to rounding.
// ---------------------------------------------------------------------------

// lane l ends with the warp-wide sum of v[l] (31 shuffles)
__device__ __forceinline__ double warp_reduce_scatter32(double (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double send = up ? v[i] : v[i + s];
      const double keep = up ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

// Vs (QNB x mp, column-major in smem, unit lower, zero columns >= nb) <- panel
template <int QNB>
__device__ void qr_stage_panel(const double* A, int lda, int j0, int nb, int mp, double* Vs) {
  BLK_FOR(e, QNB * mp) {
    const int i = e / mp, r = e - i * mp;
    Vs[e] = (i >= nb || r < i) ? 0.0 : (r == i ? 1.0 : A[(long)(j0 + i) * lda + j0 + r]);
  }
}

// a <- a - V M (V^T a) for the trailing columns c in [c0, n) (rows j0..n),
// M = T^T (geqrf) or T (orgqr); one warp per column.
template <int QNB>
__device__ void qr_trailing(double* A, int lda, int j0, int mp, int c0, int n, const double* Vs, const double* Ts,
                            bool transT, double* Wbuf) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* w2 = Wbuf + warp * QNB;
  for (int c = c0 + warp; c < n; c += nw) {
    double* Ac = A + (long)c * lda + j0;
    double acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.0;
    for (int r = lane; r < mp; r += 32) {
      const double a = Ac[r];
#pragma unroll
      for (int i = 0; i < QNB; ++i) acc[i] = fma(Vs[i * mp + r], a, acc[i]);
    }
    const double wl = warp_reduce_scatter32(acc);            // (V^T a)_lane (lanes >= QNB: 0)
    double m = 0.0;                                          // (M w)_lane
#pragma unroll
    for (int i = 0; i < QNB; ++i) {
      const double wi = __shfl_sync(0xffffffffu, wl, i);
      if (lane < QNB) m = fma(transT ? Ts[i * QNB + lane] : Ts[lane * QNB + i], wi, m);
    }
    if (lane < QNB) w2[lane] = m;
    __syncwarp();
    for (int r = lane; r < mp; r += 32) {
      double a = Ac[r];
#pragma unroll
      for (int i = 0; i < QNB; ++i) a = fma(-Vs[i * mp + r], w2[i], a);
      Ac[r] = a;
    }
    __syncwarp();
  }
}

// T (QNB x QNB upper, zero beyond nb) of the staged panel: G = V^T V, then
// T[j][j] = tau_j, T[0:j, j] = -tau_j T[0:j, 0:j] G[0:j, j]  (dlarft forward)
template <int QNB>
__device__ void qr_panel_t(const double* Vs, int mp, int nb, const double* tau, double* Gs, double* Ts) {
  constexpr unsigned PM = QNB >= 32 ? 0xffffffffu : ((1u << (QNB & 31)) - 1u);   // lanes < QNB
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = warp; j < QNB; j += nw) {
    double acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.0;
    for (int r = lane; r < mp; r += 32) {
      const double vj = Vs[j * mp + r];
#pragma unroll
      for (int i = 0; i < QNB; ++i) acc[i] = fma(Vs[i * mp + r], vj, acc[i]);
    }
    const double gl = warp_reduce_scatter32(acc);
    if (lane < QNB) Gs[lane * QNB + j] = gl;
  }
  __syncthreads();
  if (threadIdx.x < QNB) {
    const int i = threadIdx.x;
    for (int e = 0; e < QNB; ++e) Ts[i * QNB + e] = 0.0;
    __syncwarp(PM);
    for (int j = 0; j < nb; ++j) {
      double sacc = 0.0;
      if (i < j)
        for (int l = i; l < j; ++l) sacc = fma(Ts[i * QNB + l], Gs[l * QNB + j], sacc);
      __syncwarp(PM);
      if (i < j) Ts[i * QNB + j] = -tau[j] * sacc;
      if (i == j) Ts[j * QNB + j] = tau[j];
      __syncwarp(PM);
    }
  }
  __syncthreads();
}

// geqrf: A (n x n column-major) -> reflectors below the diagonal, R on and
// above, tau[n]; the panels' T kept in Tg (n/QNB+1 blocks of QNB x QNB).
// sm: >= QNB*n + 2*QNB*QNB + 16*QNB doubles of shared memory.
template <int QNB>
__device__ void blk_geqrf_cm(double* A, int lda, int n, double* tau, double* Tg, double* red, double* sm) {
  double* Vs = sm;
  double* Ts = sm + QNB * n;
  double* Gs = Ts + QNB * QNB;
  double* Wb = Gs + QNB * QNB;
  for (int j0 = 0; j0 < n; j0 += QNB) {
    const int nb = min(QNB, n - j0), mp = n - j0;
    blk_geqr2_cm(A + (long)j0 * lda + j0, lda, mp, nb, tau + j0, red);
    __syncthreads();
    qr_stage_panel<QNB>(A, lda, j0, nb, mp, Vs);
    __syncthreads();
    qr_panel_t<QNB>(Vs, mp, nb, tau + j0, Gs, Ts);
    BLK_FOR(e, QNB * QNB) Tg[(j0 / QNB) * QNB * QNB + e] = Ts[e];
    if (j0 + nb < n) qr_trailing<QNB>(A, lda, j0, mp, j0 + nb, n, Vs, Ts, true, Wb);
    __syncthreads();
  }
}

// orgqr: Q (n x n) in place from the reflectors of blk_geqrf_cm (R entries
// above the diagonal are overwritten), backward over the panels.
template <int QNB>
__device__ void blk_orgqr_cm(double* A, int lda, int n, const double* tau, const double* Tg, double* red,
                             double* sm) {
  double* Vs = sm;
  double* Ts = sm + QNB * n;
  double* Wb = Ts + 2 * QNB * QNB;
  const int last = ((n - 1) / QNB) * QNB;
  for (int j0 = last; j0 >= 0; j0 -= QNB) {
    const int nb = min(QNB, n - j0), mp = n - j0;
    qr_stage_panel<QNB>(A, lda, j0, nb, mp, Vs);
    BLK_FOR(e, QNB * QNB) Ts[e] = Tg[(j0 / QNB) * QNB * QNB + e];
    // trailing Q columns: rows j0 .. j0+nb-1 are zero before H_p is applied
    const int nt = n - j0 - nb;
    BLK_FOR(e, nb * nt) { const int c = j0 + nb + e / nb, r = j0 + e % nb; A[(long)c * lda + r] = 0.0; }
    __syncthreads();
    if (nt > 0) qr_trailing<QNB>(A, lda, j0, mp, j0 + nb, n, Vs, Ts, false, Wb);
    __syncthreads();
    // panel columns: rows above the panel are zero, then the unblocked dorg2r
    BLK_FOR(e, j0 * nb) { const int c = j0 + e / j0, r = e % j0; A[(long)c * lda + r] = 0.0; }
    __syncthreads();
    blk_org2r_cm(A + (long)j0 * lda + j0, lda, mp, nb, tau + j0, red);
    __syncthreads();
  }
}

// Modified LU (reflector.py:53-77 / paper Alg. 2) in place:
// Z -> L (strict lower, unit diag implied) and U (upper), p[n].
// signrec=true applies the LAPACK-sign-recovery variant: a pivot
// with |z_ii| == 1 exactly keeps p_i = +sign(z_ii) and skips its elimination.
__device__ void blk_mlu(double* Z, int ld, int n, double* p, bool signrec) {
  for (int i = 0; i < n; ++i) {
    __syncthreads();
    const double zi = Z[i * ld + i];
    bool skip = signrec && fabs(zi) == 1.0;
    double pi;
    if (skip) pi = (zi >= 0.0) ? 1.0 : -1.0;
    else pi = (zi >= 0.0) ? -1.0 : 1.0;
    const double uii = pi - zi;
    __syncthreads();
    if (threadIdx.x == 0) { p[i] = pi; Z[i * ld + i] = uii; }
    if (skip) {
      BLK_FOR(r, n - i - 1) Z[(i + 1 + r) * ld + i] = 0.0;
      __syncthreads();
      continue;
    }
    // U row i (c > i): u = -work ; L col i: l = -work / uii
    BLK_FOR(r, n - i - 1) {
      int rr = i + 1 + r;
      Z[i * ld + rr] = -Z[i * ld + rr];
      Z[rr * ld + i] = -Z[rr * ld + i] / uii;
    }
    __syncthreads();
    const int m = n - i - 1;
    BLK_FOR(e, m * m) {
      int a = e / m, b = e - a * m;
      int r = i + 1 + a, c = i + 1 + b;
      Z[r * ld + c] = fma(Z[r * ld + i], Z[i * ld + c], Z[r * ld + c]);
    }
  }
  __syncthreads();
}

// Cholesky (lower, in place; upper part zeroed).  Returns false on a
// non-positive pivot.
__device__ bool blk_cholesky(double* A, int ld, int n, double* red) {
  bool ok = true;
  for (int j = 0; j < n; ++j) {
    __syncthreads();
    double d = A[j * ld + j];
    if (!(d > 0.0)) { ok = false; break; }
    const double ljj = sqrt(d);
    __syncthreads();
    if (threadIdx.x == 0) A[j * ld + j] = ljj;
    BLK_FOR(r, n - j - 1) A[(j + 1 + r) * ld + j] /= ljj;
    __syncthreads();
    const int m = n - j - 1;
    BLK_FOR(e, m * m) {
      int a = e / m, b = e - a * m;
      if (b <= a) {
        int r = j + 1 + a, c = j + 1 + b;
        A[r * ld + c] = fma(-A[r * ld + j], A[c * ld + j], A[r * ld + c]);
      }
    }
  }
  __syncthreads();
  BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; if (j > i) A[i * ld + j] = 0.0; }
  __syncthreads();
  return ok;
}

// LU with partial pivoting (getrf), in place; piv[i] = row swapped with i.
// Returns false if an exactly zero pivot appears (SingularTError).
__device__ bool blk_getrf(double* A, int ld, int n, int* piv, double* red, int* ired) {
  bool ok = true;
  for (int j = 0; j < n; ++j) {
    // argmax |A[r][j]|, r >= j  (first max index, as idamax)
    double best = -1.0; int bi = j;
    for (int r = j + (int)threadIdx.x; r < n; r += blockDim.x) {
      double v = fabs(A[r * ld + j]);
      if (v > best) { best = v; bi = r; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      double ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (l == 0) { red[w] = best; ired[w] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = red[0]; int ii = ired[0];
      for (int q = 1; q < nw; ++q) if (red[q] > b || (red[q] == b && ired[q] < ii)) { b = red[q]; ii = ired[q]; }
      ired[32] = ii;
      piv[j] = ii;
    }
    __syncthreads();
    const int pr = ired[32];
    if (pr != j) BLK_FOR(c, n) { double t = A[j * ld + c]; A[j * ld + c] = A[pr * ld + c]; A[pr * ld + c] = t; }
    __syncthreads();
    const double d = A[j * ld + j];
    if (d == 0.0) { ok = false; continue; }
    BLK_FOR(r, n - j - 1) A[(j + 1 + r) * ld + j] /= d;
    __syncthreads();
    const int m = n - j - 1;
    BLK_FOR(e, m * m) {
      int a = e / m, b = e - a * m;
      int r = j + 1 + a, c = j + 1 + b;
      A[r * ld + c] = fma(-A[r * ld + j], A[j * ld + c], A[r * ld + c]);
    }
    __syncthreads();
  }
  __syncthreads();
  return ok;
}

// One-sided Jacobi (Hestenes) on the ROWS of W (n x n, row-major, ld):
// rotates row pairs until mutually orthogonal.  If Jt != null the same
// rotations are applied to the rows of Jt.  sigma[i] = ||row i|| at exit.
// Parallel round-robin ordering: n/2 disjoint pairs per step.
__device__ void blk_jacobi_rows_core(double* W, int ldw, double* Jt, int ldj, int n, double* sigma,
                                     double* red);

// Stage W (and Jt when it fits) into shared memory for the rotation sweeps.
__device__ void blk_jacobi_rows(double* W, int ldw, double* Jt, int ldj, int n, double* sigma,
                                double* red, double* sbuf = nullptr, int scap = 0) {
  const int ls = n + 1;  // odd stride: rows of a pair hit different banks
  if (sbuf && n * ls <= scap) {
    double* Ws = sbuf;
    double* Js = (Jt && 2 * n * ls <= scap) ? sbuf + n * ls : nullptr;
    __syncthreads();
    BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; Ws[i * ls + j] = W[i * ldw + j]; }
    if (Js) BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; Js[i * ls + j] = Jt[i * ldj + j]; }
    __syncthreads();
    blk_jacobi_rows_core(Ws, ls, Js ? Js : Jt, Js ? ls : ldj, n, sigma, red);
    BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; W[i * ldw + j] = Ws[i * ls + j]; }
    if (Js) BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; Jt[i * ldj + j] = Js[i * ls + j]; }
    __syncthreads();
    return;
  }
  blk_jacobi_rows_core(W, ldw, Jt, ldj, n, sigma, red);
}

__device__ void blk_jacobi_rows_core(double* W, int ldw, double* Jt, int ldj, int n, double* sigma,
                                     double* red) {
  const int ne = (n + 1) & ~1;  // even count incl. a dummy
  const int npairs = ne / 2;
  int gs = 1;
  while (gs * 2 * npairs <= (int)blockDim.x && gs < 32) gs *= 2;
  const int grp = threadIdx.x / gs, gl = threadIdx.x % gs;
  const unsigned gmask = (gs == 32) ? 0xffffffffu : (((1u << gs) - 1u) << ((threadIdx.x & 31) & ~(gs - 1)));
  const double tol = 4.0 * 2.220446049250313e-16 * (n > 4 ? n : 4);
  __shared__ int rotated;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    int my_rot = 0;
    for (int rd = 0; rd < ne - 1; ++rd) {
      if (grp < npairs) {
        int p, q;
        if (grp == 0) { p = ne - 1; q = rd; }
        else { p = (rd + grp) % (ne - 1); q = (rd - grp + (ne - 1)) % (ne - 1); }
        if (p < n && q < n) {
          double a = 0, b = 0, c = 0;
          for (int e = gl; e < n; e += gs) {
            double x = W[p * ldw + e], y = W[q * ldw + e];
            a = fma(x, x, a); b = fma(y, y, b); c = fma(x, y, c);
          }
          for (int o = gs / 2; o > 0; o >>= 1) {
            a += __shfl_xor_sync(gmask, a, o);
            b += __shfl_xor_sync(gmask, b, o);
            c += __shfl_xor_sync(gmask, c, o);
          }
          if (c != 0.0 && fabs(c) > tol * sqrt(a) * sqrt(b)) {
            double zeta = (b - a) / (2.0 * c);
            double tt;
            if (fabs(zeta) > 1e150) tt = 0.5 / zeta;
            else tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
            double cs = 1.0 / sqrt(fma(tt, tt, 1.0));
            double sn = cs * tt;
            for (int e = gl; e < n; e += gs) {
              double x = W[p * ldw + e], y = W[q * ldw + e];
              W[p * ldw + e] = cs * x - sn * y;
              W[q * ldw + e] = sn * x + cs * y;
            }
#ifndef OTS_JACOBI_NOJT
            if (Jt)
#else
            if (false)
#endif
              for (int e = gl; e < n; e += gs) {
                double x = Jt[p * ldj + e], y = Jt[q * ldj + e];
                Jt[p * ldj + e] = cs * x - sn * y;
                Jt[q * ldj + e] = sn * x + cs * y;
              }
            my_rot = 1;
          }
        }
      }
      __syncthreads();
    }
    if (my_rot) rotated = 1;
    __syncthreads();
    int any = rotated;
    __syncthreads();
#ifdef OTS_TIMING
    if (threadIdx.x == 0) atomicAdd(&g_dbg_small[15], 1ull);   // Jacobi sweeps
#endif
    if (!any) break;
  }
  // row norms
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int e = threadIdx.x; e < n; e += blockDim.x) { double x = W[i * ldw + e]; s = fma(x, x, s); }
    s = block_sum(s, red);
    if (threadIdx.x == 0) sigma[i] = sqrt(s);
  }
  __syncthreads();
}

__device__ double blk_sigma_max(double* W, int ld, int n, double* sig, double* red,
                                double* sbuf = nullptr, int scap = 0) {
  blk_jacobi_rows(W, ld, nullptr, 0, n, sig, red, sbuf, scap);
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, sig[i]);
  return block_max(m, red);
}

// Largest eigenvalue of a symmetric n x n matrix S (overwritten): Householder
// tridiagonalisation (dsytd2, lower) followed by parallel multisection on the
// Sturm count of the tridiagonal (dstebz-style, one shift per thread).
// vec: >= 4 n doubles of scratch (shared memory preferred).
__device__ void blk_tridiag(double* S, int lds, int n, double* vec, double* red) {
  double* v = vec;           // Householder vector
  double* pw = vec + n;      // p, then w
  double* d = vec + 2 * n;   // diagonal
  double* e = vec + 3 * n;   // off-diagonal
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  for (int j = 0; j + 2 < n; ++j) {
    const int m = n - j - 1;
    const double* x = S + (j + 1) * lds + j;  // column j below the diagonal, stride lds
    double s2 = 0.0;
    for (int r = 1 + (int)threadIdx.x; r < m; r += blockDim.x) { double t = x[r * lds]; s2 = fma(t, t, s2); }
    s2 = block_sum(s2, red);
    const double alpha = x[0];
    if (threadIdx.x == 0) d[j] = S[j * lds + j];
    if (s2 == 0.0) {
      if (threadIdx.x == 0) e[j] = alpha;
      __syncthreads();
      continue;
    }
    const double beta = -copysign(sqrt(fma(alpha, alpha, s2)), alpha);
    const double tau = (beta - alpha) / beta;
    const double scal = 1.0 / (alpha - beta);
    for (int r = threadIdx.x; r < m; r += blockDim.x) v[r] = (r == 0) ? 1.0 : x[r * lds] * scal;
    if (threadIdx.x == 0) e[j] = beta;
    __syncthreads();
    // p = tau S22 v  (one warp per row)
    double* S22 = S + (j + 1) * lds + (j + 1);
    double pv = 0.0;
    for (int r = w; r < m; r += nw) {
      double acc = 0.0;
      for (int c = l; c < m; c += 32) acc = fma(S22[r * lds + c], v[c], acc);
      acc = warp_sum(acc) * tau;
      if (l == 0) pw[r] = acc;
      pv = fma(acc, v[r], pv);
    }
    if (l != 0) pv = 0.0;
    pv = block_sum(pv, red);
    const double K = -0.5 * tau * pv;
    for (int r = threadIdx.x; r < m; r += blockDim.x) pw[r] = fma(K, v[r], pw[r]);
    __syncthreads();
    // S22 -= v w^T + w v^T
    for (int r = w; r < m; r += nw) {
      const double vr = v[r], wr = pw[r];
      for (int c = l; c < m; c += 32) S22[r * lds + c] -= vr * pw[c] + wr * v[c];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (n >= 2) { d[n - 2] = S[(n - 2) * lds + n - 2]; e[n - 2] = S[(n - 1) * lds + n - 2]; }
    d[n - 1] = S[(n - 1) * lds + n - 1];
  }
  __syncthreads();
}

// kth smallest eigenvalue (0-based) of the symmetric tridiagonal (d, e) left
// by blk_tridiag, in [lo, hi]: 512-way multisection on the Sturm count
// (count(x) = #eigenvalues < x), dstebz-style pivmin guard.  Uses vec+n for e^2.
__device__ double blk_sturm_kth(double* vec, int n, int kth, double lo, double hi, double pivmin) {
  double* e2 = vec + n;
  const double* d = vec + 2 * n;
  const double* e = vec + 3 * n;
  __syncthreads();
  for (int i = threadIdx.x; i + 1 < n; i += blockDim.x) e2[i] = e[i] * e[i];
  __syncthreads();
  const int NT = blockDim.x;
  __shared__ int first_hit;
  for (int it = 0; it < 64; ++it) {
    if (!(hi - lo > 2.2e-16 * fmax(fabs(lo), fabs(hi)) + pivmin)) break;
    const double xt = lo + (hi - lo) * (double)(threadIdx.x + 1) / (double)(NT + 1);
    int cnt = 0;
    double q = d[0] - xt;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += (q < 0.0);
    for (int i = 1; i < n; ++i) {
      q = (d[i] - xt) - e2[i - 1] / q;
      if (fabs(q) < pivmin) q = -pivmin;
      cnt += (q < 0.0);
    }
    if (threadIdx.x == 0) first_hit = NT;
    __syncthreads();
    if (cnt >= kth + 1) atomicMin(&first_hit, (int)threadIdx.x);
    __syncthreads();
    const int t = first_hit;
    const double nlo = (t == 0) ? lo : lo + (hi - lo) * (double)t / (double)(NT + 1);
    const double nhi = (t == NT) ? hi : lo + (hi - lo) * (double)(t + 1) / (double)(NT + 1);
    lo = nlo; hi = nhi;
    __syncthreads();
  }
  return 0.5 * (lo + hi);
}

// Gershgorin bounds of the tridiagonal and the pivmin guard
__device__ void blk_tridiag_bounds(const double* vec, int n, double* red, double& glo, double& ghi,
                                   double& dmax, double& pivmin) {
  const double* d = vec + 2 * n;
  const double* e = vec + 3 * n;
  double lo = 1.7976931348623157e308, hi = -lo, dm = -lo, e2max = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double el = (i > 0) ? fabs(e[i - 1]) : 0.0, er = (i + 1 < n) ? fabs(e[i]) : 0.0;
    lo = fmin(lo, d[i] - el - er);
    hi = fmax(hi, d[i] + el + er);
    dm = fmax(dm, d[i]);
    e2max = fmax(e2max, er * er);
  }
  glo = -block_max(-lo, red);
  ghi = block_max(hi, red);
  dmax = block_max(dm, red);
  e2max = block_max(e2max, red);
  pivmin = 2.2250738585072014e-308 * fmax(1.0, e2max);
}

// Largest eigenvalue of a symmetric n x n matrix S (overwritten): Householder
// tridiagonalisation (dsytd2, lower) followed by parallel multisection on the
// Sturm count of the tridiagonal (dstebz-style, one shift per thread).
// vec: >= 4 n doubles of scratch (shared memory preferred).
__device__ double blk_sym_lmax(double* S, int lds, int n, double* vec, double* red) {
  blk_tridiag(S, lds, n, vec, red);
  double glo, ghi, dmax, pivmin;
  blk_tridiag_bounds(vec, n, red, glo, ghi, dmax, pivmin);
  return blk_sturm_kth(vec, n, n - 1, dmax, ghi, pivmin);   // lambda_max >= max diagonal
}

// (lambda_min, lambda_max) of a symmetric S (overwritten)
__device__ void blk_sym_extremes(double* S, int lds, int n, double* vec, double* red, double& lmin,
                                 double& lmax) {
  blk_tridiag(S, lds, n, vec, red);
  double glo, ghi, dmax, pivmin;
  blk_tridiag_bounds(vec, n, red, glo, ghi, dmax, pivmin);
  lmax = blk_sturm_kth(vec, n, n - 1, dmax, ghi, pivmin);
  lmin = blk_sturm_kth(vec, n, 0, glo, ghi, pivmin);
}

// ---------------------------------------------------------------------------
// T-solver dispatch (reflector.py:80-153).  X (n x m) overwritten.
//   adjoint=false: T X = B ; adjoint=true: T^T X = B.
// ---------------------------------------------------------------------------
__device__ void t_solve_core(const SmallState& s, const double* F, int ld, double* X, int ldx, int m,
                             bool adjoint);

extern __shared__ __align__(16) double dsm[];
constexpr int SMALL_SMEM_DOUBLES = 25 * 1024;   // 200 KB dynamic smem of the small kernels

__device__ void t_solve(const SmallState& s, double* X, int ldx, int m, bool adjoint) {
  // the right-hand sides live in registers inside blk_trsm; stage the factor
  const int n = s.k0;
  if (n * (n + 1) <= SMALL_SMEM_DOUBLES) {
    __syncthreads();
    BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; dsm[i * (n + 1) + j] = s.Tf[i * s.ld + j]; }
    __syncthreads();
    t_solve_core(s, dsm, n + 1, X, ldx, m, adjoint);
    __syncthreads();
    return;
  }
  t_solve_core(s, s.Tf, s.ld, X, ldx, m, adjoint);
}

__device__ void t_solve_core(const SmallState& s, const double* F, int ld, double* X, int ldx, int m,
                             bool adjoint) {
  const int n = s.k0;
  switch (s.choice) {
    case CHOICE_QR:  // lower triangular T
      blk_trsm(F, ld, true, adjoint, false, X, ldx, n, m);
      break;

    case CHOICE_MLU:
      if (adjoint) {  // diag(p) L U x = b
        BLK_FOR(e, n * m) { int i = e / m; X[i * ldx + (e - i * m)] *= s.pvec[i]; }
        blk_trsm(F, ld, true, false, true, X, ldx, n, m);
        blk_trsm(F, ld, false, false, false, X, ldx, n, m);
      } else {        // U^T L^T diag(p) x = b
        blk_trsm(F, ld, false, true, false, X, ldx, n, m);
        blk_trsm(F, ld, true, true, true, X, ldx, n, m);
        __syncthreads();
        BLK_FOR(e, n * m) { int i = e / m; X[i * ldx + (e - i * m)] *= s.pvec[i]; }
      }
      break;
    case CHOICE_POLAR:     // pivoted LU of T = I - V_t^T P (see seed_polar)
    case CHOICE_EXPLICIT:  // P_piv L U = T (getrf); getrs semantics
      if (!adjoint) {
        for (int i = 0; i < n; ++i) {  // apply row swaps forward
          int pr = s.piv[i];
          __syncthreads();
          if (pr != i) BLK_FOR(j, m) { double t = X[i * ldx + j]; X[i * ldx + j] = X[pr * ldx + j]; X[pr * ldx + j] = t; }
        }
        blk_trsm(F, ld, true, false, true, X, ldx, n, m);
        blk_trsm(F, ld, false, false, false, X, ldx, n, m);
      } else {
        blk_trsm(F, ld, false, true, false, X, ldx, n, m);
        blk_trsm(F, ld, true, true, true, X, ldx, n, m);
        for (int i = n - 1; i >= 0; --i) {  // swaps backward
          int pr = s.piv[i];
          __syncthreads();
          if (pr != i) BLK_FOR(j, m) { double t = X[i * ldx + j]; X[i * ldx + j] = X[pr * ldx + j]; X[pr * ldx + j] = t; }
        }
      }
      break;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Polar seed on a 2-CTA cluster (k0 <= JC_NMAX): the one-sided Jacobi sweeps
// rotate the rows of W = V_t^T in CTA 0's shared memory and send each round's
// rotations (cs, sn per pair) through distributed shared memory to CTA 1,
// which applies them to the accumulated J^T held in ITS shared memory -- so
// neither matrix lives in global memory (the single-CTA version kept J^T in
// global memory: 10.5 ms of long-scoreboard stalls at k0 = 128, and W and J^T
// together exceed one CTA's 227 KB).  A ring of JC_NR rounds with
// full (CTA 1) / empty (CTA 0) mbarriers lets CTA 0 run ahead.
// ---------------------------------------------------------------------------
constexpr int JC_NR = 4, JC_NMAX = 152, JC_PAIRS = (JC_NMAX + 2) / 2;   // 152 x jc_ls(152) <= SMALL_SMEM_DOUBLES
struct JacobiLink {
  double rot[JC_NR][2 * JC_PAIRS];
  int cmd[JC_NR];                 // 0: apply round rd[slot]; 1: stop
  int rd[JC_NR];
  unsigned long long full[JC_NR];  // on CTA 1 (one remote arrival per round)
  unsigned long long empty[JC_NR]; // on CTA 0 (one remote arrival per round)
  int done;                        // CTA 0: stop already sent
};
__shared__ JacobiLink g_jlink;

__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cl_map(const void* p, unsigned rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void cl_st_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void cl_st_s32(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void cl_arrive_remote(uint32_t bar) {
  asm volatile("fence.acq_rel.cluster;\n\tmbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void cl_wait(unsigned long long* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n.reg .pred p;\nJW_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra JW_%=;\n}\n" ::"r"(a), "r"(parity)
      : "memory");
}

// both CTAs of a 2-CTA seed cluster, at kernel start
__device__ void jacobi_link_init() {
  if (threadIdx.x == 0) {
    for (int i = 0; i < JC_NR; ++i) {
      mbar_init(&g_jlink.full[i], 1);
      mbar_init(&g_jlink.empty[i], 1);
    }
    g_jlink.done = 0;
    fence_mbar_init();
  }
  __syncthreads();
  cl_sync();
}

// CTA 0: send the stop command (once) and meet CTA 1 at the closing cluster
// barrier (after which CTA 1 has written J^T to global memory)
__device__ void jacobi_link_close(long long rounds) {
  __syncthreads();
  if (g_jlink.done) return;           // closed already (uniform across the CTA)
  const int slot = (int)(rounds % JC_NR);
  if (rounds >= JC_NR) cl_wait(&g_jlink.empty[slot], (unsigned)(((rounds / JC_NR) - 1) & 1));
  if (threadIdx.x == 0) {
    cl_st_s32(cl_map(&g_jlink.cmd[slot], 1), 1);
    cl_arrive_remote(cl_map(&g_jlink.full[slot], 1));
  }
  __syncthreads();
  cl_sync();
  if (threadIdx.x == 0) g_jlink.done = 1;
  __syncthreads();
}

__device__ __forceinline__ double rcp_nr(double x) {     // 1/x: MUFU seed + 2 Newton steps
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-x, r, 2.0);
  return r * fma(-x, r, 2.0);
}
__device__ __forceinline__ double rsqrt_nr(double x) {   // 1/sqrt(x): MUFU seed + 2 Newton steps
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-0.5 * x * r, r, 1.5);
  return r * fma(-0.5 * x * r, r, 1.5);
}
// row stride of the staged W / J^T: = 8 (mod 16) doubles, so the 4 pairs of
// a warp (consecutive rows) read disjoint bank halves (2 wavefronts)
__device__ __forceinline__ int jc_ls(int n) { return ((n + 15) / 16) * 16 + 8; }

// CTA 0 side of the Jacobi (W already in shared memory); returns the number
// of rounds sent.  Same rotations and order as blk_jacobi_rows_core.
__device__ long long blk_jacobi_rows_cluster(double* W, int ldw, int n, double* sigma, double* red) {
  const int ne = (n + 1) & ~1;
  const int npairs = ne / 2;
  int gs = 1;
  while (gs * 2 * npairs <= (int)blockDim.x && gs < 32) gs *= 2;
  const int grp = threadIdx.x / gs, gl = threadIdx.x % gs;
  const unsigned gmask = (gs == 32) ? 0xffffffffu : (((1u << gs) - 1u) << ((threadIdx.x & 31) & ~(gs - 1)));
  const double tol = 4.0 * 2.220446049250313e-16 * (n > 4 ? n : 4);
  __shared__ int rotated;
  long long r = 0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    int my_rot = 0;
    for (int rd = 0; rd < ne - 1; ++rd, ++r) {
      const int slot = (int)(r % JC_NR);
      if (r >= JC_NR) cl_wait(&g_jlink.empty[slot], (unsigned)(((r / JC_NR) - 1) & 1));
      if (grp < npairs) {
        int p, q;
        if (grp == 0) { p = ne - 1; q = rd; }
        else { p = (rd + grp) % (ne - 1); q = (rd - grp + (ne - 1)) % (ne - 1); }
        double cs = 1.0, sn = 0.0;
        if (p < n && q < n) {
          double a = 0, b = 0, c = 0;
          for (int e = gl; e < n; e += gs) {
            double x = W[p * ldw + e], y = W[q * ldw + e];
            a = fma(x, x, a); b = fma(y, y, b); c = fma(x, y, c);
          }
          for (int o = gs / 2; o > 0; o >>= 1) {
            a += __shfl_xor_sync(gmask, a, o);
            b += __shfl_xor_sync(gmask, b, o);
            c += __shfl_xor_sync(gmask, c, o);
          }
          // same test and rotation as blk_jacobi_rows_core, with the divisions
          // and square roots as MUFU seeds + Newton steps (~1 ulp; the
          // rotation stays orthogonal to rounding: sn = cs tt)
          if (c != 0.0 && c * c > (tol * tol) * a * b) {
            const double zeta = (b - a) * rcp_nr(2.0 * c);
            double tt;
            if (fabs(zeta) > 1e150) tt = 0.5 * rcp_nr(zeta);
            else {
              const double h = fma(zeta, zeta, 1.0);
              const double rs = rsqrt_nr(h);
              tt = copysign(rcp_nr(fabs(zeta) + h * rs), zeta);
            }
            cs = rsqrt_nr(fma(tt, tt, 1.0));
            sn = cs * tt;
            for (int e = gl; e < n; e += gs) {
              double x = W[p * ldw + e], y = W[q * ldw + e];
              W[p * ldw + e] = cs * x - sn * y;
              W[q * ldw + e] = sn * x + cs * y;
            }
            my_rot = 1;
          }
        }
        if (gl == 0) {
          const uint32_t rot = cl_map(&g_jlink.rot[slot][2 * grp], 1);
          cl_st_f64(rot, cs);
          cl_st_f64(rot + 8, sn);
        }
      }
      if (threadIdx.x == 0) {
        cl_st_s32(cl_map(&g_jlink.cmd[slot], 1), 0);
        cl_st_s32(cl_map(&g_jlink.rd[slot], 1), rd);
      }
      __syncthreads();
      if (threadIdx.x == 0) cl_arrive_remote(cl_map(&g_jlink.full[slot], 1));
    }
    if (my_rot) rotated = 1;
    __syncthreads();
    int any = rotated;
    __syncthreads();
#ifdef OTS_TIMING
    if (threadIdx.x == 0) atomicAdd(&g_dbg_small[15], 1ull);
#endif
    if (!any) break;
  }
  for (int i = 0; i < n; ++i) {
    double sacc = 0.0;
    for (int e = threadIdx.x; e < n; e += blockDim.x) { double x = W[i * ldw + e]; sacc = fma(x, x, sacc); }
    sacc = block_sum(sacc, red);
    if (threadIdx.x == 0) sigma[i] = sqrt(sacc);
  }
  __syncthreads();
  return r;
}

// CTA 1: J^T (starting at I) in shared memory, rotated as CTA 0 dictates,
// then written to Jt (global, ldj); ends at the closing cluster barrier.
__device__ void jacobi_jt_helper(double* Jt, int ldj, int n) {
  const int ls = jc_ls(n);
  double* Js = dsm;
  BLK_FOR(e, n * n) { const int i = e / n, j = e - i * n; Js[i * ls + j] = (i == j) ? 1.0 : 0.0; }
  const int ne = (n + 1) & ~1;
  const int npairs = ne / 2;
  int gs = 1;
  while (gs * 2 * npairs <= (int)blockDim.x && gs < 32) gs *= 2;
  const int grp = threadIdx.x / gs, gl = threadIdx.x % gs;
  __syncthreads();
  for (long long r = 0;; ++r) {
    const int slot = (int)(r % JC_NR);
    cl_wait(&g_jlink.full[slot], (unsigned)((r / JC_NR) & 1));
    if (g_jlink.cmd[slot] == 1) break;
    const int rd = g_jlink.rd[slot];
    if (grp < npairs) {
      int p, q;
      if (grp == 0) { p = ne - 1; q = rd; }
      else { p = (rd + grp) % (ne - 1); q = (rd - grp + (ne - 1)) % (ne - 1); }
      const double cs = g_jlink.rot[slot][2 * grp], sn = g_jlink.rot[slot][2 * grp + 1];
      if (p < n && q < n && !(cs == 1.0 && sn == 0.0))
        for (int e = gl; e < n; e += gs) {
          const double x = Js[p * ls + e], y = Js[q * ls + e];
          Js[p * ls + e] = cs * x - sn * y;
          Js[q * ls + e] = sn * x + cs * y;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) cl_arrive_remote(cl_map(&g_jlink.empty[slot], 0));
  }
  __syncthreads();
  BLK_FOR(e, n * n) { const int i = e / n, j = e - i * n; Jt[(long)i * ldj + j] = Js[i * ls + j]; }
  __syncthreads();
  cl_sync();
}

// ---------------------------------------------------------------------------
// Kernels
// ---------------------------------------------------------------------------

// Seed: Gram check, P/T construction, W_top, Z1 = T^{-T}(W^T A), S = P^T (H^T A)_top
// polar V_t = U H via one-sided Jacobi SVD (core.py:108-120):
// P = -U, Tdense = T = I + H, Tf = chol(T).  Returns a status code.
__device__ int seed_polar(const SmallState& s, double* red, int* ired) {
  const int n = s.k0, ld = s.ld;
  int st = 0;
  long long tm0 = clock64();
  // rows of X1 := columns of V_t ; X2 := I (accumulates J^T)
  if (cl_size() == 2) {   // W in this CTA's shared memory, J^T in CTA 1's (see above)
    const int ls = jc_ls(n);
    double* Ws = dsm;
    BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; Ws[i * ls + j] = s.Vt[j * ld + i]; }
    __syncthreads();
    const long long rounds = blk_jacobi_rows_cluster(Ws, ls, n, s.sig, red);
    BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; s.X1[i * ld + j] = Ws[i * ls + j]; }
    jacobi_link_close(rounds);          // J^T now in s.X2
  } else {
    BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; s.X1[i * ld + j] = s.Vt[j * ld + i]; }
    blk_identity(s.X2, ld, n);
    __syncthreads();
    blk_jacobi_rows(s.X1, ld, s.X2, ld, n, s.sig, red, dsm, SMALL_SMEM_DOUBLES);
  }
  SMARK(10, tm0);
  // U columns u_j = X1 row j / sigma_j (null directions: v_j orthogonalised)
  // store U^T rows in X1 (normalised)
  BLK_FOR(e, n * n) {
    int j = e / n, c = e - j * n;
    double sg = s.sig[j];
    if (sg > 0.0) s.X1[j * ld + c] /= sg;
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (s.sig[j] > 0.0) continue;
    // u = v_j - sum_{i != j, done} (u_i . v_j) u_i, normalise
    BLK_FOR(c, n) s.X1[j * ld + c] = s.X2[j * ld + c];
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i < n; ++i) {
        if (i == j || (s.sig[i] == 0.0 && i > j)) continue;
        double d = 0.0;
        for (int c = threadIdx.x; c < n; c += blockDim.x) d = fma(s.X1[i * ld + c], s.X1[j * ld + c], d);
        d = block_sum(d, red);
        BLK_FOR(c, n) s.X1[j * ld + c] -= d * s.X1[i * ld + c];
        __syncthreads();
      }
    double nn = 0.0;
    for (int c = threadIdx.x; c < n; c += blockDim.x) nn = fma(s.X1[j * ld + c], s.X1[j * ld + c], nn);
    nn = sqrt(block_sum(nn, red));
    BLK_FOR(c, n) s.X1[j * ld + c] /= nn;
    __syncthreads();
  }
  SMARK(11, tm0);
  // Up = U V^T = sum_j u_j v_j^T ; H = V diag(sigma) V^T
  BLK_FOR(e, n * n) {
    int a = e / n, b = e - a * n;
    double up = 0.0, h = 0.0;
    for (int j = 0; j < n; ++j) {
      up = fma(s.X1[j * ld + a], s.X2[j * ld + b], up);
      h = fma(s.X2[j * ld + a] * s.sig[j], s.X2[j * ld + b], h);
    }
    s.P[a * ld + b] = -up;
    s.Tdense[a * ld + b] = h;
  }
  __syncthreads();
  __syncthreads();
  // One-sided Jacobi leaves U orthogonal only to its tolerance (~4 n u), and
  // the reflector is orthogonal only as far as P is and T = I - V_t^T P holds
  // (SURVEY §3.1); so refine P by one Newton-Schulz step P <- P (3I - P^T P)/2
  // (orthogonal to rounding) and form T from that P itself.  T is then
  // symmetric only up to the Jacobi error, so it is factored by pivoted LU
  // (the 'explicit' solver) rather than Cholesky; it is I + H with H PSD in
  // exact arithmetic, so positive definite.
  blk_gemm(s.X1, ld, s.P, ld, true, s.P, ld, false, n, n, n, 1.0, 0.0);
  BLK_FOR(e, n * n) { int a = e / n, b = e - a * n; s.X1[a * ld + b] = (a == b ? 1.5 : 0.0) - 0.5 * s.X1[a * ld + b]; }
  blk_gemm(s.X2, ld, s.P, ld, false, s.X1, ld, false, n, n, n, 1.0, 0.0);
  blk_copy(s.P, ld, s.X2, ld, n, n);
  blk_gemm(s.Tdense, ld, s.Vt, ld, true, s.P, ld, false, n, n, n, -1.0, 0.0);
  BLK_FOR(i, n) s.Tdense[i * ld + i] += 1.0;
  __syncthreads();
  blk_copy(s.Tf, ld, s.Tdense, ld, n, n);
  __syncthreads();
  SMARK(12, tm0);
  if (!blk_getrf(s.Tf, ld, n, s.piv, red, ired)) st = OTS_E_SINGULAR_T;
  SMARK(13, tm0);
  return st;
}

// The seed pipeline in three pieces (reflector.py:207-228 + twostage.py:90-92):
//   seed_checks  Gram-dependent validation: orthonormality defect, non-finite
//   seed_build   V_t-only: P, T (and its factors) for the chosen seed, W_t
//   seed_finish  Z1 = T^{-T}(W_t^T A_t - V_b^T A_b), S = P^T (A_t - W_t Z1)
// seed_kernel runs them in the reference's validation order; the headline
// pipeline runs seed_build on one SM while the Gram kernel streams on the
// others (seedA_kernel) and the rest after the Gram (seedB_kernel).
__device__ bool seed_checks(SmallState& s, double* red) {
  const int n = s.k0, k = s.k, ld = s.ld;
  // 1. symmetric Gram (lower blocks valid) and V_b^T A_b
  BLK_FOR(e, n * n) {
    int i = e / n, j = e - i * n;
    double g = (j <= i) ? s.Gfull[(long)i * s.ldgf + j] : s.Gfull[(long)j * s.ldgf + i];
    s.G[i * ld + j] = g;
    s.X1[i * ld + j] = g - (i == j ? 1.0 : 0.0);
  }
  BLK_FOR(e, n * k) { int i = e / k, j = e - i * k; s.VbA[i * ld + j] = s.Gfull[(long)i * s.ldgf + s.gf_acol + j]; }
  __syncthreads();
  // 2. orthonormality defect (Frobenius shortcut; exact 2-norm only if needed)
  double f = 0.0;
  BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; double x = s.X1[i * ld + j]; f = fma(x, x, f); }
  f = sqrt(block_sum(f, red));
  double defect = f;
  if (f > s.orth_tol) defect = blk_sigma_max(s.X1, ld, n, s.sig, red, dsm, SMALL_SMEM_DOUBLES);
  if (threadIdx.x == 0) s.diag[2] = defect;
  if (defect > s.orth_tol && !s.allow_defect) {
    if (threadIdx.x == 0) s.status[0] = OTS_E_ORTHONORMALITY;
    return false;
  }
  // Non-finite V or A (core.py:72-73, reached by the reference at the intra
  // QR): any NaN/Inf entry poisons the Gram block [V^T V | V_b^T A_b] or the
  // top rows A_t, so checking those k0 x (k0+k) values covers the n-row data.
  {
    int bad = 0;
    BLK_FOR(e, n * n) { if (!isfinite(s.G[(e / n) * ld + (e % n)])) bad = 1; }
    BLK_FOR(e, n * k) {
      const int i = e / k, j = e - i * k;
      if (!isfinite(s.VbA[i * ld + j]) || !isfinite(s.A[(long)i * s.lda + j])) bad = 1;
    }
    if (__syncthreads_or(bad)) {
      if (threadIdx.x == 0) s.status[0] = OTS_E_VALUE;
      return false;
    }
  }
  return true;
}

__device__ int seed_build(SmallState& s, double* red, int* ired) {
  const int n = s.k0, k = s.k, ld = s.ld;
  // 3. V_t, A_t
  BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; s.Vt[i * ld + j] = s.V[(long)i * s.ldv + j]; }
  BLK_FOR(e, n * k) { int i = e / k, j = e - i * k; s.At[i * ld + j] = s.A[(long)i * s.lda + j]; }
  __syncthreads();
  // 4. seed
  int st = 0;
  switch (s.choice) {
    case CHOICE_QR: {
      // nonneg-diagonal QR of V_t (core.py:61-84): P = -Q1, T = I + R1^T
      if (n * (n + 1) <= SMALL_SMEM_DOUBLES) {   // in shared memory
        double* Wq = dsm;
        const int lq = n + 1;
        blk_copy(Wq, lq, s.Vt, ld, n, n);
        __syncthreads();
        blk_geqr2(Wq, lq, n, n, s.tau, red);
        BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; s.X2[i * ld + j] = (j >= i) ? Wq[i * lq + j] : 0.0; }
        __syncthreads();
        blk_org2r(Wq, lq, n, n, s.tau, red);  // Q1
        blk_copy(s.X1, ld, Wq, lq, n, n);
        __syncthreads();
      } else {                                    // global memory: column-major (coalesced)
        BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; s.X1[j * ld + i] = s.Vt[i * ld + j]; }
        __syncthreads();
        // panel width 32 while the staged panel fits the shared memory, else 16
        const bool wide = 32 * n + 2 * 32 * 32 + 16 * 32 <= SMALL_SMEM_DOUBLES;
        if (wide) blk_geqrf_cm<32>(s.X1, ld, n, s.tau, s.Z2, red, dsm);   // panel T's in Z2 (free here)
        else blk_geqrf_cm<16>(s.X1, ld, n, s.tau, s.Z2, red, dsm);
        BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; s.X2[i * ld + j] = (j >= i) ? s.X1[j * ld + i] : 0.0; }
        __syncthreads();
        if (wide) blk_orgqr_cm<32>(s.X1, ld, n, s.tau, s.Z2, red, dsm);   // Q1, column-major
        else blk_orgqr_cm<16>(s.X1, ld, n, s.tau, s.Z2, red, dsm);
        BLK_FOR(e, n * n) {                        // -> row-major in place
          int i = e / n, j = e - i * n;
          if (i < j) { const double a = s.X1[i * ld + j]; s.X1[i * ld + j] = s.X1[j * ld + i]; s.X1[j * ld + i] = a; }
        }
        __syncthreads();
      }
      BLK_FOR(i, n) { double d = s.X2[i * ld + i]; s.pvec[i] = (d < 0.0) ? -1.0 : 1.0; }
      __syncthreads();
      BLK_FOR(e, n * n) {
        int i = e / n, j = e - i * n;
        s.P[i * ld + j] = -s.X1[i * ld + j] * s.pvec[j];
        double rji = (i >= j) ? s.X2[j * ld + i] * s.pvec[j] : 0.0;  // R1^T[i][j] = R1[j][i]
        if (i == j) rji = fabs(s.X2[i * ld + i]);
        double t = (i == j ? 1.0 : 0.0) + rji;
        s.Tf[i * ld + j] = t;
        s.Tdense[i * ld + j] = t;
      }
      break;
    }
    case CHOICE_MLU: {
      blk_copy(s.Tf, ld, s.Vt, ld, n, n);
      __syncthreads();
      blk_mlu(s.Tf, ld, n, s.pvec, false);
      BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; s.P[i * ld + j] = (i == j) ? s.pvec[i] : 0.0; }
      // dense T = (L U)^T diag(p):  T[i][j] = p_j * sum_l L[j][l] U[l][i]
      BLK_FOR(e, n * n) {
        int i = e / n, j = e - i * n;
        double acc = 0.0;
        int lmax = i < j ? i : j;
        for (int l = 0; l <= lmax; ++l) {
          double L = (l == j) ? 1.0 : s.Tf[j * ld + l];
          acc = fma(L, s.Tf[l * ld + i], acc);
        }
        s.Tdense[i * ld + j] = acc * s.pvec[j];
      }
      break;
    }
    case CHOICE_POLAR:
      st = seed_polar(s, red, ired);
      break;
    case CHOICE_EXPLICIT: {
      blk_copy(s.P, ld, s.Pexp, s.ldpe, n, n);
      __syncthreads();
      // unitary check ||P^T P - I||_2 <= 1e-12 k0  (reflector.py:200-201)
      blk_gemm(s.X1, ld, s.P, ld, true, s.P, ld, false, n, n, n, 1.0, 0.0);
      BLK_FOR(i, n) s.X1[i * ld + i] -= 1.0;
      __syncthreads();
      double ff = 0.0;
      BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; double x = s.X1[i * ld + j]; ff = fma(x, x, ff); }
      ff = sqrt(block_sum(ff, red));
      double pd = ff;
      const double ptol = 1e-12 * (n > 1 ? n : 1);
      if (ff > ptol) pd = blk_sigma_max(s.X1, ld, n, s.sig, red, dsm, SMALL_SMEM_DOUBLES);
      if (pd > ptol) { st = OTS_E_PARAMETER; break; }
      // T = I - V_t^T P, pivoted LU
      blk_gemm(s.Tdense, ld, s.Vt, ld, true, s.P, ld, false, n, n, n, -1.0, 0.0);
      BLK_FOR(i, n) s.Tdense[i * ld + i] += 1.0;
      __syncthreads();
      blk_copy(s.Tf, ld, s.Tdense, ld, n, n);
      __syncthreads();
      if (!blk_getrf(s.Tf, ld, n, s.piv, red, ired)) st = OTS_E_SINGULAR_T;
      break;
    }
    default:
      st = OTS_E_PARAMETER;
  }
  __syncthreads();
  return st;
}

__device__ void seed_finish(SmallState& s) {
  const int n = s.k0, k = s.k, ld = s.ld;
  // 5. W_t = fl(P - V_t)
  BLK_FOR(e, n * n) { int i = e / n, j = e - i * n; s.Wt[i * ld + j] = s.P[i * ld + j] - s.Vt[i * ld + j]; }
  __syncthreads();
  // 6. Y1 = W_t^T A_t - V_b^T A_b  -> Z1 (in place)
  blk_gemm(s.Z1, ld, s.Wt, ld, true, s.At, ld, false, n, k, n, 1.0, 0.0);
  BLK_FOR(e, n * k) { int i = e / k, j = e - i * k; s.Z1[i * ld + j] -= s.VbA[i * ld + j]; }
  __syncthreads();
  // 7. Z1 = T^{-T} Y1
  t_solve(s, s.Z1, ld, k, true);
  // 8. AH_t = A_t - W_t Z1 ; S = P^T AH_t
  blk_gemm(s.X1, ld, s.Wt, ld, false, s.Z1, ld, false, n, k, n, 1.0, 0.0);
  BLK_FOR(e, n * k) { int i = e / k, j = e - i * k; s.X1[i * ld + j] = s.At[i * ld + j] - s.X1[i * ld + j]; }
  __syncthreads();
  blk_gemm(s.Sout, s.lds_out, s.P, ld, true, s.X1, ld, false, n, k, n, 1.0, 0.0);
}

__device__ void seed_body(SmallState& s, double* red, int* ired) {
  if (threadIdx.x == 0) { s.status[0] = 0; }
  if (!seed_checks(s, red)) return;
  const int st = seed_build(s, red, ired);
  if (st != 0) {
    if (threadIdx.x == 0) s.status[0] = st;
    return;
  }
  seed_finish(s);
}

// A 2-CTA cluster launch (polar seed, k0 <= JC_NMAX): CTA 1 only serves the
// Jacobi's J^T; CTA 0 runs the seed and closes the link on every exit path.
__global__ void __launch_bounds__(SMALL_NT) seed_kernel(SmallState s) {
  __shared__ double red[64];
  __shared__ int ired[64];
  const bool clu = cl_size() == 2;
  if (clu) {
    jacobi_link_init();
    if (cl_rank() == 1) { jacobi_jt_helper(s.X2, s.ld, s.k0); return; }
  }
  seed_body(s, red, ired);
  if (clu) jacobi_link_close(0);
}

__global__ void __launch_bounds__(SMALL_NT) seedA_kernel(SmallState s) {
  __shared__ double red[64];
  __shared__ int ired[64];
  const bool clu = cl_size() == 2;
  if (clu) {
    jacobi_link_init();
    if (cl_rank() == 1) { jacobi_jt_helper(s.X2, s.ld, s.k0); return; }
  }
  const int st = seed_build(s, red, ired);
  if (threadIdx.x == 0) s.status[1] = st;
  if (clu) jacobi_link_close(0);
}

__global__ void __launch_bounds__(SMALL_NT) seedB_kernel(SmallState s) {
  __shared__ double red[64];
  if (threadIdx.x == 0) { s.status[0] = 0; }
  if (!seed_checks(s, red)) return;
  if (s.status[1] != 0) {                 // seed errors come after the Gram checks
    if (threadIdx.x == 0) s.status[0] = s.status[1];
    return;
  }
  seed_finish(s);
}

// Diagnostics from k0 x k0 data (reflector.py:241-247):
// kappa_2(T) and ||W T^{-1}||_2 = sqrt(lambda_max(T^{-T} W^T W T^{-1})),
// W^T W = W_t^T W_t + (G - V_t^T V_t).
// Diagnostics from k0 x k0 data only: kappa(T) = sigma_max(T)
// sigma_max(T^-1) and ||W T^-1||_2 = sqrt(lambda_max(T^-T W^T W T^-1)), as the
// largest eigenvalues of three symmetric matrices, one per CTA (grid 3); the
// last CTA to finish combines them.
__global__ void __launch_bounds__(SMALL_NT) diag_kernel(SmallState s) {
  __shared__ double red[64];
  __shared__ double vec_s[4 * 512];
  __shared__ int last;
  if (s.status[0] != 0) return;
  const int n = s.k0, ld = s.ld;
  long long tm0 = clock64();
  const bool fit = n * (n + 1) <= SMALL_SMEM_DOUBLES;
  // k0 > 512: the tridiagonal scratch moves to the dynamic shared memory (the
  // matrices then live in global memory, so dsm is otherwise unused)
  double* vec = (n <= 512) ? vec_s : dsm;
  const int lss = fit ? n + 1 : ld;
  double lam;
  if (blockIdx.x == 0) {  // T^T T
    double* S = fit ? dsm : s.dg[0];
    blk_gemm(S, lss, s.Tdense, ld, true, s.Tdense, ld, false, n, n, n, 1.0, 0.0);
    lam = blk_sym_lmax(S, lss, n, vec, red);
    SMARK(10, tm0);
  } else if (blockIdx.x == 1) {  // T^-T T^-1
    double* E = s.dg[1];
    blk_identity(E, ld, n);
    t_solve(s, E, ld, n, false);
    double* S = fit ? dsm : s.dg[2];
    blk_gemm(S, lss, E, ld, true, E, ld, false, n, n, n, 1.0, 0.0);
    lam = blk_sym_lmax(S, lss, n, vec, red);
    SMARK(11, tm0);
  } else {  // M = T^-T (W^T W) T^-1
    double *E = s.dg[3], *WW = s.dg[4], *H = s.dg[5];
    blk_identity(E, ld, n);
    t_solve(s, E, ld, n, false);
    SMARK(12, tm0);
    if (s.Gu == nullptr) {
      blk_gemm(WW, ld, s.Wt, ld, true, s.Wt, ld, false, n, n, n, 1.0, 0.0);
      blk_gemm(WW, ld, s.Vt, ld, true, s.Vt, ld, false, n, n, n, -1.0, 1.0);
      BLK_FOR(e2, n * n) { int i = e2 / n, j = e2 - i * n; WW[i * ld + j] += s.G[i * ld + j]; }
    } else if (s.Ltinv != nullptr) {  // B-inner, dense B = L L^T: unweighted W = u0 p - v
      const double* Vo = s.Vorig;      // original top rows (global)
      blk_gemm(H, ld, s.Ltinv, s.ldlt, false, s.P, ld, false, n, n, n, 1.0, 0.0);   // L_m^{-T} P
      BLK_FOR(e2, n * n) { int i = e2 / n, j = e2 - i * n; H[i * ld + j] -= Vo[(long)i * s.ldvo + j]; }
      __syncthreads();
      blk_gemm(WW, ld, H, ld, true, H, ld, false, n, n, n, 1.0, 0.0);
      BLK_FOR(e2, n * n) {             // - V_t^T V_t
        int i = e2 / n, j = e2 - i * n;
        double acc = 0.0;
        for (int l = 0; l < n; ++l) acc = fma(Vo[(long)l * s.ldvo + i], Vo[(long)l * s.ldvo + j], acc);
        WW[i * ld + j] -= acc;
      }
      __syncthreads();
      BLK_FOR(e2, n * n) {
        int i = e2 / n, j = e2 - i * n;
        WW[i * ld + j] += (j <= i) ? s.Gu[(long)i * s.ldgu + j] : s.Gu[(long)j * s.ldgu + i];
      }
      __syncthreads();
    } else {  // B-inner, M = diag(d): unweighted W = D^{-1/2} W'
      BLK_FOR(e2, n * n) { int i = e2 / n, j = e2 - i * n; H[i * ld + j] = s.dinv_top[i] * s.Wt[i * ld + j]; }
      blk_gemm(WW, ld, s.Wt, ld, true, H, ld, false, n, n, n, 1.0, 0.0);
      BLK_FOR(e2, n * n) { int i = e2 / n, j = e2 - i * n; H[i * ld + j] = s.dinv_top[i] * s.Vt[i * ld + j]; }
      blk_gemm(WW, ld, s.Vt, ld, true, H, ld, false, n, n, n, -1.0, 1.0);
      BLK_FOR(e2, n * n) {
        int i = e2 / n, j = e2 - i * n;
        WW[i * ld + j] += (j <= i) ? s.Gu[(long)i * s.ldgu + j] : s.Gu[(long)j * s.ldgu + i];
      }
    }
    blk_gemm(H, ld, WW, ld, false, E, ld, false, n, n, n, 1.0, 0.0);
    double* S = fit ? dsm : WW;
    blk_gemm(S, lss, E, ld, true, H, ld, false, n, n, n, 1.0, 0.0);
    BLK_FOR(e2, n * n) {  // symmetrise
      int i = e2 / n, j = e2 - i * n;
      if (j < i) {
        const double h = 0.5 * (S[i * lss + j] + S[j * lss + i]);
        S[i * lss + j] = h;
        S[j * lss + i] = h;
      }
    }
    SMARK(13, tm0);
    lam = blk_sym_lmax(S, lss, n, vec, red);
    SMARK(14, tm0);
  }
  if (threadIdx.x == 0) {
    s.dlam[blockIdx.x] = lam;
    __threadfence();
    last = (atomicAdd(s.dcount, 1) == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    const volatile double* L = s.dlam;
    const double l0 = L[0], l1 = L[1], l2 = L[2];
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    s.diag[0] = (l1 < inf) ? sqrt(fmax(l0, 0.0)) * sqrt(fmax(l1, 0.0)) : inf;
    s.diag[1] = sqrt(fmax(l2, 0.0));
  }
}

// apply_reflector (reflector.py:231-238) small part: Y = W_t^T X_t - V_b^T X_b
// (VbX from the reduced Gram block at Gfull/ldgf), Z = T^{-(*)} Y into Z1,
// top rows out_t = X_t - W_t Z into Sout (ld lds_out).  X_t = s.A (lda).
__global__ void __launch_bounds__(SMALL_NT) refl_apply_kernel(SmallState s, int adjoint) {
  const int n = s.k0, k = s.k, ld = s.ld;
  BLK_FOR(e, n * k) { int i = e / k, j = e - i * k; s.At[i * ld + j] = s.A[(long)i * s.lda + j]; }
  __syncthreads();
  blk_gemm(s.Z1, ld, s.Wt, ld, true, s.At, ld, false, n, k, n, 1.0, 0.0);
  BLK_FOR(e, n * k) { int i = e / k, j = e - i * k; s.Z1[i * ld + j] -= s.Gfull[(long)i * s.ldgf + j]; }
  __syncthreads();
  t_solve(s, s.Z1, ld, k, adjoint != 0);
  blk_gemm(s.X1, ld, s.Wt, ld, false, s.Z1, ld, false, n, k, n, 1.0, 0.0);
  BLK_FOR(e, n * k) { int i = e / k, j = e - i * k; s.Sout[(long)i * s.lds_out + j] = s.At[i * ld + j] - s.X1[i * ld + j]; }
}

// T-solver entry (reflector.py:80-153): B (k0 x m, ld ldb) <- T^{-(*)} B
__global__ void __launch_bounds__(SMALL_NT) tsolve_kernel(SmallState s, double* B, int ldb, int m, int adjoint) {
  t_solve(s, B, ldb, m, adjoint != 0);
}

// Z2 = T^{-1} Y2
// Z2 = T^{-1} Y2, Z2_COLS right-hand sides per CTA (the solves are column-separable)
constexpr int Z2_COLS = 8;
__global__ void __launch_bounds__(SMALL_NT) z2_kernel(SmallState s) {
  if (s.status[0] != 0) return;
  const int c0 = blockIdx.x * Z2_COLS;
  const int m = s.k - c0 < Z2_COLS ? s.k - c0 : Z2_COLS;
  if (m > 0) t_solve(s, s.Z2 + c0, s.ld, m, false);
}

// LAPACK sign recovery on Q_ top k x k and R output
__global__ void __launch_bounds__(SMALL_NT) sign_kernel(SmallState s, const double* Qtop, long ldq,
                                                        const double* Rfin, int ldr, double* Rout,
                                                        int ldro) {
  if (s.status[0] != 0) return;
  const int k = s.k, ld = s.ld;
  // scratch X2: the diag kernel may run concurrently on the side stream and
  // owns D1/D2/sig2.
  BLK_FOR(e, k * k) { int i = e / k, j = e - i * k; s.X2[i * ld + j] = Qtop[(long)i * ldq + j]; }
  __syncthreads();
  blk_mlu(s.X2, ld, k, s.svec, true);
  BLK_FOR(e, k * k) {
    int i = e / k, j = e - i * k;
    Rout[i * ldro + j] = (j >= i) ? s.svec[i] * Rfin[i * ldr + j] : 0.0;
  }
}

// Q_top = -(W_t Z2) diag(svec)
// Q_t = -W_t Z2 diag(s): QTOP_ROWS rows of Q_t per CTA, one output per
// thread (k <= 64 columns); W_t rows and Z2 staged through shared memory in
// chunks of QTOP_LC rows of the reduction.
constexpr int QTOP_ROWS = 8, QTOP_LC = 128;
__global__ void __launch_bounds__(QTOP_ROWS * 64) qtop_kernel(SmallState s, double* Q, long ldq) {
  if (s.status[0] != 0) return;
  const int n = s.k0, k = s.k, ld = s.ld;
  const int i0 = blockIdx.x * QTOP_ROWS;
  double* Zs = dsm;                       // QTOP_LC x k
  double* Ws = dsm + QTOP_LC * k;         // QTOP_ROWS x QTOP_LC
  const int r = threadIdx.x / 64, j = threadIdx.x % 64;
  double a0 = 0.0, a1 = 0.0;
  for (int l0 = 0; l0 < n; l0 += QTOP_LC) {
    const int lc = n - l0 < QTOP_LC ? n - l0 : QTOP_LC;
    __syncthreads();
    for (int e = threadIdx.x; e < lc * k; e += blockDim.x) Zs[e] = s.Z2[(l0 + e / k) * ld + e % k];
    for (int e = threadIdx.x; e < QTOP_ROWS * lc; e += blockDim.x) {
      const int rr = i0 + e / lc;
      Ws[e] = rr < n ? s.Wt[rr * ld + l0 + e % lc] : 0.0;
    }
    __syncthreads();
    if (j < k) {
      int l = 0;
      for (; l + 1 < lc; l += 2) {
        a0 = fma(Ws[r * lc + l], Zs[l * k + j], a0);
        a1 = fma(Ws[r * lc + l + 1], Zs[(l + 1) * k + j], a1);
      }
      if (l < lc) a0 = fma(Ws[r * lc + l], Zs[l * k + j], a0);
    }
  }
  if (i0 + r < n && j < k) Q[(long)(i0 + r) * ldq + j] = -(a0 + a1) * s.svec[j];
}

// Standalone modified LU (the `modified_lu` API, reflector.py:53-77), with
// the ||z||_2 <= 1 + 1e-8 precondition (NormBoundError).
__global__ void __launch_bounds__(SMALL_NT) mlu_kernel(const double* Z, int ldz, int n, double* LU,
                                                       double* p, double* work, int* status) {
  __shared__ double red[64];
  blk_copy(work, n, Z, ldz, n, n);
  __syncthreads();
  double nrm = blk_sigma_max(work, n, n, work + n * n, red, dsm, SMALL_SMEM_DOUBLES);
  if (nrm > 1.0 + 1e-8) { if (threadIdx.x == 0) *status = OTS_E_NORM_BOUND; return; }
  blk_copy(LU, n, Z, ldz, n, n);
  __syncthreads();
  blk_mlu(LU, n, n, p, false);
  if (threadIdx.x == 0) *status = 0;
}

// One shifted-Cholesky-QR step (core.py:177-202): from the Gram G (ld ldg,
// lower blocks valid) of the current block, L = chol(sym(G) [+ shift I]),
// Z = L^{-T} (for X <- X Z) and R <- L^T R.  shift = 11 (m k + k(k+1)) u ||G||_2.
// NotPositiveDefinite -> status OTS_E_INTRA_FAILURE (twostage.py:51-53).
__global__ void __launch_bounds__(SMALL_NT) cholqr_step_kernel(const double* Gf, int ldg, int k, long m,
                                                               int shift, double* W, int ld, double* Z,
                                                               double* R, int* status) {
  __shared__ double red[64];
  if (status[0] != 0) return;
  double* L = W;                // k x k
  double* Tm = W + k * ld;      // scratch
  BLK_FOR(e, k * k) {
    int i = e / k, j = e - i * k;
    double gij = (j <= i) ? Gf[(long)i * ldg + j] : Gf[(long)j * ldg + i];
    L[i * ld + j] = gij;
    Tm[i * ld + j] = gij;
  }
  __syncthreads();
  if (shift) {
    double nrm = blk_sigma_max(Tm, ld, k, Tm + k * ld, red, dsm, SMALL_SMEM_DOUBLES);
    const double sh = 11.0 * ((double)m * k + (double)k * (k + 1)) * 1.1102230246251565e-16 * nrm;
    BLK_FOR(i, k) L[i * ld + i] += sh;
    __syncthreads();
  }
  if (!blk_cholesky(L, ld, k, red)) {
    if (threadIdx.x == 0) status[0] = OTS_E_INTRA_FAILURE;
    return;
  }
  // Z = L^{-T}: solve L^T Z = I
  BLK_FOR(e, k * k) { int i = e / k, j = e - i * k; Z[i * ld + j] = (i == j) ? 1.0 : 0.0; }
  __syncthreads();
  blk_trsm(L, ld, true, true, false, Z, ld, k, k);
  // R <- L^T R
  blk_gemm(Tm, ld, L, ld, true, R, ld, false, k, k, k, 1.0, 0.0);
  blk_copy(R, ld, Tm, ld, k, k);
  __syncthreads();
}

cudaError_t launch_cholqr_step(const double* Gf, int ldg, int k, long m, int shift, double* W, int ld,
                               double* Z, double* R, int* status, cudaStream_t st) {
  cudaFuncSetAttribute(cholqr_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMALL_SMEM_DOUBLES * 8);
  cholqr_step_kernel<<<1, SMALL_NT, SMALL_SMEM_DOUBLES * 8, st>>>(Gf, ldg, k, m, shift, W, ld, Z, R, status);
  return cudaGetLastError();
}

bool seed_uses_cluster(const SmallState& s) {
  static const bool off = getenv("OTS_NO_SEED_CLUSTER") != nullptr;   // A/B switch
  return !off && s.choice == CHOICE_POLAR && s.k0 >= 16 && s.k0 <= JC_NMAX;
}

// the polar seed as a 2-CTA cluster (seed_uses_cluster), else one CTA
static cudaError_t launch_seed_kernel(void (*k)(SmallState), const SmallState& s, cudaStream_t st) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMALL_SMEM_DOUBLES * 8);
  if (!seed_uses_cluster(s)) {
    k<<<1, SMALL_NT, SMALL_SMEM_DOUBLES * 8, st>>>(s);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2, 1, 1);
  cfg.blockDim = dim3(SMALL_NT, 1, 1);
  cfg.dynamicSmemBytes = SMALL_SMEM_DOUBLES * 8;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, s);
}

cudaError_t launch_seed_split(const SmallState& s, int part, cudaStream_t st) {
  if (part == 0) return launch_seed_kernel(seedA_kernel, s, st);
  cudaFuncSetAttribute(seedB_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMALL_SMEM_DOUBLES * 8);
  seedB_kernel<<<1, SMALL_NT, SMALL_SMEM_DOUBLES * 8, st>>>(s);
  return cudaGetLastError();
}

cudaError_t launch_seed(const SmallState& s, cudaStream_t st) { return launch_seed_kernel(seed_kernel, s, st); }
cudaError_t launch_diag(const SmallState& s, cudaStream_t st) {
  cudaFuncSetAttribute(diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMALL_SMEM_DOUBLES * 8);
  cudaMemsetAsync(s.dcount, 0, sizeof(int), st);
  diag_kernel<<<3, SMALL_NT, SMALL_SMEM_DOUBLES * 8, st>>>(s);
  return cudaGetLastError();
}
cudaError_t launch_refl_apply(const SmallState& s, int adjoint, cudaStream_t st) {
  cudaFuncSetAttribute(refl_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMALL_SMEM_DOUBLES * 8);
  refl_apply_kernel<<<1, SMALL_NT, SMALL_SMEM_DOUBLES * 8, st>>>(s, adjoint);
  return cudaGetLastError();
}
cudaError_t launch_tsolve(const SmallState& s, double* B, int ldb, int m, int adjoint, cudaStream_t st) {
  cudaFuncSetAttribute(tsolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMALL_SMEM_DOUBLES * 8);
  tsolve_kernel<<<1, SMALL_NT, SMALL_SMEM_DOUBLES * 8, st>>>(s, B, ldb, m, adjoint);
  return cudaGetLastError();
}

cudaError_t launch_z2(const SmallState& s, cudaStream_t st) {
  cudaFuncSetAttribute(z2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMALL_SMEM_DOUBLES * 8);
  z2_kernel<<<(s.k + Z2_COLS - 1) / Z2_COLS, SMALL_NT, SMALL_SMEM_DOUBLES * 8, st>>>(s);
  return cudaGetLastError();
}
cudaError_t launch_sign(const SmallState& s, const double* Qtop, long ldq, const double* Rfin, int ldr,
                        double* Rout, int ldro, cudaStream_t st) {
  sign_kernel<<<1, SMALL_NT, 0, st>>>(s, Qtop, ldq, Rfin, ldr, Rout, ldro);
  return cudaGetLastError();
}
cudaError_t launch_qtop(const SmallState& s, double* Q, long ldq, cudaStream_t st) {
  if (s.k > 64) return cudaErrorInvalidValue;
  const int smem = (QTOP_LC * s.k + QTOP_ROWS * QTOP_LC) * 8;
  cudaFuncSetAttribute(qtop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  qtop_kernel<<<(s.k0 + QTOP_ROWS - 1) / QTOP_ROWS, QTOP_ROWS * 64, smem, st>>>(s, Q, ldq);
  return cudaGetLastError();
}
cudaError_t launch_mlu(const double* Z, int ldz, int n, double* LU, double* p, double* work, int* status,
                       cudaStream_t st) {
  cudaFuncSetAttribute(mlu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMALL_SMEM_DOUBLES * 8);
  mlu_kernel<<<1, SMALL_NT, SMALL_SMEM_DOUBLES * 8, st>>>(Z, ldz, n, LU, p, work, status);
  return cudaGetLastError();
}

void debug_counters_small(unsigned long long* out, int reset) {
#ifdef OTS_TIMING
  unsigned long long tmp[16];
  cudaMemcpyFromSymbol(tmp, g_dbg_small, sizeof tmp);
  for (int i = 10; i < 16; ++i) out[i] += tmp[i];
  if (reset) { unsigned long long z[16] = {0}; cudaMemcpyToSymbol(g_dbg_small, z, sizeof z); }
#else
  (void)out; (void)reset;
#endif
}

// Stability metrics from Gram blocks (metrics.py:25-73 restated for the GPU,
// SURVEY 8(f)): loss = max |lambda(G) - 1| over the Gram of q (or of [v, q]),
// cross = ||v^* q||_F, residual = sqrt(lambda_max(E^T E) / lambda_max(A^T A))
// with E = a - v s - q r formed explicitly.  Symmetric inputs: lower valid.
__global__ void __launch_bounds__(SMALL_NT) stability_kernel(const double* Gvv, long ldvv, const double* Gvq,
                                                             long ldvq, const double* Gqq, long ldqq,
                                                             const double* Gee, long ldee, const double* Gaa,
                                                             long ldaa, int k0, int k, int augmented,
                                                             double* work, double* out3) {
  __shared__ double red[64];
  const int m = augmented ? k0 + k : k;
  double* M = work;                 // m x m
  double* vec = work + (long)m * m; // 4 m
  auto lowsym = [](const double* G, long ld, int i, int j) { return (j <= i) ? G[i * ld + j] : G[j * ld + i]; };
  BLK_FOR(e, m * m) {
    const int i = e / m, j = e - i * m;
    double x;
    if (!augmented) x = lowsym(Gqq, ldqq, i, j);
    else if (i < k0 && j < k0) x = lowsym(Gvv, ldvv, i, j);
    else if (i < k0) x = Gvq[(long)i * ldvq + (j - k0)];
    else if (j < k0) x = Gvq[(long)j * ldvq + (i - k0)];
    else x = lowsym(Gqq, ldqq, i - k0, j - k0);
    M[e] = x - (i == j ? 1.0 : 0.0);
  }
  double cr = 0.0;
  if (Gvq) BLK_FOR(e, k0 * k) { const double x = Gvq[(long)(e / k) * ldvq + (e % k)]; cr = fma(x, x, cr); }
  cr = block_sum(cr, red);
  __syncthreads();
  double lmin = 0.0, lmax = 0.0;
  if (m > 0) blk_sym_extremes(M, m, m, vec, red, lmin, lmax);
  const double loss = fmax(fabs(lmax), fabs(lmin));
  double resid = 0.0;
  if (Gee) {
    BLK_FOR(e, k * k) { const int i = e / k, j = e - i * k; M[e] = lowsym(Gee, ldee, i, j); }
    __syncthreads();
    const double le = blk_sym_lmax(M, k, k, vec, red);
    BLK_FOR(e, k * k) { const int i = e / k, j = e - i * k; M[e] = lowsym(Gaa, ldaa, i, j); }
    __syncthreads();
    const double la = blk_sym_lmax(M, k, k, vec, red);
    resid = (la > 0.0) ? sqrt(fmax(le, 0.0) / la) : 0.0;
  }
  if (threadIdx.x == 0) { out3[0] = loss; out3[1] = sqrt(cr); out3[2] = resid; }
}

cudaError_t launch_stability(const double* Gvv, long ldvv, const double* Gvq, long ldvq, const double* Gqq,
                             long ldqq, const double* Gee, long ldee, const double* Gaa, long ldaa, int k0, int k,
                             int augmented, double* work, double* out3, cudaStream_t st) {
  stability_kernel<<<1, SMALL_NT, 0, st>>>(Gvv, ldvv, Gvq, ldvq, Gqq, ldqq, Gee, ldee, Gaa, ldaa, k0, k,
                                           augmented, work, out3);
  return cudaGetLastError();
}

// LAPACK sign vector of a QR with positive R diagonal from its
// Q's top k x k block: the modified-LU rule, with the tau = 0 / |z_jj| = 1
// exception (dlarfg's shortcut).  svec: k entries +-1 (device).
__global__ void __launch_bounds__(SMALL_NT) qr_signs_kernel(const double* Qtop, long ldq, int k, double* work,
                                                            double* svec) {
  BLK_FOR(e, k * k) { const int i = e / k, j = e - i * k; work[i * k + j] = Qtop[(long)i * ldq + j]; }
  __syncthreads();
  blk_mlu(work, k, k, svec, true);
}
cudaError_t launch_qr_signs(const double* Qtop, long ldq, int k, double* work, double* svec, cudaStream_t st) {
  qr_signs_kernel<<<1, SMALL_NT, 0, st>>>(Qtop, ldq, k, work, svec);
  return cudaGetLastError();
}

// lambda_min, lambda_max of a symmetric m x m matrix (lower triangle of G
// read; work: m*m + 4m doubles) -- spectra of Grams for orthonormality_defect
// and the weighted norms (core.py:35-49, oblique.py:70-90)
__global__ void __launch_bounds__(SMALL_NT) sym_extremes_kernel(const double* G, long ldg, int m, double* work,
                                                                double* out2) {
  __shared__ double red[64];
  double* M = work;
  double* vec = work + (long)m * m;
  BLK_FOR(e, m * m) {
    const int i = e / m, j = e - i * m;
    M[e] = (j <= i) ? G[(long)i * ldg + j] : G[(long)j * ldg + i];
  }
  double lmin = 0.0, lmax = 0.0;
  if (m == 1) {
    __syncthreads();
    lmin = lmax = M[0];
  } else if (m > 1) {
    blk_sym_extremes(M, m, m, vec, red, lmin, lmax);
  }
  if (threadIdx.x == 0) { out2[0] = lmin; out2[1] = lmax; }
}
cudaError_t launch_sym_extremes(const double* G, long ldg, int m, double* work, double* out2, cudaStream_t st) {
  sym_extremes_kernel<<<1, SMALL_NT, 0, st>>>(G, ldg, m, work, out2);
  return cudaGetLastError();
}

__global__ void neg_copy_kernel(const double* X, long ldx, int r, int c, double* Y, long ldy) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < r * c; e += gridDim.x * blockDim.x) {
    const int i = e / c, j = e - i * c;
    Y[i * ldy + j] = -X[i * ldx + j];
  }
}
cudaError_t launch_neg_copy(const double* X, long ldx, int r, int c, double* Y, long ldy, cudaStream_t st) {
  neg_copy_kernel<<<32, 256, 0, st>>>(X, ldx, r, c, Y, ldy);
  return cudaGetLastError();
}

#include "zsmall.inc"

}  // namespace ots
