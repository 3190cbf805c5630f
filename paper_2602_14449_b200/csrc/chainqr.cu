// Intra-block Householder QR of the exposed (n-k0) x k block on B200:
// flat-chain TSQR with structured [R; tile] Householder steps and a tree over
// chain R's, then explicit Q formation in reverse.  Replaces LAPACK
// dgeqrf+dorgqr behind `householder_qr` (core.py:61-84, called from
// twostage.py:93 via intra_qr twostage.py:45-54).  LAPACK's R sign convention
// is recovered afterwards (sign kernel in small.cu).
//
// Chain layout (per level):  a chain owns rows [c*RPC, (c+1)*RPC) with
// RPC = KT + L*b:  a KT-row "head" factored by a plain Householder QR, then L
// structured tiles of b rows, each factored as QR([R; tile]) with reflectors
// v_j = [e_j; y_j] (identity top).  Per tile we keep Y (in place over the
// data) and U = diag(tau) + striu(Y^T Y)  ->  T (compact-WY, dlarft).
#include "common.cuh"
#include "kernels.cuh"

namespace ots {

#ifdef OTS_TIMING
__device__ unsigned long long g_dbg[16];
#define TSTAMP(v) long long v = clock64()
#define TACC(slot, a, b) if (threadIdx.x == 0) atomicAdd(&g_dbg[slot], (unsigned long long)((b) - (a)))
#else
#define TSTAMP(v)
#define TACC(slot, a, b)
#endif

__device__ __forceinline__ int chain_real_tiles(const ChainGeom& G, int chain, int KT) {
  long r0 = (long)chain * G.rpc + KT;
  long rem = G.nrows - r0;
  if (rem <= 0) return 0;
  long t = (rem + G.b - 1) / G.b;
  return (int)(t < G.L ? t : G.L);
}

template <int KT>
struct FactorCfg {
  static constexpr int NT = 256;
  static constexpr int TPC = NT / KT;             // threads per column
  static constexpr int LDS = KT + KT / 8;         // padded row stride (bank spread)
  static constexpr int BMAX = 128;                      // = BlkCfg<KT>::B
};

// Sum over the TPC consecutive lanes that own one column (all of them take the
// same branches, so the group mask is exact even in divergent code).
template <int TPC>
__device__ __forceinline__ double tpc_sum(double v, unsigned mask) {
#pragma unroll
  for (int o = TPC / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

// plain-stride async tile load: smem rows [s0, s0+nr) <- global rows [gr0, gr0+nr)
template <int KT, int LDS>
__device__ __forceinline__ void load_rows_plain(double* S, int s0, const double* D, long ldd,
                                                long gr0, int nr, long nrows, int ncols, int tid,
                                                int nt) {
  constexpr int UPR = KT / 2;
  for (int i = tid; i < nr * UPR; i += nt) {
    int r = i / UPR, u = i - r * UPR;
    long gr = gr0 + r;
    int c = 2 * u;
    int bytes = 0;
    const double* src = D;
    if (gr < nrows && c < ncols) {
      bytes = (c + 1 < ncols) ? 16 : 8;
      src = D + gr * ldd + c;
    }
    cp_async16(S + (s0 + r) * LDS + c, src, bytes);
  }
}

template <int KT, int LDS>
__device__ __forceinline__ void store_rows_plain(const double* S, int s0, double* D, long ldd,
                                                 long gr0, int nr, long nrows, int ncols, int tid,
                                                 int nt) {
  constexpr int UPR = KT / 2;
  for (int i = tid; i < nr * UPR; i += nt) {
    int r = i / UPR, u = i - r * UPR;
    long gr = gr0 + r;
    int c = 2 * u;
    if (gr >= nrows || c >= ncols) continue;
    const double* s = S + (s0 + r) * LDS + c;
    if (c + 1 < ncols) *reinterpret_cast<double2*>(D + gr * ldd + c) = make_double2(s[0], s[1]);
    else D[gr * ldd + c] = s[0];
  }
}

// One Householder sweep over the KT columns of the smem tile.
//  head=true : rows 0..KT-1 only (plain QR of a KT x KT block)
//  head=false: top rows 0..KT-1 hold R (upper), bottom rows KT..KT+nb-1
// Writes U[c][j] = v_c^T v_j (c<j) and U[j][j] = tau_j to global `U`.
template <int KT, bool HEAD, int LDS = FactorCfg<KT>::LDS>
__device__ __forceinline__ void householder_sweep(double* S, int nb, double* U, double* tau_s) {
  using C = FactorCfg<KT>;
  constexpr int TPC = C::TPC;
  const int tid = threadIdx.x;
  const int c = tid / TPC, q = tid % TPC;
  const unsigned gmask = (TPC >= 32) ? 0xffffffffu
                                     : (((1u << TPC) - 1u) << ((tid & 31) & ~(TPC - 1)));

  auto rbeg = [&](int j) { return HEAD ? (j + 1 + q) : (KT + q); };
  const int rend = HEAD ? KT : (KT + nb);

  auto phase_a = [&](int j) {  // owners of column j: generate reflector j (dlarfg)
    double s2 = 0.0;
    for (int r = rbeg(j); r < rend; r += TPC) { double x = S[r * LDS + j]; s2 = fma(x, x, s2); }
    s2 = tpc_sum<TPC>(s2, gmask);
    const double alpha = S[j * LDS + j];
    double beta = alpha, tau = 0.0, scal = 0.0;
    if (s2 != 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, s2)), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
      for (int r = rbeg(j); r < rend; r += TPC) S[r * LDS + j] *= scal;
    }
    if (q == 0) { S[j * LDS + j] = beta; tau_s[j] = tau; }
  };

  if (c == 0) phase_a(0);
  __syncthreads();
  for (int j = 0; j < KT; ++j) {
    const double tau = tau_s[j];
    if (c != j) {
      double d = 0.0;
      for (int r = rbeg(j); r < rend; r += TPC) d = fma(S[r * LDS + j], S[r * LDS + c], d);
      d = tpc_sum<TPC>(d, gmask);
      d += S[j * LDS + c];
      if (c > j) {
        const double w = tau * d;
        for (int r = rbeg(j); r < rend; r += TPC) S[r * LDS + c] = fma(-w, S[r * LDS + j], S[r * LDS + c]);
        // row j of column c: owned by q==0 (head: row j is not in rbeg range)
        if (q == 0) S[j * LDS + c] -= w;
        if (c == j + 1) {
          __syncwarp(gmask);
          phase_a(j + 1);
        }
      } else {
        if (q == 0) U[c * (KT + 1) + j] = d;
      }
    } else {
      if (q == 0) U[j * (KT + 1) + j] = tau;
    }
    __syncthreads();
  }
}


// dlarfg arithmetic with one rsqrt and one reciprocal (no IEEE division or
// sqrt on the critical path):  h = alpha^2 + |x|^2, s = sqrt(h),
//   beta = -sign(alpha) s,  tau = (|alpha| + s)/s,  scal = sign(alpha)/(|alpha| + s)
// which equal LAPACK's (beta-alpha)/beta and 1/(alpha-beta) to ~1 ulp.
__device__ __forceinline__ void dlarfg_fast(double alpha, double s2, double& beta, double& tau,
                                            double& scal) {
  const double h = fma(alpha, alpha, s2);
  const double r = rsqrt(h);
  const double sq = h * r;
  const double aa = fabs(alpha);
  const double t = aa + sq;
  beta = -copysign(sq, alpha);
  tau = t * r;
  // 1/t: MUFU reciprocal seed + two Newton steps (~1 ulp, no IEEE slow path)
  double rt;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rt) : "d"(t));
  rt = rt * fma(-t, rt, 2.0);
  rt = rt * fma(-t, rt, 2.0);
  scal = copysign(rt, alpha);
}

// Structured step QR([R; X]) with the b x KT tile X held in REGISTERS.
// Thread (cg, rb) owns an RPB x CPT block: rows rb*RPB.., columns cg*CPT..
// The NRB threads sharing a column group are consecutive lanes, so every
// column reduction is a shuffle tree inside one warp.  Per column step a
// thread issues RPB/2 LDS.128 (v_j) for 2*RPB*CPT FMAs; only v_j
// (double-buffered, bank-padded) and R's row j go through shared memory.
// U (diag tau, strict-upper Gram, ld KT+1) -> T via the dlarft recurrence
// T[0:j, j] = -tau_j T[0:j, 0:j] U[0:j, j] (head tile only), 4 threads/row.
template <int KT>
__device__ __forceinline__ void u_to_t_block(const double* Us, double* Ts, double* Tg) {
  constexpr int UL = KT + 1;
  const int tid = threadIdx.x;
  const int i = tid >> 2, part = tid & 3;
  for (int e = tid; e < KT * KT; e += 256) Ts[e] = 0.0;
  __syncthreads();
  for (int j = 0; j < KT; ++j) {
    const double tj = Us[j * UL + j];
    double sacc = 0.0;
    if (i < j)
      for (int l = i + part; l < j; l += 4) sacc = fma(Ts[i * KT + l], Us[l * UL + j], sacc);
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
    if (i < j && part == 0) Ts[i * KT + j] = -tj * sacc;
    if (tid == 0) Ts[j * KT + j] = tj;
    __syncthreads();
  }
  for (int e = tid; e < KT * KT; e += 256) Tg[e] = Ts[e];
}

// ===========================================================================
// Structured TSQR step, blocked, register-resident (v5).  The 128 x KT tile
// lives in REGISTERS: warp w (< KT/8) owns columns 8w..8w+7, lane (g, t)
// (g = lane>>2, t = lane&3) holds x[f][h] = X[8f + 2t + h][8w + g] -- the
// C-fragment layout of m8n8k4 with X^T as the output.  R (KT x KT, upper) is
// in shared memory S, whose strictly lower part stores the Gram entries
// G[c][j] = y_c . y_j (c < j) for the tile's compact-WY T.  Per 8-column panel:
//   * warp p factors its panel: column norms and dots are 4-lane reductions
//     (a column's 128 rows sit in one lane quad), v is broadcast with 32
//     independent shuffles; Y_p goes to a double-buffered smem slot and T_p
//     (8 x 8, dlarft) to smem;
//   * one __syncthreads;
//   * warp w > p:  W^T = X_w^T Y_p + R[p rows, w cols]^T  (A from registers,
//     B = Y_p from smem), w^T = W^T T_p, R -= w, X_w^T -= w^T Y_p^T with the
//     register tile as the DMMA accumulator;  warp w < p records G blocks.
// Shared-memory traffic per DMMA is one 8-byte load per lane.
// ===========================================================================
template <int KT>
struct BlkCfg {
  static constexpr int B = 128;          // tile rows
  static constexpr int NB = 8;           // panel width
  static constexpr int NP = KT / NB;     // panels (= warps that own columns)
  static constexpr int YS = 12;          // Y slot row stride: 2 wavefronts per 32-lane access
  static constexpr int YSLOT = B * YS;
  static constexpr int NSLOT = 3;       // Y ring: a deferred apply reads Y_p one panel later
  static constexpr int XS0 = (2 * KT * KT + KT > NSLOT * YSLOT) ? 2 * KT * KT + KT : NSLOT * YSLOT;
  static constexpr int TWOFF = NSLOT * YSLOT + NP * 64;                  // packed T blocks
  static constexpr int XS1 = TWOFF + (NP * (NP - 1) / 2) * 64;   // Y slots | Gram scratch | T blocks
  static constexpr int XS2 = XS0 > XS1 ? XS0 : XS1;
  static constexpr int XS = (XS2 > KT * (KT + 4) ? XS2 : KT * (KT + 4)) + 64;  // head U|T, Y slots, Tw
  static constexpr int SMEM = (KT * KT + XS + 2 * NP * 64 + 8 * 64) * 8;
};

__device__ __forceinline__ void tile_regs_load(double (&x)[16][2], const double* D, long ldd, long gr0,
                                               int nb, int col, int ncols) {
  const int t = threadIdx.x & 3;
  const bool cv = col < ncols;
#pragma unroll
  for (int f = 0; f < 16; ++f)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = 8 * f + 2 * t + h;
      x[f][h] = (cv && r < nb) ? D[(gr0 + r) * ldd + col] : 0.0;
    }
}

__device__ __forceinline__ void tile_regs_store(const double (&x)[16][2], double* D, long ldd, long gr0,
                                                int nb, int col, int ncols) {
  const int t = threadIdx.x & 3;
  if (col >= ncols) return;
#pragma unroll
  for (int f = 0; f < 16; ++f)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = 8 * f + 2 * t + h;
      if (r < nb) D[(gr0 + r) * ldd + col] = x[f][h];
    }
}

// Sum 8 per-lane values over the warp: butterfly reduce-scatter (each step
// halves the values a lane keeps), a 2-level finish, then an indexed
// broadcast.  18 + 16 shuffles instead of 8 independent 5-level trees (80).
__device__ __forceinline__ void warp_sum8(double (&v)[8]) {
  const int lane = threadIdx.x & 31;
  double a[4], b2[2], c1;
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {          // xor 16: keep half
    double send = h16 ? v[i] : v[i + 4];
    double keep = h16 ? v[i + 4] : v[i];
    a[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {          // xor 8
    double send = h8 ? a[i] : a[i + 2];
    double keep = h8 ? a[i + 2] : a[i];
    b2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {                                      // xor 4
    double send = h4 ? b2[0] : b2[1];
    double keep = h4 ? b2[1] : b2[0];
    c1 = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  c1 += __shfl_xor_sync(0xffffffffu, c1, 2);
  c1 += __shfl_xor_sync(0xffffffffu, c1, 1);
  // lane holds total of index (h16?4:0)+(h8?2:0)+(h4?1:0); lane 4*idx' has it
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int src = ((i & 4) ? 16 : 0) + ((i & 2) ? 8 : 0) + ((i & 1) ? 4 : 0);
    v[i] = __shfl_sync(0xffffffffu, c1, src);
  }
}

// dlarfg without branches (one basic block): MUFU rsqrt/rcp seeds with two
// Newton steps each; s2 == 0 gives tau = 0, beta = alpha, scal = 0.
__device__ __forceinline__ void dlarfg_nb(double alpha, double s2, double& beta, double& tau,
                                          double& scal) {
  const double h = fma(alpha, alpha, s2);
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(h));
  r = r * fma(-0.5 * h * r, r, 1.5);
  r = r * fma(-0.5 * h * r, r, 1.5);
  const double sq = h * r;
  const double t = fabs(alpha) + sq;
  double rt;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rt) : "d"(t));
  rt = rt * fma(-t, rt, 2.0);
  rt = rt * fma(-t, rt, 2.0);
  const bool z = (s2 == 0.0);
  beta = z ? alpha : -copysign(sq, alpha);
  tau = z ? 0.0 : t * r;
  scal = z ? 0.0 : copysign(rt, alpha);
}

// One sweep over the 8 columns of a panel in the lane-per-row layout (lane
// owns rows l, l+32, l+64, l+96).  EXACT=false takes every column norm after
// the first from the downdate |x - w v|^2 = N - 2 w (x.v) + w^2 |v|^2 and is
// branch-free, so ptxas schedules the 8 steps as one block and overlaps the
// off-critical work (other dots, updates, T) with the reflector chain;
// returns true when a downdate cancelled more than half of N (then the caller
// replays the panel with EXACT=true, which reduces every norm).
template <int KT, bool EXACT>
__device__ __forceinline__ bool panel_core(int p, double (&xr)[4][8], double* S, double* T8,
                                           double* tau_s) {
  const int lane = threadIdx.x & 31;
  const int j0 = p * 8;
  const int lr = lane < 8 ? lane : 7;
  double s2n = 0.0;
  bool bad = false;
  double trow[8];       // lane ii < 8: row ii of T_p
#pragma unroll
  for (int l = 0; l < 8; ++l) trow[l] = 0.0;
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int j = j0 + jj;
    double rrow[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) rrow[cc] = (cc >= jj) ? S[j * KT + j0 + cc] : 0.0;
    // Raw dots x_jj . x_cc of the UNSCALED column: they do not depend on the
    // reflector scalars, so the warp reduction runs concurrently with dlarfg
    // and the step's critical path is one reduction, not dlarfg + reduction.
    double d[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      d[cc] = 0.0;
      if (cc != jj) {
#pragma unroll
        for (int i = 0; i < 4; ++i) d[cc] = fma(xr[i][jj], xr[i][cc], d[cc]);
      } else if (jj + 1 < 8) {   // slot jj carries |x_{jj+1}|^2 (pre-update)
#pragma unroll
        for (int i = 0; i < 4; ++i) d[cc] = fma(xr[i][jj + 1], xr[i][jj + 1], d[cc]);
      }
    }
    double s2 = s2n;
    if (EXACT || jj == 0) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int i = 0; i < 4; i += 2) { s0 = fma(xr[i][jj], xr[i][jj], s0); s1 = fma(xr[i + 1][jj], xr[i + 1][jj], s1); }
      s2 = warp_sum(s0 + s1);
    }
    warp_sum8(d);
    double beta, tj, scal;
    dlarfg_nb(rrow[jj], s2, beta, tj, scal);
#pragma unroll
    for (int i = 0; i < 4; ++i) xr[i][jj] *= scal;
#pragma unroll
    for (int cc = 0; cc < 8; ++cc)
      if (cc != jj) d[cc] *= scal;            // v . x_cc  (G entries for cc < jj)
    if (jj + 1 < 8) {
      const double N = d[jj];
      const double vv = s2 * scal * scal;
      const double w = tj * (d[jj + 1] + rrow[jj + 1]);
      const double nn = fma(w * w, vv, fma(-2.0 * w, d[jj + 1], N));
      bad = bad || !(nn >= 0.5 * N);
      s2n = fmax(nn, 0.0);
    }
    double mine = 0.0;
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      if (cc > jj) {
        const double w = tj * (d[cc] + rrow[cc]);
#pragma unroll
        for (int i = 0; i < 4; ++i) xr[i][cc] = fma(-w, xr[i][jj], xr[i][cc]);
        mine = (lane == cc) ? rrow[cc] - w : mine;
      } else if (cc < jj) {
        mine = (lane == cc) ? d[cc] : mine;      // G[j0+cc][j] in the lower part
      } else {
        mine = (lane == cc) ? beta : mine;
      }
    }
    if (lane < 8) S[j * KT + j0 + lane] = mine;
    // T_p[ii][jj] = -tau sum_{l=ii}^{jj-1} T_p[ii][l] G[l][jj]  (lane ii < 8)
    double sacc = 0.0;
#pragma unroll
    for (int l = 0; l < jj; ++l) sacc = fma((l >= lr) ? trow[l] : 0.0, d[l], sacc);
    trow[jj] = (lr == jj) ? tj : ((lr < jj) ? -tj * sacc : 0.0);
    if (lane == jj) tau_s[j] = tj;
  }
  if (lane < 8) {
#pragma unroll
    for (int l = 0; l < 8; ++l) T8[lane * 8 + l] = trow[l];
  }
  return bad;
}

// Gram-form panel sweep (the fast path).  The 8 Householder steps of the
// structured panel QR([R_pp; X_p]) only need, per step jj, the norm of the
// current tile column x_jj and its dots with the later columns; all of them
// follow from the panel Gram M = X_p^T X_p by exact rank-2 algebra:
//   y_jj = scal x_jj,  x_b <- x_b - w_b y_jj  (b > jj),  w_b = tau (R_jb + y_jj.x_b)
//   M[a][b] -= w_a c_b + w_b c_a          (jj < a <= b),  c_b = u_b - w_b yy/2
//   M[a][b] -= w_b G[a][jj]               (a < jj < b),   G[a][jj] = scal M[a][jj]
// with u_b = scal M[jj][b], yy = |y_jj|^2.  M comes from 32 DMMAs on the
// quad-layout registers (no reduction tree), the 8 steps are uniform scalar
// work in every lane (no shuffles on the step chain), and Y is formed
// afterwards from the stored w / scal with the same FMAs as the exact sweep.
// Accuracy: M's rounding is absolute in the panel-start norms, so every
// pivot must keep at least half of its panel-start norm^2 (else the caller
// replays the panel with the exact per-column reductions of panel_core<KT,true>).
#define PANEL_SCAL(jj) ((jj) == 0 ? 56 : (jj) * 9 - 1)   // strict-lower slot of scr for scal_jj

template <int KT>
__device__ __forceinline__ bool panel_gram(int p, const double (&x)[16][2], double* S, double* T8,
                                           double* tau_s, double* scr) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int j0 = p * 8;
  const int lr = lane < 8 ? lane : 7;
  {
    double acc[4][2];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
    for (int f = 0; f < 16; ++f)
#pragma unroll
      for (int h = 0; h < 2; ++h) dmma(acc[(2 * f + h) & 3], x[f][h], x[f][h]);
    scr[g * 8 + 2 * t] = (acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]);
    scr[g * 8 + 2 * t + 1] = (acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]);
  }
  __syncwarp();
  double m[8][8];   // upper triangle used (compile-time indices after unrolling)
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; b += 2) {
      if (b + 1 < a) continue;
      const double2 v = *reinterpret_cast<const double2*>(scr + a * 8 + b);
      m[a][b] = v.x;
      m[a][b + 1] = v.y;
    }
  // scr keeps the panel-start diagonal M0[a][a] (at a*9) for the checks; the
  // strict upper part then takes w[jj][b], the slot SCAL(jj) in the strict
  // lower part scal_jj.  All lanes store the same uniform values (no branch
  // splits the step chain into basic blocks).
  __syncwarp();
  double trow[8];                     // lane ii < 8: row ii of T_p
#pragma unroll
  for (int l = 0; l < 8; ++l) trow[l] = 0.0;
  bool bad = false;
  double rnext[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) rnext[b] = S[j0 * KT + j0 + b];
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int j = j0 + jj;
    double rrow[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) rrow[b] = rnext[b];
    if (jj + 1 < 8) {                 // prefetch R row j+1 (not written by this panel yet)
#pragma unroll
      for (int b = 0; b < 8; ++b) rnext[b] = (b > jj) ? S[(j + 1) * KT + j0 + b] : 0.0;
    }
    const double s2 = m[jj][jj];
    bad = bad || !(s2 >= 0.5 * scr[jj * 9]);
    double beta, tj, scal;
    dlarfg_nb(rrow[jj], s2, beta, tj, scal);
    const double yy = scal * scal * s2;
    double w[8], c[8], gcol[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      w[b] = c[b] = gcol[b] = 0.0;
      if (b > jj) {
        const double u = scal * m[jj][b];
        w[b] = tj * (rrow[b] + u);
        c[b] = fma(-0.5 * w[b], yy, u);
      } else if (b < jj) {
        gcol[b] = scal * m[b][jj];    // G[b][jj] = y_b . y_jj
      }
    }
#pragma unroll
    for (int b = jj + 1; b < 8; ++b) {
#pragma unroll
      for (int a = 0; a < jj; ++a) m[a][b] = fma(-w[b], gcol[a], m[a][b]);
      m[jj][b] = fma(-0.5 * w[b], yy, c[b]);
#pragma unroll
      for (int a = jj + 1; a <= b; ++a) m[a][b] = fma(-w[a], c[b], fma(-w[b], c[a], m[a][b]));
    }
    // outputs: S row j (G | beta | R - w), tau, T_p row per lane, w / scal
#pragma unroll
    for (int b = 0; b < 8; b += 2) {
      const double v0 = b < jj ? gcol[b] : (b == jj ? beta : rrow[b] - w[b]);
      const double v1 = b + 1 < jj ? gcol[b + 1] : (b + 1 == jj ? beta : rrow[b + 1] - w[b + 1]);
      *reinterpret_cast<double2*>(S + j * KT + j0 + b) = make_double2(v0, v1);
    }
    tau_s[j] = tj;
#pragma unroll
    for (int b = jj + 1; b < 8; ++b) scr[jj * 8 + b] = w[b];
    scr[PANEL_SCAL(jj)] = scal;
    double sacc = 0.0;
#pragma unroll
    for (int l = 0; l < jj; ++l) sacc = fma((l >= lr) ? trow[l] : 0.0, gcol[l], sacc);
    trow[jj] = (lr == jj) ? tj : ((lr < jj) ? -tj * sacc : 0.0);
  }
  if (lane < 8) {
#pragma unroll
    for (int l = 0; l < 8; ++l) T8[lane * 8 + l] = trow[l];
  }
  __syncwarp();
  return bad;
}

// Y_p from the stored w / scal (lane-per-row layout): y_jj = scal_jj x_jj,
// x_b -= w_b y_jj -- the same FMAs, in the same order, as the exact sweep.
__device__ __forceinline__ void panel_form_y(double (&xr)[4][8], const double* scr) {
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const double sc = scr[PANEL_SCAL(jj)];
#pragma unroll
    for (int i = 0; i < 4; ++i) xr[i][jj] *= sc;
#pragma unroll
    for (int b = jj + 1; b < 8; ++b) {
      const double w = scr[jj * 8 + b];
#pragma unroll
      for (int i = 0; i < 4; ++i) xr[i][b] = fma(-w, xr[i][jj], xr[i][b]);
    }
  }
}

// Panel factorization by the owning warp.  The panel is transposed through
// its Y slot into the lane-per-row layout so that v stays lane-local and the
// 7 dot products of a step are one reduce-scatter over the warp; the
// Householder vectors go back to the slot (published Y_p) and to the quad
// layout of the registers.
template <int KT>
__device__ __forceinline__ void panel_factor(int p, double (&x)[16][2], double* S, double* Ys,
                                             double* Tp, double* tau_s, double* save, double* gscr) {
  constexpr int YS = BlkCfg<KT>::YS;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int j0 = p * 8;
#ifdef OTS_TIMING
  long long pq = clock64();
#define PMARK(slot) { long long _t = clock64(); if (lane == 0) atomicAdd(&g_dbg[slot], (unsigned long long)(_t - pq)); pq = _t; }
#else
#define PMARK(slot)
#endif
#pragma unroll
  for (int f = 0; f < 16; ++f)
#pragma unroll
    for (int h = 0; h < 2; ++h) Ys[(8 * f + 2 * t + h) * YS + g] = x[f][h];
  // R rows of the panel (8 x 8 block) for a replay
  save[lane] = S[(j0 + (lane >> 3)) * KT + j0 + (lane & 7)];
  save[lane + 32] = S[(j0 + 4 + (lane >> 3)) * KT + j0 + (lane & 7)];
  __syncwarp();
  PMARK(8);
  double* T8 = Tp + p * 64;
#ifdef OTS_PANEL_EXACT
  double xr[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 8; c += 2) {
      const double2 u = *reinterpret_cast<const double2*>(Ys + (lane + 32 * i) * YS + c);
      xr[i][c] = u.x;
      xr[i][c + 1] = u.y;
    }
  const bool bad = panel_core<KT, false>(p, xr, S, T8, tau_s);
#else
  const bool bad = panel_gram<KT>(p, x, S, T8, tau_s, gscr);
  double xr[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 8; c += 2) {
      const double2 u = *reinterpret_cast<const double2*>(Ys + (lane + 32 * i) * YS + c);
      xr[i][c] = u.x;
      xr[i][c + 1] = u.y;
    }
  if (!bad) panel_form_y(xr, gscr);
#endif
  PMARK(9);
  if (__any_sync(0xffffffffu, bad)) {   // rare: replay with exact per-column reductions
    __syncwarp();
    S[(j0 + (lane >> 3)) * KT + j0 + (lane & 7)] = save[lane];
    S[(j0 + 4 + (lane >> 3)) * KT + j0 + (lane & 7)] = save[lane + 32];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < 8; c += 2) {
        const double2 u = *reinterpret_cast<const double2*>(Ys + (lane + 32 * i) * YS + c);
        xr[i][c] = u.x;
        xr[i][c + 1] = u.y;
      }
    __syncwarp();
    panel_core<KT, true>(p, xr, S, T8, tau_s);
  }
  __syncwarp();
  // Y_p -> slot (published) -> quad-layout registers
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 8; c += 2)
      *reinterpret_cast<double2*>(Ys + (lane + 32 * i) * YS + c) = make_double2(xr[i][c], xr[i][c + 1]);
  __syncwarp();
#pragma unroll
  for (int f = 0; f < 16; ++f)
#pragma unroll
    for (int h = 0; h < 2; ++h) x[f][h] = Ys[(8 * f + 2 * t + h) * YS + g];
  PMARK(12);
#undef PMARK
}

// warp w applies panel p to its register columns (w > p) or records the
// Gram block G[w cols][p cols] (w < p)
template <int KT>
__device__ __forceinline__ void panel_apply(int p, int w, double (&x)[16][2], double* S, const double* Ys,
                                            const double* Tp) {
  constexpr int YS = BlkCfg<KT>::YS;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int j0 = p * 8, c0 = w * 8;
  double acc[4][2];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = 0.0;
  // k index kk <-> tile row 8(kk>>1) + 2t + (kk&1): A = own registers
#pragma unroll
  for (int kk = 0; kk < 32; ++kk) {
    const int r = 8 * (kk >> 1) + 2 * t + (kk & 1);
    dmma(acc[kk & 3], x[kk >> 1][kk & 1], Ys[r * YS + g]);
  }
  double W0 = (acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]);
  double W1 = (acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]);
  // W^T[c0+g][j0+2t+h]
  double* r0p = S + (j0 + 2 * t) * KT + c0 + g;
  double* r1p = r0p + KT;
  if (w < p) { *r0p = W0; *r1p = W1; return; }
  W0 += *r0p;
  W1 += *r1p;
  // A operand W^T[g][k] for k = t and k = t+4 (lane quad holds k = 2t, 2t+1)
  auto regather = [&](double e0, double e1, double& lo, double& hi) {
    const int sl = 4 * g + (t >> 1), sh = sl + 2;
    const double l0 = __shfl_sync(0xffffffffu, e0, sl), l1 = __shfl_sync(0xffffffffu, e1, sl);
    const double h0 = __shfl_sync(0xffffffffu, e0, sh), h1 = __shfl_sync(0xffffffffu, e1, sh);
    lo = (t & 1) ? l1 : l0;
    hi = (t & 1) ? h1 : h0;
  };
  double alo, ahi;
  regather(W0, W1, alo, ahi);
  double o[2] = {0.0, 0.0};          // w^T[c0+g][j0+2t+h] = (W^T T_p)
  dmma(o, alo, Tp[p * 64 + t * 8 + g]);
  dmma(o, ahi, Tp[p * 64 + (t + 4) * 8 + g]);
  *r0p -= o[0];
  *r1p -= o[1];
  regather(-o[0], -o[1], alo, ahi);
  // X^T[c0+g][8f + n] -= sum_k w^T[g][k] Y[8f + n][j0 + k]
#pragma unroll
  for (int f = 0; f < 16; ++f) {
    dmma(x[f], alo, Ys[(8 * f + g) * YS + t]);
    dmma(x[f], ahi, Ys[(8 * f + g) * YS + 4 + t]);
  }
}

// T of a tile from tau (diag) and G (lower part of S), blockwise with DMMA:
//   T[q][p] = -(sum_{q'=q}^{p-1} T[q][q'] G[q'][p]) T_pp      (q < p)
// One warp per row block q.  The diagonal blocks are the panels' T_pp (Tpv);
// the off-diagonal ones are packed 8x8 blocks in Tw.  Phase p of tile t only
// reads G row block p, which tile t+1 overwrites after its panel-p barrier,
// so the phases of tile t run on the warps q < p that are idle while tile
// t+1's panel p is factored (off the chain's critical path).
__device__ __forceinline__ int tw_off(int q, int p) { return ((p * (p - 1)) / 2 + q) * 64; }

template <int KT>
__device__ __forceinline__ void t_block(int q, int p, const double* S, const double* Tpv, double* Tw,
                                        double* sc) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double m[2] = {0.0, 0.0};
  for (int qq = q; qq < p; ++qq) {
    const double* Tq = (qq == q) ? Tpv + q * 64 : Tw + tw_off(q, qq);
#pragma unroll
    for (int k0 = 0; k0 < 8; k0 += 4) dmma(m, Tq[g * 8 + k0 + t], S[(8 * p + g) * KT + 8 * qq + k0 + t]);
  }
  sc[g * 8 + 2 * t] = m[0];
  sc[g * 8 + 2 * t + 1] = m[1];
  __syncwarp();
  double o[2] = {0.0, 0.0};
#pragma unroll
  for (int k0 = 0; k0 < 8; k0 += 4) dmma(o, sc[g * 8 + k0 + t], Tpv[p * 64 + (k0 + t) * 8 + g]);
  double* dst = Tw + tw_off(q, p) + g * 8 + 2 * t;
  dst[0] = -o[0];
  dst[1] = -o[1];
  __syncwarp();
}

// T (upper block triangular) -> global.  Only the blocks on and above the
// diagonal are written: the Q-formation reads T as upper triangular.
template <int KT>
__device__ __forceinline__ void t_store(const double* Tpv, const double* Tw, double* Tg) {
  constexpr int NP = KT / 8;
  for (int e = threadIdx.x; e < (NP * (NP + 1) / 2) * 32; e += 256) {   // 2 doubles per unit
    const int blk = e >> 5, u = e & 31;
    int pj = 0;
    while ((pj + 1) * (pj + 2) / 2 <= blk) ++pj;                  // block column
    const int qi = blk - pj * (pj + 1) / 2;                       // block row (<= pj)
    const int r = (u >> 2), c = (u & 3) * 2;
    const double* src = qi == pj ? Tpv + qi * 64 : Tw + tw_off(qi, pj);
    *reinterpret_cast<double2*>(Tg + (8 * qi + r) * KT + 8 * pj + c) =
        *reinterpret_cast<const double2*>(src + r * 8 + c);
  }
}

// REDO: level-0 redo of the chains the Gram-form factor flagged (gsweep.inc;
// flag = Rout[chain][KT-1][0] != 0, an entry a chain R leaves 0).  A separate
// instantiation: the default one is unchanged (ptxas allocation).
template <int KT, bool REDO = false>
__global__ void __launch_bounds__(256, 2) chain_factor_kernel(FactorArgs a) {
  using C = BlkCfg<KT>;
  if constexpr (REDO) {
    if (a.Rout[((long)blockIdx.x * KT + KT - 1) * KT] == 0.0) return;
  }
  constexpr int NP = C::NP;
  extern __shared__ __align__(128) double S[];   // R (KT x KT), G in its lower part
  double* Xs = S + KT * KT;                       // tile (swizzled) | head U/T
  double* Tp = Xs + C::XS;                        // 2 x NP x 64: panel T_pp, by tile parity
  double* scr = Tp + 2 * NP * 64;                 // 8 warps x 64
  double* Tw = Xs + C::TWOFF;                     // packed off-diagonal T blocks (previous tile)
  __shared__ double tau_s[KT];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int chain = blockIdx.x;
  const long r0 = (long)chain * a.G.rpc;
  const int ntiles = chain_real_tiles(a.G, chain, KT);
  double* Tbase = a.U + (long)chain * (a.G.L + 1) * KT * KT;
  const int b = a.G.b;

  // ---- head: plain QR of rows [r0, r0+KT) (unblocked smem sweep, once per chain)
  load_rows_plain<KT, KT>(S, 0, a.D, a.ldd, r0, KT, a.G.nrows, a.ncols, tid, 256);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  if (a.head_tri) {
    // Tree levels: the head is an R factor (exact zeros below the diagonal),
    // so every dlarfg sees |x| = 0: tau = 0, beta = alpha (LAPACK's shortcut),
    // R = head, Y = 0, T = 0 -- the unblocked sweep would compute exactly that.
    for (int e = tid; e < KT * KT; e += 256) Tbase[e] = 0.0;
  } else {
    householder_sweep<KT, true, KT>(S, 0, Xs, tau_s);   // U -> Xs (ld KT+1)
    store_rows_plain<KT, KT>(S, 0, a.D, a.ldd, r0, KT, a.G.nrows, a.ncols, tid, 256);
    __syncthreads();
    u_to_t_block<KT>(Xs, Xs + KT * (KT + 1), Tbase);
    __syncthreads();
  }

  // ---- structured tiles (register-resident, see BlkCfg)
  const bool owner = warp < NP;
  const int mycol = 8 * warp + ((tid & 31) >> 2);
  double* Ys = Xs;                                  // NSLOT panel slots of Y
  double x[16][2];
  if (owner && ntiles > 0) {
    const long g0 = r0 + KT;
    const long rem0 = a.G.nrows - g0;
    tile_regs_load(x, a.D, a.ldd, g0, (int)(rem0 < b ? rem0 : b), mycol, a.ncols);
  }
  for (int t = 1; t <= ntiles; ++t) {
    double* Tpc = Tp + (t & 1) * NP * 64;           // this tile's T_pp
    const double* Tpp = Tp + ((t - 1) & 1) * NP * 64;   // previous tile's (its T is built now)
    const long gr0 = r0 + KT + (long)(t - 1) * b;
    const long rem = a.G.nrows - gr0;
    const int nb = (int)(rem < b ? rem : b);
    TSTAMP(t1);
    if (t < ntiles) {   // next tile -> L2 while this one is factored (its load is on the chain)
      const long g1 = gr0 + b;
      const long rem1 = a.G.nrows - g1;
      const int nb1 = (int)(rem1 < b ? rem1 : b);
      const int lpr = (a.ncols * 8 + 127) / 128;          // 128-byte lines per row
      for (int i = tid; i < nb1 * lpr; i += 256) {
        const int r = i / lpr, l = i - r * lpr;
        const double* ptr = a.D + (g1 + r) * a.ldd + l * 16;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
      }
    }
    // The owner of the next panel (p+1) shares its SM sub-partition with warp
    // (p+1)^4; that warp defers its DMMA apply of panel p by one iteration so
    // the latency-bound panel factorisation does not queue behind its DMMAs
    // on the shared FP64 pipe.  A 3-slot Y ring keeps Y_p alive for it.
    int pending = -1;
    for (int p = 0; p < NP; ++p) {
#ifdef OTS_TIMING
      long long q0 = clock64();
#endif
      if (warp == p) panel_factor<KT>(p, x, S, Ys + (p % C::NSLOT) * C::YSLOT, Tpc, tau_s, scr + warp * 64,
                                      Xs + C::NSLOT * C::YSLOT + warp * 64);
      else if (t > 1 && warp < p) t_block<KT>(warp, p, S, Tpp, Tw, scr + warp * 64);
#ifdef OTS_TIMING
      if (warp == p && (tid & 31) == 0) atomicAdd(&g_dbg[5], (unsigned long long)(clock64() - q0));
#endif
      __syncthreads();
#ifdef OTS_TIMING
      long long q1 = clock64();
#endif
      if (owner && warp != p) {
        const int defer_w = (p + 1 < NP) ? ((p + 1) ^ 4) : -1;
        if (pending >= 0) {
          panel_apply<KT>(pending, warp, x, S, Ys + (pending % C::NSLOT) * C::YSLOT, Tpc);
          pending = -1;
        }
        if (warp == defer_w) pending = p;
        else panel_apply<KT>(p, warp, x, S, Ys + (p % C::NSLOT) * C::YSLOT, Tpc);
      }
#ifdef OTS_TIMING
      if (warp == p + 1 && (tid & 31) == 0) atomicAdd(&g_dbg[6], (unsigned long long)(clock64() - q1));
      if (tid == 0) atomicAdd(&g_dbg[7], (unsigned long long)(clock64() - q0));
#endif
    }
    if (pending >= 0) panel_apply<KT>(pending, warp, x, S, Ys + (pending % C::NSLOT) * C::YSLOT, Tpc);
    __syncthreads();
    TSTAMP(t2);
    TACC(1, t1, t2);
    // Y (in place of the tile) -> global; next tile -> registers
    if (owner) {
      tile_regs_store(x, a.D, a.ldd, gr0, nb, mycol, a.ncols);
      if (t < ntiles) {
        const long g1 = gr0 + b;
        const long rem1 = a.G.nrows - g1;
        tile_regs_load(x, a.D, a.ldd, g1, (int)(rem1 < b ? rem1 : b), mycol, a.ncols);
      }
    }
    TSTAMP(t3);
    TACC(2, t2, t3);
    if (t > 1) {                    // previous tile's T is complete (phase NP-1 ran in panel NP-1)
      t_store<KT>(Tpp, Tw, Tbase + (long)(t - 1) * KT * KT);
      __syncthreads();              // Tpp is this parity's buffer for tile t+1
    }
    TSTAMP(t4);
    TACC(3, t3, t4);
    if (threadIdx.x == 0) TACC(4, 0, 1);
  }
  if (ntiles > 0) {                 // last tile: its T phases in sequence
    const double* Tpl = Tp + (ntiles & 1) * NP * 64;
    for (int p = 1; p < NP; ++p) {
      if (warp < p) t_block<KT>(warp, p, S, Tpl, Tw, scr + warp * 64);
      __syncthreads();
    }
    t_store<KT>(Tpl, Tw, Tbase + (long)ntiles * KT * KT);
  }

  // ---- chain R (upper triangle, exact zeros below)
  double* R = a.Rout + (long)chain * KT * KT;
  for (int i = tid; i < KT * KT; i += 256) {
    int r = i / KT, cc = i - r * KT;
    R[i] = (cc >= r) ? S[r * KT + cc] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Q formation (reverse chain walk).  Per structured tile (reverse order):
//   M = T C ; out_rows = -Y M ; C <- C - M
// Head:  W1 = Yt^T C ; M = T W1 ; out_rows(head) = C - Yt M   (Yt unit lower)
// ---------------------------------------------------------------------------

// ---------------------------------------------------------------------------
template <int KT>
static cudaError_t factor_t(const FactorArgs& a, cudaStream_t st) {
  using C = BlkCfg<KT>;
  if (a.G.b > C::B || a.G.nchains <= 0) return cudaErrorInvalidValue;
  if (a.head_tri == 2) {
    if constexpr (KT == 64) {
      FactorArgs b = a;
      b.head_tri = 0;
      auto k = chain_factor_kernel<KT, true>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
      k<<<a.G.nchains, 256, C::SMEM, st>>>(b);
    } else {
      return cudaErrorInvalidValue;
    }
  } else {
    auto k = chain_factor_kernel<KT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    k<<<a.G.nchains, 256, C::SMEM, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_chain_factor(const FactorArgs& a, int KT, cudaStream_t st) {
  if (KT == 16) return factor_t<16>(a, st);
  if (KT == 32) return factor_t<32>(a, st);
  if (KT == 64) return factor_t<64>(a, st);
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// Q formation, pipelined (v2): one 512-thread CTA per SM walks its chains;
// C, T, M = T C and a double-buffered whole Y tile live in shared memory
// (224 KB at KT = 64), so T and Y of tile t-1 stream in (cp.async) while tile
// t's out = -Y M runs on all 16 warps.
// ---------------------------------------------------------------------------
template <int KT>
struct Qform2Cfg {
  static constexpr int NT = 512;
  static constexpr int NW = NT / 32;
  static constexpr int B = BlkCfg<KT>::B;             // tile rows (>= any level's b)
  static constexpr int SMEM = (3 * KT * KT + 2 * B * KT) * 8;
};

// Ms = -(T C) (KT x KT) with T upper triangular; 16 warps: 8-row blocks x
// column splits.
template <int KT>
__device__ __forceinline__ void q2_tc(const double* Ts, const double* Cs, double* Ms) {
  constexpr int RB = KT / 8;              // row blocks
  constexpr int CB = KT / 8;              // 8-column blocks
  constexpr int CS = (16 / RB < CB) ? 16 / RB : CB;   // column splits per row block
  constexpr int CW = KT / CS;             // columns per warp (>= 8)
  constexpr int NJ = CW / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if (warp >= RB * CS) return;
  const int rb = warp / CS, c0 = (warp % CS) * CW;
  double acc[NJ][2];
#pragma unroll
  for (int j = 0; j < NJ; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll 4
  for (int kk = 2 * rb; kk < KT / 4; ++kk) {
    const double av = Ts[swz(8 * rb + g, 4 * kk + t, KT)];
#pragma unroll
    for (int j = 0; j < NJ; ++j) dmma(acc[j], av, Cs[swz(4 * kk + t, c0 + 8 * j + g, KT)]);
  }
#pragma unroll
  for (int j = 0; j < NJ; ++j) {   // store -M: the tall product then needs no negation
    Ms[swz(8 * rb + g, c0 + 8 * j + 2 * t, KT)] = -acc[j][0];
    Ms[swz(8 * rb + g, c0 + 8 * j + 2 * t + 1, KT)] = -acc[j][1];
  }
}

// out rows [y0, rhi) = Y Ms (Ms = -M); Y tile (B x KT) in smem; 16 warps as 4 row
// bands of 32 x 4 column quarters of KT/4.
template <int KT>
__device__ __forceinline__ void q2_ym(const double* Ys, const double* Ms, double* D, long ldd, int ncols, long y0,
                                      long rhi) {
  constexpr int B = Qform2Cfg<KT>::B;
  constexpr int WN = KT / 4;              // 16 / 8 / 4
  constexpr int NJ = WN >= 8 ? WN / 8 : 1;
  constexpr int NBANDS = B / 32;          // 4
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int band = warp / 4, wn0 = (warp % 4) * WN;
  if (band >= NBANDS || WN < 8) {
    if (WN >= 8) return;
  }
  if (WN < 8) {   // KT = 16: 4 warps per band would split 8-col fragments; use 2
    if ((warp % 4) >= 2) return;
  }
  constexpr int NJJ = WN >= 8 ? NJ : 1;
  const int c0 = WN >= 8 ? wn0 : (warp % 4) * 8;
  const int wm0 = band * 32;
  if (y0 + wm0 >= rhi) return;
  double o[4][NJJ][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJJ; ++j) o[i][j][0] = o[i][j][1] = 0.0;
#pragma unroll 4
  for (int kk = 0; kk < KT / 4; ++kk) {
    double af[4], bf[NJJ];
#pragma unroll
    for (int i = 0; i < 4; ++i) af[i] = Ys[swz(wm0 + 8 * i + g, 4 * kk + t, KT)];
#pragma unroll
    for (int j = 0; j < NJJ; ++j) bf[j] = Ms[swz(4 * kk + t, c0 + 8 * j + g, KT)];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NJJ; ++j) dmma(o[i][j], af[i], bf[j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJJ; ++j) {
      const long r = y0 + wm0 + 8 * i + g;
      const int cc = c0 + 8 * j + 2 * t;
      if (r >= rhi) continue;
      double* p = D + r * ldd + cc;
      if (cc + 1 < ncols) __stcs(reinterpret_cast<double2*>(p), make_double2(o[i][j][0], o[i][j][1]));
      else if (cc < ncols) p[0] = o[i][j][0];
    }
}

// Head rows [r0, r0 + KT) of a chain: out = C - Yt (T Yt^T) C with Yt the
// head's unit lower Householder block (smem, swizzled; its upper part is
// overwritten here), T in Ts; Ms is scratch.  Called by all threads.
template <int KT>
__device__ __forceinline__ void q2_head(double* Ts, double* Yt, double* Ms, const double* Cs, double* D, long ldd,
                                        int ncols, long r0, long nrows) {
  constexpr int NT = Qform2Cfg<KT>::NT;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  for (int e = tid; e < KT * KT; e += NT) {
    const int r = e / KT, cc = e - r * KT;
    if (cc >= r) Yt[swz(r, cc, KT)] = (cc == r) ? 1.0 : 0.0;
  }
  __syncthreads();
  // N = T Yt^T -> Ms (first 8 warps, row blocks), then M = N C -> Ts
  if (warp < KT / 8) {
    double acc[KT / 8][2];
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll 4
    for (int kk = 2 * warp; kk < KT / 4; ++kk) {
      const double av = Ts[swz(8 * warp + g, 4 * kk + t4, KT)];
#pragma unroll
      for (int j = 0; j < KT / 8; ++j) dmma(acc[j], av, Yt[swz(8 * j + g, 4 * kk + t4, KT)]);
    }
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) {
      Ms[swz(8 * warp + g, 8 * j + 2 * t4, KT)] = acc[j][0];
      Ms[swz(8 * warp + g, 8 * j + 2 * t4 + 1, KT)] = acc[j][1];
    }
  }
  __syncthreads();
  if (warp < KT / 8) {
    double acc[KT / 8][2];
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < KT / 4; ++kk) {
      const double av = Ms[swz(8 * warp + g, 4 * kk + t4, KT)];
#pragma unroll
      for (int j = 0; j < KT / 8; ++j) dmma(acc[j], av, Cs[swz(4 * kk + t4, 8 * j + g, KT)]);
    }
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) {
      Ts[swz(8 * warp + g, 8 * j + 2 * t4, KT)] = acc[j][0];
      Ts[swz(8 * warp + g, 8 * j + 2 * t4 + 1, KT)] = acc[j][1];
    }
  }
  __syncthreads();
  if (warp < KT / 8) {
    double acc[KT / 8][2];
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < KT / 4; ++kk) {
      const double av = Yt[swz(8 * warp + g, 4 * kk + t4, KT)];
#pragma unroll
      for (int j = 0; j < KT / 8; ++j) dmma(acc[j], av, Ts[swz(4 * kk + t4, 8 * j + g, KT)]);
    }
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) {
      const int r = 8 * warp + g, cc = 8 * j + 2 * t4;
      const long gr = r0 + r;
      if (gr >= nrows) continue;
      const double y0 = Cs[swz(r, cc, KT)] - acc[j][0];
      const double y1 = Cs[swz(r, cc + 1, KT)] - acc[j][1];
      double* p = D + gr * ldd + cc;
      if (cc + 1 < ncols) *reinterpret_cast<double2*>(p) = make_double2(y0, y1);
      else if (cc < ncols) p[0] = y0;
    }
  }
}

template <int KT>
__global__ void __launch_bounds__(512, 1) chain_qform2_kernel(QformArgs a) {
  using C = Qform2Cfg<KT>;
  constexpr int B = C::B;
  extern __shared__ __align__(128) double sm[];
  double* Cs = sm;
  double* Ts = Cs + KT * KT;
  double* Ms = Ts + KT * KT;
  double* Yb = Ms + KT * KT;          // 2 x (B x KT)
  const int tid = threadIdx.x;
  for (int chain = blockIdx.x; chain < a.G.nchains; chain += gridDim.x) {
    if (a.mode == 1 && !a.flags[chain]) continue;   // Gram-form level 0: accepted chain
    const long r0 = (long)chain * a.G.rpc;
    const int ntiles = chain_real_tiles(a.G, chain, KT);
    const double* Tbase = a.T + (long)chain * (a.tslots ? a.tslots : a.G.L + 1) * KT * KT;
    auto tile_rows = [&](int tt, long& gr0, long& rhi) {
      gr0 = r0 + KT + (long)(tt - 1) * a.G.b;
      rhi = gr0 + a.G.b < a.G.nrows ? gr0 + a.G.b : a.G.nrows;
    };
    auto issue_tile = [&](int tt, int buf) {   // T_tt and Y_tt (tt >= 1) or head (tt == 0)
      load_tile_async(Ts, KT, Tbase + (long)tt * KT * KT, KT, 0, KT, 0, KT, 0, KT, KT, tid, C::NT);
      if (tt >= 1) {
        long gr0, rhi;
        tile_rows(tt, gr0, rhi);
        load_tile_async(Yb + buf * B * KT, KT, a.D, a.ldd, gr0, B, gr0, rhi, 0, KT, a.ncols, tid, C::NT);
      } else {
        const long hhi = r0 + KT < a.G.nrows ? r0 + KT : a.G.nrows;
        load_tile_async(Yb + buf * B * KT, KT, a.D, a.ldd, r0, KT, r0, hhi, 0, KT, a.ncols, tid, C::NT);
      }
    };
    __syncthreads();   // previous chain done with all buffers
    load_tile_async(Cs, KT, a.Cin + (long)chain * KT * KT, KT, 0, KT, 0, KT, 0, KT, KT, tid, C::NT);
    issue_tile(ntiles, 0);
    cp_async_commit();
    int buf = 0;
    for (int tt = ntiles; tt >= 1; --tt) {
      cp_async_wait<0>();
      __syncthreads();
      q2_tc<KT>(Ts, Cs, Ms);                         // M = T C
      __syncthreads();
      issue_tile(tt - 1, buf ^ 1);                   // T, Y of the next (lower) tile
      cp_async_commit();
      for (int e = tid; e < KT * KT; e += C::NT) Cs[e] += Ms[e];   // C <- C - M (Ms = -M)
      long gr0, rhi;
      tile_rows(tt, gr0, rhi);
      q2_ym<KT>(Yb + buf * B * KT, Ms, a.D, a.ldd, a.ncols, gr0, rhi);
      buf ^= 1;
    }
    // ---- head: out = C - Yt (T Yt^T) C  (Yt unit lower)
    cp_async_wait<0>();
    __syncthreads();
    q2_head<KT>(Ts, Yb + buf * B * KT, Ms, Cs, a.D, a.ldd, a.ncols, r0, a.G.nrows);
  }
}

#include "gsweep.inc"

template <int KT>
static cudaError_t qform_t(const QformArgs& a, cudaStream_t st) {
  using C = Qform2Cfg<KT>;
  auto k = chain_qform2_kernel<KT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (a.grid_max > 0 && a.grid_max < nsm) nsm = a.grid_max;
  const int grid = a.G.nchains < nsm ? a.G.nchains : nsm;
  k<<<grid, C::NT, C::SMEM, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_chain_qform(const QformArgs& a, int KT, cudaStream_t st) {
  if (KT == 16) return qform_t<16>(a, st);
  if (KT == 32) return qform_t<32>(a, st);
  if (KT == 64) return qform_t<64>(a, st);
  return cudaErrorInvalidValue;
}

void debug_counters_small(unsigned long long* out, int reset);
int debug_counters(unsigned long long* out, int reset) {
#ifdef OTS_TIMING
  cudaMemcpyFromSymbol(out, g_dbg, sizeof(unsigned long long) * 16);
  debug_counters_small(out, reset);
  if (reset) { unsigned long long z[16] = {0}; cudaMemcpyToSymbol(g_dbg, z, sizeof z); }
  return 1;
#else
  for (int i = 0; i < 16; ++i) out[i] = 0;
  (void)reset;
  return 0;
#endif
}

int chain_bmax(int KT) {
  return KT == 16 ? FactorCfg<16>::BMAX : KT == 32 ? FactorCfg<32>::BMAX : FactorCfg<64>::BMAX;
}

}  // namespace ots
