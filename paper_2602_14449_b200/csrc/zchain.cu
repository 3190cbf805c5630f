// complex128 intra-block Householder QR (zgeqrf + zungqr semantics behind
// `householder_qr`, core.py:61-84, for complex input; twostage.py:93).
//
// Same flat-chain TSQR structure as the real path (chainqr.cu): a chain owns
// rows [c*RPC, (c+1)*RPC), a KT-row head is factored by a plain Householder
// QR, then L structured tiles QR([R; tile]) with reflectors v_j = [e_j; y_j];
// a tree over the chain R's; Q formed in reverse.  Reflectors follow zlarfg
// (beta real, tau complex) and are applied as H^H = I - conj(tau) v v^H, so
// Q = H_1 H_2 ... = I - V T V^H with the zlarft forward T.  Arithmetic is
// FP64 on CUDA cores (no complex tensor-core MMA exists); this path serves
// the complex configuration (BASELINE configs[3]), not the headline.
//
// Data: interleaved (re, im) row-major, leading dimensions in complex units.
#include "common.cuh"
#include "kernels.cuh"

namespace ots {

namespace {

typedef double2 cplx;
__device__ __forceinline__ cplx cmk(double r, double i) { return make_double2(r, i); }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cmk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return cmk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
// a * b + c
__device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx c) {
  return cmk(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// conj(a) * b + c
__device__ __forceinline__ cplx cfmac(cplx a, cplx b, cplx c) {
  return cmk(fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.x, b.y, fma(-a.y, b.x, c.y)));
}
__device__ __forceinline__ cplx conjc(cplx a) { return cmk(a.x, -a.y); }
__device__ __forceinline__ cplx cneg(cplx a) { return cmk(-a.x, -a.y); }
__device__ __forceinline__ cplx crecip(cplx b) {
  const double d = b.x * b.x + b.y * b.y;
  return cmk(b.x / d, -b.y / d);
}
__device__ __forceinline__ cplx cshfl_xor(unsigned mask, cplx v, int o) {
  return cmk(__shfl_xor_sync(mask, v.x, o), __shfl_xor_sync(mask, v.y, o));
}

#ifndef ZNT
#define ZNT 512
#endif

template <int KT>
struct ZCfg {
  static constexpr int NT = ZNT;       // factor threads per CTA
  static constexpr int B = 64;            // structured tile rows (BMAX)
  static constexpr int TPC = NT / KT;     // threads per column
  static constexpr int LDS = KT + 1;      // smem row stride (complex units)
  static constexpr int ROWS = KT + B;     // R rows + tile rows
  static constexpr int UL = KT + 1;
  static constexpr int SMEM = (ROWS * LDS + KT * UL + KT + 2 * B) * 16;
};

template <int TPC>
__device__ __forceinline__ double gsum(double v, unsigned mask) {
#pragma unroll
  for (int o = TPC / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}
template <int TPC>
__device__ __forceinline__ cplx gsumc(cplx v, unsigned mask) {
#pragma unroll
  for (int o = TPC / 2; o > 0; o >>= 1) v = cadd(v, cshfl_xor(mask, v, o));
  return v;
}

// rows [s0, s0+nr) of the smem block <- global rows [gr0, gr0+nr) (zero
// beyond nrows / ncols)
template <int KT>
__device__ void zload_rows(cplx* A, int s0, const cplx* D, long ldd, long gr0, int nr, long nrows, int ncols) {
  constexpr int LDS = ZCfg<KT>::LDS;
  for (int e = threadIdx.x; e < nr * KT; e += blockDim.x) {
    const int r = e / KT, c = e - r * KT;
    const long gr = gr0 + r;
    A[(s0 + r) * LDS + c] = (gr < nrows && c < ncols) ? D[gr * ldd + c] : cmk(0.0, 0.0);
  }
}
template <int KT>
__device__ void zstore_rows(const cplx* A, int s0, cplx* D, long ldd, long gr0, int nr, long nrows, int ncols) {
  constexpr int LDS = ZCfg<KT>::LDS;
  for (int e = threadIdx.x; e < nr * KT; e += blockDim.x) {
    const int r = e / KT, c = e - r * KT;
    const long gr = gr0 + r;
    if (gr < nrows && c < ncols) D[gr * ldd + c] = A[(s0 + r) * LDS + c];
  }
}

// One Householder sweep over the KT columns of the smem block A.
//  HEAD : plain QR of rows 0..KT-1 (reflector j spans rows j..KT-1)
//  !HEAD: rows 0..KT-1 hold R (upper, zero below), rows KT..KT+nb-1 the
//         tile; reflector j = [e_j; y_j] spans row j and the tile rows.
// U[c][j] = v_c^H v_j (c < j), U[j][j] = tau_j.
template <int KT, bool HEAD>
__device__ void zsweep(cplx* A, int nb, cplx* U, cplx* tau_s) {
  using C = ZCfg<KT>;
  constexpr int TPC = C::TPC, LDS = C::LDS, UL = C::UL;
  const int tid = threadIdx.x;
  const int c = tid / TPC, q = tid % TPC;
  const unsigned gmask = (TPC >= 32) ? 0xffffffffu : (((1u << TPC) - 1u) << ((tid & 31) & ~(TPC - 1)));
  auto rbeg = [&](int j) { return HEAD ? (j + 1 + q) : (KT + q); };
  const int rend = HEAD ? KT : (KT + nb);

  auto phase_a = [&](int j) {   // owners of column j: zlarfg
    double s2 = 0.0;
    for (int r = rbeg(j); r < rend; r += TPC) { const cplx x = A[r * LDS + j]; s2 = fma(x.x, x.x, fma(x.y, x.y, s2)); }
    s2 = gsum<TPC>(s2, gmask);
    const cplx alpha = A[j * LDS + j];
    cplx tau = cmk(0.0, 0.0);
    cplx beta = alpha;
    if (s2 != 0.0 || alpha.y != 0.0) {
      const double bt = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + s2), alpha.x);
      tau = cmk((bt - alpha.x) / bt, -alpha.y / bt);
      const cplx scal = crecip(csub(alpha, cmk(bt, 0.0)));
      for (int r = rbeg(j); r < rend; r += TPC) A[r * LDS + j] = cmul(A[r * LDS + j], scal);
      beta = cmk(bt, 0.0);
    }
    if (q == 0) { A[j * LDS + j] = beta; tau_s[j] = tau; }
  };

  if (c == 0) phase_a(0);
  __syncthreads();
  for (int j = 0; j < KT; ++j) {
    const cplx tj = tau_s[j];
    if (c != j) {
      // d = sum over reflector rows of conj(v_r) a_c  (v_j = 1 at row j)
      cplx d = cmk(0.0, 0.0);
      for (int r = rbeg(j); r < rend; r += TPC) d = cfmac(A[r * LDS + j], A[r * LDS + c], d);
      d = gsumc<TPC>(d, gmask);
      if (c > j) {
        d = cadd(d, A[j * LDS + c]);
        const cplx w = cmul(conjc(tj), d);           // conj(tau) v^H a
        for (int r = rbeg(j); r < rend; r += TPC) A[r * LDS + c] = csub(A[r * LDS + c], cmul(w, A[r * LDS + j]));
        if (q == 0) A[j * LDS + c] = csub(A[j * LDS + c], w);
        if (c == j + 1) {
          __syncwarp(gmask);
          phase_a(j + 1);
        }
      } else {
        // d = v_j^H v_c over the tile rows; the head adds v_c[j] * 1
        // (v_c[j] = A[j][c]).  U[c][j] = v_c^H v_j = conj(d).
        if (HEAD) d = cadd(d, A[j * LDS + c]);
        if (q == 0) U[c * UL + j] = conjc(d);
      }
    } else {
      if (q == 0) U[j * UL + j] = tj;
    }
    __syncthreads();
  }
}

// next structured tile -> the smem tile buffer (cp.async, zero fill beyond
// nb rows / ncols columns)
template <int KT>
__device__ __forceinline__ void zprefetch_tile(cplx* buf, const cplx* D0, long ldd, long gr0, int nb, int ncols) {
  constexpr int LDS = ZCfg<KT>::LDS, B = ZCfg<KT>::B;
  for (int e = threadIdx.x; e < B * KT; e += blockDim.x) {
    const int r = e / KT, c = e - r * KT;
    const bool ok = r < nb && c < ncols;
    cp_async16(buf + r * LDS + c, ok ? (const void*)(D0 + (gr0 + r) * ldd + c) : (const void*)D0, ok ? 16 : 0);
  }
  cp_async_commit();
}

// Structured-tile sweep.  Rows 0..KT-1 of A hold R; the tile (landed in the
// buffer rows KT..KT+B-1 by cp.async, zero beyond nb) is moved to registers:
// thread (c, q) keeps rows q+TPC*i of column c, and the buffer then receives
// the next tile while this one is swept.  Each step reads the pivot reflector
// from a two-column slot ring; a column's final reflector goes from registers
// straight to global memory.  T (zlarft forward) is built one column behind
// the Gram entries by the groups left of the pivot, T[i][l] (l > i) kept in
// U's lower triangle (U[l][i]), tau_i on the diagonal, U[l][j] (l < j) = v_l^H v_j.
template <int KT>
__device__ void zsweep_tile(cplx* A, cplx* U, cplx* tau_s, cplx* slot, cplx* D, const cplx* D0, long ldd, long gr0,
                            int nb, int ncols, long nxt_gr0, int nxt_nb, cplx* Tg) {
  using C = ZCfg<KT>;
  constexpr int TPC = C::TPC, LDS = C::LDS, UL = C::UL, B = C::B, RPT = B / TPC;
  const int tid = threadIdx.x;
  const int c = tid / TPC, q = tid % TPC;
  cplx x[RPT];
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int i = 0; i < RPT; ++i) x[i] = A[(KT + q + TPC * i) * LDS + c];
  __syncthreads();
  if (nxt_nb > 0) zprefetch_tile<KT>(A + KT * LDS, D0, ldd, nxt_gr0, nxt_nb, ncols);

  // The whole warp holding column j runs zlarfg (warp-uniform: full-mask
  // shuffles, no divergence); only the group c == j commits.
  const int warp = tid >> 5;
  const int c_first = (warp * 32) / TPC;     // first column of this warp
  constexpr unsigned FULL = 0xffffffffu;
  auto phase_a = [&](int j, cplx alpha) {
    const bool own = (c == j);
    double s2a = 0.0, s2b = 0.0;
#pragma unroll
    for (int i = 0; i < RPT; i += 2) {
      s2a = fma(x[i].x, x[i].x, fma(x[i].y, x[i].y, s2a));
      if (i + 1 < RPT) s2b = fma(x[i + 1].x, x[i + 1].x, fma(x[i + 1].y, x[i + 1].y, s2b));
    }
    const double s2 = gsum<TPC>(s2a + s2b, FULL);
    const bool nz = (s2 != 0.0 || alpha.y != 0.0);
    // beta = -sign(Re alpha) sqrt(h) via one rsqrt (1/beta comes with it);
    // 1/|alpha - beta|^2 by the MUFU reciprocal seed and two Newton steps
    // (as dlarfg_fast in chainqr.cu: ~1 ulp, no IEEE division / sqrt paths)
    const double h = fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, s2));
    const double r = rsqrt(h);
    const double bt = -copysign(h * r, alpha.x);
    const double ib = -copysign(r, alpha.x);
    const double e = bt - alpha.x;
    const double m = fma(e, e, alpha.y * alpha.y);
    double im;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(im) : "d"(m));
    im = im * fma(-m, im, 2.0);
    im = im * fma(-m, im, 2.0);
    const cplx tau = nz ? cmk(e * ib, -alpha.y * ib) : cmk(0.0, 0.0);
    const cplx scal = cmk(-e * im, -alpha.y * im);     // conj(alpha - beta) / |alpha - beta|^2
    const cplx beta = nz ? cmk(bt, 0.0) : alpha;
    if (own) {
      cplx* sl = slot + (j & 1) * B;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        if (nz) x[i] = cmul(x[i], scal);
        const int row = q + TPC * i;
        sl[row] = x[i];
        if (row < nb && j < ncols) D[(gr0 + row) * ldd + j] = x[i];
      }
      if (q == 0) { A[j * LDS + j] = beta; tau_s[j] = tau; }
    }
  };
  auto t_col = [&](int jj) {    // T[c][jj] = -tau_jj sum_{l=c}^{jj-1} T[c][l] U[l][jj]  (groups c < jj)
    if (c_first >= jj) return;  // warp-uniform
    cplx sacc = cmk(0.0, 0.0);
    if (c < jj)
      for (int l = c + q; l < jj; l += TPC) sacc = cfma(U[l * UL + c], U[l * UL + jj], sacc);
    sacc = gsumc<TPC>(sacc, FULL);
    if (c < jj && q == 0) U[jj * UL + c] = cneg(cmul(tau_s[jj], sacc));
  };

  if (warp == 0) phase_a(0, A[c * LDS + c]);
  __syncthreads();
  for (int j = 0; j < KT; ++j) {
    const bool crit = (j + 1 < KT) && (((j + 1) * TPC) >> 5) == warp;
    const cplx alpha_n = crit ? A[c * LDS + c] : cmk(0.0, 0.0);
    const cplx tj = tau_s[j];
    const cplx* vj = slot + (j & 1) * B;
    cplx v[RPT];
    cplx d = cmk(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      v[i] = vj[q + TPC * i];
      d = cfmac(v[i], x[i], d);
    }
    d = gsumc<TPC>(d, FULL);
    if (c > j) {
      d = cadd(d, A[j * LDS + c]);
      const cplx w = cmul(conjc(tj), d);               // conj(tau) v^H a
#pragma unroll
      for (int i = 0; i < RPT; ++i) x[i] = csub(x[i], cmul(w, v[i]));
      if (q == 0) A[j * LDS + c] = csub(A[j * LDS + c], w);
    } else if (c < j) {
      if (q == 0) U[c * UL + j] = conjc(d);            // U[c][j] = v_c^H v_j
    } else {
      if (q == 0) U[j * UL + j] = tj;
    }
    if (j >= 2) t_col(j - 1);
    if (crit) phase_a(j + 1, alpha_n);
#ifndef OTS_Z_NOBAR        // timing probe only (wrong results): the per-step barrier's cost
    __syncthreads();
#else
    if ((j & 3) == 3) __syncthreads();
#endif
  }
  t_col(KT - 1);
  __syncthreads();
  for (int e = tid; e < KT * KT; e += blockDim.x) {
    const int r = e / KT, cc = e - r * KT;
    Tg[e] = cc > r ? U[cc * UL + r] : (cc == r ? U[r * UL + r] : cmk(0.0, 0.0));
  }
}

// T (zlarft forward, columnwise) from U; T -> global Tg (KT x KT, row-major)
template <int KT>
__device__ void zu_to_t(cplx* U, cplx* Tg) {
  constexpr int UL = ZCfg<KT>::UL;
  constexpr int G = ZCfg<KT>::NT / KT;   // threads per row of T (a power of two)
  // in place in U: column j of T over rows i < j uses T[i][l] (l < j, already
  // final in U's upper part; U[i][i] = tau_i = T[i][i]) and U[l][j] (column j
  // still holds Gram entries); G threads share each row's dot product and the
  // new column is written after a barrier.
  const int i = threadIdx.x / G, g = threadIdx.x % G;
  const unsigned gmask = (G >= 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  for (int j = 1; j < KT; ++j) {
    const cplx tj = U[j * UL + j];
    cplx s = cmk(0.0, 0.0);
    if (i < j)
      for (int l = i + g; l < j; l += G) s = cfma(U[i * UL + l], U[l * UL + j], s);
    s = gsumc<G>(s, gmask);
    __syncthreads();
    if (i < j && g == 0) U[i * UL + j] = cneg(cmul(tj, s));
    __syncthreads();
  }
  for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
    const int r = e / KT, c = e - r * KT;
    Tg[e] = (c >= r) ? U[r * UL + c] : cmk(0.0, 0.0);
  }
}

template <int KT>
__global__ void __launch_bounds__(ZNT, 1) zchain_factor_kernel(ZFactorArgs a) {
  using C = ZCfg<KT>;
  constexpr int LDS = C::LDS, UL = C::UL;
  extern __shared__ __align__(16) unsigned char zsm_raw[];
  cplx* A = reinterpret_cast<cplx*>(zsm_raw);
  cplx* U = A + C::ROWS * LDS;
  cplx* tau_s = U + KT * UL;
  const cplx* D0 = reinterpret_cast<const cplx*>(a.D);
  cplx* D = reinterpret_cast<cplx*>(a.D);
  const int chain = blockIdx.x;
  const long r0 = (long)chain * a.G.rpc;
  const int b = a.G.b;
  long rem0 = a.G.nrows - (r0 + KT);
  int ntiles = 0;
  if (rem0 > 0) { long t = (rem0 + b - 1) / b; ntiles = (int)(t < a.G.L ? t : a.G.L); }
  cplx* Tbase = reinterpret_cast<cplx*>(a.U) + (long)chain * (a.G.L + 1) * KT * KT;

  cplx* slot = tau_s + KT;
  auto tile_rows = [&](int t, long& g0) {
    g0 = r0 + KT + (long)(t - 1) * b;
    const long rem = a.G.nrows - g0;
    return (int)(rem < b ? rem : b);
  };
  if (ntiles >= 1) {   // tile 1 lands in the buffer while the head is factored
    long g1;
    const int nb1 = tile_rows(1, g1);
    zprefetch_tile<KT>(A + KT * LDS, D0, a.ldd, g1, nb1, a.ncols);
  }
  // head
  zload_rows<KT>(A, 0, D0, a.ldd, r0, KT, a.G.nrows, a.ncols);
  __syncthreads();
  zsweep<KT, true>(A, 0, U, tau_s);
  zstore_rows<KT>(A, 0, D, a.ldd, r0, KT, a.G.nrows, a.ncols);
  __syncthreads();
  zu_to_t<KT>(U, Tbase);
  // R region: zero the strictly lower part (the head's vectors are stored)
  for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
    const int i = e / KT, j = e - i * KT;
    if (j < i) A[i * LDS + j] = cmk(0.0, 0.0);
  }
  for (int t = 1; t <= ntiles; ++t) {
    long gr0, g2 = 0;
    const int nb = tile_rows(t, gr0);
    const int nb2 = t < ntiles ? tile_rows(t + 1, g2) : 0;
    zsweep_tile<KT>(A, U, tau_s, slot, D, D0, a.ldd, gr0, nb, a.ncols, g2, nb2, Tbase + (long)t * KT * KT);
  }
  __syncthreads();
  cplx* R = reinterpret_cast<cplx*>(a.Rout) + (long)chain * KT * KT;
  for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
    const int i = e / KT, j = e - i * KT;
    R[e] = (j >= i) ? A[i * LDS + j] : cmk(0.0, 0.0);
  }
}

// acc[i][jj] += sum_l As[tr+16i][l] Bs[l][tc+16jj]  (KT x KT smem operands,
// 256 threads as a 16 x 16 grid of (KT/16) x (KT/16) register tiles)
template <int KT>
__device__ __forceinline__ void zmm(const cplx* As, const cplx* Bs, cplx (&acc)[KT / 16][KT / 16], int tr, int tc) {
  constexpr int LDS = ZCfg<KT>::LDS, MT = KT / 16;
#pragma unroll 4
  for (int l = 0; l < KT; ++l) {
    cplx av[MT], bv[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) av[i] = As[(tr + 16 * i) * LDS + l];
#pragma unroll
    for (int jj = 0; jj < MT; ++jj) bv[jj] = Bs[l * LDS + tc + 16 * jj];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int jj = 0; jj < MT; ++jj) acc[i][jj] = cfma(av[i], bv[jj], acc[i][jj]);
  }
}

// Reverse chain walk: per structured tile (reverse)  M = T C, out = -Y M,
// C <- C - M;  head: W1 = Yh^H C, M = Th W1, out = C - Yh M.
template <int KT>
__global__ void __launch_bounds__(256, 1) zchain_qform_kernel(ZQformArgs a) {
  using C = ZCfg<KT>;
  constexpr int LDS = C::LDS;
  extern __shared__ __align__(16) unsigned char zsm_raw[];
  cplx* Cs = reinterpret_cast<cplx*>(zsm_raw);
  cplx* Ms = Cs + KT * LDS;
  cplx* Ys = Ms + KT * LDS;      // 32-row chunk
  cplx* D = reinterpret_cast<cplx*>(a.D);
  const int chain = blockIdx.x;
  const long r0 = (long)chain * a.G.rpc;
  const int b = a.G.b;
  long rem0 = a.G.nrows - (r0 + KT);
  int ntiles = 0;
  if (rem0 > 0) { long t = (rem0 + b - 1) / b; ntiles = (int)(t < a.G.L ? t : a.G.L); }
  const cplx* Tbase = reinterpret_cast<const cplx*>(a.T) + (long)chain * (a.G.L + 1) * KT * KT;
  const cplx* Cin = reinterpret_cast<const cplx*>(a.Cin) + (long)chain * KT * KT;
  for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
    const int i = e / KT, j = e - i * KT;
    Cs[i * LDS + j] = Cin[e];
  }
  __syncthreads();
  constexpr int MT = KT / 16;
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
  if constexpr (KT == 64) {
    // Two smem buffers alternate roles: B1 holds T_t, then M_t = T_t C; B2
    // receives Y_t by cp.async while T_t C is formed.  After out = -Y_t M_t,
    // T_{t-1} -> B1 and Y_{t-1} -> B2 are issued as separate groups.
    cplx* B1 = Ys;
    cplx* B2 = Ms;
    auto issue_t = [&](int t) {
      const cplx* Tt = Tbase + (long)t * KT * KT;
      for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
        const int i = e / KT, j = e - i * KT;
        cp_async16(B1 + i * LDS + j, Tt + e, 16);
      }
      cp_async_commit();
    };
    auto issue_y = [&](int t) {
      const long gr0 = r0 + KT + (long)(t - 1) * b;
      const long rem = a.G.nrows - gr0;
      const int nb = (int)(rem < b ? rem : b);
      for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
        const int r = e / KT, c = e - r * KT;
        const bool ok = r < nb && c < a.ncols;
        cp_async16(B2 + r * LDS + c, ok ? (const void*)(D + (gr0 + r) * a.ldd + c) : (const void*)D, ok ? 16 : 0);
      }
      cp_async_commit();
    };
    if (ntiles >= 1) { issue_t(ntiles); issue_y(ntiles); }
    for (int t = ntiles; t >= 1; --t) {
      const long gr0 = r0 + KT + (long)(t - 1) * b;
      const long rem = a.G.nrows - gr0;
      const int nb = (int)(rem < b ? rem : b);
      cp_async_wait<1>();            // T_t landed (Y_t may still be in flight)
      __syncthreads();
      cplx acc[MT][MT];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int jj = 0; jj < MT; ++jj) acc[i][jj] = cmk(0.0, 0.0);
      zmm<KT>(B1, Cs, acc, tr, tc);   // M = T C
      __syncthreads();
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int jj = 0; jj < MT; ++jj) {
          const int o = (tr + 16 * i) * LDS + tc + 16 * jj;
          B1[o] = acc[i][jj];
          Cs[o] = csub(Cs[o], acc[i][jj]);
        }
      cp_async_wait<0>();            // Y_t
      __syncthreads();
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int jj = 0; jj < MT; ++jj) acc[i][jj] = cmk(0.0, 0.0);
      zmm<KT>(B2, B1, acc, tr, tc);   // Y M
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int jj = 0; jj < MT; ++jj) {
          const int r = tr + 16 * i, c = tc + 16 * jj;
          if (r < nb && c < a.ncols) D[(gr0 + r) * a.ldd + c] = cneg(acc[i][jj]);
        }
      __syncthreads();
      if (t > 1) { issue_t(t - 1); issue_y(t - 1); }
    }
  } else
  for (int t = ntiles; t >= 1; --t) {
    const long gr0 = r0 + KT + (long)(t - 1) * b;
    const long rem = a.G.nrows - gr0;
    const int nb = (int)(rem < b ? rem : b);
    const cplx* Tt = Tbase + (long)t * KT * KT;
    for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
      const int i = e / KT, j = e - i * KT;
      Ys[i * LDS + j] = Tt[e];
    }
    __syncthreads();
    {   // M = T C
      cplx acc[MT][MT];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int jj = 0; jj < MT; ++jj) acc[i][jj] = cmk(0.0, 0.0);
      zmm<KT>(Ys, Cs, acc, tr, tc);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int jj = 0; jj < MT; ++jj) Ms[(tr + 16 * i) * LDS + tc + 16 * jj] = acc[i][jj];
    }
    __syncthreads();
    for (int c0 = 0; c0 < nb; c0 += KT) {   // out = -Y M, KT rows at a time
      const int nr = (nb - c0 < KT) ? nb - c0 : KT;
      for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
        const int r = e / KT, c = e - r * KT;
        Ys[r * LDS + c] = (r < nr && c < a.ncols) ? D[(gr0 + c0 + r) * a.ldd + c] : cmk(0.0, 0.0);
      }
      __syncthreads();
      cplx acc[MT][MT];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int jj = 0; jj < MT; ++jj) acc[i][jj] = cmk(0.0, 0.0);
      zmm<KT>(Ys, Ms, acc, tr, tc);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int jj = 0; jj < MT; ++jj) {
          const int r = tr + 16 * i, c = tc + 16 * jj;
          if (r < nr && c < a.ncols) D[(gr0 + c0 + r) * a.ldd + c] = cneg(acc[i][jj]);
        }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
      const int i = e / KT, j = e - i * KT;
      Cs[i * LDS + j] = csub(Cs[i * LDS + j], Ms[i * LDS + j]);
    }
    __syncthreads();
  }
  // head rows [r0, r0+KT): Yh unit lower (strictly lower part of the stored head)
  const int hn = (int)((a.G.nrows - r0) < KT ? (a.G.nrows - r0) : KT);
  for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
    const int r = e / KT, c = e - r * KT;
    cplx y = cmk(0.0, 0.0);
    if (c < r && r < hn && c < a.ncols) y = D[(r0 + r) * a.ldd + c];
    if (c == r) y = cmk(1.0, 0.0);
    Ys[r * LDS + c] = y;   // Ys holds KT rows here (C::QSMEM sized for it below)
  }
  __syncthreads();
  // W1 = Yh^H C -> Ms
  for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
    const int i = e / KT, j = e - i * KT;
    cplx s = cmk(0.0, 0.0);
    for (int r = i; r < KT; ++r) s = cfmac(Ys[r * LDS + i], Cs[r * LDS + j], s);
    Ms[i * LDS + j] = s;
  }
  __syncthreads();
  // M = Th W1 -> reuse: out = C - Yh (Th W1); compute N = Th W1 into registers per entry then store into Ms
  {
    const cplx* Th = Tbase;
    cplx vals[KT * KT / 256 + 1];
    int cnt = 0;
    for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
      const int i = e / KT, j = e - i * KT;
      cplx s = cmk(0.0, 0.0);
      for (int l = i; l < KT; ++l) s = cfma(Th[i * KT + l], Ms[l * LDS + j], s);
      vals[cnt++] = s;
    }
    __syncthreads();
    cnt = 0;
    for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
      const int i = e / KT, j = e - i * KT;
      Ms[i * LDS + j] = vals[cnt++];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < hn * KT; e += blockDim.x) {
    const int r = e / KT, c = e - r * KT;
    cplx s = Cs[r * LDS + c];
    for (int l = 0; l <= r; ++l) s = csub(s, cmul(Ys[r * LDS + l], Ms[l * LDS + c]));
    if (c < a.ncols) D[(r0 + r) * a.ldd + c] = s;
  }
}

template <int KT>
cudaError_t zfactor_t(const ZFactorArgs& a, cudaStream_t st) {
  using C = ZCfg<KT>;
  if (a.G.b > C::B || a.G.nchains <= 0) return cudaErrorInvalidValue;
  auto k = zchain_factor_kernel<KT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  k<<<a.G.nchains, C::NT, C::SMEM, st>>>(a);
  return cudaGetLastError();
}
template <int KT>
cudaError_t zqform_t(const ZQformArgs& a, cudaStream_t st) {
  using C = ZCfg<KT>;
  constexpr int SM = (2 * KT * C::LDS + (KT > 32 ? KT : 32) * C::LDS) * 16;
  auto k = zchain_qform_kernel<KT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
  k<<<a.G.nchains, 256, SM, st>>>(a);
  return cudaGetLastError();
}


// ===========================================================================
// Gram-form complex tile factorization on tall tiles (KT = 64): the complex
// twin of gsweep.inc.  With alpha = R_jj real at every structured step (the
// head's and every earlier tile's diagonal is a zlarfg beta), tau_j, scal_j
// and beta_j are REAL, H_j is Hermitian, and the real identities carry over
// with conjugates on the row factors:
//   u_c = scal M[j][c],  w_c = tau (R[j][c] + u_c),  c_c = u_c - w_c yy/2,
//   M[a][b] -= conj(w_a) c_b + conj(c_a) w_b                   (a, b > j)
//   P[j][c] = u_c - w_c yy,  P[a][c] -= G[a][j] w_c,  G[a][j] = scal P[a][j]  (a < j)
//   T = D_tau (I + striu(G) D_tau)^-1,   Cc = D (I + W D)^-1,   Y = X Cc,
// where M = X^H X is recombined from the REAL Gram of the interleaved view
// (tgram_kernel's V^T V block over the 128 real columns).  Unblocked: with
// 4096-row tiles the sweep is a per-mille of the call.  A chain whose
// cancellation factor exceeds ZGS_RHO is flagged; the caller then takes the
// exact zchain_factor path for the whole call.
// ===========================================================================
#define ZGS_RHO 32.0

struct ZgsCfg {
  static constexpr int KT = 64, LDS = 65, NT = 256;
  static constexpr int SMEM = 3 * KT * LDS * 16 + (4 * KT) * 8 + (3 * KT) * 16 + 64;
};

// out (upper triangular, ld LDS) = Dg (I + S Dg)^-1, Dg = diag(dv) real, S strictly
// upper through an accessor:  out[i][j] = dv_j (delta_ij - sum_{l=i}^{j-1} out[i][l] S[l][j]).
// 4 lanes per row i; called by all 256 threads.
template <class SGet>
__device__ __forceinline__ void zgs_tri(cplx* out, const double* dv, SGet S) {
  constexpr int KT = ZgsCfg::KT, LDS = ZgsCfg::LDS;
  const int i = threadIdx.x >> 2, part = threadIdx.x & 3;
  for (int e = threadIdx.x; e < KT * KT; e += ZgsCfg::NT) out[(e >> 6) * LDS + (e & 63)] = cmk(0.0, 0.0);
  __syncthreads();
  for (int j = 0; j < KT; ++j) {
    cplx s = cmk(0.0, 0.0);
    if (i < j)
      for (int l = i + part; l < j; l += 4) s = cfma(out[i * LDS + l], S(l, j), s);
    s = gsumc<4>(s, 0xffffffffu);
    __syncthreads();
    if (part == 0) {
      if (i < j) out[i * LDS + j] = cmk(-dv[j] * s.x, -dv[j] * s.y);
      else if (i == j) out[i * LDS + j] = cmk(dv[j], 0.0);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256, 1) zgs_sweep_kernel(ZgsArgs a) {
  using C = ZgsCfg;
  constexpr int KT = C::KT, LDS = C::LDS;
  extern __shared__ __align__(16) unsigned char zsm_raw[];
  cplx* MP = reinterpret_cast<cplx*>(zsm_raw);      // M (unprocessed rows, upper) | P (processed rows) | G (processed cols)
  cplx* RW = MP + KT * LDS;                           // R (upper, diag = beta) | W^T (strictly lower)
  cplx* TB = RW + KT * LDS;                           // T, then Cc
  double* tau_v = reinterpret_cast<double*>(TB + KT * LDS);
  double* scal_v = tau_v + KT;
  double* yy_v = scal_v + KT;
  double* d0 = yy_v + KT;
  cplx* wv = reinterpret_cast<cplx*>(d0 + KT);
  cplx* cv = wv + KT;
  cplx* gv = cv + KT;
  int* flag = reinterpret_cast<int*>(gv + KT);
  const int tid = threadIdx.x;
  const int chain = blockIdx.x;
  const long r0 = (long)chain * a.G.rpc;
  long rem0 = a.G.nrows - (r0 + KT);
  int ntiles = 0;
  if (rem0 > 0) { long t = (rem0 + a.G.b - 1) / a.G.b; ntiles = (int)(t < a.G.L ? t : a.G.L); }
  const long tstride = (long)KT * KT;
  cplx* Tbase = reinterpret_cast<cplx*>(a.T) + (long)chain * (a.G.L + 1) * tstride;
  cplx* Cbase = reinterpret_cast<cplx*>(a.Cc) + (long)chain * (a.G.L + 1) * tstride;
  const cplx* Rh = reinterpret_cast<const cplx*>(a.Rh) + (long)chain * tstride;
  for (int e = tid; e < KT * KT; e += C::NT) {
    const int r = e >> 6, c = e & 63;
    RW[r * LDS + c] = (c >= r) ? Rh[e] : cmk(0.0, 0.0);
  }
  if (tid == 0) flag[0] = 0;
  __syncthreads();
  for (int t = 1; t <= ntiles; ++t) {
    // ---- M = X^H X from the real Gram of the interleaved view (ld 192)
    const double* Gr = a.TG + ((long)chain * a.G.L + t - 1) * a.tg_stride;
    for (int e = tid; e < KT * KT; e += C::NT) {
      const int j = e >> 6, l = e & 63;
      const double2 top = *reinterpret_cast<const double2*>(Gr + (long)(2 * j) * 192 + 2 * l);
      const double2 bot = *reinterpret_cast<const double2*>(Gr + (long)(2 * j + 1) * 192 + 2 * l);
      MP[j * LDS + l] = (l >= j) ? cmk(top.x + bot.y, top.y - bot.x) : cmk(0.0, 0.0);
    }
    __syncthreads();
    if (tid < KT) d0[tid] = sqrt(fmax(MP[tid * LDS + tid].x, 0.0));
    for (int j = 0; j < KT; ++j) {
      __syncthreads();
      // ---- step scalars (every thread, redundantly): real dlarfg on (alpha, s2)
      const double alpha = RW[j * LDS + j].x;
      const double s2 = fmax(MP[j * LDS + j].x, 0.0);
      double beta = alpha, tj = 0.0, scal = 0.0;
      if (s2 > 0.0) {
        beta = -copysign(sqrt(fma(alpha, alpha, s2)), alpha);
        tj = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      const double yy = scal * scal * s2;
      __syncthreads();                                // everyone has read alpha before R_jj becomes beta
      if (tid > j && tid < KT) {                      // trailing column c
        const int c = tid;
        const cplx m = MP[j * LDS + c];
        const cplx u = cmk(scal * m.x, scal * m.y);
        const cplx r = RW[j * LDS + c];
        const cplx w = cmk(tj * (r.x + u.x), tj * (r.y + u.y));
        RW[j * LDS + c] = csub(r, w);
        RW[c * LDS + j] = w;                          // W[j][c]
        wv[c] = w;
        cv[c] = cmk(fma(-0.5 * yy, w.x, u.x), fma(-0.5 * yy, w.y, u.y));
        MP[j * LDS + c] = cmk(fma(-yy, w.x, u.x), fma(-yy, w.y, u.y));   // P[j][c]
      } else if (tid == j) {
        RW[j * LDS + j] = cmk(beta, 0.0);
        tau_v[j] = tj;
        scal_v[j] = scal;
        yy_v[j] = yy;
      } else if (tid >= KT && tid < KT + j) {         // earlier row a: G[a][j]
        const int r = tid - KT;
        const cplx pj = MP[r * LDS + j];
        const cplx gg = cmk(scal * pj.x, scal * pj.y);
        MP[r * LDS + j] = gg;
        gv[r] = gg;
      }
      __syncthreads();
      // ---- rank-2 update of the trailing M and the processed rows' P
      for (int e = tid; e < KT * KT; e += C::NT) {
        const int r = e >> 6, c = e & 63;
        if (c <= j) continue;
        if (r > j) {
          if (r > c) continue;
          cplx m = MP[r * LDS + c];
          m = csub(m, cmul(conjc(wv[r]), cv[c]));
          m = csub(m, cmul(conjc(cv[r]), wv[c]));
          MP[r * LDS + c] = m;
        } else if (r < j) {
          MP[r * LDS + c] = csub(MP[r * LDS + c], cmul(gv[r], wv[c]));
        }
      }
    }
    __syncthreads();
    // ---- T = D_tau (I + striu(G) D_tau)^-1
    zgs_tri(TB, tau_v, [&](int l, int j) { return MP[l * LDS + j]; });
    {
      cplx* Tg = Tbase + (long)t * tstride;
      for (int e = tid; e < KT * KT; e += C::NT) Tg[e] = TB[(e >> 6) * LDS + (e & 63)];
    }
    __syncthreads();
    // ---- Cc = D (I + W D)^-1,  W[l][j] in RW's lower part
    zgs_tri(TB, scal_v, [&](int l, int j) { return RW[j * LDS + l]; });
    {
      cplx* Cg = Cbase + (long)t * tstride;
      for (int e = tid; e < KT * KT; e += C::NT) Cg[e] = TB[(e >> 6) * LDS + (e & 63)];
    }
    // ---- cancellation factor rho_j = sum_l |Cc[l][j]| d0[l] against |y_j|
    if (tid < KT) {
      const int j = tid;
      double rho = 0.0;
      for (int l = 0; l <= j; ++l) {
        const cplx x = TB[l * LDS + j];
        rho = fma(sqrt(x.x * x.x + x.y * x.y), d0[l], rho);
      }
      const bool ok = (tau_v[j] == 0.0) || (rho <= ZGS_RHO * sqrt(yy_v[j]));
      if (!ok) flag[0] = 1;
    }
    __syncthreads();
    if (flag[0]) {
      if (tid == 0) a.flags[chain] = 1;
      return;
    }
    // strictly lower part of RW (this tile's W) is cleared for the next tile
    for (int e = tid; e < KT * KT; e += C::NT) {
      const int r = e >> 6, c = e & 63;
      if (c < r) RW[r * LDS + c] = cmk(0.0, 0.0);
    }
    __syncthreads();
  }
  if (tid == 0) a.flags[chain] = 0;
  cplx* R = reinterpret_cast<cplx*>(a.Rout) + (long)chain * tstride;
  for (int e = tid; e < KT * KT; e += C::NT) {
    const int r = e >> 6, c = e & 63;
    R[e] = (c >= r) ? RW[r * LDS + c] : cmk(0.0, 0.0);
  }
}

// Coefficients of the accepted chains, in reverse chain order: M = T C,
// K = -Cc M, C <- C - M; K_t goes out as the 128 x 128 real right-multiplier
// of the interleaved view ([re, im] K = [re kr - im ki, re ki + im kr]), the
// chain's last C to Chead (the head rows' Q formation).
__global__ void __launch_bounds__(256, 1) zgs_coef_kernel(ZgsArgs a) {
  constexpr int KT = 64, LDS = ZCfg<64>::LDS, MT = KT / 16;
  extern __shared__ __align__(16) unsigned char zsm_raw[];
  cplx* Cs = reinterpret_cast<cplx*>(zsm_raw);
  cplx* B1 = Cs + KT * LDS;
  cplx* B2 = B1 + KT * LDS;
  const int tid = threadIdx.x, tr = tid / 16, tc = tid % 16;
  const int chain = blockIdx.x;
  const long r0 = (long)chain * a.G.rpc;
  long rem0 = a.G.nrows - (r0 + KT);
  int ntiles = 0;
  if (rem0 > 0) { long t = (rem0 + a.G.b - 1) / a.G.b; ntiles = (int)(t < a.G.L ? t : a.G.L); }
  const long tstride = (long)KT * KT;
  const cplx* Tbase = reinterpret_cast<const cplx*>(a.T) + (long)chain * (a.G.L + 1) * tstride;
  const cplx* Cbase = reinterpret_cast<const cplx*>(a.Cc) + (long)chain * (a.G.L + 1) * tstride;
  const cplx* Cin = reinterpret_cast<const cplx*>(a.Cin) + (long)chain * tstride;
  for (int e = tid; e < KT * KT; e += 256) Cs[(e >> 6) * LDS + (e & 63)] = Cin[e];
  for (int t = ntiles; t >= 1; --t) {
    __syncthreads();
    const cplx* Tt = Tbase + (long)t * tstride;
    const cplx* Ct = Cbase + (long)t * tstride;
    for (int e = tid; e < KT * KT; e += 256) {
      B1[(e >> 6) * LDS + (e & 63)] = Tt[e];
      B2[(e >> 6) * LDS + (e & 63)] = Ct[e];
    }
    __syncthreads();
    cplx acc[MT][MT];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int jj = 0; jj < MT; ++jj) acc[i][jj] = cmk(0.0, 0.0);
    zmm<KT>(B1, Cs, acc, tr, tc);                     // M = T C
    __syncthreads();
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int jj = 0; jj < MT; ++jj) {
        const int o = (tr + 16 * i) * LDS + tc + 16 * jj;
        B1[o] = acc[i][jj];
        Cs[o] = csub(Cs[o], acc[i][jj]);
        acc[i][jj] = cmk(0.0, 0.0);
      }
    __syncthreads();
    zmm<KT>(B2, B1, acc, tr, tc);                     // Cc M
    double* E = a.Kexp + ((long)chain * a.G.L + t - 1) * (4 * tstride);
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int jj = 0; jj < MT; ++jj) {
        const int ra = tr + 16 * i, cb = tc + 16 * jj;
        const double kr = -acc[i][jj].x, ki = -acc[i][jj].y;
        *reinterpret_cast<double2*>(E + (long)(2 * ra) * 128 + 2 * cb) = make_double2(kr, ki);
        *reinterpret_cast<double2*>(E + (long)(2 * ra + 1) * 128 + 2 * cb) = make_double2(-ki, kr);
      }
  }
  __syncthreads();
  cplx* Ch = reinterpret_cast<cplx*>(a.Chead) + (long)chain * tstride;
  for (int e = tid; e < KT * KT; e += 256) Ch[e] = Cs[(e >> 6) * LDS + (e & 63)];
}

// head rows of every chain <-> a side buffer (mode 0: save, 1: restore)
__global__ void zgs_heads_kernel(ZgsArgs a, double* D, long ldd, int mode) {
  const int chain = blockIdx.x;
  const long r0 = (long)chain * a.G.rpc;
  cplx* Dc = reinterpret_cast<cplx*>(D);
  cplx* S = reinterpret_cast<cplx*>(a.Hsave) + (long)chain * 64 * 64;
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
    const int r = e >> 6, c = e & 63;
    if (r0 + r >= a.G.nrows || c >= a.ncols) continue;
    if (mode == 0) S[e] = Dc[(r0 + r) * ldd + c];
    else Dc[(r0 + r) * ldd + c] = S[e];
  }
}

}  // namespace

cudaError_t launch_zgs_sweep(const ZgsArgs& a, cudaStream_t st) {
  cudaFuncSetAttribute(zgs_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ZgsCfg::SMEM);
  zgs_sweep_kernel<<<a.G.nchains, ZgsCfg::NT, ZgsCfg::SMEM, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_zgs_coef(const ZgsArgs& a, cudaStream_t st) {
  constexpr int SM = 3 * 64 * ZCfg<64>::LDS * 16;
  cudaFuncSetAttribute(zgs_coef_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
  zgs_coef_kernel<<<a.G.nchains, 256, SM, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_zgs_heads(const ZgsArgs& a, double* D, long ldd, int mode, cudaStream_t st) {
  zgs_heads_kernel<<<a.G.nchains, 256, 0, st>>>(a, D, ldd, mode);
  return cudaGetLastError();
}

int zchain_bmax() { return ZCfg<64>::B; }

cudaError_t launch_zchain_factor(const ZFactorArgs& a, int KT, cudaStream_t st) {
  if (KT == 16) return zfactor_t<16>(a, st);
  if (KT == 32) return zfactor_t<32>(a, st);
  if (KT == 64) return zfactor_t<64>(a, st);
  return cudaErrorInvalidValue;
}
cudaError_t launch_zchain_qform(const ZQformArgs& a, int KT, cudaStream_t st) {
  if (KT == 16) return zqform_t<16>(a, st);
  if (KT == 32) return zqform_t<32>(a, st);
  if (KT == 64) return zqform_t<64>(a, st);
  return cudaErrorInvalidValue;
}

}  // namespace ots
