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
  static constexpr int BMAX = 32 * TPC;           // 32 rows / thread / column step
  static constexpr int SMEM = (KT + BMAX) * LDS * 8;
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
template <int KT, bool HEAD>
__device__ __forceinline__ void householder_sweep(double* S, int nb, double* U, double* tau_s) {
  using C = FactorCfg<KT>;
  constexpr int TPC = C::TPC, LDS = C::LDS;
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
        if (q == 0) U[c * KT + j] = d;
      }
    } else {
      if (q == 0) U[j * KT + j] = tau;
    }
    __syncthreads();
  }
}


template <int KT>
__global__ void __launch_bounds__(256) chain_factor_kernel(FactorArgs a) {
  using C = FactorCfg<KT>;
  constexpr int LDS = C::LDS;
  extern __shared__ __align__(128) double S[];
  __shared__ double tau_s[KT];
  const int tid = threadIdx.x;
  const int chain = blockIdx.x;
  const long r0 = (long)chain * a.G.rpc;
  const int ntiles = chain_real_tiles(a.G, chain, KT);
  double* Ubase = a.U + (long)chain * (a.G.L + 1) * KT * KT;

  // ---- head: plain QR of rows [r0, r0+KT)
  load_rows_plain<KT, LDS>(S, 0, a.D, a.ldd, r0, KT, a.G.nrows, a.ncols, tid, C::NT);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  householder_sweep<KT, true>(S, 0, Ubase, tau_s);
  store_rows_plain<KT, LDS>(S, 0, a.D, a.ldd, r0, KT, a.G.nrows, a.ncols, tid, C::NT);
  __syncthreads();
  for (int i = tid; i < KT * KT; i += C::NT) {  // top := R (zero strictly lower part)
    int r = i / KT, cc = i - r * KT;
    if (cc < r) S[r * LDS + cc] = 0.0;
  }
  __syncthreads();

  // ---- structured tiles
  for (int t = 1; t <= ntiles; ++t) {
    const long gr0 = r0 + KT + (long)(t - 1) * a.G.b;
    load_rows_plain<KT, LDS>(S, KT, a.D, a.ldd, gr0, a.G.b, a.G.nrows, a.ncols, tid, C::NT);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    householder_sweep<KT, false>(S, a.G.b, Ubase + (long)t * KT * KT, tau_s);
    store_rows_plain<KT, LDS>(S, KT, a.D, a.ldd, gr0, a.G.b, a.G.nrows, a.ncols, tid, C::NT);
    __syncthreads();
  }

  // ---- chain R (upper triangle, exact zeros below)
  double* R = a.Rout + (long)chain * KT * KT;
  for (int i = tid; i < KT * KT; i += C::NT) {
    int r = i / KT, cc = i - r * KT;
    R[i] = (cc >= r) ? S[r * LDS + cc] : 0.0;
  }
}

// U (diag tau, strict-upper Gram) -> T via the dlarft recurrence, one CTA of
// KT threads per tile; row i of T computed by thread i.
template <int KT>
__global__ void __launch_bounds__(KT) u_to_t_kernel(double* UT, ChainGeom G) {
  extern __shared__ __align__(16) double ush[];
  double* Us = ush;             // U (KT x KT)
  double* Tt = ush + KT * KT;   // transposed T: Tt[l*KT + i] = T[i][l]
  const int tile = blockIdx.x;
  const int chain = tile / (G.L + 1), t = tile - chain * (G.L + 1);
  if (chain >= G.nchains) return;
  if (t > 0 && t > chain_real_tiles(G, chain, KT)) return;
  double* Ug = UT + (long)tile * KT * KT;
  const int i = threadIdx.x;
  for (int e = i; e < KT * KT; e += KT) Us[e] = Ug[e];
  for (int l = 0; l < KT; ++l) Tt[l * KT + i] = 0.0;
  __syncthreads();
  Tt[i * KT + i] = Us[i * KT + i];
  for (int j = i + 1; j < KT; ++j) {
    double s = 0.0;
    for (int l = i; l < j; ++l) s = fma(Tt[l * KT + i], Us[l * KT + j], s);
    Tt[j * KT + i] = -Us[j * KT + j] * s;
  }
  __syncthreads();
  for (int e = i; e < KT * KT; e += KT) {
    int r = e / KT, cc = e - r * KT;
    Ug[e] = Tt[cc * KT + r];
  }
}

// ---------------------------------------------------------------------------
// Q formation (reverse chain walk).  Per structured tile (reverse order):
//   M = T C ; out_rows = -Y M ; C <- C - M
// Head:  W1 = Yt^T C ; M = T W1 ; out_rows(head) = C - Yt M   (Yt unit lower)
// ---------------------------------------------------------------------------
template <int KT>
struct QformCfg {
  static constexpr int NT = 256;
  static constexpr int BMAX = FactorCfg<KT>::BMAX;
  static constexpr int SMEM = (3 * KT * KT + BMAX * KT) * 8;
};

// out(KT x KT, swizzled smem) = op(A) * B   [8 warps; warp w < KT/8 -> m-frag w]
template <int KT, bool TA, bool UPPER_A>
__device__ __forceinline__ void kt_gemm(const double* A, const double* B, double (&acc)[KT / 8][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int j = 0; j < KT / 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  if (warp >= KT / 8) return;
  const int kk0 = UPPER_A ? (2 * warp) : 0;  // A upper triangular: rows 8w.. need k >= 8w
#pragma unroll 4
  for (int kk = kk0; kk < KT / 4; ++kk) {
    double av = TA ? A[swz(4 * kk + t, 8 * warp + g, KT)] : A[swz(8 * warp + g, 4 * kk + t, KT)];
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) dmma(acc[j], av, B[swz(4 * kk + t, 8 * j + g, KT)]);
  }
}

template <int KT>
__device__ __forceinline__ void kt_store(double* O, const double (&acc)[KT / 8][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if (warp >= KT / 8) return;
#pragma unroll
  for (int j = 0; j < KT / 8; ++j) {
    O[swz(8 * warp + g, 8 * j + 2 * t, KT)] = acc[j][0];
    O[swz(8 * warp + g, 8 * j + 2 * t + 1, KT)] = acc[j][1];
  }
}


template <int KT>
__global__ void __launch_bounds__(256, 1) chain_qform_kernel(QformArgs a) {
  using C = QformCfg<KT>;
  extern __shared__ __align__(128) double sm[];
  double* Cs = sm;
  double* Ms = Cs + KT * KT;
  double* Ts = Ms + KT * KT;
  double* Ys = Ts + KT * KT;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int chain = blockIdx.x;
  const long r0 = (long)chain * a.G.rpc;
  const int ntiles = chain_real_tiles(a.G, chain, KT);
  const double* Tbase = a.T + (long)chain * (a.G.L + 1) * KT * KT;

  // C (chain) -> smem (swizzled)
  load_tile_async(Cs, KT, a.Cin + (long)chain * KT * KT, KT, 0, KT, 0, KT, 0, KT, KT, tid, C::NT);
  cp_async_commit();

  constexpr int WN = KT < 32 ? KT : 32;
  constexpr int NJ = WN / 8;
  constexpr int NWN = KT / WN;

  for (int tt = ntiles; tt >= 1; --tt) {
    const long gr0 = r0 + KT + (long)(tt - 1) * a.G.b;
    load_tile_async(Ts, KT, Tbase + (long)tt * KT * KT, KT, 0, KT, 0, KT, 0, KT, KT, tid, C::NT);
    const long rhi = gr0 + a.G.b < a.G.nrows ? gr0 + a.G.b : a.G.nrows;  // this tile only
    const int brows = (a.G.b + 31) / 32 * 32;
    load_tile_async(Ys, KT, a.D, a.ldd, gr0, brows, gr0, rhi, 0, KT, a.ncols, tid, C::NT);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    double acc[KT / 8][2];
    kt_gemm<KT, false, true>(Ts, Cs, acc);  // M = T C
    kt_store<KT>(Ms, acc);
    __syncthreads();
    for (int e = tid; e < KT * KT; e += C::NT) {  // C <- C - M (same swizzle positions)
      Cs[e] -= Ms[e];
    }
    // out rows = -Y M  (b x KT): warp tiles 32 x WN
    const int nwt = (brows / 32) * NWN;
    for (int wt = warp; wt < nwt; wt += 8) {
      const int wm0 = (wt / NWN) * 32, wn0 = (wt % NWN) * WN;
      double o[4][NJ][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) o[i][j][0] = o[i][j][1] = 0.0;
#pragma unroll 2
      for (int kk = 0; kk < KT / 4; ++kk) {
        double af[4], bf[NJ];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = Ys[swz(wm0 + 8 * i + g, 4 * kk + t4, KT)];
#pragma unroll
        for (int j = 0; j < NJ; ++j) bf[j] = Ms[swz(4 * kk + t4, wn0 + 8 * j + g, KT)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j) dmma(o[i][j], af[i], bf[j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          long r = gr0 + wm0 + 8 * i + g;
          int cc = wn0 + 8 * j + 2 * t4;
          if (r >= rhi) continue;
          double* p = a.D + r * a.ldd + cc;
          if (cc + 1 < a.ncols) *reinterpret_cast<double2*>(p) = make_double2(-o[i][j][0], -o[i][j][1]);
          else if (cc < a.ncols) p[0] = -o[i][j][0];
        }
    }
    __syncthreads();
  }

  // ---- head
  load_tile_async(Ts, KT, Tbase, KT, 0, KT, 0, KT, 0, KT, KT, tid, C::NT);
  load_tile_async(Ys, KT, a.D, a.ldd, r0, KT, r0, (r0 + KT < a.G.nrows ? r0 + KT : a.G.nrows), 0, KT,
                  a.ncols, tid, C::NT);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int e = tid; e < KT * KT; e += C::NT) {  // Yt: unit lower
    int r = e / KT, cc = e - r * KT;
    if (cc >= r) Ys[swz(r, cc, KT)] = (cc == r) ? 1.0 : 0.0;
  }
  __syncthreads();
  double acc[KT / 8][2];
  kt_gemm<KT, true, false>(Ys, Cs, acc);  // W1 = Yt^T C
  kt_store<KT>(Ms, acc);
  __syncthreads();
  kt_gemm<KT, false, true>(Ts, Ms, acc);  // M = T W1
  __syncthreads();
  kt_store<KT>(Ms, acc);
  __syncthreads();
  kt_gemm<KT, false, false>(Ys, Ms, acc);  // Yt M
  if (warp < KT / 8) {
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) {
      int r = 8 * warp + g;
      int cc = 8 * j + 2 * t4;
      long gr = r0 + r;
      if (gr >= a.G.nrows) continue;
      double y0 = Cs[swz(r, cc, KT)] - acc[j][0];
      double y1 = Cs[swz(r, cc + 1, KT)] - acc[j][1];
      double* p = a.D + gr * a.ldd + cc;
      if (cc + 1 < a.ncols) *reinterpret_cast<double2*>(p) = make_double2(y0, y1);
      else if (cc < a.ncols) p[0] = y0;
    }
  }
}

// ---------------------------------------------------------------------------
template <int KT>
static cudaError_t factor_t(const FactorArgs& a, cudaStream_t st) {
  using C = FactorCfg<KT>;
  if (a.G.b > C::BMAX || a.G.nchains <= 0) return cudaErrorInvalidValue;
  auto k = chain_factor_kernel<KT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  k<<<a.G.nchains, C::NT, C::SMEM, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  long tiles = (long)a.G.nchains * (a.G.L + 1);
  const int usm = 2 * KT * KT * 8;
  cudaFuncSetAttribute(u_to_t_kernel<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, usm);
  u_to_t_kernel<KT><<<(unsigned)tiles, KT, usm, st>>>(a.U, a.G);
  return cudaGetLastError();
}

cudaError_t launch_chain_factor(const FactorArgs& a, int KT, cudaStream_t st) {
  if (KT == 16) return factor_t<16>(a, st);
  if (KT == 32) return factor_t<32>(a, st);
  if (KT == 64) return factor_t<64>(a, st);
  return cudaErrorInvalidValue;
}

template <int KT>
static cudaError_t qform_t(const QformArgs& a, cudaStream_t st) {
  using C = QformCfg<KT>;
  auto k = chain_qform_kernel<KT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  k<<<a.G.nchains, C::NT, C::SMEM, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_chain_qform(const QformArgs& a, int KT, cudaStream_t st) {
  if (KT == 16) return qform_t<16>(a, st);
  if (KT == 32) return qform_t<32>(a, st);
  if (KT == 64) return qform_t<64>(a, st);
  return cudaErrorInvalidValue;
}

int chain_bmax(int KT) {
  return KT == 16 ? FactorCfg<16>::BMAX : KT == 32 ? FactorCfg<32>::BMAX : FactorCfg<64>::BMAX;
}

}  // namespace ots
