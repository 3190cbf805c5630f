// Direct-Q pipeline of the headline shape (real f64, 96 < k0 <= 128, 32 < k <= 64,
// one device or one rank's row shard): the Gram-form level-0 factor (gsweep.inc) only needs the tile
// Grams of X = A_b + V_b Z1, and its Q formation is Q_tile = X_tile K_tile
// with a 64 x 64 coefficient per tall tile, so X never has to exist:
//
//   tile Grams of [V | A]   (one pass over V and A: V^T V, V^T A, A^T A per tile)
//   X_t^T X_t = A^T A + Z1^T (V^T A + V^T V Z1) + (V^T A)^T Z1      (per tile, small)
//   V_t^T X_t = V^T A + V^T V Z1                                  (per tile, small)
//   Y2 = -V_b^T Q_ = -sum_t (V_t^T X_t) K_t                          (no pass over Q_)
//   Q_t = (A_t K_t + V_t (Z1 K_t + Z2)) diag(s)                      (one pass: V, A in, Q out)
//
// i.e. two streaming passes (this file's tgram and final kernels) instead of
// six (gram, apply1, tile Gram, Q formation, gram2, apply2): 1.09e12 executed
// flops at the headline instead of 1.58e12.  The algebra that replaces the
// passes is exact; what changes is rounding: X_t^T X_t now carries an absolute
// error u |A_t|^2, so a tile column that keeps less than FAST_KEEP of its
// norm^2 (A nearly in range(V): configs[1], configs[2]) raises the cancel
// flag, and -- like any chain the sweep flags -- sends the call to the
// materialised-X pipeline (ots_api.cu).  Head rows (64 per chain, exact
// Householder) are materialised in the Q buffer by small kernels.
//
// Reference semantics: twostage.py:90-97 (H^* A, intra QR, Q = H [0; Q_]).
// tgram_kernel (k = 0) and final_nn_kernel<128> also serve the complex128
// Gram-form intra QR on the interleaved real views (zpath.inc: zgs_intra).
#include "common.cuh"
#include "kernels.cuh"

namespace ots {

#define FAST_KEEP 0.25

// cp.async.bulk global -> shared (SASS UBLKCP), completing on an mbarrier by bytes
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}

// ============================================================================
// tgram (k0 padded to 128): per tall tile  [V^T V | V^T A]  (128 x 192)  and
// A^T A  (64 x 64), both stored as full symmetric matrices (mirrored at the
// flush), plus the per-CTA totals of [V^T V | V^T A] over every chain row
// (tiles and heads).  64-row stages through an mbarrier ring (the tsgemm_tn
// design); a CTA walks its tiles, then its heads.
//
// 20 warps (96 registers each; 21 would be allocated as 24 and spill), 300
// DMMA units per 4-row step in 8 x 8 output fragments, 75 on every SM
// sub-partition (warp w -> SMSP w % 4):
//   warps  0..3   D: diagonal block b of V^T V (10 lower fragments) + 6 A^T A fragments
//   warps  4..7   H: a 32 x 16 half of V_3^T A (8 fragments)         + 3 A^T A fragments
//   warps  8..19  F: a full 32 x 32 block (16): 6 off-diagonal V^T V, 6 V^T A
// The A^T A fragments sit in the accumulator entries the role leaves unused
// (D: the strict upper triangle of the 4 x 4 fragment grid, H: column 2).
// ============================================================================
#ifndef TG_UNROLL
#define TG_UNROLL 16
#endif
#ifndef TG_RT
#define TG_RT 64
#endif
#ifndef TG_NSTAGE
#define TG_NSTAGE 2
#endif
#ifndef TG_LA
#define TG_LA 1
#endif
struct TgCfg {
  static constexpr int PW = 128, NTASK = 20, NT = NTASK * 32, RT = TG_RT;
  // Stage rows are stored linearly with padded pitches (136 / 72 doubles: a
  // row advances 64 bytes of bank space, so the 4 rows x 8 columns of a DMMA
  // operand fragment take the 2-wavefront minimum) -- the layout a bulk
  // global->shared copy (cp.async.bulk, one per row) can write.
  static constexpr int PV = PW + 8, PA = 64 + 8;
  static constexpr int STAGE = RT * (PV + PA);
  static constexpr int NSTAGE = TG_NSTAGE;
  static constexpr int LA = TG_LA;               // stages issued ahead; NSTAGE - 1 - LA stages of slack between warps
  static constexpr int SMEM = NSTAGE * STAGE * 8;
  static constexpr int NT1 = PW + 64;
  static constexpr int UNR = TG_UNROLL;          // 4-row steps unrolled in the stage loop
};

// A^T A lower-triangle fragments (i, j) of the 8 x 8 fragment grid, packed 8 i + j:
// groups 0..3 (6 fragments, D warps), 4..7 (3 fragments, H warps).  The lists
// are data (constant memory), not code: one body per role keeps the kernel's
// hot loops inside the instruction cache (nine specialised bodies measured
// 23.0 ms at 2-step unrolling and 29.4 ms at 16).
__constant__ unsigned char c_tg_aa[8][6] = {
    {40, 41, 42, 43, 44, 45},       // row 5
    {0, 8, 9, 16, 17, 18},          // rows 0..2
    {24, 25, 26, 27, 32, 33},       // row 3, (4,0), (4,1)
    {48, 49, 50, 51, 52, 53},       // row 6, columns 0..5
    {34, 35, 36, 0, 0, 0},          // (4,2..4)
    {56, 57, 58, 0, 0, 0},          // (7,0..2)
    {59, 60, 61, 0, 0, 0},          // (7,3..5)
    {62, 63, 54, 0, 0, 0}};         // (7,6), (7,7), (6,6)
// accumulator entry of extra fragment q: D -> strict upper triangle, H -> column 2
__host__ __device__ constexpr int tg_ex_i(bool isD, int q) { return isD ? (q < 3 ? 0 : (q < 5 ? 1 : 2)) : q; }
__host__ __device__ constexpr int tg_ex_j(bool isD, int q) { return isD ? (q < 3 ? q + 1 : (q < 5 ? q - 1 : 3)) : 2; }

template <bool isD>
__device__ __forceinline__ void tg_aa_flush(double (&acc)[4][4][2], int grp, double* AA, bool store, int g, int t) {
  constexpr int N = isD ? 6 : 3;
#pragma unroll
  for (int q = 0; q < N; ++q) {
    const int fi = c_tg_aa[grp][q] >> 3, fj = c_tg_aa[grp][q] & 7;
    double (&e)[2] = acc[tg_ex_i(isD, q)][tg_ex_j(isD, q)];
    if (store) {
      const int r = 8 * fi + g, c = 8 * fj + 2 * t;
      *reinterpret_cast<double2*>(AA + r * 64 + c) = make_double2(e[0], e[1]);
      if (fi != fj) {
        AA[c * 64 + r] = e[0];
        AA[(c + 1) * 64 + r] = e[1];
      }
    }
    e[0] = e[1] = 0.0;
  }
}

// ROLE 0: D warp (diagonal block idx of V^T V + A^T A group idx), 1: H warp
// (half idx of V_3^T A + group 4 + idx), 2: F warp (block (ra, rb)).
template <int ROLE>
__device__ __forceinline__ void tg_body(const FastArgs& a, double* smem, unsigned long long* full_bar,
                                        unsigned long long* empty_bar, int idx, int ra, int rb) {
  using C = TgCfg;
  constexpr int PW = C::PW, NT1 = C::NT1, RT = C::RT, PV = C::PV, PA = C::PA;
  constexpr int NX = ROLE == 0 ? 6 : (ROLE == 1 ? 3 : 0);
  const int grp = ROLE == 0 ? idx : 4 + idx;
  const bool has_a = a.k > 0;      // k = 0 (the complex path's Gram of one 128-column view): A blocks are skipped
  const int tid = threadIdx.x, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  // in-row offsets of the two operand fragments of every extra A^T A fragment
  int xa[NX > 0 ? NX : 1], xb[NX > 0 ? NX : 1];
#pragma unroll
  for (int q = 0; q < NX; ++q) {
    const int fi = c_tg_aa[grp][q] >> 3, fj = c_tg_aa[grp][q] & 7;
    xa[q] = 8 * fi + g;
    xb[q] = 8 * fj + g;
  }
  const bool b_isV = rb < 4;
  const int boff = b_isV ? 0 : RT * PV, bW = b_isV ? PV : PA, bcol = b_isV ? 32 * rb : 32 * (rb - 4);

  // this CTA's items: tall tiles first (tile index ti = chain * L + t - 1),
  // then chain heads
  const int L = a.G.L, nch = a.G.nchains;
  const int ntl = nch * L;
  const int nitems_end = ntl + nch;
  auto item_rows = [&](int it, long& r0, long& rhi) {      // it < ntl: tile, else head it - ntl
    if (it < ntl) {
      const int chain = it / L, tt = it - chain * L;
      r0 = (long)chain * a.G.rpc + 64 + (long)tt * a.G.b;
      rhi = r0 + a.G.b;
    } else {
      r0 = (long)(it - ntl) * a.G.rpc;
      rhi = r0 + 64;
    }
    if (rhi > a.G.nrows) rhi = a.G.nrows;
  };
  auto next_item = [&](int it) {                            // successor in this CTA's sequence
    if (it < ntl) {
      it += gridDim.x;
      if (it < ntl) return it;
      return ntl + (int)blockIdx.x;
    }
    return it + (int)gridDim.x;
  };
  auto item_chunks = [&](int it) {
    if (it >= nitems_end) return 0;
    long r0, rhi;
    item_rows(it, r0, rhi);
    if (rhi <= r0) return 0;
    return (int)((rhi - r0 + RT - 1) / RT);
  };
  auto skip_empty = [&](int it) {
    while (it < nitems_end && item_chunks(it) == 0) it = next_item(it);
    return it;
  };

  const int it0 = skip_empty(blockIdx.x < ntl ? (int)blockIdx.x : ntl + (int)blockIdx.x);
  // producer.  Full stages (64 rows inside the item, even k0 and k): one bulk
  // copy per row (threads 0..63 a V row, 64..127 an A row), completing on the
  // stage's mbarrier by bytes; thread 0 posts the byte count with its arrival,
  // everyone else just arrives.  Partial stages (the last tile of the last
  // chain) and odd widths: this thread's fixed share of 16-byte cp.async units
  // with zero fill -- unit uv of rows rv0, rv0 + 10, ... of the V part (640
  // threads = 10 rows of 64 units) and unit ua of rows ra0, ra0 + 20, ... of
  // the A part.  Columns beyond k0 / k are zeroed once (bulk copies never
  // touch them).  The item's row range is worked out once per item.
  const bool bulk_ok = !(a.k0 & 1) && !(a.k & 1);
  const int uv = tid & 63, rv0 = tid >> 6, ua = tid & 31, ra0 = tid >> 5;
  const int vbytes = 2 * uv + 1 < a.k0 ? 16 : (2 * uv < a.k0 ? 8 : 0);
  const int abytes = 2 * ua + 1 < a.k ? 16 : (2 * ua < a.k ? 8 : 0);
  const double* vsrc = a.V + (vbytes ? 2 * uv : 0);
  const double* asrc = a.A + (abytes ? 2 * ua : 0);
  int p_it = it0, p_ch = 0, p_j = 0, p_n = 0;
  long p_r0 = 0, p_rhi = 0;
  if (p_it < nitems_end) {
    item_rows(p_it, p_r0, p_rhi);
    p_n = (int)((p_rhi - p_r0 + RT - 1) / RT);
  }
  auto produce = [&]() {
    if (p_it >= nitems_end) return;
    const int s = p_j % C::NSTAGE, rnd = p_j / C::NSTAGE;
    if (rnd >= 1) mbar_wait(&empty_bar[s], (rnd - 1) & 1);
    const long rr = p_r0 + (long)p_ch * RT;
    const int nr = (int)(p_rhi - rr < RT ? p_rhi - rr : RT);           // rows of this stage inside the item
    double* Ps = smem + s * C::STAGE;
    double* Bs = Ps + RT * PV;
    if (bulk_ok && nr == RT) {
      if (tid < RT) bulk_g2s(Ps + tid * PV, a.V + (rr + tid) * a.ldv, (unsigned)a.k0 * 8u, &full_bar[s]);
      else if (tid < 2 * RT && a.k > 0) bulk_g2s(Bs + (tid - RT) * PA, a.A + (rr + tid - RT) * a.lda, (unsigned)a.k * 8u, &full_bar[s]);
      if (tid == 0) mbar_arrive_expect_tx(&full_bar[s], (unsigned)(RT * (a.k0 + a.k)) * 8u);
      else mbar_arrive(&full_bar[s]);
    } else {
#pragma unroll
      for (int q = 0; q < (RT + 9) / 10; ++q) {
        const int r = rv0 + 10 * q;
        if (r < RT) {
          const bool in = r < nr;
          cp_async16(Ps + r * PV + 2 * uv, in ? vsrc + (rr + r) * a.ldv : a.V, in ? vbytes : 0);
        }
      }
#pragma unroll
      for (int q = 0; q < (RT + 19) / 20; ++q) {
        const int r = ra0 + 20 * q;
        if (r < RT) {
          const bool in = r < nr;
          cp_async16(Bs + r * PA + 2 * ua, in ? asrc + (rr + r) * a.lda : a.A, in ? abytes : 0);
        }
      }
      cp_async_mbar_arrive(&full_bar[s]);
    }
    ++p_j;
    if (++p_ch >= p_n) {
      p_ch = 0;
      p_it = skip_empty(next_item(p_it));
      if (p_it < nitems_end) {
        item_rows(p_it, p_r0, p_rhi);
        p_n = (int)((p_rhi - p_r0 + RT - 1) / RT);
      }
    }
  };
  for (int j = 0; j < C::LA; ++j) produce();

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double* tot = a.part + (long)blockIdx.x * PW * NT1;       // CTA totals [PW][NT1]
  bool tot_first = true;
  int c_it = it0, c_ch = 0, c_j = 0;
  int c_n = item_chunks(c_it);
  while (c_it < nitems_end) {
    produce();
    const int s = c_j % C::NSTAGE;
    mbar_wait(&full_bar[s], (c_j / C::NSTAGE) & 1);
    const double* Vs = smem + s * C::STAGE;
    const double* As = Vs + RT * PV;
    if (ROLE == 0) {
#pragma unroll(TgCfg::UNR)
      for (int kk = 0; kk < RT / 4; ++kk) {
        const int r = 4 * kk + t;
        double af[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = Vs[r * PV + 32 * idx + 8 * i + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j <= i; ++j) dmma(acc[i][j], af[i], af[j]);
        if (has_a) {
#pragma unroll
          for (int q = 0; q < NX; ++q)
            dmma(acc[tg_ex_i(true, q)][tg_ex_j(true, q)], As[r * PA + xa[q]], As[r * PA + xb[q]]);
        }
      }
    } else if (ROLE == 1) {
      if (has_a)
#pragma unroll(TgCfg::UNR)
      for (int kk = 0; kk < RT / 4; ++kk) {
        const int r = 4 * kk + t;
        double af[4], bf[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = Vs[r * PV + 96 + 8 * i + g];
#pragma unroll
        for (int j = 0; j < 2; ++j) bf[j] = As[r * PA + 16 * idx + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma(acc[i][j], af[i], bf[j]);
#pragma unroll
        for (int q = 0; q < NX; ++q)
          dmma(acc[tg_ex_i(false, q)][tg_ex_j(false, q)], As[r * PA + xa[q]], As[r * PA + xb[q]]);
      }
    } else {
      const double* Bs = smem + s * C::STAGE + boff;
      if (b_isV || has_a)
#pragma unroll(TgCfg::UNR)
      for (int kk = 0; kk < RT / 4; ++kk) {
        const int r = 4 * kk + t;
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = Vs[r * PV + 32 * ra + 8 * i + g];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = Bs[r * bW + bcol + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
    ++c_j;
    if (++c_ch >= c_n) {
      // ---- flush the item: tile slot (mirrored) and the CTA totals
      const bool is_tile = c_it < ntl;
      double* slot = a.TG + (long)c_it * a.tg_stride;
      if (ROLE != 2) tg_aa_flush<ROLE == 0>(acc, grp, slot + (long)PW * NT1, is_tile, g, t);
      // main block: rows 32 ra_.., cols c0_.. of [V^T V | V^T A]; D: lower fragments, H: 2 fragment columns
      const int ra_ = ROLE == 0 ? idx : (ROLE == 1 ? 3 : ra);
      const int c0_ = ROLE == 0 ? 32 * idx : (ROLE == 1 ? PW + 16 * idx : (b_isV ? 32 * rb : PW + 32 * (rb - 4)));
      const bool mirror = ROLE == 0 || (ROLE == 2 && b_isV);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (ROLE == 0 && j > i) continue;
          if (ROLE == 1 && j >= 2) continue;
          const int r = 32 * ra_ + 8 * i + g, c = c0_ + 8 * j + 2 * t;
          if (is_tile) {
            *reinterpret_cast<double2*>(slot + (long)r * NT1 + c) = make_double2(acc[i][j][0], acc[i][j][1]);
            if (mirror && !(ROLE == 0 && i == j)) {
              slot[(long)c * NT1 + r] = acc[i][j][0];
              slot[(long)(c + 1) * NT1 + r] = acc[i][j][1];
            }
          }
          double2* tp = reinterpret_cast<double2*>(tot + (long)r * NT1 + c);
          double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
          if (!tot_first) {
            const double2 o = *tp;
            v.x += o.x;
            v.y += o.y;
          }
          *tp = v;
          acc[i][j][0] = acc[i][j][1] = 0.0;
        }
      tot_first = false;
      c_ch = 0;
      c_it = skip_empty(next_item(c_it));
      c_n = item_chunks(c_it);
    }
  }
  cp_async_wait<0>();
  if (tot_first) {                                           // a CTA without items: zero totals
    const int ra_ = ROLE == 0 ? idx : (ROLE == 1 ? 3 : ra);
    const int c0_ = ROLE == 0 ? 32 * idx : (ROLE == 1 ? PW + 16 * idx : (b_isV ? 32 * rb : PW + 32 * (rb - 4)));
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (ROLE == 0 && j > i) continue;
        if (ROLE == 1 && j >= 2) continue;
        const int r = 32 * ra_ + 8 * i + g, c = c0_ + 8 * j + 2 * t;
        *reinterpret_cast<double2*>(tot + (long)r * NT1 + c) = make_double2(0.0, 0.0);
      }
  }
}

__global__ void __launch_bounds__(TgCfg::NT, 1) tgram_kernel(FastArgs a) {
  using C = TgCfg;
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) unsigned long long full_bar[C::NSTAGE], empty_bar[C::NSTAGE];
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < C::NSTAGE; ++s) {
      mbar_init(&full_bar[s], C::NT);
      mbar_init(&empty_bar[s], C::NTASK);
    }
    fence_mbar_init();
  }
  for (int e = tid; e < C::NSTAGE * C::STAGE; e += C::NT) smem[e] = 0.0;   // columns beyond k0 / k stay zero
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (warp < 4) {
    tg_body<0>(a, smem, full_bar, empty_bar, warp, 0, 0);
  } else if (warp < 8) {
    tg_body<1>(a, smem, full_bar, empty_bar, warp - 4, 0, 0);
  } else {
    // F: 6 off-diagonal blocks of V^T V, then V_b^T A for b = 0..2
    const int f = warp - 8;
    int ra, rb;
    if (f < 6) {
      ra = f < 1 ? 1 : (f < 3 ? 2 : 3);
      rb = f - (ra == 1 ? 0 : (ra == 2 ? 1 : 3));
    } else {
      ra = (f - 6) >> 1;
      rb = 4 + ((f - 6) & 1);
    }
    tg_body<2>(a, smem, full_bar, empty_bar, 0, ra, rb);
  }
}

// Gfull[PW][ldg] = sum of the CTA totals + the top rows' V_t^T V_t (rows above
// the first chain row belong to no chain; their A part is not in V_b^T A_b).
__global__ void tgram_reduce_kernel(const double* __restrict__ part, int nparts, int PW, int NT1,
                                    const double* __restrict__ Vtop, long ldv, int ntop, int k0,
                                    double* __restrict__ out, int ldg) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= PW * NT1) return;
  const int i = e / NT1, jj = e - i * NT1;
  double s = 0.0;
  for (int c = 0; c < nparts; ++c) s += part[(long)c * PW * NT1 + e];
  if (jj < PW && i < k0 && jj < k0) {
    double s2 = 0.0;
    for (int r = 0; r < ntop; ++r) s2 = fma(Vtop[(long)r * ldv + i], Vtop[(long)r * ldv + jj], s2);
    s += s2;
  }
  out[(long)i * ldg + jj] = s;
}

// ============================================================================
// Chain heads (64 rows per chain): small row-local products on CUDA cores.
//   mode 0:  D_h = A_h + V_h Z            (X rows for the head QR)
//   mode 1:  D_h = (D_h + V_h Z) diag(s)  (final Q rows)
//   mode 2:  part[cta] += V_h^T D_h       (the heads' share of V_b^T Q_)
// ============================================================================
__global__ void __launch_bounds__(256) head_rows_kernel(FastArgs a, int mode, const double* Z, int ldz,
                                                        const double* colscale, double* part) {
  extern __shared__ __align__(16) double hsm[];
  double (*Vs)[33] = reinterpret_cast<double (*)[33]>(hsm);                 // 64 x 33
  double (*Zs)[65] = reinterpret_cast<double (*)[65]>(hsm + 64 * 33);       // 32 x 65 (modes 0, 1)
  double (*Ds)[65] = reinterpret_cast<double (*)[65]>(hsm + 64 * 33);       // 64 x 65 (mode 2)
  const int tid = threadIdx.x;
  if (mode == 2) {
    // out (k0 x k) accumulated over this CTA's chains; thread -> row i, 8 cols per pass
    for (int i0 = 0; i0 < a.PW; i0 += 32) {
      double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      const int i = i0 + (tid >> 3), c0 = tid & 7;           // row i (V column), cols c0, c0 + 8, ... (bank-spread)
      for (int chain = blockIdx.x; chain < a.G.nchains; chain += gridDim.x) {
        const long r0 = (long)chain * a.G.rpc;
        __syncthreads();
#pragma unroll
        for (int e = tid; e < 64 * 64; e += 256) {             // independent loads, issued together
          const int r = e >> 6, c = e & 63;
          Ds[r][c] = (r0 + r < a.G.nrows && c < a.k) ? a.D[(r0 + r) * a.ldd + c] : 0.0;
        }
#pragma unroll
        for (int e = tid; e < 64 * 32; e += 256) {
          const int r = e >> 5, c = e & 31;
          Vs[r][c] = (r0 + r < a.G.nrows && i0 + c < a.k0) ? a.V[(r0 + r) * a.ldv + i0 + c] : 0.0;
        }
        __syncthreads();
        for (int r = 0; r < 64; ++r) {
          const double v = Vs[r][tid >> 3];
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[c] = fma(v, Ds[r][c0 + 8 * c], acc[c]);
        }
      }
      double* out = part + (long)blockIdx.x * a.PW * 64;
#pragma unroll
      for (int c = 0; c < 8; ++c) out[(long)i * 64 + c0 + 8 * c] = acc[c];
    }
    return;
  }
  for (int chain = blockIdx.x; chain < a.G.nchains; chain += gridDim.x) {
    const long r0 = (long)chain * a.G.rpc;
    const int r = tid >> 2, c0 = tid & 3;                    // row r, cols c0, c0 + 4, ... (bank-spread)
    double acc[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[c] = 0.0;
    for (int kc = 0; kc < a.k0; kc += 32) {
      __syncthreads();
#pragma unroll
      for (int e = tid; e < 64 * 32; e += 256) {
        const int rr = e >> 5, c = e & 31;
        Vs[rr][c] = (r0 + rr < a.G.nrows && kc + c < a.k0) ? a.V[(r0 + rr) * a.ldv + kc + c] : 0.0;
      }
#pragma unroll
      for (int e = tid; e < 32 * 64; e += 256) {
        const int rr = e >> 6, c = e & 63;
        Zs[rr][c] = (kc + rr < a.k0 && c < a.k) ? Z[(long)(kc + rr) * ldz + c] : 0.0;
      }
      __syncthreads();
      for (int kk = 0; kk < 32; ++kk) {
        const double v = Vs[r][kk];
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[c] = fma(v, Zs[kk][c0 + 4 * c], acc[c]);
      }
    }
    if (r0 + r < a.G.nrows) {
      const double* src = mode == 0 ? a.A + (r0 + r) * a.lda : a.D + (r0 + r) * a.ldd;
      double* dst = a.D + (r0 + r) * a.ldd;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int cc = c0 + 4 * c;
        if (cc >= a.k) continue;
        double v = src[cc] + acc[c];
        if (mode == 1 && colscale && colscale[cc] < 0.0) v = -v;
        dst[cc] = v;
      }
    }
  }
}

// ============================================================================
// tile_alg: per tall tile, from its Gram slot and Z1 (k0 x k):
//   Cx = V_t^T X_t = VA + VV Z1      (PW x 64, written over the slot's VA block)
//   M  = X_t^T X_t = AA + Z1^T Cx + VA^T Z1   (64 x 64, into the tile's Cc slot)
// and the cancellation test  M_jj >= FAST_KEEP AA_jj.  16 warps, DMMA; VV
// streams through one 32-column chunk buffer, Z1 stays resident.
// ============================================================================
template <int PW>
struct TaCfg {
  static constexpr int NT = 512;
  static constexpr int SMEM = (3 * PW * 64 + PW * 32) * 8;   // Z1 | VA | Cx | VV chunk
};

template <int PW>
__global__ void __launch_bounds__(512, 1) tile_alg_kernel(FastArgs a) {
  constexpr int NT1 = PW + 64, NT = 512;
  extern __shared__ __align__(128) double sm[];
  double* Z1s = sm;                    // PW x 64
  double* VAs = Z1s + PW * 64;         // PW x 64
  double* Cxs = VAs + PW * 64;         // PW x 64
  double* VVc = Cxs + PW * 64;         // PW x 32
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int L = a.G.L, ntl = a.G.nchains * L;
  load_tile_async(Z1s, 64, a.Z1, a.ldz, 0, PW, 0, a.k0, 0, 64, a.k, tid, NT);
  cp_async_commit();
  __shared__ int s_next;
  int ti = blockIdx.x;
  for (;;) {
    if (ti >= ntl) break;
    const int chain = ti / L, tt = ti - chain * L;
    const long r0 = (long)chain * a.G.rpc + 64 + (long)tt * a.G.b;
    if (r0 < a.G.nrows) {
      double* slot = a.TG + (long)ti * a.tg_stride;
      __syncthreads();                                       // previous tile done with VAs / Cxs / VVc
      load_tile_async(VAs, 64, slot + PW, NT1, 0, PW, 0, PW, 0, 64, 64, tid, NT);
      // ---- step 1: Cx = VA + VV Z1 ; warp -> 32 rows x 16 cols
      const int band = warp >> 2, c0 = (warp & 3) * 16;
      double o[4][2][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) o[i][j][0] = o[i][j][1] = 0.0;
      for (int ch = 0; ch < PW / 32; ++ch) {
        if (ch > 0) __syncthreads();                         // chunk buffer free
        load_tile_async(VVc, 32, slot, NT1, 0, PW, 0, PW, 32 * ch, 32, PW, tid, NT);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        if (32 * band < PW) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            double af[4], bf[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = VVc[swz(32 * band + 8 * i + g, 4 * kk + t, 32)];
#pragma unroll
            for (int j = 0; j < 2; ++j) bf[j] = Z1s[swz(32 * ch + 4 * kk + t, c0 + 8 * j + g, 64)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 2; ++j) dmma(o[i][j], af[i], bf[j]);
          }
        }
      }
      if (32 * band < PW) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int r = 32 * band + 8 * i + g, c = c0 + 8 * j + 2 * t;
            const double x0 = o[i][j][0] + VAs[swz(r, c, 64)], x1 = o[i][j][1] + VAs[swz(r, c + 1, 64)];
            Cxs[swz(r, c, 64)] = x0;
            Cxs[swz(r, c + 1, 64)] = x1;
            *reinterpret_cast<double2*>(slot + (long)r * NT1 + PW + c) = make_double2(x0, x1);
          }
      }
      __syncthreads();
      // ---- step 2: M = AA + Z1^T Cx + VA^T Z1 ; warp -> 16 x 16
      {
        const int m0 = 16 * (warp >> 2), n0 = 16 * (warp & 3);
        const double* AA = slot + (long)PW * NT1;
        double m[2][2][2], aa[2][2][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const double2 v = *reinterpret_cast<const double2*>(AA + (long)(m0 + 8 * i + g) * 64 + n0 + 8 * j + 2 * t);
            m[i][j][0] = aa[i][j][0] = v.x;
            m[i][j][1] = aa[i][j][1] = v.y;
          }
#pragma unroll 4
        for (int kk = 0; kk < PW / 4; ++kk) {
          const int r = 4 * kk + t;
          double za[2], va[2], cb[2], zb[2];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            za[i] = Z1s[swz(r, m0 + 8 * i + g, 64)];
            va[i] = VAs[swz(r, m0 + 8 * i + g, 64)];
          }
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            cb[j] = Cxs[swz(r, n0 + 8 * j + g, 64)];
            zb[j] = Z1s[swz(r, n0 + 8 * j + g, 64)];
          }
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              dmma(m[i][j], za[i], cb[j]);
              dmma(m[i][j], va[i], zb[j]);
            }
        }
        double* M = a.M + ((long)chain * (L + 1) + tt + 1) * 4096;
        bool bad = false;
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int r = m0 + 8 * i + g, c = n0 + 8 * j + 2 * t;
            *reinterpret_cast<double2*>(M + (long)r * 64 + c) = make_double2(m[i][j][0], m[i][j][1]);
            if (r == c && !(m[i][j][0] >= FAST_KEEP * aa[i][j][0])) bad = true;
            if (r == c + 1 && !(m[i][j][1] >= FAST_KEEP * aa[i][j][1])) bad = true;
          }
        if (bad) atomicOr(a.flags, 1);
      }
    }
    // next tile: dynamic ticket (CTAs that start late take fewer)
    __syncthreads();
    if (tid == 0) {
      int nx = a.ticket ? (int)gridDim.x + atomicAdd(a.ticket, 1) : ti + (int)gridDim.x;
      if (*reinterpret_cast<volatile int*>(a.flags) & 1) nx = ntl;   // cancellation seen: the call goes the other way
      s_next = nx;
    }
    __syncthreads();
    ti = s_next;
  }
  cp_async_wait<0>();
}

// ============================================================================
// coefB: per tall tile, with K_t (64 x 64, rows PW.. of the tile's coefficient
// slot, from gs_coef):   W_t = Z1 K_t  -> rows 0..PW of the slot,
//                        Y (per CTA) += Cx_t K_t       (Cx_t = V_t^T X_t)
// ============================================================================
template <int PW>
struct CbCfg {
  static constexpr int NT = 512;
  static constexpr int SMEM = (2 * PW * 64 + 64 * 64) * 8;   // Z1 | Cx | K
};

template <int PW>
__global__ void __launch_bounds__(512, 1) coef_b_kernel(FastArgs a, double* ypart) {
  constexpr int NT1 = PW + 64, NT = 512;
  extern __shared__ __align__(128) double sm[];
  double* Z1s = sm;
  double* Cxs = Z1s + PW * 64;
  double* Ks = Cxs + PW * 64;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int L = a.G.L, ntl = a.G.nchains * L;
  const int band = warp >> 2, c0 = (warp & 3) * 16;
  const bool live = 32 * band < PW;
  load_tile_async(Z1s, 64, a.Z1, a.ldz, 0, PW, 0, a.k0, 0, 64, a.k, tid, NT);
  cp_async_commit();
  double y[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) y[i][j][0] = y[i][j][1] = 0.0;
  for (int ti = blockIdx.x; ti < ntl; ti += gridDim.x) {
    const int chain = ti / L, tt = ti - chain * L;
    const long r0 = (long)chain * a.G.rpc + 64 + (long)tt * a.G.b;
    if (r0 >= a.G.nrows) continue;
    double* coef = a.Coef + (long)ti * NT1 * 64;
    const double* slot = a.TG + (long)ti * a.tg_stride;
    __syncthreads();
    load_tile_async(Cxs, 64, slot + PW, NT1, 0, PW, 0, PW, 0, 64, 64, tid, NT);
    load_tile_async(Ks, 64, coef + (long)PW * 64, 64, 0, 64, 0, 64, 0, 64, 64, tid, NT);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (live) {
      double w[4][2][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) w[i][j][0] = w[i][j][1] = 0.0;
#pragma unroll 4
      for (int kk = 0; kk < 16; ++kk) {
        double zf[4], cf[4], bf[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          zf[i] = Z1s[swz(32 * band + 8 * i + g, 4 * kk + t, 64)];
          cf[i] = Cxs[swz(32 * band + 8 * i + g, 4 * kk + t, 64)];
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) bf[j] = Ks[swz(4 * kk + t, c0 + 8 * j + g, 64)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            dmma(w[i][j], zf[i], bf[j]);
            dmma(y[i][j], cf[i], bf[j]);
          }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int r = 32 * band + 8 * i + g, c = c0 + 8 * j + 2 * t;
          *reinterpret_cast<double2*>(coef + (long)r * 64 + c) = make_double2(w[i][j][0], w[i][j][1]);
        }
    }
  }
  cp_async_wait<0>();
  if (live) {
    double* out = ypart + (long)blockIdx.x * PW * 64;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = 32 * band + 8 * i + g, c = c0 + 8 * j + 2 * t;
        *reinterpret_cast<double2*>(out + (long)r * 64 + c) = make_double2(y[i][j][0], y[i][j][1]);
      }
  }
}

// rows < k0 of every tile coefficient += Z2
__global__ void coef_add_z2_kernel(FastArgs a, const double* Z2, int ldz) {
  const int NT1 = a.PW + 64;
  const int L = a.G.L, ntl = a.G.nchains * L;
  const int per = a.k0 * 32;                                 // double2 units per tile
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < (long)ntl * per;
       e += (long)gridDim.x * blockDim.x) {
    const int ti = (int)(e / per), q = (int)(e - (long)ti * per);
    const int r = q >> 5, c = (q & 31) * 2;
    double2* p = reinterpret_cast<double2*>(a.Coef + (long)ti * NT1 * 64 + (long)r * 64 + c);
    double2 v = *p;
    if (c < a.k) v.x += Z2[(long)r * ldz + c];
    if (c + 1 < a.k) v.y += Z2[(long)r * ldz + c + 1];
    *p = v;
  }
}

// ============================================================================
// final: Q rows of every tall tile = ([V_t | A_t] Coef_t) diag(s); 128-row
// sub-tiles handed out by a ticket counter, K = PW + 64 in 32-column chunks
// (V chunks, then the two A chunks), the coefficient chunk beside it -- the
// tsgemm_nn pipeline with a per-tile right operand.
// ============================================================================
// NOUT = 64: the real pipeline (K = PW + 64: V chunks, then two A chunks).
// NOUT = 128: the complex Q formation on interleaved real views (zpath.inc):
// Q_tile' = X_tile' E_t in place, K = 128 from the V operand only, 64-row sub-tiles.
template <int NOUT>
struct FnCfg {
  static constexpr int RT = NOUT == 64 ? 128 : 64, KC = 32, NT = 256, NSTAGE = 2;
  // padded-linear stage rows (bulk-copy friendly, see TgCfg): the row-major A
  // operand (8 rows x 4 columns per fragment) wants a pitch = 32 bytes mod 128,
  // the B operand (4 rows x 8 columns) 64 bytes mod 128
  static constexpr int PP = KC + 4, PZ = NOUT + 8;
  static constexpr int STAGE = RT * PP + KC * PZ;
  static constexpr int SMEM = NSTAGE * STAGE * 8;
};

template <int NOUT>
__global__ void __launch_bounds__(256, 2) final_nn_kernel(FastArgs a, const double* colscale, double* X, long ldx,
                                                          int ncols_out) {
  using C = FnCfg<NOUT>;
  constexpr int PP = C::PP, PZ = C::PZ;
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) unsigned long long full_bar[C::NSTAGE];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = NOUT == 64 ? (warp >> 1) * 32 : (warp >> 2) * 32;
  const int wn0 = NOUT == 64 ? (warp & 1) * 32 : (warp & 3) * 32;
  const int nchA = a.k > 0 ? 2 : 0;
  const int NT1 = a.PW + 32 * nchA;
  const int L = a.G.L;
  const int spt = a.G.b / C::RT;                             // sub-tiles per tall tile
  const long nsub = (long)a.G.nchains * L * spt;
  const int nchV = a.PW / C::KC, nchunks = nchV + nchA;
  const bool bulk_ok = !(a.k0 & 1) && !(a.k & 1);
  __shared__ long s_tile[3];
  if (tid == 0) {
    s_tile[0] = blockIdx.x;
    s_tile[1] = gridDim.x + atomicAdd(a.ticket, 1);
    for (int s = 0; s < C::NSTAGE; ++s) mbar_init(&full_bar[s], C::NT);
    fence_mbar_init();
  }
  __syncthreads();
  auto tile_of = [&](long lt) { return s_tile[lt % 3]; };
  auto geom = [&](long st, int& ti, long& r0, long& rhi) {  // sub-tile -> tall tile, rows
    ti = (int)(st / spt);
    const int sub = (int)(st - (long)ti * spt);
    const int chain = ti / L, tt = ti - chain * L;
    const long g0 = (long)chain * a.G.rpc + 64 + (long)tt * a.G.b;
    rhi = g0 + a.G.b < a.G.nrows ? g0 + a.G.b : a.G.nrows;
    r0 = g0 + (long)sub * C::RT;
  };
  // Stage it: rows of V (chunks < nchV) or A columns ch * 32 .. of one 128-row
  // sub-tile and the matching 32 coefficient rows.  Full chunks: one bulk copy
  // per row (threads 0..127 an operand row, 128..159 a coefficient row),
  // completing on the stage's mbarrier by bytes; chunks cut by the sub-tile's
  // last row or by k0 / k: 16-byte cp.async units with zero fill.
  auto issue = [&](long it) {
    const long lt = it / nchunks;
    const long st = tile_of(lt);
    const int s = (int)(it % C::NSTAGE);
    if (st >= nsub) return;
    int ti;
    long r0, rhi;
    geom(st, ti, r0, rhi);
    const int ch = (int)(it - lt * nchunks);
    double* Ps = smem + s * C::STAGE;
    double* Zs = Ps + C::RT * PP;
    const bool isV = ch < nchV;
    const double* src = isV ? a.V : a.A;
    const long lds = isV ? a.ldv : a.lda;
    const int c0 = (isV ? ch : ch - nchV) * C::KC, cmax = isV ? a.k0 : a.k;
    const double* coef = a.Coef + (long)ti * NT1 * NOUT + (long)ch * C::KC * NOUT;
    if (bulk_ok && r0 + C::RT <= rhi && c0 + C::KC <= cmax) {
      if (tid < C::RT) bulk_g2s(Ps + tid * PP, src + (r0 + tid) * lds + c0, C::KC * 8, &full_bar[s]);
      else if (tid < C::RT + C::KC) bulk_g2s(Zs + (tid - C::RT) * PZ, coef + (long)(tid - C::RT) * NOUT, NOUT * 8, &full_bar[s]);
      if (tid == 0) mbar_arrive_expect_tx(&full_bar[s], (C::RT * C::KC + C::KC * NOUT) * 8);
      else mbar_arrive(&full_bar[s]);
    } else {
#pragma unroll
      for (int q = 0; q < C::RT * (C::KC / 2) / C::NT; ++q) {          // 2048 units: unit u of rows rb, rb + 16, ...
        const int i = tid + q * C::NT, r = i >> 4, u = i & 15;
        const int c = c0 + 2 * u;
        const bool in = r0 + r < rhi && c < cmax;
        cp_async16(Ps + r * PP + 2 * u, in ? src + (r0 + r) * lds + c : src, in ? (c + 1 < cmax ? 16 : 8) : 0);
      }
#pragma unroll
      for (int q = 0; q < C::KC * (NOUT / 2) / C::NT; ++q) {             // units of the coefficient rows
        const int i = tid + q * C::NT, r = i / (NOUT / 2), u = i - r * (NOUT / 2);
        cp_async16(Zs + r * PZ + 2 * u, coef + (long)r * NOUT + 2 * u, 16);
      }
      cp_async_mbar_arrive(&full_bar[s]);
    }
  };
  unsigned negmask = 0;
  if (colscale) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = wn0 + 8 * j + 2 * t;
      if (c < ncols_out && colscale[c] < 0.0) negmask |= 1u << (2 * j);
      if (c + 1 < ncols_out && colscale[c + 1] < 0.0) negmask |= 1u << (2 * j + 1);
    }
  }
  double acc[4][4][2];
  issue(0);
  for (long it = 0;; ++it) {
    const long lt = it / nchunks;
    const int ch = (int)(it - lt * nchunks);
    const long st = tile_of(lt);
    if (st >= nsub) break;
    if (ch == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    __syncthreads();                                         // everyone is done with the other stage
    if (ch == 0 && tid == 0) s_tile[(lt + 2) % 3] = gridDim.x + atomicAdd(a.ticket, 1);
    issue(it + 1);
    const int s = (int)(it % C::NSTAGE);
    mbar_wait(&full_bar[s], (unsigned)((it / C::NSTAGE) & 1));
    const double* Ps = smem + s * C::STAGE;
    const double* Zs = Ps + C::RT * PP;
#pragma unroll
    for (int kk = 0; kk < C::KC / 4; ++kk) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = Ps[(wm0 + 8 * i + g) * PP + 4 * kk + t];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Zs[(4 * kk + t) * PZ + wn0 + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
    if (ch == nchunks - 1) {
      int ti;
      long r0, rhi;
      geom(st, ti, r0, rhi);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const long r = r0 + wm0 + 8 * i + g;
          const int c = wn0 + 8 * j + 2 * t;
          if (r >= rhi) continue;
          double y0 = acc[i][j][0], y1 = acc[i][j][1];
          if (negmask) {
            const unsigned long long f0 = ((negmask >> (2 * j)) & 1u) ? 0x8000000000000000ull : 0ull;
            const unsigned long long f1 = ((negmask >> (2 * j + 1)) & 1u) ? 0x8000000000000000ull : 0ull;
            y0 = __longlong_as_double(__double_as_longlong(y0) ^ f0);
            y1 = __longlong_as_double(__double_as_longlong(y1) ^ f1);
          }
          double* p = X + r * ldx + c;
          if (c + 1 < ncols_out) __stcs(reinterpret_cast<double2*>(p), make_double2(y0, y1));
          else if (c < ncols_out) p[0] = y0;
        }
    }
  }
  cp_async_wait<0>();
}

// flags[0] |= any chain flag
__global__ void fast_flags_kernel(const int* chain_flags, int nch, int* flags) {
  if (*flags) return;                                        // the sweep did not run
  int bad = 0;
  for (int i = threadIdx.x; i < nch; i += blockDim.x) bad |= chain_flags[i];
  if (bad) atomicOr(flags, 2);
}

// ============================================================================
// launchers
// ============================================================================
static int fast_nsm() {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return nsm;
}

cudaError_t launch_tgram(const FastArgs& a, int grid, cudaStream_t st) {
  if (a.G.L < 1 || a.PW != 128) return cudaErrorInvalidValue;
  cudaFuncSetAttribute(tgram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TgCfg::SMEM);
  tgram_kernel<<<grid, TgCfg::NT, TgCfg::SMEM, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_tgram_reduce(const FastArgs& a, int nparts, const double* Vtop, int ntop, double* out, int ldg,
                                cudaStream_t st) {
  const int NT1 = a.PW + 64, count = a.PW * NT1;
  tgram_reduce_kernel<<<(count + 127) / 128, 128, 0, st>>>(a.part, nparts, a.PW, NT1, Vtop, a.ldv, ntop, a.k0, out,
                                                          ldg);
  return cudaGetLastError();
}

cudaError_t launch_head_rows(const FastArgs& a, int mode, const double* Z, int ldz, const double* colscale,
                             double* part, int grid, cudaStream_t st) {
  const int smem = (64 * 33 + 64 * 65) * 8;
  cudaFuncSetAttribute(head_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  head_rows_kernel<<<grid, 256, smem, st>>>(a, mode, Z, ldz, colscale, part);
  return cudaGetLastError();
}

template <int PW>
static cudaError_t launch_tile_alg_t(const FastArgs& a, cudaStream_t st) {
  auto k = tile_alg_kernel<PW>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TaCfg<PW>::SMEM);
  const int ntl = a.G.nchains * a.G.L, nsm = fast_nsm();
  if (a.ticket) {
    cudaError_t e = cudaMemsetAsync(a.ticket, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
  }
  k<<<ntl < nsm ? ntl : nsm, 512, TaCfg<PW>::SMEM, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_tile_alg(const FastArgs& a, cudaStream_t st) {
  switch (a.PW) {
    case 32: return launch_tile_alg_t<32>(a, st);
    case 64: return launch_tile_alg_t<64>(a, st);
    case 96: return launch_tile_alg_t<96>(a, st);
    case 128: return launch_tile_alg_t<128>(a, st);
  }
  return cudaErrorInvalidValue;
}

template <int PW>
static cudaError_t launch_coef_b_t(const FastArgs& a, double* ypart, int grid, cudaStream_t st) {
  auto k = coef_b_kernel<PW>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, CbCfg<PW>::SMEM);
  k<<<grid, 512, CbCfg<PW>::SMEM, st>>>(a, ypart);
  return cudaGetLastError();
}

cudaError_t launch_coef_b(const FastArgs& a, double* ypart, int grid, cudaStream_t st) {
  switch (a.PW) {
    case 32: return launch_coef_b_t<32>(a, ypart, grid, st);
    case 64: return launch_coef_b_t<64>(a, ypart, grid, st);
    case 96: return launch_coef_b_t<96>(a, ypart, grid, st);
    case 128: return launch_coef_b_t<128>(a, ypart, grid, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_coef_add_z2(const FastArgs& a, const double* Z2, int ldz, cudaStream_t st) {
  coef_add_z2_kernel<<<fast_nsm() * 4, 256, 0, st>>>(a, Z2, ldz);
  return cudaGetLastError();
}

template <int NOUT>
static cudaError_t launch_final_nn_t(const FastArgs& a, const double* colscale, double* X, long ldx, int ncols_out,
                                     cudaStream_t st) {
  using C = FnCfg<NOUT>;
  if (a.G.b % C::RT || !a.ticket) return cudaErrorInvalidValue;
  auto k = final_nn_kernel<NOUT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  const long nsub = (long)a.G.nchains * a.G.L * (a.G.b / C::RT);
  const int nsm = fast_nsm();
  const int grid = (int)(nsub < 2L * nsm ? nsub : 2L * nsm);
  cudaError_t e = cudaMemsetAsync(a.ticket, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  k<<<grid, C::NT, C::SMEM, st>>>(a, colscale, X, ldx, ncols_out);
  return cudaGetLastError();
}

cudaError_t launch_final_nn(const FastArgs& a, const double* colscale, double* X, long ldx, cudaStream_t st) {
  return launch_final_nn_t<64>(a, colscale, X, ldx, a.k, st);
}

// complex Q formation on real views: X (rows x ncols_out, in place) <- X E_t per
// tall tile, E_t = a.Coef + tile * 128 * 128 (a.V = X, a.k0 = a.PW = 128, a.k = 0)
cudaError_t launch_final_nn128(const FastArgs& a, double* X, long ldx, int ncols_out, cudaStream_t st) {
  if (a.PW != 128 || a.k != 0) return cudaErrorInvalidValue;
  return launch_final_nn_t<128>(a, nullptr, X, ldx, ncols_out, st);
}

cudaError_t launch_fast_flags(const int* chain_flags, int nch, int* flags, cudaStream_t st) {
  fast_flags_kernel<<<1, 256, 0, st>>>(chain_flags, nch, flags);
  return cudaGetLastError();
}

}  // namespace ots
