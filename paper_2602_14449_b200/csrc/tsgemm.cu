// Tall-skinny FP64 contractions on DMMA (sm_100a).
//
//  tsgemm_tn : C(PW x NTOT) = sum_rows  P^T [P | B]   (reduction over n rows)
//              -- the inner-product blocks V^*V, V^*A (reflector.py:220,236)
//                 and V^*Q_ (reflector.py:236 via twostage.py:96).
//  tsgemm_nn : X = (B + P Z) * diag(colscale)         (row-local update)
//              -- the reflector update  x - W (T-solve) y  (reflector.py:238)
//                 on the n-row part, with W_bottom = -V implicit.
//
// Both stream row tiles HBM -> smem with multi-stage cp.async (16 B, zero
// fill), swizzled so every m8n8k4 fragment load is conflict-minimal, and keep
// the k0 x k accumulators in registers for the whole CTA lifetime (tn) or per
// row tile (nn).  Cross-CTA sums go through a fixed-order reduction
// (deterministic, run-to-run bit reproducible).
#include "common.cuh"
#include "kernels.cuh"

namespace ots {

// cp.async.bulk global -> shared row copy completing on an mbarrier by bytes,
// and the arrival that posts a stage's byte count
__device__ __forceinline__ void nn_bulk_g2s(void* smem, const void* gmem, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void nn_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}

// ============================================================================
// TN: per-CTA partial inner products
// ============================================================================

template <int PW, int BW, bool ALIAS, bool SYM>
struct TnCfg {
  static constexpr int MB = PW / 32;
  static constexpr int NBV = ALIAS ? PW / 32 : 0;
  static constexpr int NBB = BW / 32;
  static constexpr int NVT = ALIAS ? (SYM ? MB * (MB + 1) / 2 : MB * MB) : 0;
  static constexpr int NFULL = NVT + MB * NBB;
  // Balance DMMA work over the 4 SM sub-partitions (warp w -> SMSP w % 4):
  // when NFULL = 2 mod 4, split the last two 32x32 tasks into 32x16 halves.
  static constexpr int NSPLIT = (NFULL % 4 == 2 && NFULL > 4) ? 2 : 0;
  static constexpr int NTASK = NFULL + NSPLIT;      // warps
  static constexpr int NT = NTASK * 32;
  // 64-row stages (two in flight) for the wide headline shapes: half the
  // ring hand-offs per DMMA of 32-row stages (measured: gram 19.5 -> 18.4 ms)
  // (for the cross product V^T Q_ it measured slower: 8.87 -> 9.15 ms)
  static constexpr int RT = (PW == 128 && BW == 64 && ALIAS) ? 64 : 32;
  // Stage rows are stored linearly with padded pitches (a row advances 64
  // bytes of bank space: the 4 rows x 8 columns of an operand fragment take
  // the 2-wavefront minimum), the layout bulk row copies (cp.async.bulk) write.
  static constexpr int PPW = PW + 8, PBW = BW > 0 ? BW + 8 : 0;
  static constexpr int STAGE = RT * (PPW + PBW);
  static constexpr int NSTAGE_RAW = (220 * 1024) / (STAGE * 8);
  static constexpr int NSTAGE = NSTAGE_RAW > 4 ? 4 : (NSTAGE_RAW < 2 ? 2 : NSTAGE_RAW);
  static constexpr int SMEM = NSTAGE * STAGE * 8;
  static constexpr int NTOT = NBV * 32 + BW;
};

template <int PW, int BW, bool ALIAS, bool SYM>
__global__ void __launch_bounds__(TnCfg<PW, BW, ALIAS, SYM>::NT, 1)
tsgemm_tn_kernel(TnArgs a) {
  using C = TnCfg<PW, BW, ALIAS, SYM>;
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;

  // task decode: V-part (mi, ni<=mi or all) then B-part; the last NSPLIT
  // full tasks become 2*NSPLIT half tasks (n-range of 16 columns each)
  int mi = 0, ni = 0, nhalf = 0;
  bool fromP = false, half = false;
  {
    // Diagonal Gram blocks only form their lower-triangular fragments (10 of
    // 16 DMMAs; every consumer reads the lower triangle), which unbalances the
    // SM sub-partitions (warp w -> SMSP w % 4); for the hot 128 | 64 shape a
    // swap of tasks 3 and 9 restores 66 DMMA units on each SMSP.
    int w = warp;
    if (PW == 128 && BW == 64 && ALIAS && SYM) w = (warp == 3) ? 9 : (warp == 9 ? 3 : warp);
    if (C::NSPLIT && w >= C::NFULL - C::NSPLIT) {
      const int hw = w - (C::NFULL - C::NSPLIT);     // 0 .. 2*NSPLIT-1
      w = C::NFULL - C::NSPLIT + hw / 2;
      half = true;
      nhalf = hw & 1;
    }
    if (w < C::NVT) {
      fromP = true;
      for (int m = 0; m < C::MB; ++m) {
        int cnt = SYM ? (m + 1) : C::MB;
        if (w < cnt) { mi = m; ni = w; break; }
        w -= cnt;
      }
    } else {
      w -= C::NVT;
      mi = w / (C::NBB > 0 ? C::NBB : 1);
      ni = w - mi * C::NBB;
    }
  }

  const long r_lo = a.row_begin + (long)blockIdx.x * a.rows_per_cta;
  long r_hi = r_lo + a.rows_per_cta;
  if (r_hi > a.row_end) r_hi = a.row_end;
  const int ntiles = r_hi > r_lo ? (int)((r_hi - r_lo + C::RT - 1) / C::RT) : 0;
  const long plo = a.row_begin > a.p_row_begin ? a.row_begin : a.p_row_begin;
  const long blo = a.row_begin > a.b_row_begin ? a.row_begin : a.b_row_begin;

  auto stage_p = [&](int s) { return smem + s * C::STAGE; };
  auto stage_b = [&](int s) { return smem + s * C::STAGE + C::RT * C::PPW; };
  // mbarrier ring instead of a CTA barrier per stage: every thread issues its
  // share of tile it+LA (cp.async, then cp.async.mbarrier.arrive on full[s])
  // once all warps have released that stage (empty[s], one arrival per warp);
  // a warp computes tile it after full[s].  Warps may drift LA tiles apart, so
  // per-stage work imbalance no longer stalls the whole CTA.
  // tiles issued ahead: the Gram (ALIAS) warps are balanced, the cross-product
  // warps gain from 2 tiles of slack (measured: gram2 10.1 -> 8.9 ms)
  constexpr int LA = ALIAS ? C::NSTAGE - 1 : (C::NSTAGE - 2 > 0 ? C::NSTAGE - 2 : 1);
  __shared__ __align__(8) unsigned long long full_bar[C::NSTAGE], empty_bar[C::NSTAGE];
  if (tid == 0) {
    for (int s = 0; s < C::NSTAGE; ++s) {
      mbar_init(&full_bar[s], C::NT);
      mbar_init(&empty_bar[s], C::NTASK);
    }
    fence_mbar_init();
  }
  // Full stages: one bulk copy per row (threads 0 .. RT-1 a P row, RT .. 2RT-1 a
  // B row), completing on the stage's mbarrier by bytes, thread 0 posts the byte
  // count; stages cut by the row ranges, odd widths / offsets: 16-byte cp.async
  // units with zero fill.  Columns beyond pcols / bcols are zeroed once (bulk
  // copies never touch them).
  constexpr bool BULK_T = C::NT >= C::RT * (BW > 0 ? 2 : 1);
  const bool bulk_ok = BULK_T && !(a.pcols & 1) && !(a.pc0 & 1) && !(a.ldp & 1) &&
                       (reinterpret_cast<uintptr_t>(a.P) & 15) == 0 &&
                       (BW == 0 || (!(a.bcols & 1) && !(a.bc0 & 1) && !(a.ldb & 1) &&
                                    (reinterpret_cast<uintptr_t>(a.B) & 15) == 0));
  if (bulk_ok) {
    for (int e = tid; e < C::NSTAGE * C::STAGE; e += C::NT) smem[e] = 0.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  auto produce = [&](int j) {
    if (j >= ntiles) return;
    const int s = j % C::NSTAGE, rnd = j / C::NSTAGE;
    if (rnd >= 1) mbar_wait(&empty_bar[s], (rnd - 1) & 1);
    const long r0 = r_lo + (long)j * C::RT;
    double* Ps = stage_p(s);
    double* Bs = stage_b(s);
    if (bulk_ok && r0 >= plo && r0 + C::RT <= r_hi && (BW == 0 || r0 >= blo)) {
      if (tid < C::RT)
        nn_bulk_g2s(Ps + tid * C::PPW, a.P + (r0 + tid) * a.ldp + a.pc0, (unsigned)a.pcols * 8u, &full_bar[s]);
      else if (BW > 0 && tid < 2 * C::RT)
        nn_bulk_g2s(Bs + (tid - C::RT) * C::PBW, a.B + (r0 + tid - C::RT) * a.ldb + a.bc0, (unsigned)a.bcols * 8u,
                    &full_bar[s]);
      if (tid == 0) nn_arrive_expect_tx(&full_bar[s], (unsigned)(C::RT * (a.pcols + (BW > 0 ? a.bcols : 0))) * 8u);
      else mbar_arrive(&full_bar[s]);
    } else {
      for (int i = tid; i < C::RT * (PW / 2); i += C::NT) {
        const int r = i / (PW / 2), u = i - r * (PW / 2);
        const long gr = r0 + r;
        const int c = 2 * u;
        const bool in = gr >= plo && gr < r_hi && c < a.pcols;
        cp_async16(Ps + r * C::PPW + c, in ? a.P + gr * a.ldp + a.pc0 + c : a.P, in ? (c + 1 < a.pcols ? 16 : 8) : 0);
      }
      if (BW > 0) {
        for (int i = tid; i < C::RT * (BW / 2 > 0 ? BW / 2 : 1); i += C::NT) {
          const int r = i / (BW / 2 > 0 ? BW / 2 : 1), u = i - r * (BW / 2 > 0 ? BW / 2 : 1);
          const long gr = r0 + r;
          const int c = 2 * u;
          const bool in = gr >= blo && gr < r_hi && c < a.bcols;
          cp_async16(Bs + r * C::PBW + c, in ? a.B + gr * a.ldb + a.bc0 + c : a.B, in ? (c + 1 < a.bcols ? 16 : 8) : 0);
        }
      }
      cp_async_mbar_arrive(&full_bar[s]);
    }
  };
  for (int j = 0; j < LA; ++j) produce(j);

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int it = 0; it < ntiles; ++it) {
    produce(it + LA);
    const int s = it % C::NSTAGE;
    mbar_wait(&full_bar[s], (it / C::NSTAGE) & 1);
    const double* Ps = stage_p(s);
    const double* Bs = fromP ? Ps : stage_b(s);
    const int BWs = fromP ? C::PPW : (BW > 0 ? C::PBW : 32);
    const int nb0 = fromP ? 32 * ni : 32 * ni;
    if (SYM && fromP && mi == ni && !half) {   // diagonal block: fragments i >= j only
#pragma unroll
      for (int kk = 0; kk < C::RT / 4; ++kk) {
        const int r = 4 * kk + t;
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = Ps[r * C::PPW + 32 * mi + 8 * i + g];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = Bs[r * BWs + nb0 + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j <= i; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
    } else if (!half) {
#pragma unroll
      for (int kk = 0; kk < C::RT / 4; ++kk) {
        const int r = 4 * kk + t;
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = Ps[r * C::PPW + 32 * mi + 8 * i + g];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = Bs[r * BWs + nb0 + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
    } else {
      const int nbh = nb0 + 16 * nhalf;
#pragma unroll
      for (int kk = 0; kk < C::RT / 4; ++kk) {
        const int r = 4 * kk + t;
        double af[4], bf[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = Ps[r * C::PPW + 32 * mi + 8 * i + g];
#pragma unroll
        for (int j = 0; j < 2; ++j) bf[j] = Bs[r * BWs + nbh + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
  }
  cp_async_wait<0>();

  // partial write
  double* out = a.partial + (long)blockIdx.x * PW * C::NTOT;
  const int ncol0 = (fromP ? 32 * ni : C::NBV * 32 + 32 * ni) + (half ? 16 * nhalf : 0);
  const int nj = half ? 2 : 4;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= nj) continue;
      int m = 32 * mi + 8 * i + g;
      int n = ncol0 + 8 * j + 2 * t;
      *reinterpret_cast<double2*>(out + (long)m * C::NTOT + n) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

// Fixed-order reduction of per-CTA partials: out[m][n] = sum_c partial[c][m][n]
// (optionally scaled by alpha and added to an existing value when accumulate).
__global__ void reduce_partials_kernel(const double* __restrict__ partial, int nparts, long count,
                                       double* __restrict__ out, double alpha) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int c = 0; c < nparts; ++c) s += partial[(long)c * count + i];
  out[i] = alpha * s;
}

// ============================================================================
// NN: X = (B + P Z) * diag(colscale) on rows [row_begin, row_end)
// ============================================================================

template <int KT>
struct NnCfg {
  static constexpr int WN = KT < 32 ? KT : 32;
  static constexpr int NWN = KT / WN;
  static constexpr int NWM = 8 / NWN;
  static constexpr int RT = NWM * 32;
  static constexpr int NT = 256;
  static constexpr int KC = 32;
  // Stage rows are stored linearly with padded pitches (the row-major A operand,
  // 8 rows x 4 columns per fragment, wants 32 bytes mod 128 per row, the B
  // operand, 4 rows x 8 columns, 64 bytes mod 128: two wavefronts per operand
  // load either way) so that full chunks can be written by bulk row copies
  // (cp.async.bulk, SASS UBLKCP) completing on an mbarrier by bytes.
  static constexpr int PP = KC + 4, PZ = KT + 8;
  static constexpr int STAGE = RT * PP + KC * PZ;
  static constexpr int NSTAGE = 2;                    // 2 CTAs / SM share the SM
  static constexpr int SMEM = NSTAGE * STAGE * 8;
};

template <int KT>
__global__ void __launch_bounds__(256, 2) tsgemm_nn_kernel(NnArgs a) {
  using C = NnCfg<KT>;
  constexpr int WN = C::WN;
  constexpr int NJ = WN / 8;
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp / C::NWN) * 32;
  const int wn0 = (warp % C::NWN) * WN;

  const long nrows = a.row_end - a.row_begin;
  const long ntiles_total = (nrows + C::RT - 1) / C::RT;
  const int nchunks = (a.kdim + C::KC - 1) / C::KC;
  // Tiles: the CTA's first tile is blockIdx.x; with a ticket counter the later
  // ones are handed out dynamically (gridDim.x + ticket), so CTAs that start
  // late -- e.g. on SMs held by the concurrent diagnostics kernel -- take fewer
  // tiles instead of stretching the tail.  Without it: static stride.
  // 3-slot ring: slot (lt % 3) holds local tile lt; tile lt+2 is fetched at
  // chunk 0 of tile lt, after a barrier that retires tile lt-1's slot.
  __shared__ long s_tile[3];
  __shared__ __align__(8) unsigned long long full_bar[C::NSTAGE];
  const bool dyn = a.tile_counter != nullptr;
  if (tid == 0) {
    s_tile[0] = blockIdx.x;
    s_tile[1] = dyn ? gridDim.x + atomicAdd(a.tile_counter, 1) : blockIdx.x + (long)gridDim.x;
    for (int s = 0; s < C::NSTAGE; ++s) mbar_init(&full_bar[s], C::NT);
    fence_mbar_init();
  }
  __syncthreads();
  constexpr int PP = C::PP, PZ = C::PZ;
  // bulk copies need 16-byte row pieces: even widths, and a full Z row (ncols = KT)
  const bool bulk_ok = !(a.kdim & 1) && a.ncols == KT && C::RT + C::KC <= C::NT && !(a.ldz & 1) && !(a.ldp & 1) &&
                       ((reinterpret_cast<uintptr_t>(a.Z) | reinterpret_cast<uintptr_t>(a.P)) & 15) == 0;
  auto tile_of = [&](long lt) { return s_tile[lt % 3]; };
  auto tile_r0 = [&](long lt) { return a.row_begin + tile_of(lt) * (long)C::RT; };
  // Stage it: columns ch * 32 .. of one RT-row tile of P and the matching 32
  // rows of Z.  Full chunks: one bulk copy per row (threads 0 .. RT-1 a P row,
  // RT .. RT+31 a Z row), thread 0 posts the byte count; chunks cut by the last
  // row or by kdim: 16-byte cp.async units with zero fill.
  auto issue = [&](long it) {
    const long lt = it / nchunks;
    if (tile_of(lt) >= ntiles_total) return;
    const int s = (int)(it % C::NSTAGE);
    const int ch = (int)(it - lt * nchunks);
    double* Ps = smem + s * C::STAGE;
    double* Zs = Ps + C::RT * PP;
    const long r0 = tile_r0(lt);
    if (bulk_ok && r0 + C::RT <= a.row_end && (ch + 1) * C::KC <= a.kdim) {
      if (tid < C::RT) nn_bulk_g2s(Ps + tid * PP, a.P + (r0 + tid) * a.ldp + ch * C::KC, C::KC * 8, &full_bar[s]);
      else if (tid < C::RT + C::KC)
        nn_bulk_g2s(Zs + (tid - C::RT) * PZ, a.Z + (long)(ch * C::KC + tid - C::RT) * a.ldz, KT * 8, &full_bar[s]);
      if (tid == 0) nn_arrive_expect_tx(&full_bar[s], (C::RT * C::KC + C::KC * KT) * 8);
      else mbar_arrive(&full_bar[s]);
    } else {
      for (int i = tid; i < C::RT * (C::KC / 2); i += C::NT) {
        const int r = i / (C::KC / 2), u = i - r * (C::KC / 2);
        const int c = ch * C::KC + 2 * u;
        const bool in = r0 + r < a.row_end && c < a.kdim;
        cp_async16(Ps + r * PP + 2 * u, in ? a.P + (r0 + r) * a.ldp + c : a.P, in ? (c + 1 < a.kdim ? 16 : 8) : 0);
      }
      for (int i = tid; i < C::KC * (KT / 2); i += C::NT) {
        const int r = i / (KT / 2), u = i - r * (KT / 2);
        const int zr = ch * C::KC + r, c = 2 * u;
        const bool in = zr < a.kdim && c < a.ncols;
        cp_async16(Zs + r * PZ + 2 * u, in ? a.Z + (long)zr * a.ldz + c : a.Z, in ? (c + 1 < a.ncols ? 16 : 8) : 0);
      }
      cp_async_mbar_arrive(&full_bar[s]);
    }
  };

  double acc[4][NJ][2];
  // this thread's output columns with a negative colscale (bit 2j+h)
  unsigned negmask = 0;
  if (a.colscale) {
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = wn0 + 8 * j + 2 * t;
      if (c < a.ncols && a.colscale[c] < 0.0) negmask |= 1u << (2 * j);
      if (c + 1 < a.ncols && a.colscale[c + 1] < 0.0) negmask |= 1u << (2 * j + 1);
    }
  }

  // accumulators start from B (so the epilogue is a plain store)
  auto acc_from_b = [&](long r0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        long r = r0 + wm0 + 8 * i + g;
        int c = wn0 + 8 * j + 2 * t;
        double x0 = 0.0, x1 = 0.0;
        if (a.B != nullptr && r < a.row_end) {
          const double* p = a.B + r * a.ldb + c;
          if (c + 1 < a.ncols) { double2 v = __ldcs(reinterpret_cast<const double2*>(p)); x0 = v.x; x1 = v.y; }
          else if (c < a.ncols) x0 = p[0];
        }
        acc[i][j][0] = x0; acc[i][j][1] = x1;
      }
  };
  auto epilogue_store = [&](long r0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        long r = r0 + wm0 + 8 * i + g;
        int c = wn0 + 8 * j + 2 * t;
        if (r >= a.row_end) continue;
        // colscale entries are +-1 (LAPACK sign recovery): flip the sign bit
        // with integer ops instead of DMULs competing with DMMA for the FP64 pipe
        double y0 = acc[i][j][0], y1 = acc[i][j][1];
        if (negmask) {
          const unsigned long long f0 = ((negmask >> (2 * j)) & 1u) ? 0x8000000000000000ull : 0ull;
          const unsigned long long f1 = ((negmask >> (2 * j + 1)) & 1u) ? 0x8000000000000000ull : 0ull;
          y0 = __longlong_as_double(__double_as_longlong(y0) ^ f0);
          y1 = __longlong_as_double(__double_as_longlong(y1) ^ f1);
        }
        double* p = a.X + r * a.ldx + c;
        if (c + 1 < a.ncols) __stcs(reinterpret_cast<double2*>(p), make_double2(y0, y1));
        else if (c < a.ncols) p[0] = y0;
      }
  };

  if (nchunks == 0) {  // X = B * colscale
    for (long r0 = a.row_begin + (long)blockIdx.x * C::RT; r0 < a.row_end; r0 += (long)gridDim.x * C::RT) {
      acc_from_b(r0);
      epilogue_store(r0);
    }
    return;
  }

#pragma unroll
  for (int s = 0; s < C::NSTAGE - 1; ++s) issue(s);

  for (long it = 0;; ++it) {
    const long lt = it / nchunks;
    const int ch = (int)(it - lt * nchunks);
    if (tile_of(lt) >= ntiles_total) break;
    if (ch == 0) acc_from_b(tile_r0(lt));
    __syncthreads();                                   // everyone is done with the other stage
    if (ch == 0 && tid == 0)
      s_tile[(lt + 2) % 3] = dyn ? gridDim.x + atomicAdd(a.tile_counter, 1) : tile_of(lt + 1) + gridDim.x;
    issue(it + C::NSTAGE - 1);
    if (ch == 1 && a.B != nullptr) {        // next tile's B rows -> L2 (acc_from_b reads them straight
      const long lt1 = lt + 1;             // into registers at its chunk 0)
      if (tile_of(lt1) < ntiles_total) {
        const long r1 = tile_r0(lt1);
        const int lpr = (a.ncols * 8 + 127) / 128;
        for (int i = tid; i < C::RT * lpr; i += C::NT) {
          const long r = r1 + i / lpr;
          if (r < a.row_end) {
            const double* ptr = a.B + r * a.ldb + (i % lpr) * 16;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
          }
        }
      }
    }
    const int s = (int)(it % C::NSTAGE);
    mbar_wait(&full_bar[s], (unsigned)((it / C::NSTAGE) & 1));
    const double* Ps = smem + s * C::STAGE;
    const double* Zs = Ps + C::RT * PP;
#pragma unroll
    for (int kk = 0; kk < C::KC / 4; ++kk) {
      double af[4], bf[NJ];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = Ps[(wm0 + 8 * i + g) * PP + 4 * kk + t];
#pragma unroll
      for (int j = 0; j < NJ; ++j) bf[j] = Zs[(4 * kk + t) * PZ + wn0 + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
    if (ch == nchunks - 1) epilogue_store(tile_r0(lt));
  }
  cp_async_wait<0>();
}

// ============================================================================
// host launchers
// ============================================================================
template <int PW, int BW, bool ALIAS, bool SYM>
static cudaError_t launch_tn_t(const TnArgs& a0, int grid, cudaStream_t st) {
  using C = TnCfg<PW, BW, ALIAS, SYM>;
  auto k = tsgemm_tn_kernel<PW, BW, ALIAS, SYM>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  TnArgs a = a0;
  long rows = a.row_end - a.row_begin;
  long per = (rows + grid - 1) / grid;
  per = (per + C::RT - 1) / C::RT * C::RT;
  if (per < C::RT) per = C::RT;
  a.rows_per_cta = per;
  k<<<grid, C::NT, C::SMEM, st>>>(a);
  return cudaGetLastError();
}

// Dispatch on padded widths.  PW in {32,64,96,128}; BW in {0,32,64}.
cudaError_t launch_tsgemm_tn(const TnArgs& a, int PW, int BW, bool alias, bool sym, int grid,
                             cudaStream_t st) {
#define OTS_TN(pw, bw, al, sy)                                                   \
  if (PW == pw && BW == bw && alias == al && sym == sy)                          \
    return launch_tn_t<pw, bw, al, sy>(a, grid, st);
  OTS_TN(32, 32, true, true) OTS_TN(32, 64, true, true) OTS_TN(64, 32, true, true) OTS_TN(64, 64, true, true)
  OTS_TN(96, 32, true, true) OTS_TN(96, 64, true, true)
  OTS_TN(128, 32, true, true) OTS_TN(128, 64, true, true)
  OTS_TN(32, 0, true, true) OTS_TN(64, 0, true, true) OTS_TN(96, 0, true, true) OTS_TN(128, 0, true, true)
  OTS_TN(32, 32, false, false) OTS_TN(64, 32, false, false) OTS_TN(96, 32, false, false)
  OTS_TN(128, 32, false, false) OTS_TN(32, 64, false, false) OTS_TN(64, 64, false, false)
  OTS_TN(96, 64, false, false) OTS_TN(128, 64, false, false)
  OTS_TN(128, 128, false, false) OTS_TN(128, 96, false, false) OTS_TN(96, 96, false, false)
  OTS_TN(64, 128, false, false) OTS_TN(96, 128, false, false) OTS_TN(32, 128, false, false)
#undef OTS_TN
  return cudaErrorInvalidValue;
}

// out[(m0+i)*ldo + n0 + j] = alpha * sum_c partial[c][i][j]   (i < rows, j < cols of a rows x ldp block)
__global__ void reduce_partials_strided_kernel(const double* __restrict__ partial, int nparts, int rows,
                                               int cols, int ldp, int prow, double* __restrict__ out,
                                               long ldo, double alpha) {
  long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long)rows * cols) return;
  const int i = (int)(e / cols), j = (int)(e - (long)i * cols);
  const long stride = (long)prow * ldp;   // per-CTA partial = padded rows x ldp
  double s = 0.0;
  for (int c = 0; c < nparts; ++c) s += partial[c * stride + (long)i * ldp + j];
  out[(long)i * ldo + j] = alpha * s;
}

cudaError_t launch_reduce_strided(const double* partial, int nparts, int rows, int cols, int ldp, double* out,
                                  long ldo, double alpha, cudaStream_t st) {
  long count = (long)rows * cols;
  const int prow = (rows + 31) / 32 * 32;
  reduce_partials_strided_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(partial, nparts, rows, cols,
                                                                                  ldp, prow, out, ldo, alpha);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const double* partial, int nparts, long count, double* out, double alpha,
                          cudaStream_t st) {
  int bs = 256;
  long nb = (count + bs - 1) / bs;
  reduce_partials_kernel<<<(unsigned)nb, bs, 0, st>>>(partial, nparts, count, out, alpha);
  return cudaGetLastError();
}

template <int KT>
static cudaError_t launch_nn_t(const NnArgs& a, int nsm, cudaStream_t st) {
  using C = NnCfg<KT>;
  auto k = tsgemm_nn_kernel<KT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  long rows = a.row_end - a.row_begin;
  if (rows <= 0) return cudaSuccess;
  long tiles = (rows + C::RT - 1) / C::RT;
  int grid = (int)(tiles < 2L * nsm ? tiles : 2L * nsm);
  if (a.tile_counter) {
    cudaError_t e = cudaMemsetAsync(a.tile_counter, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
  }
  k<<<grid, C::NT, C::SMEM, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_tsgemm_nn(const NnArgs& a, int KT, int nsm, cudaStream_t st) {
  if (KT == 16) return launch_nn_t<16>(a, nsm, st);
  if (KT == 32) return launch_nn_t<32>(a, nsm, st);
  if (KT == 64) return launch_nn_t<64>(a, nsm, st);
  if (KT == 128) return launch_nn_t<128>(a, nsm, st);   // 64-row tiles (complex real views)
  return cudaErrorInvalidValue;
}

}  // namespace ots
