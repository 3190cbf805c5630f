// C-ABI of the B200 two-stage orthogonalization (include/ots.h).
//
// Host orchestration of Algorithm 1 (twostage.py:57-97) as a fixed sequence of
// stream-ordered phases over row-sharded data:
//
//   gram    K1  G = [V^T V | V_b^T A_b]              (tsgemm_tn, DMMA)
//   seed    K2  defect check, P, T, W_t, Z1 = T^{-T}(W^T A), S   (small.cu)
//   diag        kappa(T), ||W T^{-1}||  -- side stream, overlaps the passes
//   apply1  K3a X = A_b + V_b Z1  (= (H^T A)_{k0+1:n})   (tsgemm_nn)
//   factor  K3b chain TSQR of X (+ tree levels)          (chainqr.cu)
//   qform   K5a explicit Q_ (tree levels down to rows)   (chainqr.cu)
//   sign        LAPACK sign recovery, R                  (small.cu)
//   gram2   K5c Y2 = -V_b^T Q_                           (tsgemm_tn)
//   z2          Z2 = T^{-1} Y2                           (small.cu)
//   apply2  K5b Q_b = (Q_ + V_b Z2) diag(s)              (tsgemm_nn)
//   qtop        Q_t = -W_t Z2 diag(s)                    (small.cu)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <cstdlib>

#include "common.cuh"
#include "small.cuh"
#include "ots.h"

#include "kernels.cuh"
namespace ots { cudaError_t fp64_peak(int nsm, cudaStream_t st, double* tflops); }

using namespace ots;

namespace {

inline int pad32(long x) { return (int)((x + 31) / 32 * 32); }
inline int kt_for(long k) { return k <= 16 ? 16 : (k <= 32 ? 32 : 64); }

__global__ void set_identity_kernel(double* D, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n * n) D[i] = (i / n == i % n) ? 1.0 : 0.0;
}
// core.py:75-83 phase fix for real: Q columns times sign(R_jj) (0 -> +1),
// then (second launch, one block) R rows likewise with |R_jj| on the diagonal
// -- two launches so no block reads a diagonal another block already rewrote.
__global__ void nonneg_q_kernel(double* Q, long ldq, long m, int k, const double* R, long ldr) {
  __shared__ double ph[64];
  for (int j = threadIdx.x; j < k; j += blockDim.x) ph[j] = (R[j * ldr + j] < 0.0) ? -1.0 : 1.0;
  __syncthreads();
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < m * k; e += (long)gridDim.x * blockDim.x) {
    long i = e / k; int j = (int)(e - i * k);
    Q[i * ldq + j] *= ph[j];
  }
}
__global__ void nonneg_r_kernel(int k, double* R, long ldr) {
  __shared__ double ph[64];
  for (int j = threadIdx.x; j < k; j += blockDim.x) ph[j] = (R[j * ldr + j] < 0.0) ? -1.0 : 1.0;
  __syncthreads();
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    int i = e / k, j = e - i * k;
    R[i * ldr + j] = (i == j) ? fabs(R[i * ldr + j]) : R[i * ldr + j] * ph[i];
  }
}
// complex: ph_j = R_jj / |R_jj| (1 for 0); Q <- Q diag(ph), R <- diag(conj ph) R
__device__ __forceinline__ double2 zphase(double2 d) {
  const double mg = hypot(d.x, d.y);
  return (mg != 0.0) ? make_double2(d.x / mg, d.y / mg) : make_double2(1.0, 0.0);
}
__global__ void zc_nonneg_q_kernel(double2* Q, long ldq, long m, int k, const double2* R, long ldr) {
  __shared__ double2 ph[64];
  for (int j = threadIdx.x; j < k; j += blockDim.x) ph[j] = zphase(R[j * ldr + j]);
  __syncthreads();
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < m * k; e += (long)gridDim.x * blockDim.x) {
    long i = e / k; int j = (int)(e - i * k);
    const double2 q = Q[i * ldq + j], p = ph[j];
    Q[i * ldq + j] = make_double2(q.x * p.x - q.y * p.y, q.x * p.y + q.y * p.x);
  }
}
__global__ void zc_nonneg_r_kernel(int k, double2* R, long ldr) {
  __shared__ double2 ph[64];
  for (int j = threadIdx.x; j < k; j += blockDim.x) ph[j] = zphase(R[j * ldr + j]);
  __syncthreads();
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    int i = e / k, j = e - i * k;
    const double2 r = R[i * ldr + j], p = ph[i];
    R[i * ldr + j] = (i == j) ? make_double2(hypot(r.x, r.y), 0.0)
                              : make_double2(r.x * p.x + r.y * p.y, r.y * p.x - r.x * p.y);
  }
}

struct Level {
  double* D; long ldd; int ncols;
  ChainGeom G;
  double* UT;     // per-tile U -> T
  double* R;      // stacked chain R's (nchains * KT rows, ld KT)
  double* CC = nullptr;   // level 0, KT = 64: per-tile Cc of the Gram-form factor
  double* HS = nullptr;   //   head rows per chain
  int* FL = nullptr;      //   per-chain redo flags
  ChainGeom G128{};       //   the same chains on 128-row tiles (exact redo)
};

}  // namespace

struct ots_ctx {
  int device = 0;
  int nsm = 148;
  cudaStream_t side = nullptr;   // highest priority: its few CTAs go first, the
                                 // dynamically scheduled apply1 tiles fill around them
  cudaEvent_t ev_seed = nullptr, ev_diag = nullptr, ev_seedA = nullptr, ev_fast = nullptr;
  int fast_taken = 0;            // last two_stage call went through the direct-Q pipeline
  int* nn_counter = nullptr;     // tile tickets of the NN updates
  char* ws = nullptr;
  size_t ws_size = 0;
  int* h_status = nullptr;   // pinned
  double* h_diag = nullptr;  // pinned
  std::string err;
  // profiling
  bool profile = false;
  std::vector<std::string> pnames;
  std::vector<cudaEvent_t> pev;
  std::vector<float> pms;
  std::vector<std::string> last_names;
  int launches = 0;
  char* b_ws = nullptr;      // B-inner scaled copies
  size_t b_size = 0;
  char* z_ws = nullptr;      // complex cholshift ping-pong buffer
  char* zgs_ws = nullptr;    // complex Gram-form intra QR workspace (zpath.inc)
  size_t zgs_size = 0;
  size_t z_size = 0;
  // distributed job state
  struct Job* job = nullptr;
};

namespace {

struct Arena {
  char* base; size_t off = 0, cap;
  Arena(char* b, size_t c) : base(b), cap(c) {}
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~(size_t)255;
    T* p = reinterpret_cast<T*>(base + off);
    off += n * sizeof(T);
    return p;
  }
};

int fail(ots_ctx* c, int code, const std::string& msg) { c->err = msg; return code; }

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess)                                                      \
      return fail(ctx, OTS_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

void prof_mark(ots_ctx* ctx, cudaStream_t st, const char* name) {
  if (!ctx->profile) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  ctx->pev.push_back(e);
  ctx->pnames.push_back(name);
}

void prof_begin(ots_ctx* ctx, cudaStream_t st) {
  for (auto e : ctx->pev) cudaEventDestroy(e);
  ctx->pev.clear();
  ctx->pnames.clear();
  prof_mark(ctx, st, "start");
}

void prof_end(ots_ctx* ctx) {
  if (!ctx->profile || ctx->pev.empty()) return;
  cudaEventSynchronize(ctx->pev.back());
  ctx->pms.clear();
  ctx->last_names.clear();
  for (size_t i = 1; i < ctx->pev.size(); ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, ctx->pev[i - 1], ctx->pev[i]);
    ctx->pms.push_back(ms);
    ctx->last_names.push_back(ctx->pnames[i]);
  }
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// -------------------------------------------------------------------------
// Job: one two-stage factorisation on this rank's rows.
// -------------------------------------------------------------------------
struct JobCfg {
  long n_local, row0, k0, k;
  const double* V; long ldv;
  const double* A; long lda;
  double* Q; long ldq;
  int choice; const double* Pexp; long ldp;
  double orth_tol; int allow_defect;
  cudaStream_t st;
  bool distributed;
  int nsm_avail = 0;     // SMs the row-parallel phases may plan for (0: all)
  const double* gram_in = nullptr; long ldgi = 0;   // caller's V^T V (incremental Gram), or null
  int ld_min = 0;        // small-state leading dimension at least this (reflector objects: fixed ld)
  // Row-weighted callers (B = diag(d), rows scaled by d^1/2 and the result by
  // d^-1/2): every row has to be accurate relative to its OWN norm, and the
  // register-tile kernel's constant there is about half the Gram form's
  // (tools/gs_accuracy.py), so those calls keep the exact level-0 factor.
  bool exact_intra = false;
  bool fast_try = false;   // caller allows the direct-Q pipeline (fastpath.cu) when the shape qualifies
};

}  // namespace

struct Job {
  JobCfg c;
  int PW = 32, BWa = 32, KT = 16, NTOT1 = 64, ld = 32;
  int grid_tn = 148, grid_tn2 = 148;
  int gram_nsm = 0;      // SMs of the Gram kernels (nsm - 1 when the seed runs beside them)
  bool seeded_early = false;   // row-sharded path: seedA already launched beside the Gram
  int nsm_use = 0;             // SMs the row-parallel phases are planned for
  long qrow0 = 0;        // first local row of the QR block (k0 on rank 0)
  long m = 0;            // local QR rows
  double *partial = nullptr, *Gfull = nullptr, *Y2full = nullptr, *top = nullptr;
  double *ident = nullptr, *svec = nullptr, *Cglob = nullptr;
  SmallState s{};
  std::vector<Level> lv;        // local levels (0 = data rows)
  std::vector<Level> glv;       // global tree levels over gathered rank R's
  double* Rall = nullptr;       // gathered R's copy (nranks*KT x KT)
  double* chol_ws = nullptr;    // 3 ld x ld scratch of the cholshift step
  double* Rfinal = nullptr;
  // direct-Q pipeline (fastpath.cu)
  bool fast = false;
  bool fast_active = false;     // row-sharded phases: this rank's factor took the direct-Q route
  double *fTG = nullptr, *fCoef = nullptr, *fpart = nullptr;
  long ftg_stride = 0;
  int* fflags = nullptr;        // [0] flags, [1] ticket
};

namespace ots { void gs_event_log(long long* out); }
namespace {

// level-0 chains per SM (2 = the two CTAs an SM holds); OTS_CHAINS_PER_SM
// overrides it for experiments
long chains_per_sm() {
  static long v = [] {
    const char* e = getenv("OTS_CHAINS_PER_SM");
    long x = e ? atol(e) : 2;
    return x >= 1 ? x : 2;
  }();
  return v;
}

// The Gram-form level-0 factor (gsweep.inc) for KT = 64 on tall tiles of
// gs_tile_rows() rows (2048 .. 8192 by size; OTS_GS_B overrides, a multiple of 128);
// OTS_GSWEEP=0 selects the register-tile kernel for every chain.
bool gsweep_on(int KT, int b) {
  static int v = [] {
    const char* e = getenv("OTS_GSWEEP");
    return e ? atoi(e) : 1;
  }();
  return v != 0 && KT == 64 && b == 128;
}

// The direct-Q pipeline (fastpath.cu): OTS_FAST=0 turns it off; calls with
// fewer QR rows than OTS_FAST_MIN_ROWS (default 2^19) keep the materialised-X
// pipeline (the extra small kernels and the host hand-off do not pay there).
bool fast_on() {
  static int v = [] {
    const char* e = getenv("OTS_FAST");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}
long fast_min_rows() {
  static long v = [] {
    const char* e = getenv("OTS_FAST_MIN_ROWS");
    long x = e ? atol(e) : (1L << 19);
    return x > 0 ? x : (1L << 19);
  }();
  return v;
}

// Tall-tile height of the Gram-form factor.  The sweep, the per-tile algebra
// and the coefficient kernels cost one unit per tile, so taller is cheaper
// (headline: 2048 -> 42.0 ms, 4096 -> 39.8, 8192 -> 38.7, parity unchanged),
// as long as every SM still gets a dozen tiles to balance over: 2048 rows,
// doubled up to 8192 while m / b >= 12 nsm.  OTS_GS_B overrides it.
int gs_tile_rows(long m, int nsm) {
  static int env = [] {
    const char* e = getenv("OTS_GS_B");
    int x = e ? atoi(e) : 0;
    return (x >= 128 && x % 128 == 0) ? x : 0;
  }();
  if (env) return env;
  int b = 2048;
  while (b < 8192 && m / (2 * b) >= 12L * nsm) b *= 2;
  return b;
}

// level-0 chain geometry: tiles of b rows, rows split over chains_per_sm * nsm chains
// fan-in of the reduction tree over the chain R's (OTS_TREE_G, default 4)
int tree_fanin() {
  static int v = [] {
    const char* e = getenv("OTS_TREE_G");
    int x = e ? atoi(e) : 4;
    return (x >= 2 && x <= 4) ? x : 4;
  }();
  return v;
}

ChainGeom level0_geom(long m, int KT, int b, int nsm) {
  long target = chains_per_sm() * nsm;
  long per = (m + target - 1) / target;
  long Lt = per > KT ? (per - KT + b - 1) / b : 0;
  long rpc = KT + Lt * b;
  long nch = (m + rpc - 1) / rpc;
  if (nch < 1) nch = 1;
  return ChainGeom{m, b, (int)Lt, rpc, (int)nch};
}

std::vector<Level> plan_levels(Arena& ar, double* D0, long ldd0, int ncols0, long m, int KT, int nsm,
                                bool exact = false) {
  std::vector<Level> lv;
  // level 0
  {
    Level L{};
    L.D = D0; L.ldd = ldd0; L.ncols = ncols0;
    int b = chain_bmax(KT);
    if (b > 128 && KT == 64) b = 128;
    const bool gs = !exact && gsweep_on(KT, b);
    L.G = level0_geom(m, KT, gs ? gs_tile_rows(m, nsm) : b, nsm);
    const long nch = L.G.nchains;
    if (gs) {
      const int f = L.G.b / b;
      L.G128 = ChainGeom{m, b, L.G.L * f, L.G.rpc, L.G.nchains};
      L.UT = ar.take<double>((size_t)nch * (L.G128.L + 1) * KT * KT);
      L.CC = ar.take<double>((size_t)nch * (L.G.L + 1) * KT * KT);
      L.HS = ar.take<double>((size_t)nch * KT * KT);
      L.FL = ar.take<int>((size_t)nch);
    } else {
      L.UT = ar.take<double>((size_t)nch * (L.G.L + 1) * KT * KT);
    }
    L.R = ar.take<double>((size_t)nch * KT * KT);
    lv.push_back(L);
  }
  while (lv.back().G.nchains > 1) {
    const Level& P = lv.back();
    Level L{};
    L.D = P.R; L.ldd = KT; L.ncols = KT;
    long nrows = (long)P.G.nchains * KT;
    int g = tree_fanin();
    long rpc = (long)KT * g;
    long nch = (nrows + rpc - 1) / rpc;
    L.G = ChainGeom{nrows, KT, g - 1, rpc, (int)nch};
    L.UT = ar.take<double>((size_t)nch * g * KT * KT);
    L.R = ar.take<double>((size_t)nch * KT * KT);
    lv.push_back(L);
  }
  return lv;
}

size_t plan_levels_bytes(long m, int KT, int nsm, bool exact = false) {
  // mirror of plan_levels' allocations (+ alignment slack)
  size_t tot = 0;
  int b = chain_bmax(KT);
  if (b > 128 && KT == 64) b = 128;
  const bool gs = !exact && gsweep_on(KT, b);
  const ChainGeom G = level0_geom(m, KT, gs ? gs_tile_rows(m, nsm) : b, nsm);
  long nch = G.nchains;
  const long tslots = gs ? (long)G.L * (G.b / b) + 1 : G.L + 1;
  tot += ((size_t)nch * tslots * KT * KT + (size_t)nch * KT * KT) * 8 + 512;
  if (gs) tot += ((size_t)nch * (G.L + 1) * KT * KT + (size_t)nch * KT * KT) * 8 + nch * 4 + 1536;
  while (nch > 1) {
    long nrows = nch * KT;
    long rpc2 = (long)KT * tree_fanin();
    long n2 = (nrows + rpc2 - 1) / rpc2;
    tot += ((size_t)n2 * 4 * KT * KT + (size_t)n2 * KT * KT) * 8 + 512;
    nch = n2;
  }
  return tot;
}

int ensure_ws(ots_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->ws_size) return OTS_OK;
  if (ctx->ws) cudaFree(ctx->ws);
  ctx->ws = nullptr;
  ctx->ws_size = 0;
  size_t b = bytes + (bytes >> 3) + (1 << 20);
  CK(cudaMalloc(&ctx->ws, b));
  ctx->ws_size = b;
  return OTS_OK;
}

// tri_first: level 0's rows are already stacked R factors (the global tree);
// levels >= 1 always are.
int run_factor_levels(ots_ctx* ctx, std::vector<Level>& lv, int KT, cudaStream_t st, bool tri_first = false) {
  for (size_t l = 0; l < lv.size(); ++l) {
    Level& L = lv[l];
    FactorArgs fa{L.D, L.ldd, L.ncols, L.G, L.UT, L.R, (l > 0 || tri_first) ? 1 : 0};
    if (l == 0 && !tri_first && L.CC) {
      // Gram-form tall tiles (X untouched); chains beyond the cancellation
      // bound are redone by the register-tile kernel on 128-row tiles
      GsweepArgs ga{L.D, L.ldd, L.ncols, L.G, L.UT, L.R, L.CC, L.HS, L.FL, (long)L.G128.L + 1};
      CK(launch_gs_gram(ga, st));
      prof_mark(ctx, st, "gs_gram");
      CK(launch_chain_gsweep(ga, st));
      prof_mark(ctx, st, "gs_sweep");
      fa.G = L.G128;
      fa.head_tri = 2;                                 // redo the flagged chains exactly
      CK(launch_chain_factor(fa, KT, st));
      continue;
    }
    CK(launch_chain_factor(fa, KT, st));
  }
  return OTS_OK;
}

// Q-form from the top level (whose single chain gets C = Ctop) down to level 0.
int run_qform_levels(ots_ctx* ctx, std::vector<Level>& lv, int KT, const double* Ctop, cudaStream_t st,
                     int grid_max = 0) {
  const double* Cin = Ctop;
  for (int l = (int)lv.size() - 1; l >= 0; --l) {
    Level& L = lv[l];
    QformArgs qa{L.D, L.ldd, L.ncols, L.G, L.UT, Cin, grid_max};
    if (L.CC) {
      // Gram-form level 0: flagged chains from Y (128-row tiles), accepted
      // ones from X and Cc (tall tiles)
      qa.G = L.G128;
      qa.mode = 1;
      qa.flags = L.FL;
      qa.tslots = (long)L.G128.L + 1;
      CK(launch_chain_qform(qa, KT, st));
      qa.G = L.G;
      qa.mode = 2;
      qa.Cc = L.CC;
      qa.Hs = L.HS;
      CK(launch_gs_qform(qa, st));
    } else {
      CK(launch_chain_qform(qa, KT, st));
    }
    Cin = L.D;  // output rows of level l are the C's of level l-1's chains
  }
  return OTS_OK;
}

int grid_for_tn(int PW, int BW, bool alias, bool sym, int nsm) {
  // warps per CTA = number of 32x32 tasks; smem-limited residency.
  int mb = PW / 32;
  int nt = (alias ? (sym ? mb * (mb + 1) / 2 : mb * mb) : 0) + mb * (BW / 32);
  if (nt % 4 == 2 && nt > 4) nt += 2;   // mirrors TnCfg::NSPLIT
  const int RT = 32;                                   // mirrors TnCfg (padded pitches, 220 KB budget)
  int stage = RT * (PW + 8 + (BW > 0 ? BW + 8 : 0)) * 8;
  int nst = std::min(4, std::max(2, (220 * 1024) / stage));
  int smem = nst * stage;
  int by_smem = std::max(1, (227 * 1024) / (smem + 1024));
  int by_threads = std::max(1, 2048 / (nt * 32));
  int per = std::min(by_smem, by_threads);
  (void)nt;
  return nsm * per;
}

// Build the job (workspace layout + small-state pointers).
int job_setup(ots_ctx* ctx, Job& j, const JobCfg& c) {
  j.c = c;
  const long k0 = c.k0, k = c.k;
  j.PW = pad32(std::max<long>(k0, 1));
  j.BWa = k <= 32 ? 32 : 64;
  j.KT = kt_for(k);
  j.NTOT1 = j.PW + j.BWa;
  j.ld = std::max(std::max(j.PW, j.KT), c.ld_min);
  j.qrow0 = (c.row0 == 0) ? k0 : 0;
  j.m = c.n_local - j.qrow0;
  j.grid_tn = grid_for_tn(j.PW, j.BWa, true, true, ctx->nsm);
  const int nsm_use = (c.nsm_avail > 0 && c.nsm_avail < ctx->nsm) ? c.nsm_avail : ctx->nsm;
  j.nsm_use = nsm_use;
  j.grid_tn2 = grid_for_tn(j.PW, j.BWa, false, false, nsm_use);
  const int ld = j.ld, KT = j.KT;
  const int gmax = std::max(j.grid_tn, j.grid_tn2);
  const int PWk = pad32(std::max<long>(k, 1));
  size_t part_n = std::max((size_t)gmax * j.PW * j.NTOT1,
                           (size_t)grid_for_tn(PWk, 0, true, true, ctx->nsm) * PWk * PWk);
  if (k0 > 128) {
    part_n = std::max(part_n, (size_t)grid_for_tn(128, 0, true, true, ctx->nsm) * 128 * 128);
    part_n = std::max(part_n, (size_t)grid_for_tn(128, 128, false, false, ctx->nsm) * 128 * 128);
    part_n = std::max(part_n, (size_t)grid_for_tn(128, j.BWa, false, false, ctx->nsm) * 128 * j.BWa);
  }
  const size_t gf_n = std::max((size_t)j.PW * j.NTOT1, (size_t)PWk * PWk);
  size_t bytes = 0;
  bytes += part_n * 8 + 256;
  bytes += gf_n * 8 * 2 + 512;                                       // Gfull, Y2full
  bytes += (size_t)3 * ld * ld * 8 + 256;                            // cholshift scratch
  bytes += (size_t)k0 * (k0 + k + 2) * 8 + 256;                    // top rows
  bytes += (size_t)22 * ld * ld * 8 + 22 * 256;                    // small matrices + diag scratch
  bytes += (size_t)8 * ld * 8 + 10 * 256;                          // vectors, dlam, dcount
  bytes += (size_t)KT * KT * 8 * 2 + 1024;                         // ident, svec
  bytes += plan_levels_bytes(std::max<long>(j.m, 1), KT, nsm_use, c.exact_intra);
  // direct-Q pipeline: per-tall-tile Grams of [V | A] and coefficients
  j.fast = false;
  size_t f_tg = 0, f_coef = 0, f_part = 0;
  // (callers that bring their own V^T V are Krylov-type drivers whose new block A = L Q_prev lies
  // mostly in range(V): the attempt would be rejected after a wasted tile pass -- measured +13 ms
  // on the k0 = 128 step of configs[4] -- so they keep the materialised-X pipeline)
  if (c.fast_try && fast_on() && !c.gram_in && !c.exact_intra && c.ld_min == 0 &&
      k0 > 96 && k0 <= 128 && KT == 64 && gsweep_on(KT, 128) && j.m >= fast_min_rows()) {
    const ChainGeom G = level0_geom(j.m, KT, gs_tile_rows(j.m, nsm_use), nsm_use);
    if (G.L >= 1) {
      j.fast = true;
      const size_t ntl = (size_t)G.nchains * G.L;
      j.ftg_stride = (long)j.PW * (j.PW + 64) + 64 * 64;
      f_tg = ntl * (size_t)j.ftg_stride;
      f_coef = ntl * (size_t)(j.PW + 64) * 64;
      f_part = (size_t)2 * ctx->nsm * j.PW * (j.PW + 64);
      bytes += (f_tg + f_coef + f_part) * 8 + 1024 + 64;
    }
  }
  bytes += (size_t)64 * KT * KT * 8 * 4 + 4096;                    // global tree (<=64 ranks)
  bytes += 64;
  int rc = ensure_ws(ctx, bytes);
  if (rc) return rc;
  Arena ar(ctx->ws, ctx->ws_size);
  j.partial = ar.take<double>(part_n);
  j.Gfull = ar.take<double>(gf_n);
  j.Y2full = ar.take<double>(gf_n);
  j.chol_ws = ar.take<double>((size_t)3 * ld * ld);
  j.top = ar.take<double>((size_t)std::max<long>(k0, 1) * (k0 + k + 2));
  SmallState& s = j.s;
  s = SmallState{};
  s.k0 = (int)k0; s.k = (int)k; s.ld = ld;
  s.choice = c.choice; s.allow_defect = c.allow_defect; s.orth_tol = c.orth_tol;
  s.V = c.V; s.ldv = c.ldv; s.A = c.A; s.lda = c.lda;
  s.Gfull = j.Gfull; s.ldgf = j.NTOT1; s.gf_acol = j.PW;
  s.Pexp = c.Pexp; s.ldpe = (int)c.ldp;
  double** mats[] = {&s.G, &s.Vt, &s.At, &s.VbA, &s.P, &s.Tf, &s.Tdense, &s.Wt,
                     &s.Z1, &s.Z2, &s.X1, &s.X2, &s.D1, &s.D2, &s.Sd};
  for (auto m : mats) *m = ar.take<double>((size_t)ld * ld);
  for (auto& m : s.dg) m = ar.take<double>((size_t)ld * ld);
  s.dlam = ar.take<double>(4);
  s.dcount = ar.take<int>(4);
  s.pvec = ar.take<double>(ld); s.tau = ar.take<double>(ld); s.sig = ar.take<double>(ld);
  s.sig2 = ar.take<double>(ld); s.svec = ar.take<double>(std::max(ld, KT));
  s.piv = ar.take<int>(ld);
  s.diag = ar.take<double>(4);
  s.status = ar.take<int>(4);
  j.ident = ar.take<double>((size_t)KT * KT);
  j.svec = s.svec;
  j.lv = plan_levels(ar, c.Q + j.qrow0 * c.ldq, c.ldq, (int)k, std::max<long>(j.m, 1), KT, nsm_use, c.exact_intra);
  if (j.fast) {
    j.fTG = ar.take<double>(f_tg);
    j.fCoef = ar.take<double>(f_coef);
    j.fpart = ar.take<double>(f_part);
    j.fflags = ar.take<int>(16);
  }
  // (last: ots_dist_tree carves the global tree's levels from the workspace behind Cglob)
  j.Rall = ar.take<double>((size_t)64 * KT * KT);
  j.Cglob = ar.take<double>((size_t)64 * KT * KT);
  if (ar.off > ctx->ws_size) return fail(ctx, OTS_E_CUDA, "workspace plan overflow");
  return OTS_OK;
}

// K1: Gfull = [V^T V | V_b^T A_b] (PW x NTOT1).  k0 <= 128: one launch.  Larger
// k0: 128-column blocks of V -- diagonal blocks (alias, symmetric), lower
// off-diagonal blocks V_a^T V_b, and V_a^T A_b -- each reduced in place.
int phase_gram(ots_ctx* ctx, Job& j) {
  const JobCfg& c = j.c;
  const int k0 = (int)c.k0, k = (int)c.k;
  const int gnsm = j.gram_nsm > 0 ? j.gram_nsm : ctx->nsm;   // SMs the Gram kernels may use
  if (c.gram_in) {
    // V^T V supplied by the caller (assembled incrementally by the Alg. 3
    // driver from earlier blocks): only V_b^T A_b streams over V here
    CK(cudaMemcpy2DAsync(j.Gfull, (size_t)j.NTOT1 * 8, c.gram_in, (size_t)c.ldgi * 8, (size_t)k0 * 8, k0,
                         cudaMemcpyDeviceToDevice, c.st));
    for (int a0 = 0; a0 < k0; a0 += 128) {
      const int aw = std::min(128, k0 - a0), PWa = pad32(aw);
      TnArgs a{};
      a.P = c.V; a.ldp = c.ldv; a.pc0 = a0; a.pcols = aw;
      a.B = c.A; a.ldb = c.lda; a.bc0 = 0; a.bcols = k;
      a.row_begin = 0; a.row_end = c.n_local; a.b_row_begin = j.qrow0; a.p_row_begin = 0;
      a.partial = j.partial;
      const int grid = grid_for_tn(PWa, j.BWa, false, false, gnsm);
      CK(launch_tsgemm_tn(a, PWa, j.BWa, false, false, grid, c.st));
      CK(launch_reduce_strided(j.partial, grid, aw, k, j.BWa, j.Gfull + (long)a0 * j.NTOT1 + j.PW, j.NTOT1, 1.0,
                               c.st));
    }
    return OTS_OK;
  }
  if (k0 <= 128) {
    TnArgs a{};
    a.P = c.V; a.ldp = c.ldv; a.pc0 = 0; a.pcols = k0;
    a.B = c.A; a.ldb = c.lda; a.bc0 = 0; a.bcols = k;
    a.row_begin = 0; a.row_end = c.n_local;
    a.b_row_begin = j.qrow0; a.p_row_begin = 0;
    a.partial = j.partial;
    CK(launch_tsgemm_tn(a, j.PW, j.BWa, true, true, j.grid_tn, c.st));
    CK(launch_reduce(j.partial, j.grid_tn, (long)j.PW * j.NTOT1, j.Gfull, 1.0, c.st));
    return OTS_OK;
  }
  const int nbk = (k0 + 127) / 128;
  for (int ab = 0; ab < nbk; ++ab) {
    const int a0 = 128 * ab, aw = std::min(128, k0 - a0), PWa = pad32(aw);
    for (int bb = 0; bb <= ab; ++bb) {
      const int b0 = 128 * bb, bw = std::min(128, k0 - b0), PWb = pad32(bw);
      TnArgs a{};
      a.P = c.V; a.ldp = c.ldv; a.pc0 = a0; a.pcols = aw;
      a.row_begin = 0; a.row_end = c.n_local; a.b_row_begin = 0; a.p_row_begin = 0;
      a.partial = j.partial;
      int grid, ldp;
      if (ab == bb) {
        a.B = nullptr; a.ldb = 0; a.bc0 = 0; a.bcols = 0;
        grid = grid_for_tn(PWa, 0, true, true, gnsm);
        ldp = PWa;
        CK(launch_tsgemm_tn(a, PWa, 0, true, true, grid, c.st));
      } else {
        a.B = c.V; a.ldb = c.ldv; a.bc0 = b0; a.bcols = bw;
        grid = grid_for_tn(PWa, PWb, false, false, gnsm);
        ldp = PWb;
        CK(launch_tsgemm_tn(a, PWa, PWb, false, false, grid, c.st));
      }
      CK(launch_reduce_strided(j.partial, grid, aw, bw, ldp, j.Gfull + (long)a0 * j.NTOT1 + b0, j.NTOT1, 1.0,
                               c.st));
    }
    TnArgs a{};
    a.P = c.V; a.ldp = c.ldv; a.pc0 = a0; a.pcols = aw;
    a.B = c.A; a.ldb = c.lda; a.bc0 = 0; a.bcols = k;
    a.row_begin = 0; a.row_end = c.n_local; a.b_row_begin = j.qrow0; a.p_row_begin = 0;
    a.partial = j.partial;
    const int grid = grid_for_tn(PWa, j.BWa, false, false, gnsm);
    CK(launch_tsgemm_tn(a, PWa, j.BWa, false, false, grid, c.st));
    CK(launch_reduce_strided(j.partial, grid, aw, k, j.BWa, j.Gfull + (long)a0 * j.NTOT1 + j.PW, j.NTOT1, 1.0,
                             c.st));
  }
  return OTS_OK;
}

int phase_apply1(ots_ctx* ctx, Job& j) {
  const JobCfg& c = j.c;
  NnArgs a{};
  a.P = c.V; a.ldp = c.ldv; a.kdim = (int)c.k0;
  a.Z = j.s.Z1; a.ldz = j.ld;
  a.B = c.A; a.ldb = c.lda;
  a.X = c.Q; a.ldx = c.ldq;
  a.ncols = (int)c.k;
  a.row_begin = j.qrow0; a.row_end = c.n_local;
  a.colscale = nullptr;
  a.tile_counter = ctx->nn_counter;
  CK(launch_tsgemm_nn(a, j.KT, ctx->nsm, c.st));
  return OTS_OK;
}

int phase_vtb(ots_ctx* ctx, Job& j, const double* Bm, long ldb, double alpha);
int phase_gram2(ots_ctx* ctx, Job& j) { return phase_vtb(ctx, j, j.c.Q, j.c.ldq, -1.0); }

// Y2full (k0 x k, ld BWa) = alpha * V_b^T B_b over this rank's QR rows
int phase_vtb(ots_ctx* ctx, Job& j, const double* Bm, long ldb, double alpha) {
  const JobCfg& c = j.c;
  const int k0 = (int)c.k0, k = (int)c.k;
  const int nbk = (k0 + 127) / 128;
  for (int ab = 0; ab < nbk; ++ab) {
    const int a0 = 128 * ab, aw = std::min(128, k0 - a0), PWa = pad32(aw);
    TnArgs a{};
    a.P = c.V; a.ldp = c.ldv; a.pc0 = a0; a.pcols = aw;
    a.B = Bm; a.ldb = ldb; a.bc0 = 0; a.bcols = k;
    a.row_begin = j.qrow0; a.row_end = c.n_local;
    a.b_row_begin = j.qrow0; a.p_row_begin = j.qrow0;
    a.partial = j.partial;
    const int grid = (nbk == 1) ? j.grid_tn2 : grid_for_tn(PWa, j.BWa, false, false, j.nsm_use > 0 ? j.nsm_use : ctx->nsm);
    CK(launch_tsgemm_tn(a, PWa, j.BWa, false, false, grid, c.st));
    CK(launch_reduce_strided(j.partial, grid, aw, k, j.BWa, j.Y2full + (long)a0 * j.BWa, j.BWa, alpha, c.st));
  }
  return OTS_OK;
}

__global__ void copy_y2_kernel(const double* Y2full, int ldy, double* Z2, int ld, int k0, int k) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k0 * k; e += gridDim.x * blockDim.x) {
    int i = e / k, jj = e - i * k;
    Z2[i * ld + jj] = Y2full[i * ldy + jj];
  }
}

int phase_apply2(ots_ctx* ctx, Job& j) {
  const JobCfg& c = j.c;
  NnArgs a{};
  a.P = c.V; a.ldp = c.ldv; a.kdim = (int)c.k0;
  a.Z = j.s.Z2; a.ldz = j.ld;
  a.B = c.Q; a.ldb = c.ldq;
  a.X = c.Q; a.ldx = c.ldq;
  a.ncols = (int)c.k;
  a.row_begin = j.qrow0; a.row_end = c.n_local;
  a.colscale = j.svec;
  a.tile_counter = ctx->nn_counter;
  CK(launch_tsgemm_nn(a, j.KT, ctx->nsm, c.st));
  return OTS_OK;
}

__global__ void set_identity_ld_kernel(double* D, int n, int ld) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    int i = e / n, jj = e - i * n;
    D[i * ld + jj] = (i == jj) ? 1.0 : 0.0;
  }
}
__global__ void triu_copy_kernel(const double* Rs, int lds, double* R, long ldr, int k) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) {
    int i = e / k, jj = e - i * k;
    R[i * ldr + jj] = (jj >= i) ? Rs[i * lds + jj] : 0.0;
  }
}
__global__ void ones_kernel(double* v, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = 1.0;
}

// Shifted Cholesky-QR with two refinements on X (m x k, in place):
// core.py:177-202.  R (k x k, ldr) written; status <- INTRA_FAILURE on breakdown.
int run_cholshift(ots_ctx* ctx, Job& j, double* X, long ldx, long m, int k, double* R, long ldr,
                  cudaStream_t st, int refine_passes = 2) {
  const int PWk = pad32(k);
  const int grid = grid_for_tn(PWk, 0, true, true, ctx->nsm);
  double* W = j.chol_ws;   // small scratch (2 k x ld + k)
  double* Z = j.s.X2;
  double* Racc = j.s.Sd;
  set_identity_ld_kernel<<<4, 256, 0, st>>>(Racc, k, j.ld);
  for (int pass = 0; pass < 1 + std::max(0, refine_passes); ++pass) {
    TnArgs a{};
    a.P = X; a.ldp = ldx; a.pc0 = 0; a.pcols = k;
    a.B = nullptr; a.ldb = 0; a.bc0 = 0; a.bcols = 0;
    a.row_begin = 0; a.row_end = m; a.b_row_begin = 0; a.p_row_begin = 0;
    a.partial = j.partial;
    CK(launch_tsgemm_tn(a, PWk, 0, true, true, grid, st));
    CK(launch_reduce(j.partial, grid, (long)PWk * PWk, j.Gfull, 1.0, st));
    CK(launch_cholqr_step(j.Gfull, PWk, k, m, pass == 0, W, j.ld, Z, Racc, j.s.status, st));
    NnArgs b{};
    b.P = X; b.ldp = ldx; b.kdim = k; b.Z = Z; b.ldz = j.ld; b.B = nullptr; b.ldb = 0;
    b.X = X; b.ldx = ldx; b.ncols = k; b.row_begin = 0; b.row_end = m; b.colscale = nullptr;
    CK(launch_tsgemm_nn(b, j.KT, ctx->nsm, st));
  }
  triu_copy_kernel<<<4, 256, 0, st>>>(Racc, j.ld, R, ldr, k);
  CK(cudaGetLastError());
  return OTS_OK;
}

// status <- OTS_E_VALUE when the (real view of the) k x k R holds a
// non-finite entry: a NaN/Inf anywhere in the input reaches every R of the
// TSQR chain that holds it and from there the final R (core.py:72-73 check,
// done on k^2 data instead of a pass over the n-length input)
__global__ void nonfinite_status_kernel(const double* R, long ldr, int rows, int cols, int* status) {
  int bad = 0;
  for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
    const int i = e / cols, j = e - i * cols;
    if (!isfinite(R[(long)i * ldr + j])) bad = 1;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicCAS(status, 0, OTS_E_VALUE);
}

int read_status(ots_ctx* ctx, Job& j, double* diag_host) {
  const JobCfg& c = j.c;
  CK(cudaMemcpyAsync(ctx->h_status, j.s.status, sizeof(int), cudaMemcpyDeviceToHost, c.st));
  CK(cudaMemcpyAsync(ctx->h_diag, j.s.diag, 3 * sizeof(double), cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  if (diag_host) std::memcpy(diag_host, ctx->h_diag, 3 * sizeof(double));
  int st = ctx->h_status[0];
  if (st != 0) {
    char buf[256];
    if (st == OTS_E_ORTHONORMALITY)
      snprintf(buf, sizeof buf, "||v^* v - I||_2 = %.3e exceeds %.1e", ctx->h_diag[2], c.orth_tol);
    else if (st == OTS_E_NOT_PD)
      snprintf(buf, sizeof buf, "Cholesky factor of T: matrix is not positive definite");
    else if (st == OTS_E_SINGULAR_T)
      snprintf(buf, sizeof buf, "T is numerically singular");
    else if (st == OTS_E_VALUE)
      snprintf(buf, sizeof buf, "input contains non-finite entries");
    else if (st == OTS_E_INTRA_FAILURE)
      snprintf(buf, sizeof buf, "shifted Cholesky-QR broke down: Cholesky factorization failed (matrix not positive definite)");
    else if (st == OTS_E_PARAMETER)
      snprintf(buf, sizeof buf, "explicit seed p is not unitary to tolerance");
    else
      snprintf(buf, sizeof buf, "status %d", st);
    return fail(ctx, st, buf);
  }
  return OTS_OK;
}

int validate_layout(ots_ctx* ctx, const void* p, long ld, const char* name) {
  if (p == nullptr) return OTS_OK;
  if ((ld & 1) || !aligned16(p))
    return fail(ctx, OTS_E_VALUE, std::string(name) + ": rows must be 16-byte aligned (even ld)");
  return OTS_OK;
}

}  // namespace

struct BHook {                 // B-inner extension of the pipeline
  const double* Gu; int ldgu;   // unweighted Gram of the original V
  const double* dinv_top;       // diagonal M: 1/d on the top k0 rows
  const double* d; long n;      // diagonal M: full weights (for the Q epilogue)
  const double* L = nullptr; long ldl = 0;          // dense B = L L^T (Q epilogue: L^{-T})
  const double* Ltinv = nullptr; int ldlt = 0;      // dense: L_m^{-T} (diagnostics)
  const double* Vorig = nullptr; long ldvo = 0;     // dense: original V (diagnostics)
};

// Y = D^(+-1/2) X, row-oriented (real views, even leading dimensions: 16-byte
// accesses): one warp per row, the row factor computed once per row, no
// per-element index division (the element-wise form ran at ~4 TB/s).
__global__ void row_scale_pairs_kernel(const double* X, long ldx, long n, int cols, const double* d, int inv,
                                       double* Y, long ldy) {
  const int lane = threadIdx.x & 31;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  const int np = cols >> 1;
  for (long i = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    const double s = inv ? rsqrt(d[i]) : sqrt(d[i]);
    const double2* xr = reinterpret_cast<const double2*>(X + i * ldx);
    double2* yr = reinterpret_cast<double2*>(Y + i * ldy);
    for (int q = lane; q < np; q += 32) {
      const double2 v = __ldcs(xr + q);
      __stcs(yr + q, make_double2(v.x * s, v.y * s));
    }
    if ((cols & 1) && lane == 0) Y[i * ldy + cols - 1] = X[i * ldx + cols - 1] * s;
  }
}
__global__ void b_unscale_kernel(double* Q, long ldq, long n, int k, const double* d, const double* R,
                                 long ldr) {
  // Q <- D^{-1/2} Q diag(sg), sg_j = sign(R_jj) (0 -> +1): the B-path's
  // positive-diagonal convention (oblique.py:232).
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < n * k; e += (long)gridDim.x * blockDim.x) {
    long i = e / k; int j = (int)(e - i * k);
    const double sg = (R[(long)j * ldr + j] < 0.0) ? -1.0 : 1.0;
    Q[i * ldq + j] *= sg * rsqrt(d[i]);
  }
}
static int row_grid(long n) { return (int)std::min<long>(148L * 16, (n + 7) / 8); }

__global__ void b_rsign_kernel(double* R, long ldr, int k) {
  // R <- diag(sg) R  (rows), sg from its own diagonal; one block, ordered so
  // the diagonal is read before it is rewritten.
  __shared__ double sg[64];
  for (int j = threadIdx.x; j < k; j += blockDim.x) sg[j] = (R[(long)j * ldr + j] < 0.0) ? -1.0 : 1.0;
  __syncthreads();
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    int i = e / k, j = e - i * k;
    R[(long)i * ldr + j] *= sg[i];
  }
}
__global__ void inv_top_kernel(const double* d, int k0, double* out) {
  for (int i = threadIdx.x; i < k0; i += blockDim.x) out[i] = 1.0 / d[i];
}

// ---------------------------------------------------------------------------
// Direct-Q pipeline (fastpath.cu) between the seed and qtop.  Returns 1 when
// the cancellation test or the sweep flagged the input (nothing the caller
// keeps was written: the materialised-X pipeline then runs from apply1), 0
// when Q's bottom rows, R and Z2 are done, < 0 on errors.
// ---------------------------------------------------------------------------
FastArgs fast_args(ots_ctx* ctx, Job& j) {
  const JobCfg& c = j.c;
  const Level& L0 = j.lv[0];
  FastArgs fa{};
  fa.V = c.V + j.qrow0 * c.ldv; fa.ldv = c.ldv;
  fa.A = c.A + j.qrow0 * c.lda; fa.lda = c.lda;
  fa.D = L0.D; fa.ldd = L0.ldd;
  fa.k0 = (int)c.k0; fa.k = (int)c.k; fa.PW = j.PW;
  fa.G = L0.G;
  fa.TG = j.fTG; fa.tg_stride = j.ftg_stride;
  fa.part = j.fpart;
  fa.Z1 = j.s.Z1; fa.ldz = j.ld;
  fa.M = L0.CC;
  fa.Coef = j.fCoef;
  fa.flags = j.fflags;
  fa.ticket = j.fflags + 1;
  (void)ctx;
  return fa;
}

int fast_gram(ots_ctx* ctx, Job& j) {
  const JobCfg& c = j.c;
  FastArgs fa = fast_args(ctx, j);
  const int grid = j.gram_nsm > 0 ? j.gram_nsm : ctx->nsm;
  CK(cudaMemsetAsync(j.fflags, 0, 16 * sizeof(int), c.st));
  CK(launch_tgram(fa, grid, c.st));
  CK(launch_tgram_reduce(fa, grid, c.V, (int)j.qrow0, j.Gfull, j.NTOT1, c.st));
  return OTS_OK;
}

// stage 1: heads' X rows, X^T X / V^T X per tile, Gram-form sweep, route
// decision (returns 1: rejected), local tree over the chain R's
int fast_factor(ots_ctx* ctx, Job& j) {
  const JobCfg& c = j.c;
  cudaStream_t st = c.st;
  const int KT = j.KT;
  FastArgs fa = fast_args(ctx, j);
  Level& L0 = j.lv[0];
  const int nch = L0.G.nchains;
  const int ghead = std::min(nch, 2 * ctx->nsm);
  CK(launch_head_rows(fa, 0, j.s.Z1, j.ld, nullptr, nullptr, ghead, st));     // X rows of the heads
  CK(launch_tile_alg(fa, st));
  prof_mark(ctx, st, "tile_alg");
  GsweepArgs ga{L0.D, L0.ldd, L0.ncols, L0.G, L0.UT, L0.R, L0.CC, L0.HS, L0.FL, (long)L0.G128.L + 1};
  ga.abort_flag = j.fflags;
  CK(launch_chain_gsweep(ga, st));
  CK(launch_fast_flags(L0.FL, nch, j.fflags, st));
  CK(cudaMemcpyAsync(ctx->h_status + 8, j.fflags, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(ctx->ev_fast, st));
  prof_mark(ctx, st, "gs_sweep");
  // one int through pinned memory decides the route (a rejected attempt
  // leaves nothing queued behind it)
  CK(cudaEventSynchronize(ctx->ev_fast));
  if (ctx->h_status[8] != 0) return 1;
  for (size_t l = 1; l < j.lv.size(); ++l) {          // tree over the chain R's
    Level& L = j.lv[l];
    FactorArgs fl{L.D, L.ldd, L.ncols, L.G, L.UT, L.R, 1};
    CK(launch_chain_factor(fl, KT, st));
  }
  prof_mark(ctx, st, "factor");
  return 0;
}

// stage 2: C's down the local tree from Ctop, per-tile coefficients, heads'
// Q_ rows, LAPACK signs (on the rank that owns the top rows: Rfin -> Rout),
// and this rank's Y2 = -V_b^T Q_ into Y2full
int fast_coef(ots_ctx* ctx, Job& j, const double* Ctop, bool do_sign, double* Q, long ldq, const double* Rfin,
              double* Rout, long ldr) {
  const JobCfg& c = j.c;
  cudaStream_t st = c.st;
  const int KT = j.KT;
  const long k0 = c.k0, k = c.k;
  FastArgs fa = fast_args(ctx, j);
  Level& L0 = j.lv[0];
  const int nch = L0.G.nchains;
  const double* Cin = Ctop;
  for (int l = (int)j.lv.size() - 1; l >= 1; --l) {
    Level& L = j.lv[l];
    QformArgs qa{L.D, L.ldd, L.ncols, L.G, L.UT, Cin, 0};
    CK(launch_chain_qform(qa, KT, st));
    Cin = L.D;
  }
  {
    QformArgs qa{L0.D, L0.ldd, L0.ncols, L0.G, L0.UT, Cin, 0};
    qa.mode = 2;
    qa.Cc = L0.CC; qa.Hs = L0.HS; qa.flags = L0.FL;
    qa.tslots = (long)L0.G128.L + 1;
    qa.Kout = j.fCoef; qa.kstride = (long)(j.PW + 64) * 64; qa.koff = (long)j.PW * 64;
    qa.grid_max = j.nsm_use;
    CK(launch_gs_coef(qa, st));
  }
  if (do_sign) CK(launch_sign(j.s, Q + k0 * ldq, ldq, Rfin, KT, Rout, (int)ldr, st));
  // Y2 = -V_b^T Q_ = -(sum_t Cx_t K_t + sum_heads V_h^T Q_h)
  const int gb = j.nsm_use, gh = std::min(nch, j.nsm_use);
  CK(launch_coef_b(fa, j.fpart, gb, st));
  CK(launch_head_rows(fa, 2, nullptr, 0, nullptr, j.fpart + (size_t)gb * j.PW * 64, gh, st));
  CK(launch_reduce_strided(j.fpart, gb + gh, (int)k0, (int)k, 64, j.Y2full, j.BWa, -1.0, st));
  return 0;
}

// stage 3 (Z2 and the signs known): coefficient rows += Z2, the final pass and
// the heads' final rows
int fast_final(ots_ctx* ctx, Job& j, bool diag_side) {
  cudaStream_t st = j.c.st;
  FastArgs fa = fast_args(ctx, j);
  Level& L0 = j.lv[0];
  const int ghead = std::min(L0.G.nchains, 2 * ctx->nsm);
  CK(launch_coef_add_z2(fa, j.s.Z2, j.ld, st));
  prof_mark(ctx, st, "coef");
  if (diag_side) {
    // the diagnostics already run on the side stream (launched behind the seed)
    CK(launch_final_nn(fa, j.svec, L0.D, L0.ldd, st));
    CK(launch_head_rows(fa, 1, j.s.Z2, j.ld, j.svec, nullptr, ghead, st));
  } else {
    // diagnostics (3 CTAs) on the main stream ahead of the final pass on the
    // side stream (dynamic sub-tiles: the SMs they hold take fewer), as apply1
    CK(cudaEventRecord(ctx->ev_seed, st));
    CK(launch_diag(j.s, st));
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_seed, 0));
    CK(launch_final_nn(fa, j.svec, L0.D, L0.ldd, ctx->side));
    CK(launch_head_rows(fa, 1, j.s.Z2, j.ld, j.svec, nullptr, ghead, ctx->side));
    CK(cudaEventRecord(ctx->ev_diag, ctx->side));
    CK(cudaStreamWaitEvent(st, ctx->ev_diag, 0));
  }
  prof_mark(ctx, st, "final");
  return 0;
}

int fast_pipeline(ots_ctx* ctx, Job& j, double* Q, long ldq, double* R, long ldr, bool diag_side) {
  const JobCfg& c = j.c;
  cudaStream_t st = c.st;
  const int KT = j.KT;
  int rc = fast_factor(ctx, j);
  if (rc) return rc;
  set_identity_kernel<<<(KT * KT + 255) / 256, 256, 0, st>>>(j.ident, KT);
  if ((rc = fast_coef(ctx, j, j.ident, true, Q, ldq, j.lv.back().R, R, ldr))) return rc;
  copy_y2_kernel<<<16, 256, 0, st>>>(j.Y2full, j.BWa, j.s.Z2, j.ld, (int)c.k0, (int)c.k);
  CK(launch_z2(j.s, st));
  return fast_final(ctx, j, diag_side);
}

int two_stage_pipeline(ots_ctx* ctx, const JobCfg& c, int intra, double* Q, long ldq, double* R, long ldr,
                       double* S, long lds, double* diag_host, const BHook* bh) {
  const long n = c.n_local, k0 = c.k0, k = c.k;
  cudaStream_t st = c.st;
  Job j;
  int rc;
  // k0 > 128: the k0 x k0 diagnostics take tens of ms on three single-CTA
  // eigenvalue problems; they then run on the side stream beside everything
  // after the seed, and the row-parallel phases are planned for nsm - 3 SMs
  // (chains, qform and Gram grids; the NN updates balance dynamically).
  // Small calls (apply1 well under the diagnostics' fixed ~0.3-0.6 ms) take
  // the same route: the diagnostics then hide behind factor..apply2.
  const bool small_call = (double)n * (double)k0 * (double)k < 2.5e10;
  const bool diag_side = (k0 > 128 || small_call) && ctx->nsm > 16;
  JobCfg c2 = c;
  if (diag_side) c2.nsm_avail = ctx->nsm - 3;
  c2.fast_try = intra == OTS_INTRA_HOUSEHOLDER && bh == nullptr;
  ctx->fast_taken = 0;
  if ((rc = job_setup(ctx, j, c2))) return rc;
  const int KT = j.KT;
  if (bh) {
    j.s.Gu = bh->Gu; j.s.ldgu = bh->ldgu; j.s.dinv_top = bh->dinv_top;
    j.s.Ltinv = bh->Ltinv; j.s.ldlt = bh->ldlt; j.s.Vorig = bh->Vorig; j.s.ldvo = bh->ldvo;
  }
  prof_begin(ctx, st);
  j.s.Sout = S; j.s.lds_out = (int)lds;
  // The V_t-only part of the seed (QR / LU / polar of the k0 x k0 top block)
  // runs on one SM, on the side stream, while the single-wave Gram kernel
  // streams on the other nsm-1 SMs; the Gram-dependent checks and Z1, S
  // follow the Gram (validation order kept: defect > non-finite > seed).
  const bool split_seed = ctx->nsm > 8;
  if (split_seed) {
    CK(cudaEventRecord(ctx->ev_seedA, st));          // inputs ready on st
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_seedA, 0));
    CK(launch_seed_split(j.s, 0, ctx->side));
    CK(cudaEventRecord(ctx->ev_seedA, ctx->side));
    j.gram_nsm = ctx->nsm - (seed_uses_cluster(j.s) ? 2 : 1);
    j.grid_tn = grid_for_tn(j.PW, j.BWa, true, true, j.gram_nsm);
  }
  if ((rc = j.fast ? fast_gram(ctx, j) : phase_gram(ctx, j))) return rc;
  prof_mark(ctx, st, "gram");
  if (split_seed) {
    CK(cudaStreamWaitEvent(st, ctx->ev_seedA, 0));
    CK(launch_seed_split(j.s, 1, st));
  } else {
    CK(launch_seed(j.s, st));
  }
  CK(cudaEventRecord(ctx->ev_seed, st));
  prof_mark(ctx, st, "seed");
  // The diagnostics (3 CTAs, ~2 ms) go on the main stream right behind the
  // seed so they own their SMs before apply1's CTAs (side stream, released by
  // an event a little later) fill the rest; apply1 hands out its tiles
  // dynamically, so those 3 SMs simply take fewer.  The factor then starts on
  // an idle GPU instead of waiting for the diagnostics' SMs.
  bool fast_done = false;
  if (diag_side) {
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_seed, 0));
    CK(launch_diag(j.s, ctx->side));
    CK(cudaEventRecord(ctx->ev_diag, ctx->side));   // waited for before the status read
  }
  if (j.fast) {
    rc = fast_pipeline(ctx, j, Q, ldq, R, ldr, diag_side);
    if (rc < 0) return rc;
    fast_done = rc == 0;
    ctx->fast_taken = fast_done ? 1 : 0;
  }
  if (fast_done) {
    // Q's bottom rows, R, Z2 done
  } else if (diag_side) {
    if ((rc = phase_apply1(ctx, j))) return rc;
  } else {
    // (re-recorded: after a rejected direct-Q attempt the side stream must not
    // run ahead of the diagnostics' launch)
    CK(cudaEventRecord(ctx->ev_seed, st));
    CK(launch_diag(j.s, st));
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_seed, 0));
    JobCfg c1 = j.c;
    j.c.st = ctx->side;
    rc = phase_apply1(ctx, j);
    j.c = c1;
    if (rc) return rc;
    CK(cudaEventRecord(ctx->ev_diag, ctx->side));   // apply1 done
    CK(cudaStreamWaitEvent(st, ctx->ev_diag, 0));
  }
  if (!fast_done) {
  prof_mark(ctx, st, "apply1");
  if (intra == OTS_INTRA_HOUSEHOLDER) {
    if ((rc = run_factor_levels(ctx, j.lv, KT, st))) return rc;
    prof_mark(ctx, st, "factor");
    set_identity_kernel<<<(KT * KT + 255) / 256, 256, 0, st>>>(j.ident, KT);
    if ((rc = run_qform_levels(ctx, j.lv, KT, j.ident, st, diag_side ? j.nsm_use : 0))) return rc;
    prof_mark(ctx, st, "qform");
    CK(launch_sign(j.s, Q + k0 * ldq, ldq, j.lv.back().R, KT, R, (int)ldr, st));
  } else {
    if ((rc = run_cholshift(ctx, j, Q + k0 * ldq, ldq, n - k0, (int)k, R, ldr, st))) return rc;
    ones_kernel<<<1, 64, 0, st>>>(j.svec, (int)k);
    prof_mark(ctx, st, "cholshift");
  }
  if ((rc = phase_gram2(ctx, j))) return rc;
  prof_mark(ctx, st, "gram2");
  copy_y2_kernel<<<16, 256, 0, st>>>(j.Y2full, j.BWa, j.s.Z2, j.ld, (int)k0, (int)k);
  CK(launch_z2(j.s, st));
  prof_mark(ctx, st, "z2");
  if ((rc = phase_apply2(ctx, j))) {
    return rc;
  }
  prof_mark(ctx, st, "apply2");
  }  // !fast_done
  CK(launch_qtop(j.s, Q, ldq, st));
  if (bh) {
    if (bh->L != nullptr) {       // dense B: Q = L^{-T} Q' sgn
      CK(launch_colsign(Q, ldq, n, (int)k, R, ldr, st));
      CK(launch_trsm_lt(bh->L, bh->ldl, Q, ldq, (int)n, (int)k, st));
    } else {
      b_unscale_kernel<<<(int)std::min<long>(4096, (n * k + 255) / 256), 256, 0, st>>>(Q, ldq, n, (int)k, bh->d, R, ldr);
    }
    b_rsign_kernel<<<1, 256, 0, st>>>(R, ldr, (int)k);
    prof_mark(ctx, st, "b_epilogue");
  }
  if (diag_side) CK(cudaStreamWaitEvent(st, ctx->ev_diag, 0));
  prof_mark(ctx, st, "tail");
  // gram, reduce, seed(B), diag, apply1, identity, sign, gram2, reduce, copy_y2,
  // z2, apply2, qtop + a factor and a qform launch per level (+ seedA, B epilogue)
  ctx->launches = 13 + 2 * (int)j.lv.size() + (bh ? 2 : 0) + (split_seed ? 1 : 0);
  // direct-Q: tgram, reduce, seed(B), head x3, tile_alg, gsweep, flags, identity, gs_coef, sign, coef_b,
  // reduce, copy_y2, z2, add_z2, diag, final, qtop + a factor and a qform launch per tree level (+ seedA)
  if (fast_done) ctx->launches = 20 + 2 * ((int)j.lv.size() - 1) + (split_seed ? 1 : 0);
  rc = read_status(ctx, j, diag_host);
  prof_end(ctx);
  return rc;
}

// ===========================================================================
// exported C-ABI
// ===========================================================================
extern "C" {

int ots_version(void) { return 1; }

void ots_gs_event_log(long long* out) { ots::gs_event_log(out); }

int ots_ctx_create(int device, ots_ctx** out) {
  if (!out) return OTS_E_VALUE;
  ots_ctx* c = new ots_ctx();
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { c->err = cudaGetErrorString(e); *out = c; return OTS_E_CUDA; }
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device);
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi);
  }
  cudaMalloc(&c->nn_counter, 256);
  cudaEventCreateWithFlags(&c->ev_seed, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_diag, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_seedA, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_fast, cudaEventDisableTiming);
  cudaMallocHost(&c->h_status, 64);
  cudaMallocHost(&c->h_diag, 64);
  *out = c;
  e = cudaGetLastError();
  if (e != cudaSuccess) { c->err = cudaGetErrorString(e); return OTS_E_CUDA; }
  return OTS_OK;
}

void ots_ctx_destroy(ots_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->ws) cudaFree(c->ws);
  if (c->b_ws) cudaFree(c->b_ws);
  if (c->z_ws) cudaFree(c->z_ws);
  if (c->zgs_ws) cudaFree(c->zgs_ws);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->nn_counter) cudaFree(c->nn_counter);
  if (c->ev_seed) cudaEventDestroy(c->ev_seed);
  if (c->ev_diag) cudaEventDestroy(c->ev_diag);
  if (c->ev_seedA) cudaEventDestroy(c->ev_seedA);
  if (c->ev_fast) cudaEventDestroy(c->ev_fast);
  if (c->h_status) cudaFreeHost(c->h_status);
  if (c->h_diag) cudaFreeHost(c->h_diag);
  for (auto e : c->pev) cudaEventDestroy(e);
  delete c->job;
  delete c;
}

const char* ots_last_error(const ots_ctx* c) { return c ? c->err.c_str() : "null context"; }
int ots_sm_count(const ots_ctx* c) { return c ? c->nsm : 0; }
int ots_last_fast(const ots_ctx* c) { return c ? c->fast_taken : 0; }

int ots_set_profiling(ots_ctx* c, int enable) { c->profile = enable != 0; return OTS_OK; }

int ots_last_launch_count(const ots_ctx* c) { return c ? c->launches : 0; }

int ots_debug_counters(unsigned long long* out, int reset) { return ots::debug_counters(out, reset); }

int ots_fp64_peak(ots_ctx* ctx, double* tflops) {
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();   // a stale error from unrelated earlier work is not ours
  CK(fp64_peak(ctx->nsm, nullptr, tflops));
  return OTS_OK;
}

int ots_last_profile(const ots_ctx* c, char* names, int cap, float* ms, int mcap) {
  std::string all;
  int n = (int)c->pms.size();
  for (int i = 0; i < n; ++i) {
    if (i < mcap) ms[i] = c->pms[i];
    all += c->last_names[i];
    all += "\n";
  }
  if (names && cap > 0) {
    strncpy(names, all.c_str(), cap - 1);
    names[cap - 1] = 0;
  }
  return n;
}

int ots_two_stage_f64(ots_ctx* ctx, int64_t n, int64_t k0, int64_t k, const double* V, int64_t ldv,
                      const double* A, int64_t lda, int choice, int intra, const double* P, int64_t ldp,
                      double orth_tol, int allow_defect, double* Q, int64_t ldq, double* R, int64_t ldr,
                      double* S, int64_t lds, double* diag_host, void* stream) {
  return ots_two_stage_gram_f64(ctx, n, k0, k, V, ldv, A, lda, choice, intra, P, ldp, orth_tol, allow_defect,
                                nullptr, 0, Q, ldq, R, ldr, S, lds, diag_host, stream);
}

int ots_two_stage_gram_f64(ots_ctx* ctx, int64_t n, int64_t k0, int64_t k, const double* V, int64_t ldv,
                           const double* A, int64_t lda, int choice, int intra, const double* P, int64_t ldp,
                           double orth_tol, int allow_defect, const double* gram, int64_t ldg, double* Q,
                           int64_t ldq, double* R, int64_t ldr, double* S, int64_t lds, double* diag_host,
                           void* stream) {
  if (!ctx) return OTS_E_VALUE;
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();   // a stale error from unrelated earlier work is not ours
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || k0 < 0 || k < 0) return fail(ctx, OTS_E_DIMENSION, "negative dimension");
  if (k0 + k > n) return fail(ctx, OTS_E_DIMENSION, "need k0 + k <= n");
  if (k > 64) return fail(ctx, OTS_E_UNSUPPORTED, "k > 64 not supported by this build");
  if (k0 > 1024) return fail(ctx, OTS_E_UNSUPPORTED, "k0 > 1024 not supported by this build");
  if (intra != OTS_INTRA_HOUSEHOLDER && intra != OTS_INTRA_CHOLSHIFT)
    return fail(ctx, OTS_E_PARAMETER, "unknown intra method");
  if (choice < 0 || choice > 3) return fail(ctx, OTS_E_PARAMETER, "unknown choice");
  if (choice == OTS_CHOICE_EXPLICIT && P == nullptr)
    return fail(ctx, OTS_E_PARAMETER, "choice='explicit' requires a seed matrix p");
  int rc;
  if ((rc = validate_layout(ctx, V, ldv, "V"))) return rc;
  if ((rc = validate_layout(ctx, A, lda, "A"))) return rc;
  if ((rc = validate_layout(ctx, Q, ldq, "Q"))) return rc;
  if (k == 0) return OTS_OK;
  if (k0 == 0) {   // intra_qr(a, intra) (twostage.py:81-84 -> :45-54)
    rc = (intra == OTS_INTRA_CHOLSHIFT) ? ots_shifted_cholesky_qr_f64(ctx, n, k, A, lda, Q, ldq, R, ldr, stream)
                                        : ots_householder_qr_f64(ctx, n, k, A, lda, Q, ldq, R, ldr, 0, stream);
    if (rc == OTS_E_NOT_PD && intra == OTS_INTRA_CHOLSHIFT)
      rc = fail(ctx, OTS_E_INTRA_FAILURE, "shifted Cholesky-QR broke down: " + ctx->err);
    if (diag_host) { diag_host[0] = 1.0; diag_host[1] = 0.0; diag_host[2] = 0.0; }
    return rc;
  }
  JobCfg c{n, 0, k0, k, V, ldv, A, lda, Q, ldq, choice, P, ldp, orth_tol, allow_defect, st, false};
  c.gram_in = gram; c.ldgi = ldg;
  return two_stage_pipeline(ctx, c, intra, Q, ldq, R, ldr, S, lds, diag_host, nullptr);
}

}  // extern "C"

// ----------------------------- reflector objects ---------------------------
struct ots_refl {
  int device = 0;
  long n = 0, k0 = 0, ldv = 0;
  const double* V = nullptr;
  int choice = 1, ld = 32;
  double* buf = nullptr;       // persistent small state
  SmallState s{};
  double defect = 0.0;
};

namespace {
// copy the reflector-defining small matrices of a job into the object
void refl_capture(ots_refl* r, const Job& j, cudaStream_t st) {
  const size_t m2 = (size_t)j.ld * j.ld;
  double** dst[] = {&r->s.G, &r->s.Vt, &r->s.P, &r->s.Tf, &r->s.Tdense, &r->s.Wt};
  const double* src[] = {j.s.G, j.s.Vt, j.s.P, j.s.Tf, j.s.Tdense, j.s.Wt};
  for (int i = 0; i < 6; ++i) {
    *dst[i] = r->buf + i * m2;
    cudaMemcpyAsync(*dst[i], src[i], m2 * 8, cudaMemcpyDeviceToDevice, st);
  }
  r->s.pvec = r->buf + 6 * m2;
  cudaMemcpyAsync(r->s.pvec, j.s.pvec, j.ld * 8, cudaMemcpyDeviceToDevice, st);
  r->s.piv = reinterpret_cast<int*>(r->buf + 6 * m2 + j.ld);
  cudaMemcpyAsync(r->s.piv, j.s.piv, j.ld * sizeof(int), cudaMemcpyDeviceToDevice, st);
}
// point a job's small state at the reflector's matrices
void refl_attach(const ots_refl* r, Job& j) {
  j.s.G = r->s.G; j.s.Vt = r->s.Vt; j.s.P = r->s.P; j.s.Tf = r->s.Tf; j.s.Tdense = r->s.Tdense;
  j.s.Wt = r->s.Wt; j.s.pvec = r->s.pvec; j.s.piv = r->s.piv; j.s.choice = r->choice;
}
}  // namespace

extern "C" {

/* build_reflector(v, choice, p, orth_tol, allow_defect)  -- reflector.py:207-228 */
int ots_build_reflector_f64(ots_ctx* ctx, int64_t n, int64_t k0, const double* V, int64_t ldv, int choice,
                            const double* P, int64_t ldp, double orth_tol, int allow_defect, ots_refl** out,
                            double* defect_host, void* stream) {
  if (!ctx || !out) return OTS_E_VALUE;
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();   // a stale error from unrelated earlier work is not ours
  cudaStream_t st = (cudaStream_t)stream;
  if (k0 > n) return fail(ctx, OTS_E_DIMENSION, "v must be tall");
  if (k0 == 0) return fail(ctx, OTS_E_DIMENSION, "v must have at least one column");
  if (k0 > 1024) return fail(ctx, OTS_E_UNSUPPORTED, "k0 > 1024 not supported by this build");
  if (choice < 0 || choice > 3) return fail(ctx, OTS_E_PARAMETER, "unknown choice");
  int rc;
  if ((rc = validate_layout(ctx, V, ldv, "V"))) return rc;
  // a one-column job on A = V gives the Gram, the defect check and the seed
  JobCfg c{n, 0, k0, 1, V, ldv, V, ldv, nullptr, 0, choice, P, ldp, orth_tol, allow_defect, st, false};
  c.ld_min = std::max(pad32(k0), 64);   // the ld every later job on this object uses (any m <= 64)
  Job j;
  if ((rc = job_setup(ctx, j, c))) return rc;
  if ((rc = phase_gram(ctx, j))) return rc;
  j.s.Sout = j.s.Sd; j.s.lds_out = j.ld;
  CK(launch_seed(j.s, st));
  ots_refl* r = new ots_refl();
  r->device = ctx->device; r->n = n; r->k0 = k0; r->ldv = ldv; r->V = V; r->choice = choice; r->ld = j.ld;
  r->s = j.s;
  CK(cudaMalloc(&r->buf, ((size_t)6 * j.ld * j.ld + 2 * j.ld + 64) * 8));
  refl_capture(r, j, st);
  double diag[3];
  rc = read_status(ctx, j, diag);
  r->defect = diag[2];
  if (defect_host) *defect_host = diag[2];
  if (rc) { cudaFree(r->buf); delete r; return rc; }
  *out = r;
  return OTS_OK;
}

void ots_reflector_destroy(ots_refl* r) {
  if (!r) return;
  cudaSetDevice(r->device);
  cudaFree(r->buf);
  delete r;
}

/* apply_reflector(h, x, adjoint)                   -- reflector.py:231-238
 * Y (n x m) = X - W T^{-(*)} (W^T X); Y may alias X. m <= 64 per call. */
int ots_apply_reflector_f64(ots_ctx* ctx, const ots_refl* r, int64_t m, const double* X, int64_t ldx,
                            double* Y, int64_t ldy, int adjoint, void* stream) {
  if (!ctx || !r) return OTS_E_VALUE;
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();   // a stale error from unrelated earlier work is not ours
  cudaStream_t st = (cudaStream_t)stream;
  if (m == 0) return OTS_OK;
  if (m > 64) return fail(ctx, OTS_E_UNSUPPORTED, "apply_reflector: at most 64 columns per call");
  int rc;
  if ((rc = validate_layout(ctx, X, ldx, "X"))) return rc;
  if ((rc = validate_layout(ctx, Y, ldy, "Y"))) return rc;
  JobCfg c{r->n, 0, r->k0, m, r->V, r->ldv, X, ldx, Y, ldy, r->choice, nullptr, 0, 1.0, 1, st, false};
  c.ld_min = r->ld;   // the object's small matrices are stored at r->ld (refl_attach points at them)
  Job j;
  if ((rc = job_setup(ctx, j, c))) return rc;
  refl_attach(r, j);
  CK(cudaMemsetAsync(j.s.status, 0, sizeof(int), st));
  if ((rc = phase_vtb(ctx, j, X, ldx, 1.0))) return rc;        // V_b^T X_b
  j.s.Gfull = j.Y2full; j.s.ldgf = j.BWa;
  j.s.Sout = j.s.D2; j.s.lds_out = j.ld;                       // out_t staged (Y may alias X)
  CK(launch_refl_apply(j.s, adjoint, st));
  if ((rc = phase_apply1(ctx, j))) return rc;                  // Y_b = X_b + V_b Z
  CK(cudaMemcpy2DAsync(Y, ldy * 8, j.s.D2, j.ld * 8, m * 8, r->k0, cudaMemcpyDeviceToDevice, st));
  CK(cudaStreamSynchronize(st));
  ctx->launches = 5;
  return OTS_OK;
}

/* reflector_diagnostics(h) -> [kappa_t, wt_inv_norm]  -- reflector.py:241-247 */
int ots_reflector_diagnostics_f64(ots_ctx* ctx, const ots_refl* r, double* diag_host, void* stream) {
  if (!ctx || !r) return OTS_E_VALUE;
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();   // a stale error from unrelated earlier work is not ours
  cudaStream_t st = (cudaStream_t)stream;
  JobCfg c{r->n, 0, r->k0, 1, r->V, r->ldv, r->V, r->ldv, nullptr, 0, r->choice, nullptr, 0, 1.0, 1, st, false};
  c.ld_min = r->ld;
  Job j;
  int rc;
  if ((rc = job_setup(ctx, j, c))) return rc;
  refl_attach(r, j);
  CK(cudaMemsetAsync(j.s.status, 0, sizeof(int), st));
  CK(launch_diag(j.s, st));
  double d3[3];
  rc = read_status(ctx, j, d3);
  if (diag_host) { diag_host[0] = d3[0]; diag_host[1] = d3[1]; }
  return rc;
}

/* t_solver.solve(b, adjoint) (reflector.py:80-153): B (k0 x m, device) in place.
 * t_solver.reconstruct() / seed p: ots_reflector_get (which 0 = P, 1 = T). */
int ots_reflector_tsolve_f64(ots_ctx* ctx, const ots_refl* r, int64_t m, double* B, int64_t ldb, int adjoint,
                             void* stream) {
  if (!ctx || !r) return OTS_E_VALUE;
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();   // a stale error from unrelated earlier work is not ours
  SmallState s = r->s;
  CK(launch_tsolve(s, B, (int)ldb, (int)m, adjoint, (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return OTS_OK;
}

int ots_reflector_get_f64(ots_ctx* ctx, const ots_refl* r, int which, double* out, int64_t ldo, void* stream) {
  if (!ctx || !r) return OTS_E_VALUE;
  const double* src = which == 0 ? r->s.P : r->s.Tdense;
  CK(cudaMemcpy2DAsync(out, ldo * 8, src, r->ld * 8, r->k0 * 8, r->k0, cudaMemcpyDeviceToDevice,
                       (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return OTS_OK;
}

int ots_householder_qr_f64(ots_ctx* ctx, int64_t m, int64_t k, const double* A, int64_t lda, double* Q,
                           int64_t ldq, double* R, int64_t ldr, int nonneg_diag, void* stream) {
  if (!ctx) return OTS_E_VALUE;
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();   // a stale error from unrelated earlier work is not ours
  cudaStream_t st = (cudaStream_t)stream;
  if (m < k) return fail(ctx, OTS_E_DIMENSION, "need rows >= cols");
  if (k > 64) return fail(ctx, OTS_E_UNSUPPORTED, "k > 64 not supported by this build");
  int rc;
  if ((rc = validate_layout(ctx, A, lda, "A"))) return rc;
  if ((rc = validate_layout(ctx, Q, ldq, "Q"))) return rc;
  if (k == 0) return OTS_OK;
  JobCfg c{m, 1 /*row0!=0: no top block*/, 0, k, nullptr, 0, A, lda, Q, ldq, OTS_CHOICE_QR, nullptr, 0,
           1e-8, 0, st, false};
  Job j;
  if ((rc = job_setup(ctx, j, c))) return rc;
  const int KT = j.KT;
  prof_begin(ctx, st);
  if (A != Q) CK(cudaMemcpy2DAsync(Q, ldq * 8, A, lda * 8, k * 8, m, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(j.s.status, 0, sizeof(int), st));
  if ((rc = run_factor_levels(ctx, j.lv, KT, st))) return rc;
  prof_mark(ctx, st, "factor");
  set_identity_kernel<<<(KT * KT + 255) / 256, 256, 0, st>>>(j.ident, KT);
  if ((rc = run_qform_levels(ctx, j.lv, KT, j.ident, st))) return rc;
  prof_mark(ctx, st, "qform");
  CK(launch_sign(j.s, Q, ldq, j.lv.back().R, KT, R, (int)ldr, st));
  // Q <- Q diag(s)
  NnArgs a{};
  a.P = nullptr; a.ldp = 0; a.kdim = 0; a.Z = nullptr; a.ldz = 0;
  a.B = Q; a.ldb = ldq; a.X = Q; a.ldx = ldq; a.ncols = (int)k;
  a.row_begin = 0; a.row_end = m; a.colscale = j.svec;
  CK(launch_tsgemm_nn(a, KT, ctx->nsm, st));
  if (nonneg_diag) {
    nonneg_q_kernel<<<std::min<long>(1024, (m * k + 255) / 256), 256, 0, st>>>(Q, ldq, m, (int)k, R, ldr);
    nonneg_r_kernel<<<1, 256, 0, st>>>((int)k, R, ldr);
  }
  nonfinite_status_kernel<<<1, 256, 0, st>>>(R, ldr, (int)k, (int)k, j.s.status);
  prof_mark(ctx, st, "sign");
  ctx->launches = 4 + 3 * (int)j.lv.size() + (nonneg_diag ? 1 : 0);
  CK(cudaMemcpyAsync(ctx->h_status, j.s.status, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  prof_end(ctx);
  CK(cudaGetLastError());
  if (ctx->h_status[0] == OTS_E_VALUE) return fail(ctx, OTS_E_VALUE, "input contains non-finite entries");
  return OTS_OK;
}

// Dense SPD weight B (n x n): lower Cholesky factor into L (B unchanged when
// L != B).  OTS_E_NOT_PD when a pivot is not positive.
int ots_dense_cholesky_f64(ots_ctx* ctx, int64_t n, const double* B, int64_t ldb, double* L, int64_t ldl,
                           void* stream) {
  if (!ctx) return OTS_E_VALUE;
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0) return fail(ctx, OTS_E_DIMENSION, "n must be >= 0");
  if (n == 0) return OTS_OK;
  if (L != B) CK(cudaMemcpy2DAsync(L, ldl * 8, B, ldb * 8, n * 8, n, cudaMemcpyDeviceToDevice, st));
  int* dstat = ctx->nn_counter + 16;   // spare device word of the context
  CK(launch_dense_cholesky(L, ldl, (int)n, dstat, st));
  CK(cudaMemcpyAsync(ctx->h_status, dstat, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (ctx->h_status[0] == OTS_E_NOT_PD) return fail(ctx, OTS_E_NOT_PD, "weight matrix is not positive definite");
  return OTS_OK;
}

// X (n x m) <- L^{-T} X  (L lower, from ots_dense_cholesky_f64)
int ots_dense_trsm_lt_f64(ots_ctx* ctx, int64_t n, int64_t m, const double* L, int64_t ldl, double* X,
                          int64_t ldx, void* stream) {
  if (!ctx) return OTS_E_VALUE;
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();
  CK(launch_trsm_lt(L, ldl, X, ldx, (int)n, (int)m, (cudaStream_t)stream));
  return OTS_OK;
}

// Y (n x m) = L^T X
int ots_dense_trmm_lt_f64(ots_ctx* ctx, int64_t n, int64_t m, const double* L, int64_t ldl, const double* X,
                          int64_t ldx, double* Y, int64_t ldy, void* stream) {
  if (!ctx) return OTS_E_VALUE;
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();
  CK(launch_trmm_lt(L, ldl, X, ldx, Y, ldy, (int)n, (int)m, (cudaStream_t)stream));
  return OTS_OK;
}

// b_two_stage_qr (oblique.py:279-315) for a dense SPD B = L L^T with the
// canonical basis u = initial_b_basis(B, k0+k) = [L_m^{-T}; 0]: Algorithm 1 on
// (L^T V, L^T A), Q = L^{-T} Q' sgn, R = sgn R', S unchanged.
int ots_b_two_stage_dense_f64(ots_ctx* ctx, int64_t n, int64_t k0, int64_t k, const double* V, int64_t ldv,
                              const double* A, int64_t lda, const double* L, int64_t ldl, int choice,
                              const double* P, int64_t ldp, double orth_tol, double* Q, int64_t ldq, double* R,
                              int64_t ldr, double* S, int64_t lds, double* diag_host, void* stream) {
  if (!ctx) return OTS_E_VALUE;
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();
  cudaStream_t st = (cudaStream_t)stream;
  if (k0 + k > n) return fail(ctx, OTS_E_DIMENSION, "need k0 + k <= n");
  if (k > 64 || k0 > 1024) return fail(ctx, OTS_E_UNSUPPORTED, "shape not supported by this build");
  if (k0 < 1 || k < 1) return fail(ctx, OTS_E_UNSUPPORTED, "b_two_stage_dense needs k0, k >= 1");
  if (choice < 0 || choice > 3) return fail(ctx, OTS_E_PARAMETER, "unknown choice");
  int rc;
  if ((rc = validate_layout(ctx, V, ldv, "V"))) return rc;
  if ((rc = validate_layout(ctx, A, lda, "A"))) return rc;
  if ((rc = validate_layout(ctx, Q, ldq, "Q"))) return rc;
  const long ldv2 = (k0 + 1) & ~1L, lda2 = (k + 1) & ~1L, ldt = (k0 + 1) & ~1L;
  const int PWv = pad32(k0);
  const int gridu = grid_for_tn(PWv, 0, true, true, ctx->nsm);
  size_t need = ((size_t)n * (ldv2 + lda2) + (size_t)gridu * PWv * PWv + (size_t)PWv * PWv +
                 (size_t)k0 * ldt + 256) * 8 + 4096;
  if (need > ctx->b_size) {
    if (ctx->b_ws) cudaFree(ctx->b_ws);
    ctx->b_ws = nullptr; ctx->b_size = 0;
    CK(cudaMalloc(&ctx->b_ws, need));
    ctx->b_size = need;
  }
  double* V2 = reinterpret_cast<double*>(ctx->b_ws);
  double* A2 = V2 + (size_t)n * ldv2;
  double* part = A2 + (size_t)n * lda2;
  double* Gu = part + (size_t)gridu * PWv * PWv;
  double* Lti = Gu + (size_t)PWv * PWv;                 // L_m^{-T}, k0 x k0
  CK(launch_trmm_lt(L, ldl, V, ldv, V2, ldv2, (int)n, (int)k0, st));
  CK(launch_trmm_lt(L, ldl, A, lda, A2, lda2, (int)n, (int)k, st));
  set_identity_ld_kernel<<<16, 256, 0, st>>>(Lti, (int)k0, (int)ldt);
  CK(launch_trsm_lt(L, ldl, Lti, ldt, (int)k0, (int)k0, st));     // (L^{-T})_{top} = L_m^{-T}
  TnArgs a{};
  a.P = V; a.ldp = ldv; a.pc0 = 0; a.pcols = (int)k0;
  a.row_begin = 0; a.row_end = n; a.partial = part;
  CK(launch_tsgemm_tn(a, PWv, 0, true, true, gridu, st));
  CK(launch_reduce(part, gridu, (long)PWv * PWv, Gu, 1.0, st));
  BHook bh{Gu, PWv, nullptr, nullptr, n, L, ldl, Lti, (int)ldt, V, ldv};
  JobCfg c{n, 0, k0, k, V2, ldv2, A2, lda2, Q, ldq, choice, P, ldp, orth_tol, 0, st, false};
  return two_stage_pipeline(ctx, c, OTS_INTRA_HOUSEHOLDER, Q, ldq, R, ldr, S, lds, diag_host, &bh);
}

int ots_b_two_stage_diag_f64(ots_ctx* ctx, int64_t n, int64_t k0, int64_t k, const double* V, int64_t ldv,
                             const double* A, int64_t lda, const double* d, int choice, const double* P,
                             int64_t ldp, double orth_tol, double* Q, int64_t ldq, double* R, int64_t ldr,
                             double* S, int64_t lds, double* diag_host, void* stream) {
  if (!ctx) return OTS_E_VALUE;
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();   // a stale error from unrelated earlier work is not ours
  cudaStream_t st = (cudaStream_t)stream;
  if (k0 + k > n) return fail(ctx, OTS_E_DIMENSION, "need k0 + k <= n");
  if (k > 64 || k0 > 1024) return fail(ctx, OTS_E_UNSUPPORTED, "shape not supported by this build");
  if (k0 < 1 || k < 1) return fail(ctx, OTS_E_UNSUPPORTED, "b_two_stage_diag needs k0, k >= 1");
  if (choice < 0 || choice > 3) return fail(ctx, OTS_E_PARAMETER, "unknown choice");
  int rc;
  if ((rc = validate_layout(ctx, V, ldv, "V"))) return rc;
  if ((rc = validate_layout(ctx, A, lda, "A"))) return rc;
  if ((rc = validate_layout(ctx, Q, ldq, "Q"))) return rc;
  // scaled copies D^{1/2} V, D^{1/2} A and the unweighted Gram live in a
  // second buffer owned by the context
  const long ldv2 = (k0 + 1) & ~1L, lda2 = (k + 1) & ~1L;
  const int PWv = pad32(k0);
  const int gridu = grid_for_tn(PWv, 0, true, true, ctx->nsm);
  size_t need = ((size_t)n * (ldv2 + lda2) + (size_t)gridu * PWv * PWv + (size_t)PWv * PWv + 256) * 8 + 4096;
  if (need > ctx->b_size) {
    if (ctx->b_ws) cudaFree(ctx->b_ws);
    ctx->b_ws = nullptr; ctx->b_size = 0;
    CK(cudaMalloc(&ctx->b_ws, need));
    ctx->b_size = need;
  }
  double* V2 = reinterpret_cast<double*>(ctx->b_ws);
  double* A2 = V2 + (size_t)n * ldv2;
  double* part = A2 + (size_t)n * lda2;
  double* Gu = part + (size_t)gridu * PWv * PWv;
  double* dinv = Gu + (size_t)PWv * PWv;
  row_scale_pairs_kernel<<<row_grid(n), 256, 0, st>>>(V, ldv, n, (int)k0, d, 0, V2, ldv2);
  row_scale_pairs_kernel<<<row_grid(n), 256, 0, st>>>(A, lda, n, (int)k, d, 0, A2, lda2);
  inv_top_kernel<<<1, 128, 0, st>>>(d, (int)k0, dinv);
  TnArgs a{};
  a.P = V; a.ldp = ldv; a.pc0 = 0; a.pcols = (int)k0;
  a.row_begin = 0; a.row_end = n; a.partial = part;
  CK(launch_tsgemm_tn(a, PWv, 0, true, true, gridu, st));
  CK(launch_reduce(part, gridu, (long)PWv * PWv, Gu, 1.0, st));
  BHook bh{Gu, PWv, dinv, d, n};
  JobCfg c{n, 0, k0, k, V2, ldv2, A2, lda2, Q, ldq, choice, P, ldp, orth_tol, 0, st, false};
  c.exact_intra = true;
  return two_stage_pipeline(ctx, c, OTS_INTRA_HOUSEHOLDER, Q, ldq, R, ldr, S, lds, diag_host, &bh);
}

int ots_shifted_cholesky_qr_f64(ots_ctx* ctx, int64_t m, int64_t k, const double* A, int64_t lda, double* Q,
                                int64_t ldq, double* R, int64_t ldr, void* stream) {
  return ots_shifted_cholesky_qr_ex_f64(ctx, m, k, A, lda, Q, ldq, R, ldr, 2, stream);
}

int ots_shifted_cholesky_qr_ex_f64(ots_ctx* ctx, int64_t m, int64_t k, const double* A, int64_t lda, double* Q,
                                   int64_t ldq, double* R, int64_t ldr, int refine_passes, void* stream) {
  if (!ctx) return OTS_E_VALUE;
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();   // a stale error from unrelated earlier work is not ours
  cudaStream_t st = (cudaStream_t)stream;
  if (m < k) return fail(ctx, OTS_E_DIMENSION, "need rows >= cols");
  if (k > 64) return fail(ctx, OTS_E_UNSUPPORTED, "k > 64 not supported by this build");
  int rc;
  if ((rc = validate_layout(ctx, A, lda, "A"))) return rc;
  if ((rc = validate_layout(ctx, Q, ldq, "Q"))) return rc;
  if (k == 0) return OTS_OK;
  JobCfg c{m, 1, 0, k, nullptr, 0, A, lda, Q, ldq, OTS_CHOICE_QR, nullptr, 0, 1e-8, 0, st, false};
  Job j;
  if ((rc = job_setup(ctx, j, c))) return rc;
  if (A != Q) CK(cudaMemcpy2DAsync(Q, ldq * 8, A, lda * 8, k * 8, m, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(j.s.status, 0, sizeof(int), st));
  if ((rc = run_cholshift(ctx, j, Q, ldq, m, (int)k, R, ldr, st, refine_passes))) return rc;
  ctx->launches = 1 + 4 * (1 + std::max(0, refine_passes));
  CK(cudaMemcpyAsync(ctx->h_status, j.s.status, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (ctx->h_status[0] == OTS_E_INTRA_FAILURE)
    return fail(ctx, OTS_E_NOT_PD, "Cholesky factorization failed (matrix not positive definite)");
  return OTS_OK;
}

int ots_modified_lu_f64(ots_ctx* ctx, int64_t n, const double* Z, int64_t ldz, double* LU, double* p,
                        void* stream) {
  if (!ctx) return OTS_E_VALUE;
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();   // a stale error from unrelated earlier work is not ours
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0) return OTS_OK;
  if (n > 512) return fail(ctx, OTS_E_UNSUPPORTED, "n > 512");
  int rc = ensure_ws(ctx, (size_t)(n * n + 2 * n + 64) * 8);
  if (rc) return rc;
  double* work = reinterpret_cast<double*>(ctx->ws);
  int* status = reinterpret_cast<int*>(work + n * n + 2 * n + 8);
  CK(launch_mlu(Z, (int)ldz, (int)n, LU, p, work, status, st));
  CK(cudaMemcpyAsync(ctx->h_status, status, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (ctx->h_status[0] == OTS_E_NORM_BOUND) return fail(ctx, OTS_E_NORM_BOUND, "||z||_2 exceeds 1 beyond tolerance");
  return OTS_OK;
}

// ----------------------------- distributed phases -------------------------
int ots_dist_begin(ots_ctx* ctx, int64_t n_local, int64_t row0, int64_t k0, int64_t k, const double* V,
                   int64_t ldv, const double* A, int64_t lda, double* Q, int64_t ldq, int choice,
                   const double* P, int64_t ldp, double orth_tol, void* stream) {
  cudaSetDevice(ctx->device);
  (void)cudaGetLastError();   // a stale error from unrelated earlier work is not ours
  if (k > 64 || k0 > 1024 || k0 < 1 || k < 1) return fail(ctx, OTS_E_UNSUPPORTED, "shape not in this build");
  if (row0 == 0 && n_local < k0 + k) return fail(ctx, OTS_E_DIMENSION, "rank 0 must own >= k0+k rows");
  int rc;
  if ((rc = validate_layout(ctx, V, ldv, "V"))) return rc;
  if ((rc = validate_layout(ctx, A, lda, "A"))) return rc;
  if ((rc = validate_layout(ctx, Q, ldq, "Q"))) return rc;
  delete ctx->job;
  ctx->job = new Job();
  JobCfg c{n_local, row0, k0, k, V, ldv, A, lda, Q, ldq, choice, P, ldp, orth_tol, 0,
           (cudaStream_t)stream, true};
  // per rank the row-parallel work is short, so the diagnostics (side stream,
  // three CTAs) run beside apply1 and the factor, which are planned for the
  // remaining SMs
  if (ctx->nsm > 16) c.nsm_avail = ctx->nsm - 3;
  c.fast_try = true;     // each rank picks its route on its own rows: R, C and Y2 are exchanged either way
  ctx->fast_taken = 0;
  return job_setup(ctx, *ctx->job, c);
}

int ots_dist_sizes(ots_ctx* ctx, int64_t* out4) {
  if (!ctx->job) return fail(ctx, OTS_E_VALUE, "ots_dist_begin not called");
  Job& j = *ctx->job;
  out4[0] = (int64_t)j.PW * j.NTOT1;                          // gram partial
  out4[1] = j.c.k0 * ((j.c.k0 + j.c.k + 1) & ~1L);            // packed top rows
  out4[2] = j.KT;                                              // R block is KT x KT
  out4[3] = (int64_t)j.PW * j.BWa;                             // Y2 partial
  return OTS_OK;
}

int ots_dist_gram(ots_ctx* ctx, double* gram_out) {
  Job& j = *ctx->job;
  int rc = j.fast ? fast_gram(ctx, j) : phase_gram(ctx, j);
  if (rc) return rc;
  long cnt = (long)j.PW * j.NTOT1;
  if (gram_out) CK(cudaMemcpyAsync(gram_out, j.Gfull, cnt * 8, cudaMemcpyDeviceToDevice, j.c.st));
  return OTS_OK;
}

__global__ void pack_top_kernel(const double* V, long ldv, const double* A, long lda, int k0, int k,
                                double* top, int ldt) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k0 * (k0 + k); e += gridDim.x * blockDim.x) {
    int i = e / (k0 + k), jj = e - i * (k0 + k);
    top[i * ldt + jj] = jj < k0 ? V[(long)i * ldv + jj] : A[(long)i * lda + (jj - k0)];
  }
}

int ots_dist_top_rows(ots_ctx* ctx, double* top_out) {
  Job& j = *ctx->job;
  const long k0 = j.c.k0, k = j.c.k;
  const int ldt = (int)((k0 + k + 1) & ~1L);
  if (top_out && j.c.row0 == 0)
    pack_top_kernel<<<32, 256, 0, j.c.st>>>(j.c.V, j.c.ldv, j.c.A, j.c.lda, (int)k0, (int)k, top_out, ldt);
  CK(cudaGetLastError());
  return OTS_OK;
}

// V_t-only seed (seedA) from the broadcast top rows, on the side stream; the
// Gram that follows uses nsm-1 CTAs so seedA has its SM (as in the one-GPU
// pipeline).  Optional: ots_dist_seed then runs only the Gram-dependent part.
int ots_dist_seed_early(ots_ctx* ctx, const double* top_rows) {
  Job& j = *ctx->job;
  if (!top_rows || ctx->nsm <= 8) return OTS_OK;
  const long k0 = j.c.k0, k = j.c.k;
  const int ldt = (int)((k0 + k + 1) & ~1L);
  CK(cudaMemcpyAsync(j.top, top_rows, (size_t)k0 * ldt * 8, cudaMemcpyDeviceToDevice, j.c.st));
  j.s.V = j.top; j.s.ldv = ldt; j.s.A = j.top + k0; j.s.lda = ldt;
  CK(cudaEventRecord(ctx->ev_seedA, j.c.st));
  CK(cudaStreamWaitEvent(ctx->side, ctx->ev_seedA, 0));
  CK(launch_seed_split(j.s, 0, ctx->side));
  CK(cudaEventRecord(ctx->ev_seedA, ctx->side));
  j.gram_nsm = ctx->nsm - (seed_uses_cluster(j.s) ? 2 : 1);
  j.grid_tn = grid_for_tn(j.PW, j.BWa, true, true, j.gram_nsm);
  j.seeded_early = true;
  return OTS_OK;
}

int ots_dist_seed(ots_ctx* ctx, const double* gram_sum, const double* top_rows) {
  Job& j = *ctx->job;
  const long k0 = j.c.k0, k = j.c.k;
  const int ldt = (int)((k0 + k + 1) & ~1L);
  if (gram_sum && gram_sum != j.Gfull)
    CK(cudaMemcpyAsync(j.Gfull, gram_sum, (size_t)j.PW * j.NTOT1 * 8, cudaMemcpyDeviceToDevice, j.c.st));
  if (top_rows && !j.seeded_early) {
    CK(cudaMemcpyAsync(j.top, top_rows, (size_t)k0 * ldt * 8, cudaMemcpyDeviceToDevice, j.c.st));
    j.s.V = j.top; j.s.ldv = ldt; j.s.A = j.top + k0; j.s.lda = ldt;
  }
  j.s.Sout = j.s.Sd;  // S kept on device until finish
  j.s.lds_out = j.ld;
  if (j.seeded_early) {
    CK(cudaStreamWaitEvent(j.c.st, ctx->ev_seedA, 0));
    CK(launch_seed_split(j.s, 1, j.c.st));
  } else {
    CK(launch_seed(j.s, j.c.st));
  }
  CK(cudaEventRecord(ctx->ev_seed, j.c.st));
  CK(cudaStreamWaitEvent(ctx->side, ctx->ev_seed, 0));
  CK(launch_diag(j.s, ctx->side));   // beside apply1 / factor; waited for in ots_dist_finish
  CK(cudaEventRecord(ctx->ev_diag, ctx->side));
  return OTS_OK;
}

int ots_dist_factor(ots_ctx* ctx, double* r_local_out) {
  Job& j = *ctx->job;
  // apply1 (dynamic tiles) and the factor (chains planned for nsm - 3 SMs)
  // run beside the diagnostics launched by ots_dist_seed
  int rc;
  j.fast_active = false;
  if (j.fast) {
    rc = fast_factor(ctx, j);
    if (rc < 0) return rc;
    j.fast_active = rc == 0;
    ctx->fast_taken = j.fast_active ? 1 : 0;
  }
  if (!j.fast_active) {
    if ((rc = phase_apply1(ctx, j))) return rc;
    if ((rc = run_factor_levels(ctx, j.lv, j.KT, j.c.st))) return rc;
  }
  if (r_local_out)
    CK(cudaMemcpyAsync(r_local_out, j.lv.back().R, (size_t)j.KT * j.KT * 8, cudaMemcpyDeviceToDevice, j.c.st));
  return OTS_OK;
}

int ots_dist_tree(ots_ctx* ctx, const double* r_all, int nranks, int rank) {
  Job& j = *ctx->job;
  const int KT = j.KT;
  cudaStream_t st = j.c.st;
  if (nranks > 64) return fail(ctx, OTS_E_UNSUPPORTED, "more than 64 ranks");
  CK(cudaMemcpyAsync(j.Rall, r_all, (size_t)nranks * KT * KT * 8, cudaMemcpyDeviceToDevice, st));
  // global levels over the gathered rank R's (rows = nranks*KT)
  std::vector<Level> g;
  {
    // reuse the tail of the workspace: carve from a fresh arena after Cglob
    size_t used = (reinterpret_cast<char*>(j.Cglob + (size_t)64 * KT * KT) - ctx->ws);
    size_t need = plan_levels_bytes((long)nranks * KT, KT, 1) + 4096;
    if (used + need > ctx->ws_size) return fail(ctx, OTS_E_CUDA, "workspace too small for tree");
    Arena ar(ctx->ws + used, ctx->ws_size - used);
    // one chain per 4 R's (same shape as the local tree levels)
    Level L{};
    L.D = j.Rall; L.ldd = KT; L.ncols = KT;
    long nrows = (long)nranks * KT;
    long rpc = (long)KT * 4;
    L.G = ChainGeom{nrows, KT, 3, rpc, (int)((nrows + rpc - 1) / rpc)};
    L.UT = ar.take<double>((size_t)L.G.nchains * 4 * KT * KT);
    L.R = ar.take<double>((size_t)L.G.nchains * KT * KT);
    g.push_back(L);
    while (g.back().G.nchains > 1) {
      const Level& P = g.back();
      Level M{};
      M.D = P.R; M.ldd = KT; M.ncols = KT;
      long nr = (long)P.G.nchains * KT;
      M.G = ChainGeom{nr, KT, 3, rpc, (int)((nr + rpc - 1) / rpc)};
      M.UT = ar.take<double>((size_t)M.G.nchains * 4 * KT * KT);
      M.R = ar.take<double>((size_t)M.G.nchains * KT * KT);
      g.push_back(M);
    }
  }
  j.glv = g;
  int rc;
  if ((rc = run_factor_levels(ctx, j.glv, KT, st, true))) return rc;
  j.Rfinal = j.glv.back().R;
  set_identity_kernel<<<(KT * KT + 255) / 256, 256, 0, st>>>(j.ident, KT);
  if ((rc = run_qform_levels(ctx, j.glv, KT, j.ident, st))) return rc;
  // this rank's C block: rows [rank*KT, rank*KT+KT) of Rall (now output rows)
  CK(cudaMemcpyAsync(j.Cglob, j.Rall + (size_t)rank * KT * KT, (size_t)KT * KT * 8, cudaMemcpyDeviceToDevice, st));
  return OTS_OK;
}

int ots_dist_qform(ots_ctx* ctx, double* y2_out, double* sign_out) {
  Job& j = *ctx->job;
  cudaStream_t st = j.c.st;
  int rc;
  if (j.fast_active) {
    if ((rc = fast_coef(ctx, j, j.Cglob, j.c.row0 == 0, j.c.Q, j.c.ldq, j.Rfinal, j.s.D1 /*scratch R*/, j.ld)))
      return rc;
    if (j.c.row0 == 0 && sign_out)
      CK(cudaMemcpyAsync(sign_out, j.svec, j.c.k * 8, cudaMemcpyDeviceToDevice, st));
  } else {
    if ((rc = run_qform_levels(ctx, j.lv, j.KT, j.Cglob, st, j.nsm_use))) return rc;
    if (j.c.row0 == 0) {
      CK(launch_sign(j.s, j.c.Q + j.c.k0 * j.c.ldq, j.c.ldq, j.Rfinal, j.KT, j.s.D1 /*scratch R*/, j.ld, st));
      if (sign_out) CK(cudaMemcpyAsync(sign_out, j.svec, j.c.k * 8, cudaMemcpyDeviceToDevice, st));
    }
    if ((rc = phase_gram2(ctx, j))) return rc;
  }
  long cnt = (long)j.PW * j.BWa;
  if (y2_out) CK(cudaMemcpyAsync(y2_out, j.Y2full, cnt * 8, cudaMemcpyDeviceToDevice, st));
  return OTS_OK;
}

__global__ void rscale_kernel(const double* Rfin, int ldr, const double* s, double* R, long ldro, int k) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) {
    int i = e / k, jj = e - i * k;
    R[i * ldro + jj] = (jj >= i) ? s[i] * Rfin[i * ldr + jj] : 0.0;
  }
}
__global__ void copy_s_kernel(const double* Sd, int ld, double* S, long lds, int k0, int k) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k0 * k; e += gridDim.x * blockDim.x) {
    int i = e / k, jj = e - i * k;
    S[i * lds + jj] = Sd[i * ld + jj];
  }
}

int ots_dist_finish(ots_ctx* ctx, const double* y2_sum, const double* sign, double* R, int64_t ldr, double* S,
                    int64_t lds, double* diag_host) {
  Job& j = *ctx->job;
  cudaStream_t st = j.c.st;
  const int k0 = (int)j.c.k0, k = (int)j.c.k;
  if (y2_sum && y2_sum != j.Y2full)
    CK(cudaMemcpyAsync(j.Y2full, y2_sum, (size_t)j.PW * j.BWa * 8, cudaMemcpyDeviceToDevice, st));
  if (sign && sign != j.svec) CK(cudaMemcpyAsync(j.svec, sign, (size_t)k * 8, cudaMemcpyDeviceToDevice, st));
  copy_y2_kernel<<<16, 256, 0, st>>>(j.Y2full, j.BWa, j.s.Z2, j.ld, k0, k);
  CK(launch_z2(j.s, st));
  int rc;
  if ((rc = j.fast_active ? fast_final(ctx, j, true) : phase_apply2(ctx, j))) return rc;
  if (j.c.row0 == 0) CK(launch_qtop(j.s, j.c.Q, j.c.ldq, st));
  if (R) rscale_kernel<<<8, 256, 0, st>>>(j.Rfinal, j.KT, j.svec, R, ldr, k);
  if (S) copy_s_kernel<<<8, 256, 0, st>>>(j.s.Sd, j.ld, S, lds, k0, k);
  {  // kernels this rank launched for the call (ots_last_launch_count)
    const int nb = (k0 + 127) / 128;
    const int gram = (k0 <= 128) ? 2 : nb * (nb + 1) + 2 * nb;
    const bool top = j.c.row0 == 0;
    ctx->launches = gram + (top ? 1 : 0) + 2 + 1 + 2 * (int)j.lv.size() + 2 * (int)j.glv.size() + 1 +
                    (top ? 1 : 0) + 2 * nb + 3 + (top ? 1 : 0) + (R ? 1 : 0) + (S ? 1 : 0);
  }
  CK(cudaStreamWaitEvent(st, ctx->ev_diag, 0));   // diagnostics (side stream)
  return read_status(ctx, j, diag_host);
}

}  // extern "C"

#include "zpath.inc"
#include "metrics.inc"
