// Shared device helpers for the B200 (sm_100a) two-stage orthogonalization path.
//
// FP64 math uses the warp-level DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4):
// on sm_100a tcgen05 has no f64 kind, and DMMA and DFMA share the same
// ~37 TF/s peak (profiles/r01_fp64_peak.json), so DMMA is chosen for its
// operand reuse (8 FMAs per register operand instead of 1) and low issue cost.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef OTS_HD
#define OTS_HD __host__ __device__ __forceinline__
#endif

namespace ots {

// ---------------------------------------------------------------------------
// DMMA m8n8k4 (f64).  Fragment ownership (PTX ISA, mma.m8n8k4 .f64):
//   A (8x4 row):  a  = A[g][t]          g = lane>>2, t = lane&3
//   B (4x8 col):  b  = B[t][g]
//   C (8x8):      c0 = C[g][2t], c1 = C[g][2t+1]
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// Shared-memory tile layout.  Row-major tiles of W doubles per row (W a
// multiple of 16), 16-byte units XOR-swizzled by ((row & 3) << 1).  This makes
// both fragment access patterns of m8n8k4 run at the 2-wavefront minimum for a
// 256-byte warp access:
//   P1: 4 consecutive rows x 8 consecutive columns (A^T / B operands)
//   P2: 8 consecutive rows x 4 consecutive columns (row-major A operand)
// ---------------------------------------------------------------------------
OTS_HD int swz(int r, int c, int W) {
  return r * W + ((((c >> 1) ^ ((r & 3) << 1)) << 1) | (c & 1));
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) with zero fill: src_bytes in {0, 8, 16}.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Load `rows` x `cols` doubles (global row-major, ld) starting at (r0, c0)
// into a swizzled smem tile of width W (W >= padded cols).  Rows outside
// [rlo, rhi) and columns >= cmax are zero-filled.  16-byte units; requires
// 16-byte aligned global rows (ld even, base 16B aligned) -- enforced on host.
__device__ __forceinline__ void load_tile_async(double* sm, int W, const double* g, long ld,
                                                long r0, int nrows, long rlo, long rhi,
                                                int c0, int ncols_pad, int cmax,
                                                int tid, int nthreads) {
  const int upr = ncols_pad >> 1;  // 16B units per row
  const int total = nrows * upr;
  for (int i = tid; i < total; i += nthreads) {
    int r = i / upr;
    int u = i - r * upr;
    long gr = r0 + r;
    int c = c0 + 2 * u;
    int bytes = 0;
    const double* src = g;
    if (gr >= rlo && gr < rhi && c < cmax) {
      bytes = (c + 1 < cmax) ? 16 : 8;
      src = g + gr * ld + c;
    }
    cp_async16(sm + swz(r, 2 * u, W), src, bytes);
  }
}

// mbarrier helpers (shared::cta)
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// arrive on `bar` when all prior cp.async of this thread have completed
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace ots

// Status codes (C-ABI).  One negative code per exception class of the
// reference's errors.py:4-65 (the Python facade maps them back).
#define OTS_OK 0
#define OTS_E_DIMENSION -1
#define OTS_E_NOT_HERMITIAN -2
#define OTS_E_NOT_PD -3
#define OTS_E_CONVERGENCE -4
#define OTS_E_SINGULAR -5
#define OTS_E_NORM_BOUND -6
#define OTS_E_SINGULAR_T -7
#define OTS_E_ORTHONORMALITY -8
#define OTS_E_INTRA_FAILURE -9
#define OTS_E_BREAKDOWN -10
#define OTS_E_PARAMETER -12
#define OTS_E_VALUE -20
#define OTS_E_CUDA -30
#define OTS_E_UNSUPPORTED -31
