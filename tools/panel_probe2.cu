// Latency probe of the full panel_factor<64> (transposes + Gram sweep + Y)
// for one warp in isolation, optionally with DMMA-busy warps beside it.
#include "../paper_2602_14449_b200/csrc/chainqr.cu"
#include <cstdio>
namespace ots {
__global__ void probe_pf(const double* xin, double* out, long long* cyc, int reps, int nbusy) {
  using C = BlkCfg<64>;
  extern __shared__ __align__(128) double S[];
  double* Xs = S + 64 * 64;
  double* Tp = Xs + C::XS;
  double* scr = Tp + C::NP * 64;
  __shared__ double tau_s[64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) S[i] = (i % 65 == 0) ? 3.0 : 0.01 * (i % 7);
  __syncthreads();
  if (warp != 0) {
    if (warp <= nbusy) {
      double acc[2] = {0, 0};
      for (int i = 0; i < reps * 400; ++i) dmma(acc, 1.0 + lane, 0.5);
      out[threadIdx.x] = acc[0] + acc[1];
    }
    return;
  }
  double x[16][2];
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int f = 0; f < 16; ++f)
      for (int h = 0; h < 2; ++h) x[f][h] = xin[(f * 2 + h) * 32 + lane];
    __syncwarp();
    const int p = r & 7;
    long long t0 = clock64();
    panel_factor<64>(p, x, S, Xs + (p % 3) * C::YSLOT, Tp, tau_s, scr, Xs + C::NSLOT * C::YSLOT);
    __syncwarp();
    long long t1 = clock64();
    tot += t1 - t0;
    for (int f = 0; f < 16; ++f) out[64 + (f * 2) * 32 + lane] = x[f][0] + x[f][1];
  }
  if (lane == 0) cyc[0] = tot;
}
}
namespace ots { void debug_counters_small(unsigned long long*, int) {} }
int main() {
  double *xin, *o; long long* c;
  cudaMalloc(&xin, 32 * 32 * 8); cudaMalloc(&o, 65536); cudaMalloc(&c, 64);
  double h[1024];
  unsigned s = 1;
  for (int i = 0; i < 1024; ++i) { s = s * 1664525u + 1013904223u; h[i] = ((s >> 8) / 16777216.0) - 0.5; }
  cudaMemcpy(xin, h, 8192, cudaMemcpyHostToDevice);
  const int smem = ots::BlkCfg<64>::SMEM;
  cudaFuncSetAttribute(ots::probe_pf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int busy = 0; busy <= 7; busy += 7) {
    ots::probe_pf<<<1, 256, smem>>>(xin, o, c, 64, busy); cudaDeviceSynchronize();
    ots::probe_pf<<<1, 256, smem>>>(xin, o, c, 64, busy);
    long long hc; cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("busy warps %d: %.0f cycles per panel (%.0f per column)  err=%s\n", busy, hc / 64.0, hc / 512.0,
           cudaGetErrorString(cudaGetLastError()));
#ifdef OTS_TIMING
    unsigned long long d[16];
    cudaMemcpyFromSymbol(d, ots::g_dbg, sizeof(d));
    printf("   (2 launches) transpose-in %.0f  sweep %.0f  y-out %.0f per panel\n", d[8] / 128.0, d[9] / 128.0, d[12] / 128.0);
    cudaMemset(o, 0, 8);
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(ots::g_dbg, z, sizeof(z));
#endif
  }
  return 0;
}
