// Latency probe: panel_core (8-column structured Householder panel, one warp)
// in isolation, to separate its intrinsic dependency chain from contention.
#include "../paper_2602_14449_b200/csrc/chainqr.cu"
#include <cstdio>
namespace ots {
__global__ void probe_panel(double* out, long long* cyc, int reps, int nwarps_busy) {
  __shared__ double S[64 * 64];
  __shared__ double T8[64 * 8];
  __shared__ double tau[64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) S[i] = (i % 65 == 0) ? 1.0 : 0.01 * (i % 7);
  __syncthreads();
  if (warp != 0) {   // optional DMMA load on other warps
    if (warp < nwarps_busy) {
      double acc[2] = {0, 0};
      for (int i = 0; i < reps * 600; ++i) dmma(acc, 1.0 + lane, 0.5);
      out[threadIdx.x] = acc[0] + acc[1];
    }
    return;
  }
  double xr[4][8];
  for (int i = 0; i < 4; ++i)
    for (int c = 0; c < 8; ++c) xr[i][c] = 0.001 * ((lane * 7 + i * 13 + c * 5) % 17) + (c == i ? 1.0 : 0.0);
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    panel_core<64, false>(r & 7, xr, S, T8, tau);
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[0] = t1 - t0;
  double s = 0;
  for (int i = 0; i < 4; ++i) for (int c = 0; c < 8; ++c) s += xr[i][c];
  out[lane] = s;
}
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8192); cudaMalloc(&c, 64);
  for (int busy = 1; busy <= 8; busy *= 2) {
    ots::probe_panel<<<1, 256>>>(o, c, 64, busy); cudaDeviceSynchronize();
    ots::probe_panel<<<1, 256>>>(o, c, 64, busy);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("busy warps %d: %.0f cycles per column\n", busy - 1, h / 64.0 / 8.0);
  }
  return 0;
}
