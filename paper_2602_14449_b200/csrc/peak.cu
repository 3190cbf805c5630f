// FP64 DMMA peak probe (the roofline denominator for the FP64 path; the
// driver-written MEASURED_PEAKS.json carries HBM and bf16 only).
#include "common.cuh"

namespace ots {

template <int NACC>
__global__ void dmma_peak_kernel(double* out, int iters) {
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = 0.0;
  const double a = 1e-3 * (threadIdx.x & 7), b = 1e-3 * (threadIdx.x >> 3);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) dmma(acc[j], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

cudaError_t fp64_peak(int nsm, cudaStream_t st, double* tflops) {
  double* out;
  cudaError_t e = cudaMalloc(&out, sizeof(double) * nsm * 1024);
  if (e != cudaSuccess) return e;
  const int tpb = 256, blocks = nsm * 4, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_peak_kernel<8><<<blocks, tpb, 0, st>>>(out, 64);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0, st);
    dmma_peak_kernel<8><<<blocks, tpb, 0, st>>>(out, iters);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (tpb / 32);
  *tflops = flops / (best * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError();
}

}  // namespace ots
