// Do DMMA (mma.sync m8n8k4 f64) and DFMA share one FP64 unit on sm_100a?
// Warps 0..W/2-1 run a DMMA loop, the rest a DFMA loop, in the same CTAs;
// compare the combined rate with each alone.  Also dependent-chain latencies.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void mix(double* out, int iters, int mode) {   // mode 0: all DMMA, 1: all DFMA, 2: half/half
  const int warp = threadIdx.x >> 5;
  const bool do_mma = mode == 0 || (mode == 2 && (warp & 1) == 0);
  double s = 0;
  if (do_mma) {
    double acc[8][2];
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0;
    double a = 1e-3 * (threadIdx.x & 7), b = 1e-3 * (threadIdx.x >> 3);
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(acc[j][0], acc[j][1], a, b);
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  } else {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double bb = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {   // 32 FMA per iteration = 64 flop/thread = 2048 flop/warp = 4 DMMA
        a0 = fma(a0, bb, c); a1 = fma(a1, bb, c); a2 = fma(a2, bb, c); a3 = fma(a3, bb, c);
        a4 = fma(a4, bb, c); a5 = fma(a5, bb, c); a6 = fma(a6, bb, c); a7 = fma(a7, bb, c);
      }
    s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void lat(double* out, int iters, long long* cyc) {
  double d0 = 0, d1 = 0, a = 1e-3 * (threadIdx.x & 7), b = 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) dmma(d0, d1, a, b);
  long long t1 = clock64();
  double x = threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) x = fma(x, 0.9999, 1e-7);
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / iters; cyc[1] = (t2 - t1) / iters; }
  out[threadIdx.x] = d0 + d1 + x;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 4 * 1024);
  long long* cyc; cudaMallocManaged(&cyc, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int tpb = 512, blocks = sms * 2, iters = 8192;
  printf("{");
  for (int mode = 0; mode < 3; ++mode) {
    mix<<<blocks, tpb>>>(out, 64, mode);
    cudaEventRecord(e0); mix<<<blocks, tpb>>>(out, iters, mode); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warps = (double)blocks * tpb / 32;
    double fl_mma = 512.0 * 8 * iters, fl_fma = 2048.0 * iters;   // per warp
    double flops = mode == 0 ? warps * fl_mma : mode == 1 ? warps * fl_fma : warps / 2 * (fl_mma + fl_fma);
    printf("%s\"mode%d_ms\": %.3f, \"mode%d_tflops\": %.2f", mode ? ", " : "", mode, ms, mode, flops / ms / 1e9);
  }
  lat<<<1, 32>>>(out, 4096, cyc); cudaDeviceSynchronize();
  printf(", \"dmma_dep_latency_cyc\": %lld, \"dfma_dep_latency_cyc\": %lld}\n", cyc[0], cyc[1]);
  return 0;
}
