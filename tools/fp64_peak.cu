// FP64 peak microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync m8n8k4 f64).
// Prints JSON with measured TFLOP/s; used as the FP64 roofline denominator
// (MEASURED_PEAKS.json carries no FP64 figure).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = 1e-3 * (threadIdx.x & 7), b = 1e-3 * (threadIdx.x >> 3);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) dmma(acc[j][0], acc[j][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  // DFMA
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb); int iters = 4096;
    dfma_loop<<<blocks, tpb>>>(out, 16);
    cudaEventRecord(e0); dfma_loop<<<blocks, tpb>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * tpb;
    printf(", \"dfma_tpb%d_tflops\": %.3f", tpb, flops / ms / 1e9);
  }
  // DMMA with various accum counts / warps
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * (1024 / tpb); int iters = 8192;
    dmma_loop<8><<<blocks, tpb>>>(out, 16);
    cudaEventRecord(e0); dmma_loop<8><<<blocks, tpb>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (tpb / 32);
    printf(", \"dmma8_tpb%d_tflops\": %.3f", tpb, flops / ms / 1e9);
  }
  for (int tpb : {256, 512}) {
    int blocks = sms * (1024 / tpb); int iters = 4096;
    dmma_loop<16><<<blocks, tpb>>>(out, 16);
    cudaEventRecord(e0); dmma_loop<16><<<blocks, tpb>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 16 * (double)iters * blocks * (tpb / 32);
    printf(", \"dmma16_tpb%d_tflops\": %.3f", tpb, flops / ms / 1e9);
  }
  // HBM copy (double)
  size_t N = (size_t)1 << 30; double *x, *y; cudaMalloc(&x, N * 8); cudaMalloc(&y, N * 8);
  cudaMemset(x, 0, N * 8);
  cudaMemcpy(y, x, N * 8, cudaMemcpyDeviceToDevice);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); cudaMemcpy(y, x, N * 8, cudaMemcpyDeviceToDevice); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf(", \"copy_gbs\": %.1f", 2.0 * N * 8 / best / 1e6);
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
