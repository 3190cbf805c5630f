// DMMA (mma.sync m8n8k4 f64) issue-rate probe on sm_100a: TFLOP/s versus
// warps per SM, independent accumulators per warp and shared-memory operand
// loads per DMMA -- sizes the streaming kernels' warp layouts (gs_gram,
// gs_qform).  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
#include <cstdio>
#include <cuda_runtime.h>

// NACC accumulators, NLD fragment loads from smem per step, all NACC DMMAs per step
template <int NACC, int NLD>
__global__ void probe(double* out, int iters) {
  __shared__ double sm[64 * 64];
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) sm[i] = 1e-3 * (i & 15);
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = 1e-3 * g, b = 1e-3 * t;
  for (int it = 0; it < iters; ++it) {
    const int kk = it & 15;
    double f[NLD > 0 ? NLD : 1];
#pragma unroll
    for (int q = 0; q < NLD; ++q) f[q] = sm[(4 * kk + t) * 64 + ((8 * q + g) ^ (t << 1))];
#pragma unroll
    for (int j = 0; j < NACC; ++j) {
      const double x = NLD > 0 ? f[j % (NLD > 0 ? NLD : 1)] : a;
      const double y = NLD > 0 ? f[(j / 2) % (NLD > 0 ? NLD : 1)] : b;
      dmma(acc[j], x, y);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC, int NLD>
void run(const char* name, int warps_per_sm, int sms, double* out, cudaEvent_t e0, cudaEvent_t e1) {
  const int tpb = warps_per_sm * 32 > 1024 ? 512 : warps_per_sm * 32;
  const int bps = warps_per_sm * 32 / tpb;
  const int blocks = sms * bps;
  const int iters = 4096 * 16 / NACC;
  probe<NACC, NLD><<<blocks, tpb>>>(out, 64);
  cudaEventRecord(e0);
  probe<NACC, NLD><<<blocks, tpb>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 512.0 * NACC * (double)iters * blocks * (tpb / 32);
  printf(", \"%s_w%d\": %.2f", name, warps_per_sm, flops / ms / 1e9);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 2048);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"gpu\": \"%s\"", p.name);
  for (int w : {4, 8, 12, 16, 32}) {
    run<4, 0>("acc4", w, sms, out, e0, e1);
    run<18, 0>("acc18", w, sms, out, e0, e1);
    run<18, 8>("acc18_ld8", w, sms, out, e0, e1);
    run<9, 8>("acc9_ld8", w, sms, out, e0, e1);
    run<4, 4>("acc4_ld4", w, sms, out, e0, e1);
    run<8, 6>("acc8_ld6", w, sms, out, e0, e1);
  }
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
