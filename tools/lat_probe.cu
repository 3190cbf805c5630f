// Dependent-chain latency probe for FP64 ops on sm_100a (one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* cyc, double seed) {
  double a = seed + threadIdx.x, b = 1.0000001, c = 1e-9;
  long long t0, t1;
  const int N = 1024;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = fma(a, b, c);
  t1 = clock64(); cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = a + c;
  t1 = clock64(); cyc[1] = t1 - t0;
  // SHFL (double) chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1) + c;
  t1 = clock64(); cyc[2] = t1 - t0;
  // rsqrt chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = rsqrt(a) + 1.0;
  t1 = clock64(); cyc[3] = t1 - t0;
  // rcp.approx + 2 newton chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) {
    double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    r = r * fma(-a, r, 2.0); r = r * fma(-a, r, 2.0);
    a = r + 1.5;
  }
  t1 = clock64(); cyc[4] = t1 - t0;
  // DMMA chain
  double acc[2] = {a, c};
  t0 = clock64();
  for (int i = 0; i < N; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(acc[0]), "+d"(acc[1]) : "d"(b), "d"(c));
  t1 = clock64(); cyc[5] = t1 - t0;
  // LDS dependent chain (pointer chasing through smem values)
  __shared__ double sm[64];
  sm[threadIdx.x] = 0.0; sm[threadIdx.x + 32] = 0.0;
  __syncwarp();
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < N; ++i) { double v = sm[idx]; idx = (idx + (int)v + 1) & 63; }
  t1 = clock64(); cyc[6] = t1 - t0;
  // double division chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = 1.0 / a + 1.0;
  t1 = clock64(); cyc[7] = t1 - t0;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) a = sqrt(a) + 1.0;
  t1 = clock64(); cyc[8] = t1 - t0;
  out[threadIdx.x] = a + acc[0] + acc[1] + idx;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 16 * 8);
  probe<<<1, 32>>>(o, c, 1.0); cudaDeviceSynchronize();
  probe<<<1, 32>>>(o, c, 1.0);
  long long h[16]; cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"dfma", "dadd", "shfl_f64+dadd", "rsqrt_f64+dadd", "rcp+2newton+dadd", "dmma", "lds(+iadd)", "ddiv+dadd", "dsqrt+dadd"};
  for (int i = 0; i < 9; ++i) printf("%-20s %.1f cyc/iter\n", nm[i], h[i] / 1024.0);
  return 0;
}
