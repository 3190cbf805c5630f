// Latency of one dependent dlarfg step (the pivot chain of the Gram-form
// panels) for three formulations: f64 MUFU seeds + Newton (dlarfg_nb), IEEE
// sqrt / division, and f32 MUFU seeds + f64 Newton.  One warp, dependent chain.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void v_mufu64(double alpha, double s2, double& beta, double& tau, double& scal) {
  const double h = fma(alpha, alpha, s2);
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(h));
  r = r * fma(-0.5 * h * r, r, 1.5);
  r = r * fma(-0.5 * h * r, r, 1.5);
  const double sq = h * r;
  const double t = fabs(alpha) + sq;
  double rt;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rt) : "d"(t));
  rt = rt * fma(-t, rt, 2.0);
  rt = rt * fma(-t, rt, 2.0);
  beta = -copysign(sq, alpha);
  tau = t * r;
  scal = copysign(rt, alpha);
}
__device__ __forceinline__ void v_ieee(double alpha, double s2, double& beta, double& tau, double& scal) {
  const double sq = sqrt(fma(alpha, alpha, s2));
  beta = -copysign(sq, alpha);
  tau = (beta - alpha) / beta;
  scal = 1.0 / (alpha - beta);
}
__device__ __forceinline__ void v_mufu32(double alpha, double s2, double& beta, double& tau, double& scal) {
  const double h = fma(alpha, alpha, s2);
  double r = (double)rsqrtf((float)h);
  r = r * fma(-0.5 * h * r, r, 1.5);
  r = r * fma(-0.5 * h * r, r, 1.5);
  const double sq = h * r;
  const double t = fabs(alpha) + sq;
  double rt = (double)__frcp_rn((float)t);
  rt = rt * fma(-t, rt, 2.0);
  rt = rt * fma(-t, rt, 2.0);
  beta = -copysign(sq, alpha);
  tau = t * r;
  scal = copysign(rt, alpha);
}

template <int V>
__global__ void probe(double* out, long long* cyc, int n) {
  double alpha = 1.0 + threadIdx.x * 1e-3, s2 = 0.5;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double beta, tau, scal;
    if (V == 0) v_mufu64(alpha, s2, beta, tau, scal);
    else if (V == 1) v_ieee(alpha, s2, beta, tau, scal);
    else v_mufu32(alpha, s2, beta, tau, scal);
    s2 = fma(scal * 1e-3, tau, 0.5);          // dependent
    alpha = fma(beta, 1e-9, alpha);
  }
  const long long t1 = clock64();
  out[threadIdx.x] = s2 + alpha;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void fma_chain(double* out, long long* cyc, int n) {
  double x = threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-7);
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void shfl_chain(double* out, long long* cyc, int n) {
  double x = threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1.0;
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d; long long* c; long long h;
  cudaMalloc(&d, 1024 * 8); cudaMalloc(&c, 8);
  const int n = 4096;
  const char* names[3] = {"mufu64+newton", "ieee sqrt/div", "mufu32+newton"};
  for (int rep = 0; rep < 2; ++rep) {
    probe<0><<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("%s: %.1f cycles/step\n", names[0], (double)h / n);
    probe<1><<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("%s: %.1f cycles/step\n", names[1], (double)h / n);
    probe<2><<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("%s: %.1f cycles/step\n", names[2], (double)h / n);
    fma_chain<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("dfma chain: %.1f cycles/op\n", (double)h / n);
    shfl_chain<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("shfl64+dadd chain: %.1f cycles/op\n", (double)h / n);
  }
  return 0;
}
