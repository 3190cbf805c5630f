// Check launch_tsgemm_tn sym instances against a CPU Gram.
#include "../paper_2602_14449_b200/csrc/tsgemm.cu"
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
using namespace ots;
int main() {
  int nsm = 148;
  for (int pcols : {40, 64, 80, 96, 112, 128}) {
    const long n = 20000;
    const int PW = (pcols + 31) / 32 * 32;
    const long ld = pcols + (pcols & 1);
    std::vector<double> h(n * ld);
    srand(1);
    for (auto& x : h) x = rand() / (double)RAND_MAX - 0.5;
    double *d, *part, *out;
    cudaMalloc(&d, h.size() * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    int grid = 2 * nsm;
    cudaMalloc(&part, (size_t)grid * PW * PW * 8);
    cudaMalloc(&out, (size_t)PW * PW * 8);
    TnArgs a{};
    a.P = d; a.ldp = ld; a.pc0 = 0; a.pcols = pcols; a.B = nullptr; a.ldb = 0; a.bc0 = 0; a.bcols = 0;
    a.row_begin = 0; a.row_end = n; a.b_row_begin = 0; a.p_row_begin = 0; a.partial = part;
    cudaError_t e = launch_tsgemm_tn(a, PW, 0, true, true, grid, 0);
    launch_reduce_strided(part, grid, pcols, pcols, PW, out, pcols, 1.0, 0);
    cudaDeviceSynchronize();
    std::vector<double> g(pcols * pcols);
    cudaMemcpy(g.data(), out, g.size() * 8, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < pcols; ++i)
      for (int j = 0; j <= i; ++j) {
        double s = 0;
        for (long r = 0; r < n; ++r) s += h[r * ld + i] * h[r * ld + j];
        err = fmax(err, fabs(s - g[i * pcols + j]));
      }
    printf("pcols %d PW %d launch=%d maxerr %.3e\n", pcols, PW, (int)e, err);
  }
  return 0;
}
