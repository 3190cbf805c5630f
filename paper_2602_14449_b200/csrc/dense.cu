// Dense SPD weight B for the B-inner-product extension (oblique.py:36-90,
// 93-108, 279-315).  With B = L L^T (lower L, the reference's chol_b), the
// B-inner product is the Euclidean one of L^T x, and the canonical initial
// basis initial_b_basis(B, m) = [L_m^{-T}; 0] maps to [I_m; 0].  So Algorithm 4
// on (V, A) equals the Euclidean Algorithm 1 on (L^T V, L^T A), mapped back by
// Q = L^{-T} Q' sgn, R = sgn R' (SURVEY Appendix A.2 with D^1/2 -> L^T).
// Kernels here: blocked right-looking Cholesky, Y = L^T X, X <- L^{-T} X.
// All matrices row-major with leading dimensions; L's strict upper triangle is
// stored as exact zeros.  Sizes are those of a dense n x n weight (n up to a
// few thousand), so these are simple shared-memory tiled kernels.
#include "common.cuh"
#include "kernels.cuh"

namespace ots {

constexpr int DB = 32;   // panel / tile width

// factor the nb x nb diagonal block at j0 and solve the rows below:
// L21 = A21 L11^{-T}.  One CTA.
__global__ void __launch_bounds__(512) chol_panel_kernel(double* A, long ld, int n, int j0, int* status) {
  __shared__ double Dm[DB][DB + 1];
  const int nb = n - j0 < DB ? n - j0 : DB;
  const int tid = threadIdx.x;
  for (int e = tid; e < nb * nb; e += blockDim.x) Dm[e / nb][e % nb] = A[(long)(j0 + e / nb) * ld + j0 + e % nb];
  __syncthreads();
  for (int c = 0; c < nb; ++c) {
    if (tid == 0) {
      const double d = Dm[c][c];
      if (!(d > 0.0)) atomicExch(status, OTS_E_NOT_PD);
      Dm[c][c] = sqrt(fmax(d, 0.0));
    }
    __syncthreads();
    const double dc = Dm[c][c];
    for (int r = c + 1 + tid; r < nb; r += blockDim.x) Dm[r][c] = dc > 0.0 ? Dm[r][c] / dc : 0.0;
    __syncthreads();
    const int w = nb - c - 1;
    for (int e = tid; e < w * w; e += blockDim.x) {
      const int r = c + 1 + e / w, cc = c + 1 + e % w;
      if (cc <= r) Dm[r][cc] -= Dm[r][c] * Dm[cc][c];
    }
    __syncthreads();
  }
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int r = e / nb, cc = e % nb;
    A[(long)(j0 + r) * ld + j0 + cc] = cc <= r ? Dm[r][cc] : 0.0;
  }
  for (long i = j0 + nb + tid; i < n; i += blockDim.x) {   // forward substitution per row
    double x[DB];
    double* row = A + i * ld + j0;
#pragma unroll
    for (int c = 0; c < DB; ++c) {
      if (c < nb) {
        double s = row[c];
#pragma unroll
        for (int l = 0; l < c; ++l) s -= x[l] * Dm[c][l];
        x[c] = Dm[c][c] > 0.0 ? s / Dm[c][c] : 0.0;
        row[c] = x[c];
      }
    }
  }
}

// trailing update A[i][c] -= sum_l L[i][l] L[c][l], j0+nb <= c <= i
__global__ void __launch_bounds__(1024) chol_update_kernel(double* A, long ld, int n, int j0, int nb) {
  const int t0 = j0 + nb;
  const int bi = t0 + blockIdx.y * DB, bc = t0 + blockIdx.x * DB;
  if (bc > bi + DB - 1) return;   // tile strictly above the diagonal
  __shared__ double Li[DB][DB + 1], Lc[DB][DB + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;
  Li[ty][tx] = (bi + ty < n && tx < nb) ? A[(long)(bi + ty) * ld + j0 + tx] : 0.0;
  Lc[ty][tx] = (bc + ty < n && tx < nb) ? A[(long)(bc + ty) * ld + j0 + tx] : 0.0;
  __syncthreads();
  const int i = bi + ty, c = bc + tx;
  if (i >= n || c >= n || c > i) return;
  double s = 0.0;
#pragma unroll
  for (int l = 0; l < DB; ++l) s = fma(Li[ty][l], Lc[tx][l], s);
  A[(long)i * ld + c] -= s;
}

__global__ void zero_upper_kernel(double* A, long ld, int n) {
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < (long)n * n; e += (long)gridDim.x * blockDim.x) {
    const long i = e / n, c = e - i * n;
    if (c > i) A[i * ld + c] = 0.0;
  }
}

cudaError_t launch_dense_cholesky(double* A, long ld, int n, int* status, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(status, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  for (int j0 = 0; j0 < n; j0 += DB) {
    const int nb = n - j0 < DB ? n - j0 : DB;
    chol_panel_kernel<<<1, 512, 0, st>>>(A, ld, n, j0, status);
    const int rem = n - j0 - nb;
    if (rem > 0) {
      dim3 grid((rem + DB - 1) / DB, (rem + DB - 1) / DB);
      chol_update_kernel<<<grid, dim3(DB, DB), 0, st>>>(A, ld, n, j0, nb);
    }
  }
  zero_upper_kernel<<<256, 256, 0, st>>>(A, ld, n);
  return cudaGetLastError();
}

// Y (n x m) = L^T X with L lower: Y[i][c] = sum_{j >= i} L[j][i] X[j][c]
__global__ void __launch_bounds__(256) trmm_lt_kernel(const double* L, long ldl, const double* X, long ldx,
                                                      double* Y, long ldy, int n, int m) {
  __shared__ double Ls[DB][DB + 1], Xs[DB][DB + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
  const int i0 = blockIdx.y * DB, c0 = blockIdx.x * DB;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int j0 = i0; j0 < n; j0 += DB) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int jj = ty + 8 * r;
      Ls[jj][tx] = (j0 + jj < n && i0 + tx < n) ? L[(long)(j0 + jj) * ldl + i0 + tx] : 0.0;
      Xs[jj][tx] = (j0 + jj < n && c0 + tx < m) ? X[(long)(j0 + jj) * ldx + c0 + tx] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < DB; ++jj) {
      const double xv = Xs[jj][tx];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = fma(Ls[jj][ty + 8 * r], xv, acc[r]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = i0 + ty + 8 * r, c = c0 + tx;
    if (i < n && c < m) Y[(long)i * ldy + c] = acc[r];
  }
}

cudaError_t launch_trmm_lt(const double* L, long ldl, const double* X, long ldx, double* Y, long ldy, int n, int m,
                           cudaStream_t st) {
  if (n <= 0 || m <= 0) return cudaSuccess;
  dim3 grid((m + DB - 1) / DB, (n + DB - 1) / DB);
  trmm_lt_kernel<<<grid, dim3(DB, 8), 0, st>>>(L, ldl, X, ldx, Y, ldy, n, m);
  return cudaGetLastError();
}

// L^T X = Y in place, rows [i0, i0+nb): back substitution, one thread per column
__global__ void trsm_lt_diag_kernel(const double* L, long ldl, double* X, long ldx, int i0, int nb, int m) {
  __shared__ double Dm[DB][DB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) Dm[e / nb][e % nb] = L[(long)(i0 + e / nb) * ldl + i0 + e % nb];
  __syncthreads();
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < m; c += gridDim.x * blockDim.x) {
    double x[DB];
#pragma unroll
    for (int ii = DB - 1; ii >= 0; --ii) {
      if (ii < nb) {
        double s = X[(long)(i0 + ii) * ldx + c];
#pragma unroll
        for (int j = ii + 1; j < DB; ++j)
          if (j < nb) s -= Dm[j][ii] * x[j];
        x[ii] = s / Dm[ii][ii];
        X[(long)(i0 + ii) * ldx + c] = x[ii];
      }
    }
  }
}

// rows r < i0: X[r][c] -= sum_{j in block} L[j][r] X[j][c]
__global__ void __launch_bounds__(256) trsm_lt_update_kernel(const double* L, long ldl, double* X, long ldx, int i0,
                                                             int nb, int m) {
  __shared__ double Ls[DB][DB + 1], Xs[DB][DB + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
  const int r0 = blockIdx.y * DB, c0 = blockIdx.x * DB;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int jj = ty + 8 * q;
    Ls[jj][tx] = (jj < nb && r0 + tx < i0) ? L[(long)(i0 + jj) * ldl + r0 + tx] : 0.0;
    Xs[jj][tx] = (jj < nb && c0 + tx < m) ? X[(long)(i0 + jj) * ldx + c0 + tx] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = r0 + ty + 8 * q, c = c0 + tx;
    if (r >= i0 || c >= m) continue;
    double s = 0.0;
#pragma unroll
    for (int jj = 0; jj < DB; ++jj) s = fma(Ls[jj][ty + 8 * q], Xs[jj][tx], s);
    X[(long)r * ldx + c] -= s;
  }
}

cudaError_t launch_trsm_lt(const double* L, long ldl, double* X, long ldx, int n, int m, cudaStream_t st) {
  if (n <= 0 || m <= 0) return cudaSuccess;
  const int nblk = (n + DB - 1) / DB;
  for (int b = nblk - 1; b >= 0; --b) {
    const int i0 = b * DB, nb = n - i0 < DB ? n - i0 : DB;
    trsm_lt_diag_kernel<<<(m + 255) / 256, 256, 0, st>>>(L, ldl, X, ldx, i0, nb, m);
    if (i0 > 0) {
      dim3 grid((m + DB - 1) / DB, (i0 + DB - 1) / DB);
      trsm_lt_update_kernel<<<grid, dim3(DB, 8), 0, st>>>(L, ldl, X, ldx, i0, nb, m);
    }
  }
  return cudaGetLastError();
}

// Q <- Q diag(sg), sg_j = sign(R_jj) (0 -> +1)  (the B path's positive R diagonal)
__global__ void colsign_kernel(double* Q, long ldq, long n, int k, const double* R, long ldr) {
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < n * k; e += (long)gridDim.x * blockDim.x) {
    const long i = e / k;
    const int j = (int)(e - i * k);
    if (R[(long)j * ldr + j] < 0.0) Q[i * ldq + j] = -Q[i * ldq + j];
  }
}

cudaError_t launch_colsign(double* Q, long ldq, long n, int k, const double* R, long ldr, cudaStream_t st) {
  const int nb = (int)((n * k + 255) / 256 < 4096 ? (n * k + 255) / 256 : 4096);
  colsign_kernel<<<nb > 0 ? nb : 1, 256, 0, st>>>(Q, ldq, n, k, R, ldr);
  return cudaGetLastError();
}

}  // namespace ots
