// CholeskyQR2 factorization of a tall 128-column Householder block, returned in LAPACK form.
//
// The blocked QR (qr.cu) factors each 128-column block of a tall matrix (m in the millions) and
// then applies it to the trailing columns as a compact-WY product. Factoring the block with 8
// sixteen-column TSQR panels is a chain of ~100 latency-bound launches (the critical path of the
// tall QR, DESIGN.md (f)). For a well-conditioned block the same outputs come from four GEMM
// passes over the block instead:
//   G1 = P^T P,  P = Q1 R1 (Cholesky of G1),  G2 = Q1^T Q1,  Q1 = Q R2,  R = R2 R1   (CholeskyQR2)
// followed by Householder reconstruction (Ballard, Demmel, Grigori, Jacquelin, Nguyen, Solomonik
// 2014): the LU factorization without pivoting of Y = [I; 0] - Q S, with the sign matrix S chosen
// column by column so every pivot is 1 + |w| >= 1, gives the unit-lower reflector block V = L,
// T = U L_top^{-T}, tau = diag(T) and R_h = S R, i.e. exactly what dgeqrf + dlarft produce (up
// to roundoff). CholeskyQR2 needs cond(P) well below eps^{-1/2}; the Cholesky pivots are checked
// (min/max diagonal of R1, R2 >= 1e-5; the second Gram Q1^T Q1 within 0.1 of I entrywise) and the
// caller falls back to the TSQR panels otherwise.
#include "common.cuh"

TTB_API int ttb_dgemm(void* stream, int tA, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
                      long long sA, const double* B, long long ldb, long long sB, double beta, double* C,
                      long long ldc, long long sC, int batch);

constexpr int TTB_CHOLQR_FALLBACK = -50;

namespace {

constexpr int CQT = 1024;

// G (b x b row-major, symmetric) = R^T R with R upper; R and R^{-1} row-major. flag |= bit on a
// non-positive pivot or min/max diagonal of R below 1e-5. 32 x 32 thread grid over the trailing
// triangle; R^{-1} row by row (bottom up, columns in parallel) with X^T kept in W's lower triangle.
__global__ void __launch_bounds__(CQT) chol_inv_kernel(int b, const double* __restrict__ G, double* R, double* Ri,
                                                       int* flag, int bit) {
  extern __shared__ double W[];  // b x (b + 1)
  __shared__ double xd[128];
  __shared__ int bad;
  const int ld = b + 1;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < b * b; e += CQT) {
    const double g = G[e];
    W[(e / b) * ld + e % b] = g;
    // the second pass (bit 2) factors Q1^T Q1: accepted only within 0.1 of I entrywise (the rule of
    // linalg.cholqr2_colmajor); a min/max pivot ratio alone does not bound how far Q1 is from orthogonal
    if (bit == 2 && !(fabs(g - (e / b == e % b ? 1.0 : 0.0)) <= 0.1)) bad = 1;
  }
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) atomicOr(flag, bit);
    return;
  }
  for (int k = 0; k < b; ++k) {
    const double piv = W[k * ld + k];
    if (!(piv > 0.0) || !isfinite(piv)) {
      if (threadIdx.x == 0) bad = 1;
      break;
    }
    const double rkk = sqrt(piv), inv = 1.0 / rkk, ipiv = 1.0 / piv;
    // trailing update from the unscaled row k, then row k of R
    for (int i = k + 1 + ty; i < b; i += 32)
      for (int j = i + tx; j < b; j += 32) W[i * ld + j] -= W[k * ld + i] * W[k * ld + j] * ipiv;
    __syncthreads();
    for (int j = k + 1 + threadIdx.x; j < b; j += CQT) W[k * ld + j] *= inv;
    if (threadIdx.x == 0) W[k * ld + k] = rkk;
    __syncthreads();
  }
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) atomicOr(flag, bit);
    return;
  }
  if (threadIdx.x == 0) {
    double mn = W[0], mx = W[0];
    for (int k = 1; k < b; ++k) { mn = fmin(mn, W[k * ld + k]); mx = fmax(mx, W[k * ld + k]); }
    if (!(mn >= 1e-5 * mx)) { bad = 1; atomicOr(flag, bit); }
  }
  for (int e = threadIdx.x; e < b * b; e += CQT) {
    const int i = e / b, j = e % b;
    R[e] = (j >= i) ? W[i * ld + j] : 0.0;
  }
  __syncthreads();
  if (bad) return;
  // X = R^{-1}: row i from the rows below it; X[l][j] (l < j) lives at W[j][l], diagonal in xd
  for (int i = b - 1; i >= 0; --i) {
    const double rii = W[i * ld + i];
    for (int j = i + threadIdx.x; j < b; j += CQT) {
      if (j == i) {
        xd[i] = 1.0 / rii;
      } else {
        double acc = W[i * ld + j] * xd[j];
        for (int l = i + 1; l < j; ++l) acc += W[i * ld + l] * W[j * ld + l];
        W[j * ld + i] = -acc / rii;
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < b * b; e += CQT) {
    const int i = e / b, j = e % b;
    Ri[e] = (j > i) ? W[j * ld + i] : (j == i ? xd[i] : 0.0);
  }
}

// Householder reconstruction of the top block. Qtop (row-major b x b: Qtop[c * b + r] = Q(r, c)),
// R (b x b row-major upper). Writes the factored top block of P (col-major, ld lda: S R on and above
// the diagonal, L strictly below), tau, Vtop (col-major unit lower), T (row-major upper) and
// SUi = S U^{-1} (row-major) for the bottom rows V_bot = -Q_bot S U^{-1}.
__global__ void __launch_bounds__(CQT) recon_kernel(int b, const double* __restrict__ Qtop,
                                                    const double* __restrict__ R, double* P, long long lda,
                                                    double* tau, double* Vtop, double* T, double* SUi) {
  extern __shared__ double M[];  // b x (b + 1): L below the diagonal, U on and above it
  __shared__ double sg[128], pv[128], xd[128];
  const int ld = b + 1;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < b * b; e += CQT) {
    const int r = e % b, c = e / b;
    M[r * ld + c] = Qtop[e];
  }
  __syncthreads();
  // LU of Y = I - Q S without pivoting, s_k chosen at step k so that the pivot is 1 + |w| >= 1;
  // the updates act on the Q part only (the identity part stays e_j), U's rows are stored unsigned
  for (int k = 0; k < b; ++k) {
    const double w = M[k * ld + k];
    const double s = (w > 0.0) ? -1.0 : 1.0;
    const double piv = 1.0 - s * w;
    const double f = -s / piv;
    for (int i = k + 1 + ty; i < b; i += 32) {
      const double l = f * M[i * ld + k];
      for (int j = k + 1 + tx; j < b; j += 32) M[i * ld + j] -= l * M[k * ld + j];
    }
    __syncthreads();
    for (int i = k + 1 + threadIdx.x; i < b; i += CQT) M[i * ld + k] *= f;
    if (threadIdx.x == 0) { sg[k] = s; pv[k] = piv; }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < b * b; e += CQT) {
    const int k = e / b, j = e % b;
    if (j > k) M[k * ld + j] *= -sg[j];
    else if (j == k) M[k * ld + k] = pv[k];
  }
  __syncthreads();
  // keep U (row-major) in SUi's slot while T = U L^{-T} overwrites it in place (row i by one thread,
  // left to right: X L^T = U)
  for (int e = threadIdx.x; e < b * b; e += CQT) {
    const int i = e / b, j = e % b;
    SUi[e] = (j >= i) ? M[i * ld + j] : 0.0;
  }
  for (int i = threadIdx.x; i < b; i += CQT) {
    for (int j = i + 1; j < b; ++j) {
      double x = M[i * ld + j];
      for (int l = i; l < j; ++l) x -= M[i * ld + l] * M[j * ld + l];
      M[i * ld + j] = x;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < b * b; e += CQT) {
    const int r = e % b, c = e / b;
    P[(long long)c * lda + r] = (r <= c) ? sg[r] * R[(long long)r * b + c] : M[r * ld + c];
    Vtop[(long long)c * b + r] = (r == c) ? 1.0 : (r > c ? M[r * ld + c] : 0.0);
    const int i = e / b, j = e % b;
    T[e] = (j >= i) ? M[i * ld + j] : 0.0;
  }
  for (int c = threadIdx.x; c < b; c += CQT) tau[c] = M[c * ld + c];
  __syncthreads();
  // U back into smem; X = U^{-1} row by row (bottom up, columns in parallel), X^T in the lower
  // triangle, diagonal in xd; then SUi = S X
  for (int e = threadIdx.x; e < b * b; e += CQT) {
    const int i = e / b, j = e % b;
    if (j >= i) M[i * ld + j] = SUi[e];
  }
  __syncthreads();
  for (int i = b - 1; i >= 0; --i) {
    const double uii = M[i * ld + i];
    for (int j = i + threadIdx.x; j < b; j += CQT) {
      if (j == i) {
        xd[i] = 1.0 / uii;
      } else {
        double acc = M[i * ld + j] * xd[j];
        for (int l = i + 1; l < j; ++l) acc += M[i * ld + l] * M[j * ld + l];
        M[j * ld + i] = -acc / uii;
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < b * b; e += CQT) {
    const int i = e / b, j = e % b;
    SUi[e] = sg[i] * ((j > i) ? M[j * ld + i] : (j == i ? xd[i] : 0.0));
  }
}

}  // namespace

// Doubles of workspace for cholqr_block: one m x b buffer (Q1) + 12 b x b blocks + flags.
long long cholqr_workspace(long long m, int b) { return m * b + 12LL * b * b + 16; }

// Factor the col-major mp x b block P (ld lda, b <= 128) in place as dgeqrf would, writing tau,
// the explicit unit-lower top block Vtop (col-major b x b) and the block T (row-major b x b).
// Returns 0 on success, TTB_CHOLQR_FALLBACK when the block is too ill-conditioned for CholeskyQR2
// (P untouched; the caller uses its panel path), otherwise an error code. Four passes over the
// block: G1 = P^T P, Q1 = P R1^-1, G2 = Q1^T Q1, and V_bot = -Q1_bot (R2^-1 S U^-1) (Q = Q1 R2^-1
// is only formed for its top b x b block).
int cholqr_block(cudaStream_t st, long long mp, int b, double* P, long long lda, double* tau, double* Vtop,
                 double* T, double* ws) {
  if (b > 128 || b < 1 || mp < 2LL * b) return TTB_EARG;
  void* s = (void*)st;
  double* Q1 = ws;
  double* sm = ws + mp * b;
  const long long bb = (long long)b * b;
  double *G1 = sm, *R1 = sm + bb, *R1i = sm + 2 * bb, *G2 = sm + 3 * bb, *R2 = sm + 4 * bb, *R2i = sm + 5 * bb;
  double *Rr = sm + 6 * bb, *SUi = sm + 7 * bb, *Qt = sm + 8 * bb, *Mb = sm + 9 * bb;
  int* flag = reinterpret_cast<int*>(sm + 12 * bb);
  const size_t smem = (size_t)b * (b + 1) * sizeof(double);
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 132 * 1024);
    cudaFuncSetAttribute(recon_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 132 * 1024);
    cfg = true;
  }
  cudaMemsetAsync(flag, 0, sizeof(int), st);
  int rc = ttb_dgemm(s, 0, 1, b, b, (int)mp, 1.0, P, lda, 0, P, lda, 0, 0.0, G1, b, 0, 1);  // P^T P
  if (rc) return rc;
  chol_inv_kernel<<<1, CQT, smem, st>>>(b, G1, R1, R1i, flag, 1); ttb_count();
  rc = ttb_dgemm(s, 1, 0, b, (int)mp, b, 1.0, R1i, b, 0, P, lda, 0, 0.0, Q1, mp, 0, 1);     // Q1 = P R1^-1
  if (rc) return rc;
  rc = ttb_dgemm(s, 0, 1, b, b, (int)mp, 1.0, Q1, mp, 0, Q1, mp, 0, 0.0, G2, b, 0, 1);      // Q1^T Q1
  if (rc) return rc;
  chol_inv_kernel<<<1, CQT, smem, st>>>(b, G2, R2, R2i, flag, 2); ttb_count();
  int hflag = 0;
  cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return (int)e;
  if (hflag) return TTB_CHOLQR_FALLBACK;
  rc = ttb_dgemm(s, 1, 0, b, b, b, 1.0, R2i, b, 0, Q1, mp, 0, 0.0, Qt, b, 0, 1);             // Q top block
  if (rc) return rc;
  rc = ttb_dgemm(s, 0, 0, b, b, b, 1.0, R2, b, 0, R1, b, 0, 0.0, Rr, b, 0, 1);              // R = R2 R1
  if (rc) return rc;
  recon_kernel<<<1, CQT, smem, st>>>(b, Qt, Rr, P, lda, tau, Vtop, T, SUi); ttb_count();
  rc = ttb_dgemm(s, 0, 0, b, b, b, 1.0, R2i, b, 0, SUi, b, 0, 0.0, Mb, b, 0, 1);            // R2^-1 S U^-1
  if (rc) return rc;
  // V_bot = -Q_bot S U^-1 = -Q1_bot (R2^-1 S U^-1), written below the top block of P
  rc = ttb_dgemm(s, 1, 0, b, (int)(mp - b), b, -1.0, Mb, b, 0, Q1 + b, mp, 0, 0.0, P + b, lda, 0, 1);
  if (rc) return rc;
  return ttb_last_error();
}
