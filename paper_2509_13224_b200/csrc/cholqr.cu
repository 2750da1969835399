// CholeskyQR2 factorization of a tall 128-column Householder block, returned in LAPACK form.
//
// The blocked QR (qr.cu) factors each 128-column block of a tall matrix (m in the millions) and
// then applies it to the trailing columns as a compact-WY product. Factoring the block with 8
// sixteen-column TSQR panels is a chain of ~100 latency-bound launches (the critical path of the
// tall QR, DESIGN.md (f)). For a well-conditioned block the same outputs come from five GEMM
// passes instead:
//   G1 = P^T P,  P = Q1 R1 (Cholesky of G1),  G2 = Q1^T Q1,  Q1 = Q R2,  R = R2 R1   (CholeskyQR2)
// followed by Householder reconstruction (Ballard, Demmel, Grigori, Jacquelin, Nguyen, Solomonik
// 2014): the LU factorization without pivoting of Y = [I; 0] - Q S, with the sign matrix S chosen
// column by column so every pivot is 1 + |w| >= 1, gives the unit-lower reflector block V = L,
// T = U L_top^{-T}, tau = diag(T) and R_h = S R, i.e. exactly what dgeqrf + dlarft produce (up
// to roundoff). CholeskyQR2 needs cond(P) well below eps^{-1/2}; the Cholesky pivots are checked
// (min/max diagonal of R1, R2 >= 1e-5) and the caller falls back to the TSQR panels otherwise.
#include "common.cuh"

TTB_API int ttb_dgemm(void* stream, int tA, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
                      long long sA, const double* B, long long ldb, long long sB, double beta, double* C,
                      long long ldc, long long sC, int batch);

constexpr int TTB_CHOLQR_FALLBACK = -50;

namespace {

constexpr int CQT = 1024;

// G (b x b row-major, symmetric) = R^T R with R upper; R and R^{-1} row-major. flag |= bit on a
// non-positive pivot or min/max diagonal of R below 1e-5.
__global__ void __launch_bounds__(CQT) chol_inv_kernel(int b, const double* __restrict__ G, double* R, double* Ri,
                                                       int* flag, int bit) {
  extern __shared__ double W[];  // b x (b + 1)
  __shared__ int bad;
  const int ld = b + 1;
  for (int e = threadIdx.x; e < b * b; e += CQT) W[(e / b) * ld + e % b] = G[e];
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int k = 0; k < b; ++k) {
    const double piv = W[k * ld + k];
    if (!(piv > 0.0) || !isfinite(piv)) {
      if (threadIdx.x == 0) bad = 1;
      break;
    }
    const double rkk = sqrt(piv), inv = 1.0 / rkk;
    __syncthreads();
    for (int j = k + 1 + threadIdx.x; j < b; j += CQT) W[k * ld + j] *= inv;
    if (threadIdx.x == 0) W[k * ld + k] = rkk;
    __syncthreads();
    const int nt = b - k - 1;
    for (int e = threadIdx.x; e < nt * nt; e += CQT) {
      const int i = k + 1 + e / nt, j = k + 1 + e % nt;
      if (j >= i) W[i * ld + j] -= W[k * ld + i] * W[k * ld + j];
    }
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
  // R^{-1}: column j by back substitution (thread j)
  for (int j = threadIdx.x; j < b; j += CQT) {
    for (int i = b - 1; i >= 0; --i) {
      double x = 0.0;
      if (i <= j) {
        double s = (i == j) ? 1.0 : 0.0;
        for (int l = i + 1; l <= j; ++l) s -= W[i * ld + l] * Ri[(long long)l * b + j];
        x = s / W[i * ld + i];
      }
      Ri[(long long)i * b + j] = x;
    }
  }
}

// Householder reconstruction of the top block. Q (b columns, row-major (b x ldq): Qrm[c * ldq + r] =
// Q(r, c)), R (b x b row-major upper). Writes the factored top block of P (col-major, ld lda: S R on
// and above the diagonal, L strictly below), tau, Vtop (col-major unit lower), T (row-major upper)
// and SUi = S U^{-1} (row-major) for the bottom rows V_bot = -Q_bot S U^{-1}.
__global__ void __launch_bounds__(CQT) recon_kernel(int b, const double* __restrict__ Qrm, long long ldq,
                                                    const double* __restrict__ R, double* P, long long lda,
                                                    double* tau, double* Vtop, double* T, double* SUi) {
  extern __shared__ double M[];  // b x (b + 1): L below the diagonal, unsigned U rows above
  __shared__ double sg[128], pv[128];
  const int ld = b + 1;
  for (int e = threadIdx.x; e < b * b; e += CQT) {
    const int r = e % b, c = e / b;
    M[r * ld + c] = Qrm[(long long)c * ldq + r];
  }
  __syncthreads();
  for (int k = 0; k < b; ++k) {
    const double w = M[k * ld + k];
    const double s = (w > 0.0) ? -1.0 : 1.0;   // pivot 1 - s w = 1 + |w|
    const double piv = 1.0 - s * w;
    __syncthreads();
    if (threadIdx.x == 0) { sg[k] = s; pv[k] = piv; }
    for (int i = k + 1 + threadIdx.x; i < b; i += CQT) M[i * ld + k] = -s * M[i * ld + k] / piv;
    __syncthreads();
    const int nt = b - k - 1;
    for (int e = threadIdx.x; e < nt * nt; e += CQT) {
      const int i = k + 1 + e / nt, j = k + 1 + e % nt;
      M[i * ld + j] -= M[i * ld + k] * M[k * ld + j];
    }
    __syncthreads();
  }
  // U[k][j] = -s_j M[k][j] (j > k), U[k][k] = piv_k; keep U in M's upper part from here on
  for (int e = threadIdx.x; e < b * b; e += CQT) {
    const int k = e / b, j = e % b;
    if (j > k) M[k * ld + j] *= -sg[j];
  }
  for (int k = threadIdx.x; k < b; k += CQT) M[k * ld + k] = pv[k];
  __syncthreads();
  // T = U L^{-T}: X L^T = U, row i by thread i, columns left to right
  for (int i = threadIdx.x; i < b; i += CQT) {
    for (int j = 0; j < b; ++j) {
      double x = 0.0;
      if (j >= i) {
        x = M[i * ld + j];
        for (int l = i; l < j; ++l) x -= T[(long long)i * b + l] * M[j * ld + l];
      }
      T[(long long)i * b + j] = x;
    }
  }
  // SUi = S U^{-1}: column j of U^{-1} by back substitution (thread j)
  for (int j = threadIdx.x; j < b; j += CQT) {
    for (int i = b - 1; i >= 0; --i) {
      double x = 0.0;
      if (i <= j) {
        double s = (i == j) ? 1.0 : 0.0;
        for (int l = i + 1; l <= j; ++l) s -= M[i * ld + l] * SUi[(long long)l * b + j] * sg[l];
        x = s / M[i * ld + i];
      }
      SUi[(long long)i * b + j] = sg[i] * x;
    }
  }
  __syncthreads();
  // outputs: P top block, tau, Vtop
  for (int e = threadIdx.x; e < b * b; e += CQT) {
    const int r = e % b, c = e / b;
    double v;
    if (r <= c) v = sg[r] * R[(long long)r * b + c];
    else v = M[r * ld + c];
    P[(long long)c * lda + r] = v;
    Vtop[(long long)c * b + r] = (r == c) ? 1.0 : (r > c ? M[r * ld + c] : 0.0);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < b; c += CQT) tau[c] = T[(long long)c * b + c];
}

}  // namespace

// Doubles of workspace for cholqr_block: one m x b buffer (Q1) + 12 b x b blocks + flags.
long long cholqr_workspace(long long m, int b) { return m * b + 12LL * b * b + 16; }

// Factor the col-major mp x b block P (ld lda, b <= 128) in place as dgeqrf would, writing tau,
// the explicit unit-lower top block Vtop (col-major b x b) and the block T (row-major b x b).
// Q2: an mp x b scratch buffer (may be the caller's). Returns 0 on success, TTB_CHOLQR_FALLBACK when
// the block is too ill-conditioned for CholeskyQR2 (P untouched; the caller uses its panel path),
// otherwise an error code.
int cholqr_block(cudaStream_t st, long long mp, int b, double* P, long long lda, double* tau, double* Vtop,
                 double* T, double* ws, double* Q2) {
  if (b > 128 || b < 1 || mp < 2LL * b) return TTB_EARG;
  void* s = (void*)st;
  double* Q1 = ws;
  double* sm = ws + mp * b;
  const long long bb = (long long)b * b;
  double *G1 = sm, *R1 = sm + bb, *R1i = sm + 2 * bb, *G2 = sm + 3 * bb, *R2 = sm + 4 * bb, *R2i = sm + 5 * bb;
  double *Rr = sm + 6 * bb, *SUi = sm + 7 * bb;
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
  rc = ttb_dgemm(s, 1, 0, b, (int)mp, b, 1.0, R2i, b, 0, Q1, mp, 0, 0.0, Q2, mp, 0, 1);     // Q = Q1 R2^-1
  if (rc) return rc;
  rc = ttb_dgemm(s, 0, 0, b, b, b, 1.0, R2, b, 0, R1, b, 0, 0.0, Rr, b, 0, 1);              // R = R2 R1
  if (rc) return rc;
  recon_kernel<<<1, CQT, smem, st>>>(b, Q2, mp, Rr, P, lda, tau, Vtop, T, SUi); ttb_count();
  // V_bot = -Q_bot S U^{-1}, written below the top block of P
  rc = ttb_dgemm(s, 1, 0, b, (int)(mp - b), b, -1.0, SUi, b, 0, Q2 + b, mp, 0, 0.0, P + b, lda, 0, 1);
  if (rc) return rc;
  return ttb_last_error();
}
