// Inverse of a lower-triangular matrix (the Cholesky factors of the CholeskyQR2 orthogonalization of
// very tall TT unfoldings, linalg.cholqr2_colmajor): Q = X R^{-1} is then one Ozaki-scheme GEMM
// instead of a triangular solve with a million right-hand sides.
//
// n % 128 == 0, row-major. The 128 x 128 diagonal blocks are inverted by one CTA each (forward
// substitution, one thread per column of the inverse, the block's lower triangle packed in shared
// memory); block row i of the inverse then follows from the blocked recurrence
//   Linv[i, :i] = -Linv[i, i] (L[i, :i] Linv[:i, :i])
// as two small GEMMs per block row.
#include "common.cuh"

TTB_API int ttb_dgemm(void* stream, int tA, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
                      long long sA, const double* B, long long ldb, long long sB, double beta, double* C,
                      long long ldc, long long sC, int batch);

namespace {

constexpr int TB = 128;

__global__ void __launch_bounds__(TB) tri_inv_diag_kernel(int n, const double* __restrict__ L, long long ldl,
                                                          double* Li, long long ldi) {
  extern __shared__ double sm[];
  double* Lp = sm;                       // packed lower triangle: row i at i (i + 1) / 2
  double* X = sm + TB * (TB + 1) / 2;    // X[i][j], column j owned by thread j
  const int b0 = blockIdx.x * TB, j = threadIdx.x;
  for (int i = 0; i < TB; ++i)
    for (int k = j; k <= i; k += TB) Lp[i * (i + 1) / 2 + k] = L[(long long)(b0 + i) * ldl + b0 + k];
  __syncthreads();
  for (int i = 0; i < TB; ++i) {
    double s = 0.0;
    if (i >= j) {
      s = i == j ? 1.0 : 0.0;
      const double* li = Lp + i * (i + 1) / 2;
      for (int k = j; k < i; ++k) s -= li[k] * X[k * TB + j];
      s /= li[i];
    }
    X[i * TB + j] = s;
  }
  for (int i = 0; i < TB; ++i) Li[(long long)(b0 + i) * ldi + b0 + j] = X[i * TB + j];
}

}  // namespace

// Linv (n x n, ldi) = L^{-1} for a lower-triangular row-major L (ldl; the strict upper triangle is
// ignored); n % 128 == 0. ws: n * n doubles.
TTB_API int ttb_trtri_lower(void* stream, int n, const double* L, long long ldl, double* Li, long long ldi, double* ws) {
  if (n <= 0 || n % TB) return TTB_EARG;
  cudaStream_t st = as_stream(stream);
  const size_t smem = (size_t)(TB * (TB + 1) / 2 + TB * TB) * sizeof(double);
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(tri_inv_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cfg = true;
  }
  cudaMemset2DAsync(Li, sizeof(double) * ldi, 0, sizeof(double) * n, n, st);
  tri_inv_diag_kernel<<<n / TB, TB, smem, st>>>(n, L, ldl, Li, ldi); ttb_count();
  for (int bi = 1; bi < n / TB; ++bi) {
    const int r0 = bi * TB;
    // W (128 x r0) = L[r0:r0+128, :r0] Linv[:r0, :r0]
    int rc = ttb_dgemm(stream, 0, 0, TB, r0, r0, 1.0, L + (long long)r0 * ldl, ldl, 0, Li, ldi, 0, 0.0, ws, r0, 0, 1);
    if (rc) return rc;
    // Linv[r0:r0+128, :r0] = -Linv[r0:, r0:] W
    rc = ttb_dgemm(stream, 0, 0, TB, r0, TB, -1.0, Li + (long long)r0 * ldi + r0, ldi, 0, ws, r0, 0, 0.0,
                   Li + (long long)r0 * ldi, ldi, 0, 1);
    if (rc) return rc;
  }
  return ttb_last_error();
}
