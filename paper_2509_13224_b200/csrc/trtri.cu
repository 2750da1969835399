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

// ---- small helpers of the CholeskyQR / Gram-SVD routes (linalg.py), replacing eager tensor ops

namespace {
// L (row-major, ldl) = lower triangle of the col-major potrf factor stored in G (its row-major view holds
// L^T in the upper triangle and the untouched Gram entries in the strict lower one); zero above the
// diagonal. offmax (nullable): max |G_rm[i][j]| over i > j, as an order-preserving 64-bit key.
__global__ void tri_from_potrf_kernel(int n, const double* __restrict__ G, long long ldg, double* __restrict__ L,
                                      long long ldl, unsigned long long* offmax) {
  __shared__ double t[32][33];
  const int bi = blockIdx.y * 32, bj = blockIdx.x * 32;   // output tile rows bi.., cols bj..
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5; // 32 x 8 threads
  // read the transposed tile G_rm[bj + r][bi + c] (the L^T upper triangle of the source)
  for (int r = ty; r < 32; r += 8) {
    const int gi = bj + r, gj = bi + tx;
    t[r][tx] = (gi < n && gj < n) ? G[(long long)gi * ldg + gj] : 0.0;
  }
  __syncthreads();
  double m = 0.0;
  for (int r = ty; r < 32; r += 8) {
    const int i = bi + r, j = bj + tx;
    if (i < n && j < n) {
      L[(long long)i * ldl + j] = j <= i ? t[tx][r] : 0.0;
      if (offmax && i > j) m = fmax(m, fabs(G[(long long)i * ldg + j]));
    }
  }
  if (offmax) {
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (tx == 0) atomicMax(offmax, (unsigned long long)__double_as_longlong(m));   // m >= 0
  }
}

// ||A||_2 (square n x n, row-major) by power iteration on B = A^T A (formed by one DMMA GEMM beforehand) from
// a fixed start vector, one cooperative launch: per step y = B v (a warp per row, coalesced), v = y / ||y||.
__global__ void __launch_bounds__(256) norm2_power_kernel(int n, const double* __restrict__ B, int iters, double* v,
                                                          double* y, double* red, double* out) {
  cg::grid_group grid = cg::this_grid();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31, gw = tid >> 5, nw = nth >> 5;
  __shared__ double sred[8];
  for (int i = tid; i < n; i += nth) v[i] = 1.0 + 0.5 * sin(0.37 * i + 1.0);   // deterministic start
  if (tid == 0) { red[0] = 0.0; red[1] = 0.0; }
  grid.sync();
  double nrm = 0.0;
  for (int it = 0; it < iters; ++it) {
    double loc = 0.0;
    for (int i = gw; i < n; i += nw) {
      double s = 0.0;
      for (int k = lane; k < n; k += 32) s += B[(long long)i * n + k] * v[k];
      s = warp_sum(s);
      if (lane == 0) { y[i] = s; loc += s * s; }
    }
    if (lane == 0) sred[threadIdx.x >> 5] = loc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = 0.0;
      for (int w = 0; w < 8; ++w) b += sred[w];
      atomicAdd(red + (it & 1), b);
    }
    grid.sync();
    nrm = sqrt(red[it & 1]);
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int j = tid; j < n; j += nth) v[j] = y[j] * inv;
    if (tid == 0) red[(it + 1) & 1] = 0.0;
    grid.sync();
  }
  if (tid == 0) *out = sqrt(nrm);
}
}  // namespace

TTB_API int ttb_tri_from_potrf(void* stream, int n, const double* G, long long ldg, double* L, long long ldl,
                               double* offmax) {
  if (n < 1) return TTB_EARG;
  cudaStream_t st = as_stream(stream);
  if (offmax) cudaMemsetAsync(offmax, 0, sizeof(double), st);
  tri_from_potrf_kernel<<<dim3(ceil_div(n, 32), ceil_div(n, 32)), 256, 0, st>>>(
      n, G, ldg, L, ldl, reinterpret_cast<unsigned long long*>(offmax)); ttb_count();
  return ttb_last_error();
}

// out (device double): the power-iteration estimate of ||A||_2 (a lower bound, within a few percent
// after 24 steps for the clustered spectra of the CholeskyQR factors). ws: n^2 + 2 n + 2 doubles.
TTB_API int ttb_norm2_est(void* stream, int n, const double* A, long long lda, int iters, double* ws, double* out) {
  if (n < 1 || iters < 1) return TTB_EARG;
  cudaStream_t st = as_stream(stream);
  double* Bm = ws;
  double* v = ws + (long long)n * n;
  double* y = v + n;
  double* red = y + n;
  int rc = ttb_dgemm(stream, 1, 0, n, n, n, 1.0, A, lda, 0, A, lda, 0, 0.0, Bm, n, 0, 1);   // B = A^T A
  if (rc) return rc;
  static int gmax = 0;
  if (!gmax) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, norm2_power_kernel, 256, 0);
    gmax = ttb_num_sms() * (per > 0 ? (per < 2 ? per : 2) : 1);
  }
  int grid = ceil_div((long long)n * 32, 256);    // a warp per row
  if (grid > gmax) grid = gmax;
  void* args[] = {&n, &Bm, &iters, &v, &y, &red, &out};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)norm2_power_kernel, dim3(grid), dim3(256), args, 0, st);
  ttb_count();
  return e == cudaSuccess ? ttb_last_error() : (int)e;
}
