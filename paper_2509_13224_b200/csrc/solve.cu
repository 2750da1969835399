// Dense FP64 solvers: LU with partial pivoting, blocked Cholesky, triangular
// solves, and the cooperative maxvol kernel that drives TT-cross pivoting.
#include "common.cuh"

TTB_API int ttb_dgemm(void* stream, int tA, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
                      long long sA, const double* B, long long ldb, long long sB, double beta, double* C,
                      long long ldc, long long sC, int batch);

namespace {

constexpr int ST = 1024;

// ---------------------------------------------------------------------------
// LU (getrf, partial pivoting, first-max pivot like LAPACK idamax), single CTA.
__global__ void __launch_bounds__(ST) lu_kernel(int n, double* A, long long lda, int* piv, int* info) {
  __shared__ double sv[32];
  __shared__ long long si[32];
  __shared__ int sp;
  if (threadIdx.x == 0) *info = 0;
  for (int k = 0; k < n; ++k) {
    AbsMax best{-1.0, (long long)1 << 62};
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
      AbsMax c{fabs(A[(long long)k * lda + i]), i};
      best = absmax_merge(best, c);
    }
    best = block_absmax(best, sv, si);
    if (threadIdx.x == 0) {
      sp = (int)best.i;
      piv[k] = sp;
      if (best.v == 0.0 && *info == 0) *info = k + 1;
    }
    __syncthreads();
    const int p = sp;
    if (p != k)
      for (int c = threadIdx.x; c < n; c += blockDim.x) {
        double t = A[(long long)c * lda + k];
        A[(long long)c * lda + k] = A[(long long)c * lda + p];
        A[(long long)c * lda + p] = t;
      }
    __syncthreads();
    const double d = A[(long long)k * lda + k];
    if (d != 0.0)
      for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) A[(long long)k * lda + i] /= d;
    __syncthreads();
    const int m = n - k - 1;
    for (long long e = threadIdx.x; e < (long long)m * m; e += blockDim.x) {
      int c = k + 1 + (int)(e / m), i = k + 1 + (int)(e % m);
      A[(long long)c * lda + i] -= A[(long long)k * lda + i] * A[(long long)c * lda + k];
    }
    __syncthreads();
  }
}

// Solve op(A) X = B for the LU factors (col-major), one RHS column per thread.
__global__ void lu_apply_kernel(int n, const double* __restrict__ LU, long long lda, const int* __restrict__ piv,
                                int nrhs, double* B, long long ldb, int trans) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nrhs) return;
  double* b = B + (long long)c * ldb;
  if (!trans) {
    for (int k = 0; k < n; ++k) {
      int p = piv[k];
      if (p != k) { double t = b[k]; b[k] = b[p]; b[p] = t; }
    }
    for (int k = 0; k < n; ++k) {  // L y = b (unit lower)
      double x = b[k];
      for (int i = k + 1; i < n; ++i) b[i] -= LU[(long long)k * lda + i] * x;
    }
    for (int k = n - 1; k >= 0; --k) {  // U x = y
      double x = b[k] / LU[(long long)k * lda + k];
      b[k] = x;
      for (int i = 0; i < k; ++i) b[i] -= LU[(long long)k * lda + i] * x;
    }
  } else {
    // A^T = U^T L^T P^T : U^T y = b, L^T z = y, x = P z
    for (int k = 0; k < n; ++k) {
      double s = b[k];
      for (int i = 0; i < k; ++i) s -= LU[(long long)k * lda + i] * b[i];
      b[k] = s / LU[(long long)k * lda + k];
    }
    for (int k = n - 1; k >= 0; --k) {
      double s = b[k];
      for (int i = k + 1; i < n; ++i) s -= LU[(long long)k * lda + i] * b[i];
      b[k] = s;
    }
    for (int k = n - 1; k >= 0; --k) {
      int p = piv[k];
      if (p != k) { double t = b[k]; b[k] = b[p]; b[p] = t; }
    }
  }
}

// ---------------------------------------------------------------------------
// Cholesky panel: factor diagonal block (nb x nb) and solve the rows below, single CTA.
constexpr int CNB = 64;

__global__ void __launch_bounds__(256) chol_panel_kernel(int n, int j0, double* A, long long lda, int* info) {
  __shared__ double L11[CNB * CNB];
  const int nb = min(CNB, n - j0);
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int c = e / nb, i = e % nb;
    L11[c * CNB + i] = A[(long long)(j0 + c) * lda + j0 + i];
  }
  __syncthreads();
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  // left-looking column sweep: at step k thread i >= k finishes L(i, k) = A(i, k) - sum_{j<k} L(i, j) L(k, j)
  // (the same subtractions in the same order as the right-looking update, so the same bits), then the
  // column is scaled by the pivot: one dot product of length k per thread instead of a rank-1 update of
  // the whole trailing block by all threads every step
  for (int k = 0; k < nb; ++k) {
    const int i = threadIdx.x;
    if (i >= k && i < nb) {
      double sacc = L11[k * CNB + i];
#pragma unroll 8
      for (int j = 0; j < k; ++j) sacc -= L11[j * CNB + i] * L11[j * CNB + k];
      L11[k * CNB + i] = sacc;
    }
    __syncthreads();
    double d = L11[k * CNB + k];
    if (d <= 0.0 || !isfinite(d)) {
      if (threadIdx.x == 0) { bad = 1; if (blockIdx.x == 0) *info = j0 + k + 1; }
      __syncthreads();
      break;
    }
    d = sqrt(d);
    __syncthreads();
    if (i > k && i < nb) L11[k * CNB + i] /= d;
    if (i == k) L11[k * CNB + k] = d;
    __syncthreads();
  }
  if (bad) return;
  // every CTA factors the (tiny) diagonal block redundantly; CTA 0 writes it back
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
      int c = e / nb, i = e % nb;
      if (i >= c) A[(long long)(j0 + c) * lda + j0 + i] = L11[c * CNB + i];
    }
  // rows below: x L11^T = a  (one row per thread, rows spread over the grid)
  for (int r = j0 + nb + blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double x[CNB];
#pragma unroll
    for (int k = 0; k < CNB; ++k) {
      if (k < nb) {
        double s = A[(long long)(j0 + k) * lda + r];
        for (int q = 0; q < k; ++q) s -= x[q] * L11[q * CNB + k];
        x[k] = s / L11[k * CNB + k];
      }
    }
#pragma unroll
    for (int k = 0; k < CNB; ++k)
      if (k < nb) A[(long long)(j0 + k) * lda + r] = x[k];
  }
}

// Solve L L^T x = b with b in shared memory, single CTA, 32-row blocks.
__global__ void __launch_bounds__(ST) chol_solve_kernel(int n, const double* __restrict__ L, long long lda, double* bg) {
  extern __shared__ double b[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < n; i += blockDim.x) b[i] = bg[i];
  __syncthreads();
  // forward
  for (int b0 = 0; b0 < n; b0 += 32) {
    const int nb = min(32, n - b0);
    if (wid == 0) {
      double v = lane < nb ? b[b0 + lane] : 0.0;
      for (int j = 0; j < nb; ++j) {
        double yj = __shfl_sync(0xffffffffu, v, j) / L[(long long)(b0 + j) * lda + b0 + j];
        if (lane == j) v = yj;
        if (lane > j && lane < nb) v -= L[(long long)(b0 + j) * lda + b0 + lane] * yj;
      }
      if (lane < nb) b[b0 + lane] = v;
    }
    __syncthreads();
    for (int i = b0 + nb + threadIdx.x; i < n; i += blockDim.x) {
      double s = b[i];
      for (int j = 0; j < nb; ++j) s -= L[(long long)(b0 + j) * lda + i] * b[b0 + j];
      b[i] = s;
    }
    __syncthreads();
  }
  // backward with L^T
  const int last = ((n - 1) / 32) * 32;
  for (int b0 = last; b0 >= 0; b0 -= 32) {
    const int nb = min(32, n - b0);
    // b[b0+j] -= sum_{i >= b0+nb} L[i, b0+j] x[i]
    for (int j = wid; j < nb; j += nw) {
      double s = 0.0;
      for (int i = b0 + nb + lane; i < n; i += 32) s += L[(long long)(b0 + j) * lda + i] * b[i];
      s = warp_sum(s);
      if (lane == 0) b[b0 + j] -= s;
    }
    __syncthreads();
    if (wid == 0) {
      double v = lane < nb ? b[b0 + lane] : 0.0;
      for (int j = nb - 1; j >= 0; --j) {
        double xj = __shfl_sync(0xffffffffu, v, j) / L[(long long)(b0 + j) * lda + b0 + j];
        if (lane == j) v = xj;
        if (lane < j) v -= L[(long long)(b0 + lane) * lda + b0 + j] * xj;
      }
      if (lane < nb) b[b0 + lane] = v;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) bg[i] = b[i];
}

// ---------------------------------------------------------------------------
// maxvol (reference maxvol.py): GEPP row choice, C = M inv(M[rows]), greedy swaps.
constexpr int MT_ = 512;  // 16 warps per CTA: the update passes are HBM-bound, keep enough loads in flight
constexpr int RMAX = 128;

// every CTA merges the per-CTA (value, index) partials: warp 0, lanes stride over CTAs
__device__ __forceinline__ AbsMax grid_absmax(const double* pv, const long long* pi, int nblk, double* sv,
                                              long long* si) {
  __shared__ AbsMax res;
  if (threadIdx.x < 32) {
    AbsMax g{-1.0, (long long)1 << 62};
    for (int b = threadIdx.x; b < nblk; b += 32) g = absmax_merge(g, AbsMax{pv[b], pi[b]});
    g = warp_absmax(g);
    if (threadIdx.x == 0) res = g;
  }
  __syncthreads();
  AbsMax r = res;
  __syncthreads();
  return r;
}

// One grid barrier per elimination step and per swap: the matrix is double-buffered (every step
// reads buffer A and writes buffer B, so the pivot row can be read by all CTAs while its owner
// writes the updated copy), and each update pass also produces the per-CTA argmax partials the
// next step needs (parity-double-buffered). Same operations, same order and the same tie-break
// (lowest physical / flattened index) as the reference's numpy code (maxvol.py:19-62).
__global__ void __launch_bounds__(MT_) maxvol_kernel(int n, int r, const double* __restrict__ Q, double* W0,
                                                      int* perm, double* W1, double* Ainv, double* pv,
                                                      long long* pi, double tol, int max_iters, int* rows_out,
                                                      int* status, int ainv_smem) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double mv_dyn[];   // ainv_smem: the 2 r^2 Gauss-Jordan tableau of phase 2 (block 0)
  __shared__ double sv[32];
  __shared__ long long si[32];
  __shared__ double srow[RMAX];
  __shared__ double sA[RMAX * RMAX / 4];  // holds Ainv when r <= 64
  const int nblk = gridDim.x;
  const int chunk = (n + nblk - 1) / nblk;
  const int i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  double* pvs[2] = {pv, pv + 296};
  long long* pis[2] = {pi, pi + 296};
  double* scl = pv + 2 * 296;  // per-CTA |max| for the degeneracy scale
  // copy; partials: global |max| (scale) and the step-0 pivot search over column 0
  AbsMax mx{0.0, 0};
  AbsMax b0{-1.0, (long long)1 << 62};
  for (int i = i0 + threadIdx.x; i < i1; i += MT_) {
    perm[i] = i;
    for (int c = 0; c < r; ++c) {
      double v = Q[(long long)c * n + i];
      W0[(long long)c * n + i] = v;
      mx.v = fmax(mx.v, fabs(v));
    }
    b0 = absmax_merge(b0, AbsMax{fabs(Q[i]), i});
  }
  mx.i = 0;
  mx = block_absmax(mx, sv, si);
  b0 = block_absmax(b0, sv, si);
  if (threadIdx.x == 0) { scl[blockIdx.x] = mx.v; pvs[0][blockIdx.x] = b0.v; pis[0][blockIdx.x] = b0.i; }
  grid.sync();
  double scale = 0.0;
  for (int b = 0; b < nblk; ++b) scale = fmax(scale, scl[b]);
  // phase 1: Gaussian elimination with partial pivoting, physical row swaps (A -> B each step)
  double* A = W0;
  double* B = W1;
  for (int k = 0; k < r; ++k) {
    AbsMax g = grid_absmax(pvs[k & 1], pis[k & 1], nblk, sv, si);
    if (g.v <= 1e-14 * fmax(scale, 1e-300)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) *status = 1;
      return;  // uniform across the grid
    }
    const int p = (int)g.i;
    if (p != k && blockIdx.x == 0 && threadIdx.x == 0) { int t = perm[k]; perm[k] = perm[p]; perm[p] = t; }
    for (int c = k + threadIdx.x; c < r; c += MT_) srow[c] = A[(long long)c * n + p];  // pivot row
    __syncthreads();
    const double d = srow[k];
    AbsMax best{-1.0, (long long)1 << 62};
    for (int i = max(i0, k) + threadIdx.x; i < i1; i += MT_) {
      if (i == k) {  // the pivot row moves to position k unchanged
        for (int c = k + 1; c < r; ++c) B[(long long)c * n + k] = srow[c];
        continue;
      }
      const int src = (i == p) ? k : i;  // old row k moves to position p
      const double l = A[(long long)k * n + src] / d;
      for (int c = k + 1; c < r; ++c) B[(long long)c * n + i] = A[(long long)c * n + src] - l * srow[c];
      if (k + 1 < r) best = absmax_merge(best, AbsMax{fabs(B[(long long)(k + 1) * n + i]), i});
    }
    best = block_absmax(best, sv, si);
    if (threadIdx.x == 0) { pvs[(k + 1) & 1][blockIdx.x] = best.v; pis[(k + 1) & 1][blockIdx.x] = best.i; }
    grid.sync();
    double* t = A; A = B; B = t;
  }
  // phase 2: Ainv = inv(Q[rows]) by Gauss-Jordan with partial pivoting (block 0), C = Q Ainv. The
  // tableau lives in shared memory when it fits (the r steps are a chain of small dependent passes:
  // shared-memory latency instead of L2 round trips; same operations in the same order), the inverse
  // is then copied out for the other CTAs.
  if (blockIdx.x == 0) {
    double* Aw = ainv_smem ? mv_dyn : Ainv;
    for (int e = threadIdx.x; e < r * r; e += MT_) {
      int c = e / r, i = e % r;
      Aw[(long long)c * r + i] = Q[(long long)c * n + perm[i]];
      Aw[(long long)(c + r) * r + i] = (c == i) ? 1.0 : 0.0;
    }
    __syncthreads();
    __shared__ int sp;
    for (int k = 0; k < r; ++k) {
      if (threadIdx.x < 32) {   // first row index of the largest |column k| entry at or below the diagonal
        int p = k;
        double bv = -1.0;
        for (int i = k + (int)threadIdx.x; i < r; i += 32) {
          double v = fabs(Aw[(long long)k * r + i]);
          if (v > bv) { bv = v; p = i; }
        }
        for (int o = 16; o; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int op = __shfl_xor_sync(0xffffffffu, p, o);
          if (ov > bv || (ov == bv && op < p)) { bv = ov; p = op; }
        }
        if (threadIdx.x == 0) sp = p;
      }
      __syncthreads();
      const int p = sp;
      if (p != k)
        for (int c = threadIdx.x; c < 2 * r; c += MT_) {
          double t = Aw[(long long)c * r + k];
          Aw[(long long)c * r + k] = Aw[(long long)c * r + p];
          Aw[(long long)c * r + p] = t;
        }
      __syncthreads();
      const double d = Aw[(long long)k * r + k];
      __syncthreads();
      for (int c = threadIdx.x; c < 2 * r; c += MT_) Aw[(long long)c * r + k] /= d;
      __syncthreads();
      for (int e = threadIdx.x; e < r * 2 * r; e += MT_) {
        int c = e / r, i = e % r;
        if (i != k && c != k) Aw[(long long)c * r + i] -= Aw[(long long)k * r + i] * Aw[(long long)c * r + k];
      }
      __syncthreads();
      for (int i = threadIdx.x; i < r; i += MT_)
        if (i != k) Aw[(long long)k * r + i] = 0.0;
      __syncthreads();
    }
    if (ainv_smem)
      for (int e = threadIdx.x; e < r * r; e += MT_) Ainv[(long long)r * r + e] = Aw[(long long)r * r + e];
  }
  grid.sync();
  // inverse sits in columns r..2r-1; C (buffer Ca) = Q Ainv, with the first swap's argmax partials
  const double* Ai = Ainv + (long long)r * r;
  const bool in_smem = r <= 64;
  if (in_smem) {
    for (int e = threadIdx.x; e < r * r; e += MT_) sA[e] = Ai[e];
    __syncthreads();
  }
  double* Ca = W0;
  double* Cb = W1;
  {
    AbsMax best{-1.0, (long long)1 << 62};
    for (int i = i0 + threadIdx.x; i < i1; i += MT_) {
      for (int c = 0; c < r; ++c) {
        double s = 0.0;
        for (int k = 0; k < r; ++k) s += Q[(long long)k * n + i] * (in_smem ? sA[c * r + k] : Ai[(long long)c * r + k]);
        Ca[(long long)c * n + i] = s;
        best = absmax_merge(best, AbsMax{fabs(s), (long long)i * r + c});
      }
    }
    best = block_absmax(best, sv, si);
    if (threadIdx.x == 0) { pvs[0][blockIdx.x] = best.v; pis[0][blockIdx.x] = best.i; }
  }
  int* rows = perm;  // rows[0..r) live in perm[0..r)
  grid.sync();
  // phase 3: greedy swaps (Sherman-Morrison), Ca -> Cb each iteration
  for (int it = 0; it < max_iters; ++it) {
    AbsMax g = grid_absmax(pvs[it & 1], pis[it & 1], nblk, sv, si);
    if (g.v <= tol) break;
    const int bi = (int)(g.i / r), bj = (int)(g.i % r);
    for (int c = threadIdx.x; c < r; c += MT_) srow[c] = Ca[(long long)c * n + bi] - (c == bj ? 1.0 : 0.0);
    const double pivv = Ca[(long long)bj * n + bi];
    __syncthreads();
    AbsMax best{-1.0, (long long)1 << 62};
    for (int i = i0 + threadIdx.x; i < i1; i += MT_) {
      const double f = Ca[(long long)bj * n + i] / pivv;
      for (int c = 0; c < r; ++c) {
        const double v = Ca[(long long)c * n + i] - f * srow[c];
        Cb[(long long)c * n + i] = v;
        best = absmax_merge(best, AbsMax{fabs(v), (long long)i * r + c});
      }
    }
    best = block_absmax(best, sv, si);
    if (threadIdx.x == 0) { pvs[(it + 1) & 1][blockIdx.x] = best.v; pis[(it + 1) & 1][blockIdx.x] = best.i; }
    if (blockIdx.x == 0 && threadIdx.x == 0) rows[bj] = bi;
    grid.sync();
    double* t = Ca; Ca = Cb; Cb = t;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int a = 0; a < r; ++a) rows_out[a] = rows[a];
    for (int a = 1; a < r; ++a) {
      int v = rows_out[a], b = a - 1;
      while (b >= 0 && rows_out[b] > v) { rows_out[b + 1] = rows_out[b]; --b; }
      rows_out[b + 1] = v;
    }
    *status = 0;
  }
}

constexpr size_t MV_DYN_MAX = 160 * 1024;   // dynamic shared memory the phase-2 tableau may take (r <= 101)

int maxvol_grid(int n, size_t dyn) {
  // one row per thread, up to the co-resident limit of the cooperative launch (<= 296 partials)
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(maxvol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)MV_DYN_MAX);
  }
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, maxvol_kernel, MT_, dyn);
  int maxb = sms * (per > 0 ? per : 1);
  if (maxb > 296) maxb = 296;
  int want = ceil_div(n, MT_);
  if (want < 1) want = 1;
  return want < maxb ? want : maxb;
}

}  // namespace

// LU factorization (in place, col-major) + solve of op(A) X = B (B col-major n x nrhs, overwritten).
TTB_API int ttb_lu_solve(void* stream, int n, double* A, long long lda, int* piv, int nrhs, double* B, long long ldb,
                         int trans, int* info) {
  if (n < 1 || nrhs < 0) return TTB_EARG;
  cudaStream_t st = as_stream(stream);
  lu_kernel<<<1, ST, 0, st>>>(n, A, lda, piv, info); ttb_count();
  if (nrhs > 0) lu_apply_kernel<<<ceil_div(nrhs, 128), 128, 0, st>>>(n, A, lda, piv, nrhs, B, ldb, trans); ttb_count();
  return ttb_last_error();
}

// Cholesky factorization of SPD col-major A (lower triangle used/overwritten). info: 0 ok, k>0 failed pivot.
TTB_API int ttb_potrf(void* stream, int n, double* A, long long lda, int* info) {
  if (n < 1) return TTB_EARG;
  cudaStream_t st = as_stream(stream);
  cudaMemsetAsync(info, 0, sizeof(int), st);
  for (int j0 = 0; j0 < n; j0 += CNB) {
    const int nb = n - j0 < CNB ? n - j0 : CNB;
    {
      int g = ceil_div(n - j0 - nb, 256);
      if (g < 1) g = 1;
      if (g > ttb_num_sms()) g = ttb_num_sms();
      chol_panel_kernel<<<g, 256, 0, st>>>(n, j0, A, lda, info); ttb_count();
    }
    const int m2 = n - j0 - nb;
    if (m2 > 0) {
      const double* Lp = A + (long long)j0 * lda + j0 + nb;  // col-major m2 x nb == row-major nb x m2 (ld lda)
      double* A22 = A + (long long)(j0 + nb) * lda + j0 + nb;
      int rc = ttb_dgemm(stream, 1, 0, m2, m2, nb, -1.0, Lp, lda, 0, Lp, lda, 0, 1.0, A22, lda, 0, 1);
      if (rc) return rc;
    }
  }
  return ttb_last_error();
}

TTB_API int ttb_potrs(void* stream, int n, const double* L, long long lda, double* b) {
  if (n < 1) return TTB_EARG;
  size_t smem = (size_t)n * sizeof(double);
  if (smem > 200 * 1024) return TTB_EARG;
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(chol_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cfg = true;
  }
  chol_solve_kernel<<<1, ST, smem, as_stream(stream)>>>(n, L, lda, b); ttb_count();
  return ttb_last_error();
}

TTB_API long long ttb_maxvol_workspace(int n, int r) {
  // two n*r buffers, Ainv (2 r^2), partials: values 2 x 296 + scale 296, indices 2 x 296 (int64)
  return 2LL * n * r + 2LL * r * r + 5 * 296 + 64;
}

// rows_out: r sorted row indices of a tol-dominant submatrix of Q (n x r col-major, ld n), n > r.
// iws: n + 1 ints (perm + status). Returns TTB_ESINGULAR when Q is column-rank deficient.
TTB_API int ttb_maxvol(void* stream, int n, int r, const double* Q, double tol, int max_iters, int* rows_out, double* ws,
                       int* iws) {
  if (r < 1 || r > RMAX || n <= r) return TTB_EARG;
  double* W = ws;
  double* C = W + (long long)n * r;
  double* Ainv = C + (long long)n * r;
  double* pv = Ainv + 2LL * r * r;
  long long* pi = reinterpret_cast<long long*>(pv + 3 * 296);
  int* perm = iws;
  int* status = iws + n;
  size_t dyn = 2 * (size_t)r * r * sizeof(double);
  int ainv_smem = dyn <= MV_DYN_MAX ? 1 : 0;
  if (!ainv_smem) dyn = 0;
  int nblk = maxvol_grid(n, dyn);
  void* args[] = {&n, &r, &Q, &W, &perm, &C, &Ainv, &pv, &pi, &tol, &max_iters, &rows_out, &status, &ainv_smem};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)maxvol_kernel, dim3(nblk), dim3(MT_), args, dyn, as_stream(stream)); ttb_count();
  return e == cudaSuccess ? 0 : (int)e;
}

// ---------------------------------------------------------------------------
// Banded LU without pivoting (stable for totally positive matrices such as B-spline
// collocation at Greville points) + parallel solves of many right-hand sides.
namespace {

__global__ void band_lu_kernel(int n, int kl, int ku, double* A, long long lda) {
  // one warp: the k-th step touches at most kl x ku entries
  const int lane = threadIdx.x;
  for (int k = 0; k < n; ++k) {
    const double piv = A[(long long)k * lda + k];
    const int i1 = min(n - 1, k + kl), j1 = min(n - 1, k + ku);
    for (int i = k + 1 + lane; i <= i1; i += 32) A[(long long)k * lda + i] /= piv;
    __syncwarp();
    const int ni = i1 - k, nj = j1 - k;
    for (int e = lane; e < ni * nj; e += 32) {
      const int i = k + 1 + e / nj, j = k + 1 + e % nj;
      A[(long long)j * lda + i] -= A[(long long)k * lda + i] * A[(long long)j * lda + k];
    }
    __syncwarp();
  }
}

__global__ void band_lu_apply_kernel(int n, int kl, int ku, const double* __restrict__ LU, long long lda, int nrhs,
                                     double* B, long long ldb) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nrhs) return;
  double* b = B + (long long)c * ldb;
  for (int k = 0; k < n; ++k) {
    double s = b[k];
    for (int i = max(0, k - kl); i < k; ++i) s -= LU[(long long)i * lda + k] * b[i];
    b[k] = s;
  }
  for (int k = n - 1; k >= 0; --k) {
    double s = b[k];
    for (int j = k + 1; j <= min(n - 1, k + ku); ++j) s -= LU[(long long)j * lda + k] * b[j];
    b[k] = s / LU[(long long)k * lda + k];
  }
}

}  // namespace

// A (n x n col-major, band kl/ku) is factored in place without pivoting; B (n x nrhs col-major) <- A^-1 B.
TTB_API int ttb_band_lu_solve(void* stream, int n, int kl, int ku, double* A, long long lda, int nrhs, double* B,
                              long long ldb) {
  if (n < 1 || kl < 0 || ku < 0) return TTB_EARG;
  cudaStream_t st = as_stream(stream);
  band_lu_kernel<<<1, 32, 0, st>>>(n, kl, ku, A, lda); ttb_count();
  if (nrhs > 0) { band_lu_apply_kernel<<<ceil_div(nrhs, 128), 128, 0, st>>>(n, kl, ku, A, lda, nrhs, B, ldb); ttb_count(); }
  return ttb_last_error();
}
