// Blocked Householder QR (LAPACK dgeqrf/dorgqr conventions) on column-major FP64 matrices.
//
// Panels of NB columns are factored by one cooperative kernel (grid-wide
// reductions for the column norms and the reflector/column dot products,
// deterministic: every CTA re-sums the per-CTA partials in the same order);
// the trailing matrix is updated with the compact-WY form
// A2 -= V (T^T (V^T A2)) through three DMMA GEMMs, which carry the flops.
#include "common.cuh"
#include <stdlib.h>

TTB_API int ttb_dgemm(void* stream, int tA, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
                      long long sA, const double* B, long long ldb, long long sB, double beta, double* C,
                      long long ldc, long long sC, int batch);
// tsqr.cu
long long tsqr_workspace(long long m);
long long cholqr_workspace(long long m, int b);
// blas.cu: large WY products (W = C V^T over the long dimension, C -= W2 V) as Ozaki-scheme FP64 on the
// int8 tensor cores when the shape allows, else ttb_dgemm
int dgemm_wy(void* stream, int tB, int M, int N, int K, double alpha, const double* A, long long lda, const double* B,
             long long ldb, double beta, double* C, long long ldc);
int cholqr_block(cudaStream_t st, long long mp, int b, double* P, long long lda, double* tau, double* Vtop,
                 double* T, double* ws);
constexpr int TTB_CHOLQR_FALLBACK = -50;
bool tsqr_applies(long long m, int jb);
int tsqr_panel(long long m, int jb, double* P, long long ld, double* tau, double* V, double* Tout, double* ws,
               cudaStream_t st);

namespace {

constexpr int NB = 16;  // inner Householder panel width (memory-bound part)
constexpr int PT = 256;  // threads per CTA of the panel kernel
constexpr int kMaxPanelBlocks = 1024;  // sizing of the per-CTA partial buffers

// Factor the m x jb panel P (col-major, ld) in place. Writes tau[0..jb), the explicit
// reflectors V (m x jb col-major, ld m: unit diagonal, zeros above) and the WY factor T
// (jb x jb row-major, upper triangular). part: gridDim.x * (NB*NB + NB) doubles.
__global__ void __launch_bounds__(PT, 2) panel_qr_kernel(int m, int jb, double* P, long long ld, double* tau, double* V,
                                                      double* T, double* part) {
  // One pass over the panel and ONE grid-wide barrier per column. While column j's reflector
  // is applied to a row, the row's updated entries are already folded into the next column's
  // statistics (its squared norm and z_c = x^T P[:, c]), so the reflector of column j+1 is
  // known right after the barrier: w_c = v^T P[:, c] = P[j+1, c] + scal * z_c. Writes of the
  // pivot row j are deferred by one column (it is read by every CTA at the start of column j).
  cg::grid_group grid = cg::this_grid();
  constexpr int ZW = NB + 1;  // z_c for c < NB, norm at index NB
  __shared__ double swarp[PT / 32][ZW];
  __shared__ double sz[ZW];
  __shared__ double sw[NB];
  __shared__ double srow[NB];
  __shared__ double sbeta[NB];
  const int nblk = gridDim.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int chunk = (m + nblk - 1) / nblk;
  const int r0 = blockIdx.x * chunk;
  const int r1 = min(m, r0 + chunk);
  double* zpart = part;  // [2][nblk][ZW]

  auto reduce_store = [&](double* acc, double nz, int buf) {
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      double v = warp_sum(acc[c]);
      if (lane == 0) swarp[wid][c] = v;
    }
    {
      double v = warp_sum(nz);
      if (lane == 0) swarp[wid][NB] = v;
    }
    __syncthreads();
    if (threadIdx.x < ZW) {
      double v = 0.0;
      for (int w = 0; w < PT / 32; ++w) v += swarp[w][threadIdx.x];
      zpart[((long long)buf * nblk + blockIdx.x) * ZW + threadIdx.x] = v;
    }
  };

  {  // statistics of column 0: ||x||^2 and z_c = x^T P[:, c] over rows > 0
    double acc[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) acc[c] = 0.0;
    double nz = 0.0;
    for (int i = max(r0, 1) + threadIdx.x; i < r1; i += PT) {
      const double x = P[i];
      nz += x * x;
#pragma unroll
      for (int c = 1; c < NB; ++c)
        if (c < jb) acc[c] += x * P[(long long)c * ld + i];
    }
    reduce_store(acc, nz, 0);
    grid.sync();
  }
  for (int j = 0; j < jb; ++j) {
    const int buf = j & 1;
    // every CTA re-sums the per-CTA partials (same order everywhere -> identical results):
    // one warp per statistic, lanes stride over the CTAs, then a shuffle reduction
    for (int t = wid; t < ZW; t += PT / 32) {
      double v = 0.0;
      for (int b = lane; b < nblk; b += 32) v += zpart[((long long)buf * nblk + b) * ZW + t];
      v = warp_sum(v);
      if (lane == 0) sz[t] = v;
    }
    // deferred write of pivot row j-1 (nobody reads it during column j)
    if (j >= 1 && (j - 1) >= r0 && (j - 1) < r1)
      for (int c = j + threadIdx.x; c < jb; c += PT) P[(long long)c * ld + (j - 1)] = srow[c];
    __syncthreads();
    const double xn2 = sz[NB];
    const double alpha = P[(long long)j * ld + j];
    double beta, t, scal;
    if (xn2 == 0.0) {
      beta = alpha; t = 0.0; scal = 0.0;
    } else {
      const double nrm = sqrt(alpha * alpha + xn2);
      beta = alpha >= 0.0 ? -nrm : nrm;
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (threadIdx.x < NB) {
      const int c = threadIdx.x;
      if (c > j && c < jb) {
        const double pjc = P[(long long)c * ld + j];
        const double w = pjc + scal * sz[c];
        sw[c] = w;
        srow[c] = pjc - t * w;   // new pivot-row entry (written one column later by its owner)
      }
      if (c == 0) sbeta[j] = beta;
    }
    __syncthreads();
    double acc[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) acc[c] = 0.0;
    double nz = 0.0;
    for (int i = max(r0, j + 1) + threadIdx.x; i < r1; i += PT) {
      const double v = scal * P[(long long)j * ld + i];
      P[(long long)j * ld + i] = v;
      const double tv = t * v;
      double vals[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c > j && c < jb) vals[c] = P[(long long)c * ld + i];
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c > j && c < jb) {
          vals[c] -= tv * sw[c];
          P[(long long)c * ld + i] = vals[c];
        }
      if (i > j + 1 && j + 1 < jb) {
        double xn = 0.0;
#pragma unroll
        for (int c = 0; c < NB; ++c)
          if (c == j + 1) xn = vals[c];
        nz += xn * xn;
#pragma unroll
        for (int c = 0; c < NB; ++c)
          if (c > j + 1 && c < jb) acc[c] += xn * vals[c];
      }
    }
    reduce_store(acc, nz, buf ^ 1);
    if (blockIdx.x == 0 && threadIdx.x == 0) tau[j] = t;
    grid.sync();
  }
  // the diagonal (beta) of every owned pivot row (the last pivot row has no entries right of it)
  for (int j = threadIdx.x; j < jb; j += PT)
    if (j >= r0 && j < r1) P[(long long)j * ld + j] = sbeta[j];
  grid.sync();
  // explicit V (unit diagonal, zeros above); its Gram and the WY factor T follow on the host side
  for (int i = r0 + threadIdx.x; i < r1; i += PT) {
    for (int c = 0; c < jb; ++c) {
      double v = (i < c) ? 0.0 : (i == c ? 1.0 : P[(long long)c * ld + i]);
      V[(long long)c * m + i] = v;
    }
  }
}

// V from the stored panel (for dorgqr) -- unit diagonal, zeros above
__global__ void extract_v_kernel(int m, int jb, const double* P, long long ld, double* V) {
  long long tot = (long long)m * jb;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    int c = (int)(e / m), i = (int)(e % m);
    V[e] = (i < c) ? 0.0 : (i == c ? 1.0 : P[(long long)c * ld + i]);
  }
}

__global__ void eye_kernel(int m, int k, double* Q, long long ld) {
  long long tot = (long long)m * k;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    int c = (int)(e / m), i = (int)(e % m);
    Q[(long long)c * ld + i] = (i == c) ? 1.0 : 0.0;
  }
}

// R (k x n, col-major ld k) = upper triangle of A
__global__ void extract_r_kernel(int k, int n, const double* A, long long lda, double* R) {
  long long tot = (long long)k * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    int c = (int)(e / k), i = (int)(e % k);
    R[e] = (i <= c) ? A[(long long)c * lda + i] : 0.0;
  }
}

int panel_grid(int m) {
  static int max_blocks = 0;
  if (!max_blocks) {
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, panel_qr_kernel, PT, 0);
    max_blocks = sms * (per_sm > 0 ? (per_sm > 4 ? 4 : per_sm) : 1);
  }
  int want = ceil_div(m, 4 * PT);  // >= 1024 rows per CTA before going wider
  if (want < 1) want = 1;
  return want < max_blocks ? want : max_blocks;
}

// Panel small enough for one CTA's shared memory (m * jb <= kSmallPanel): no grid barriers,
// factorization + explicit V + Gram + T in one launch (latency-bound medium-sized QRs).
constexpr int kSmallPanel = 20480;
constexpr int SPT = 512;

__global__ void __launch_bounds__(SPT) panel_small_kernel(int m, int jb, double* P, long long ld, double* tau,
                                                           double* V, double* T) {
  extern __shared__ double S[];  // m x jb col-major, ld m
  __shared__ double red[32];
  __shared__ double w[NB], taus[NB], betas[NB], G[NB * NB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = SPT / 32;
  for (int e = threadIdx.x; e < m * jb; e += SPT) S[e] = P[(long long)(e / m) * ld + (e % m)];
  __syncthreads();
  for (int j = 0; j < jb; ++j) {
    double* col = S + (long long)j * m;
    double s = 0.0;
    for (int i = j + 1 + threadIdx.x; i < m; i += SPT) s += col[i] * col[i];
    s = block_sum(s, red);
    const double alpha = col[j];
    double beta, t, scal;
    if (s == 0.0) { beta = alpha; t = 0.0; scal = 0.0; }
    else {
      const double nrm = sqrt(alpha * alpha + s);
      beta = alpha >= 0.0 ? -nrm : nrm;
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    for (int i = j + 1 + threadIdx.x; i < m; i += SPT) col[i] *= scal;
    __syncthreads();
    for (int c = j + 1 + wid; c < jb; c += nw) {
      const double* sc = S + (long long)c * m;
      double acc = 0.0;
      for (int i = j + lane; i < m; i += 32) acc += (i == j ? 1.0 : col[i]) * sc[i];
      acc = warp_sum(acc);
      if (lane == 0) w[c] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < (jb - j - 1) * (m - j); e += SPT) {
      const int c = j + 1 + e / (m - j), i = j + e % (m - j);
      S[(long long)c * m + i] -= t * (i == j ? 1.0 : col[i]) * w[c];
    }
    if (threadIdx.x == 0) { taus[j] = t; betas[j] = beta; }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * jb; e += SPT) {
    const int c = e / m, i = e % m;
    P[(long long)c * ld + i] = (i == c) ? betas[c] : S[e];
    V[e] = (i < c) ? 0.0 : (i == c ? 1.0 : S[e]);
  }
  if (threadIdx.x < jb) tau[threadIdx.x] = taus[threadIdx.x];
  // Gram of the unit-lower V (one warp per pair a < b), then dlarft
  for (int pr = wid; pr < jb * jb; pr += nw) {
    const int a = pr / jb, b = pr % jb;
    if (a >= b) continue;
    double acc = 0.0;
    for (int i = b + lane; i < m; i += 32) {
      const double va = (i == a) ? 1.0 : S[(long long)a * m + i];
      const double vb = (i == b) ? 1.0 : S[(long long)b * m + i];
      acc += va * vb;
    }
    acc = warp_sum(acc);
    if (lane == 0) G[a * NB + b] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int e = 0; e < jb * jb; ++e) T[e] = 0.0;
    for (int i = 0; i < jb; ++i) {
      const double ti = taus[i];
      T[i * jb + i] = ti;
      for (int r = 0; r < i; ++r) {
        double v = 0.0;
        for (int c = r; c < i; ++c) v += T[r * jb + c] * G[c * NB + i];
        T[r * jb + i] = -ti * v;
      }
    }
  }
}

bool panel_is_small(int m, int jb) { return (long long)m * jb <= kSmallPanel; }

// Register-resident single-CTA panel (m <= CPT * CRPT rows): thread t holds rows t + CPT s. One
// batched reduction per column (the look-ahead statistics of tsqr.cu: z_c = x^T A[:, c] with
// x = A[j+1:, j], giving the reflector application and the dlarft column), two barriers per column.
constexpr int CPT = 256, CRPT = 5;
template <int JB>
__global__ void __launch_bounds__(CPT, 1) panel_cta_kernel(int m, int jb_rt, double* P, long long ld, double* tau,
                                                           double* V, double* T) {
  __shared__ double red[CPT / 32][NB];
  __shared__ double zf[NB];
  __shared__ double rowb[2][NB];
  __shared__ double Ts[NB][NB + 1];
  const int jb = JB ? JB : jb_rt;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  double a[CRPT][NB];
#pragma unroll
  for (int s = 0; s < CRPT; ++s) {
    const int i = t + CPT * s;
#pragma unroll
    for (int c = 0; c < NB; ++c) a[s][c] = (i < m && c < jb) ? P[(long long)c * ld + i] : 0.0;
  }
  for (int e = t; e < NB * (NB + 1); e += CPT) (&Ts[0][0])[e] = 0.0;
  auto stats = [&](int col, int buf) {  // z_c = sum_{i > col} A[i, col] A[i, c]; row col -> rowb[buf]
    double z[NB];
    double x[CRPT];
#pragma unroll
    for (int s = 0; s < CRPT; ++s) {
      const int i = t + CPT * s;
      double xv = 0.0;
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c == col) xv = a[s][c];
      x[s] = (i > col && i < m) ? xv : 0.0;
    }
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      z[c] = 0.0;
#pragma unroll
      for (int s = 0; s < CRPT; ++s) z[c] += x[s] * a[s][c];
    }
    warp_allreduce16(z, lane);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < NB; ++c) red[w][c] = z[c];
    if (t == col)
#pragma unroll
      for (int c = 0; c < NB; ++c) rowb[buf][c] = a[0][c];
    __syncthreads();
    if (t < NB) {
      double v = 0.0;
      for (int q = 0; q < CPT / 32; ++q) v += red[q][t];
      zf[t] = v;
    }
    __syncthreads();
  };
  stats(0, 0);
  for (int j = 0; j < jb; ++j) {
    double rowj[NB], zj[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) { rowj[c] = rowb[j & 1][c]; zj[c] = zf[c]; }
    double alpha = 0.0, s2 = 0.0;
#pragma unroll
    for (int c = 0; c < NB; ++c)
      if (c == j) { alpha = rowj[c]; s2 = zj[c]; }
    double beta, tj, scal;
    if (s2 == 0.0) {
      beta = alpha; tj = 0.0; scal = 0.0;
    } else {
      const double nrm = sqrt(alpha * alpha + s2);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tj = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    double wv[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) wv[c] = rowj[c] + scal * zj[c];
    if (t < j) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (b >= t && b < j) acc += Ts[t][b] * wv[b];
      Ts[t][j] = -tj * acc;
    }
    if (t == 0) Ts[j][j] = tj;
#pragma unroll
    for (int s = 0; s < CRPT; ++s) {
      const int i = t + CPT * s;
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        if (c == j) {
          const double vi = (i > j && i < m) ? a[s][c] * scal : (i == j ? 1.0 : 0.0);
          if (i > j) a[s][c] = vi;
          const double tv = tj * vi;
#pragma unroll
          for (int c2 = 0; c2 < NB; ++c2)
            if (c2 > c) a[s][c2] -= tv * wv[c2];
        }
      }
    }
    if (t == j)
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c == j) a[0][c] = beta;
    if (j + 1 < jb) stats(j + 1, (j + 1) & 1);
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < CRPT; ++s) {
    const int i = t + CPT * s;
    if (i < m)
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c < jb) {
          P[(long long)c * ld + i] = a[s][c];
          V[(long long)c * m + i] = (i < c) ? 0.0 : (i == c ? 1.0 : a[s][c]);
        }
  }
  for (int e = t; e < jb * jb; e += CPT) T[e] = Ts[e / jb][e % jb];
  if (t < jb) tau[t] = Ts[t][t];
}

int launch_panel_small(int m, int jb, double* P, long long ld, double* tau, double* V, double* T, cudaStream_t st) {
  static int legacy = getenv("TTB_PANEL_SMALL") ? 1 : 0;
  if (!legacy && m <= CPT * CRPT && jb <= NB) {
    if (jb == NB) panel_cta_kernel<NB><<<1, CPT, 0, st>>>(m, jb, P, ld, tau, V, T);
    else panel_cta_kernel<0><<<1, CPT, 0, st>>>(m, jb, P, ld, tau, V, T);
    ttb_count();
    return ttb_last_error();
  }
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(panel_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmallPanel * 8);
    cfg = true;
  }
  panel_small_kernel<<<1, SPT, (size_t)m * jb * sizeof(double), st>>>(m, jb, P, ld, tau, V, T); ttb_count();
  return ttb_last_error();
}

int launch_panel(int m, int jb, double* P, long long ld, double* tau, double* V, double* T, double* part, cudaStream_t st) {
  int nblk = panel_grid(m);
  void* args[] = {&m, &jb, &P, &ld, &tau, &V, &T, &part};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)panel_qr_kernel, dim3(nblk), dim3(PT), args, 0, st); ttb_count();
  return e == cudaSuccess ? 0 : (int)e;
}

}  // namespace

namespace {

#ifndef TTB_NB2
#define TTB_NB2 128
#endif
constexpr int NB2 = TTB_NB2;  // outer WY block (trailing-update GEMMs have K = 128)

// T (nb x nb row-major, upper, nb <= NB) from the Gram G = V^T V (upper triangle read, row-major
// ld ldg) and tau (dlarft, forward, columnwise); staged in shared memory.
__global__ void larft_kernel(int nb, const double* G, int ldg, const double* tau, double* T) {
  __shared__ double Ts[NB][NB + 1], Gs[NB][NB + 1];
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    Ts[r][c] = 0.0;
    Gs[r][c] = (r < nb && c < nb && r <= c) ? G[(long long)r * ldg + c] : 0.0;
  }
  __syncthreads();
  for (int i = 0; i < nb; ++i) {
    const double ti = tau[i];
    if (threadIdx.x == 0) Ts[i][i] = ti;
    for (int r = threadIdx.x; r < i; r += blockDim.x) {
      double v = 0.0;
      for (int c = r; c < i; ++c) v += Ts[r][c] * Gs[c][i];
      Ts[r][i] = -ti * v;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) T[e] = Ts[e / nb][e % nb];
}

// Outer-block T (JB x JB row-major) from the inner panels' T factors (NB x NB each, row-major ld
// jb_p, at Tin + p NB NB) and the outer Gram G (row-major ld ldg) by block merges:
// T[0:c0, c0:c0+jb] = -T[0:c0, 0:c0] (G[0:c0, c0:c0+jb] T_pp)   (I - V1 T1 V1^T)(I - V2 T2 V2^T)
constexpr int LBT = 256;
__global__ void __launch_bounds__(LBT) larft_block_kernel(int JB, const double* __restrict__ G, int ldg,
                                                           const double* __restrict__ Tin, double* T) {
  extern __shared__ double sm[];
  const int LDT = JB + 1;
  double* Ts = sm;                       // JB x LDT
  double* Ps = sm + (long long)JB * LDT; // JB x NB
  for (int e = threadIdx.x; e < JB * LDT; e += LBT) Ts[e] = 0.0;
  __syncthreads();
  const int np = (JB + NB - 1) / NB;
  for (int p = 0; p < np; ++p) {
    const int c0 = p * NB, jb = min(NB, JB - c0);
    const double* Tp = Tin + (long long)p * NB * NB;
    for (int e = threadIdx.x; e < jb * jb; e += LBT) Ts[(c0 + e / jb) * LDT + c0 + e % jb] = Tp[e];
  }
  __syncthreads();
  for (int p = 1; p < np; ++p) {
    const int c0 = p * NB, jb = min(NB, JB - c0);
    const double* Tp = Ts + (long long)c0 * LDT + c0;
    for (int e = threadIdx.x; e < c0 * jb; e += LBT) {  // P = G[0:c0, c0:c0+jb] T_pp (T_pp upper)
      const int r = e / jb, c = e % jb;
      double acc = 0.0;
      for (int b = 0; b <= c; ++b) acc += G[(long long)r * ldg + c0 + b] * Tp[b * LDT + c];
      Ps[r * NB + c] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < c0 * jb; e += LBT) {  // T[0:c0, c0:] = -T[0:c0, 0:c0] P
      const int r = e / jb, c = e % jb;
      double acc = 0.0;
      for (int b = r; b < c0; ++b) acc += Ts[r * LDT + b] * Ps[b * NB + c];
      Ts[r * LDT + c0 + c] = -acc;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < JB * JB; e += LBT) T[e] = Ts[(e / JB) * LDT + e % JB];
}

int launch_larft_block(int JB, const double* G, int ldg, const double* Tin, double* T, cudaStream_t st) {
  const size_t smem = ((size_t)JB * (JB + 1) + (size_t)JB * NB) * sizeof(double);
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(larft_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cfg = true;
  }
  larft_block_kernel<<<1, LBT, smem, st>>>(JB, G, ldg, Tin, T); ttb_count();
  return ttb_last_error();
}

// G (nb x nb row-major, nb <= NB) = V^T V for a tall col-major V (m x nb, ld m): every CTA
// stages 128-row tiles in shared memory, one thread per (a, b) pair accumulates; per-CTA
// partials are summed by a second kernel in a fixed order (deterministic).
__global__ void __launch_bounds__(256) gram_partial_kernel(int m, int nb, const double* __restrict__ V,
                                                           double* __restrict__ part) {
  __shared__ double tile[NB][129];
  const int pairs = nb * nb;
  double acc = 0.0;
  const int a = threadIdx.x / nb, b = threadIdx.x % nb;
  for (int r0 = blockIdx.x * 128; r0 < m; r0 += gridDim.x * 128) {
    const int rn = min(128, m - r0);
    __syncthreads();
    for (int e = threadIdx.x; e < nb * 128; e += 256) {
      const int c = e / 128, i = e % 128;
      tile[c][i] = i < rn ? V[(long long)c * m + r0 + i] : 0.0;
    }
    __syncthreads();
    if (threadIdx.x < pairs && a <= b)
      for (int i = 0; i < 128; ++i) acc += tile[a][i] * tile[b][i];
  }
  if (threadIdx.x < pairs) part[(long long)blockIdx.x * pairs + threadIdx.x] = (a <= b) ? acc : 0.0;
}

// one CTA per Gram entry (upper triangle a <= b; larft reads only that): fixed-order block sum
__global__ void gram_final_kernel(int nb, int nblk, const double* __restrict__ part, double* G) {
  __shared__ double red[32];
  const int pairs = nb * nb;
  const int e = blockIdx.x;
  if ((e / nb) > (e % nb)) return;  // uniform per CTA
  double v = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) v += part[(long long)b * pairs + e];
  v = block_sum(v, red);
  if (threadIdx.x == 0) G[e] = v;
}

int launch_gram(int m, int nb, const double* V, double* G, double* part, cudaStream_t st) {
  int blocks = ceil_div(m, 128);
  if (blocks > 592) blocks = 592;
  gram_partial_kernel<<<blocks, 256, 0, st>>>(m, nb, V, part); ttb_count();
  gram_final_kernel<<<nb * nb, 128, 0, st>>>(nb, blocks, part, G); ttb_count();
  return ttb_last_error();
}

struct QrWs {
  double *part, *Vp, *Vb, *W, *W2, *G, *Tin, *Tout, *ts;
  double *Wb, *W2b, *Gb, *Vt2;  // second set for the look-ahead stream split
  double* cq;                    // CholeskyQR2 block factorization (cholqr.cu)
};

QrWs carve(double* ws, int m, int n) {
  const int k = m < n ? m : n;
  const long long wn = (long long)(n > k ? n : k);
  QrWs w;
  w.part = ws;
  w.Vp = w.part + (long long)kMaxPanelBlocks * (NB * NB + NB + 2);
  w.Vb = w.Vp + (long long)m * NB;
  w.W = w.Vb + (long long)m * NB2;
  w.W2 = w.W + wn * NB2;
  w.G = w.W2 + wn * NB2;
  w.Tin = w.G + (long long)NB2 * NB2;
  w.Tout = w.Tin + (long long)((k + NB - 1) / NB) * NB * NB;
  w.ts = w.Tout + (long long)((k + NB2 - 1) / NB2) * NB2 * NB2;
  w.Wb = w.ts + tsqr_workspace(m);
  w.W2b = w.Wb + wn * NB2;
  w.Gb = w.W2b + wn * NB2;
  w.Vt2 = w.Gb + (long long)NB2 * NB2;  // 2 x NB2 x NB2: Vtop of block parity 0 / 1
  w.cq = w.Vt2 + 2LL * NB2 * NB2;
  return w;
}

// TTB_PANEL=coop selects the cooperative column-by-column panel for tall panels (A/B testing)
bool coop_panels() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TTB_PANEL");
    v = (e && e[0] == 'c') ? 1 : 0;
  }
  return v == 1;
}

int grid_v(long long tot) {
  int b = ceil_div(tot, 256);
  if (b > ttb_num_sms() * 8) b = ttb_num_sms() * 8;
  return b < 1 ? 1 : b;
}

// C (rows mp, cols nq, col-major ld) := (I - V T V^T)^{op} C, V col-major (mp x jb, ld mp), T row-major jb x jb.
// transT = 1 applies Q^T (geqrf trailing update), 0 applies Q (orgqr).
int apply_wy(void* stream, int mp, int nq, int jb, const double* V, const double* T, int transT, double* C,
             long long ldc, double* W, double* W2) {
  int rc = dgemm_wy(stream, 1, nq, jb, mp, 1.0, C, ldc, V, mp, 0.0, W, jb);
  if (rc) return rc;
  rc = ttb_dgemm(stream, 0, transT ? 0 : 1, nq, jb, jb, 1.0, W, jb, 0, T, jb, 0, 0.0, W2, jb, 0, 1);
  if (rc) return rc;
  return dgemm_wy(stream, 0, nq, mp, jb, -1.0, W2, jb, V, mp, 1.0, C, ldc);
}

// Same update with V read in place from the factored panel Ap (col-major, ld lda): rows >= jb of V
// are the stored reflector entries; only the unit-lower top jb x jb block (Vtop, ld jb) is explicit.
int apply_wy_panel(void* stream, int mp, int nq, int jb, const double* Ap, long long lda, const double* Vtop,
                   const double* T, int transT, double* C, long long ldc, double* W, double* W2) {
  const int mb = mp - jb;
  int rc = 0;
  if (mb > 0) rc = dgemm_wy(stream, 1, nq, jb, mb, 1.0, C + jb, ldc, Ap + jb, lda, 0.0, W, jb);
  if (rc) return rc;
  rc = ttb_dgemm(stream, 0, 1, nq, jb, jb, 1.0, C, ldc, 0, Vtop, jb, 0, mb > 0 ? 1.0 : 0.0, W, jb, 0, 1);
  if (rc) return rc;
  rc = ttb_dgemm(stream, 0, transT ? 0 : 1, nq, jb, jb, 1.0, W, jb, 0, T, jb, 0, 0.0, W2, jb, 0, 1);
  if (rc) return rc;
  rc = ttb_dgemm(stream, 0, 0, nq, jb, jb, -1.0, W2, jb, 0, Vtop, jb, 0, 1.0, C, ldc, 0, 1);
  if (rc || mb <= 0) return rc;
  return dgemm_wy(stream, 0, nq, mb, jb, -1.0, W2, jb, Ap + jb, lda, 1.0, C + jb, ldc);
}

// W[q][p] = V[q][p] (rows q < nid of W = C^T V when C's first nid columns are still e_q: orgqr)
__global__ void w_identity_kernel(int nid, int jb, const double* __restrict__ Vtop, double* W) {
  for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < nid * jb; e += blockDim.x * gridDim.x) {
    const int q = e / jb, p = e % jb;
    W[e] = Vtop[(long long)p * jb + q];
  }
}

// apply_wy_panel for orgqr: the first nid columns of C are untouched identity columns (rows < nid),
// so their rows of W = C^T V are rows of V and only the remaining columns need the long GEMM.
int apply_wy_panel_orgqr(void* stream, int mp, int nq, int jb, int nid, const double* Ap, long long lda,
                         const double* Vtop, const double* T, double* C, long long ldc, double* W, double* W2) {
  cudaStream_t st = as_stream(stream);
  const int mb = mp - jb;
  const int nr = nq - nid;
  w_identity_kernel<<<ceil_div((long long)nid * jb, 256), 256, 0, st>>>(nid, jb, Vtop, W); ttb_count();
  int rc = 0;
  if (nr > 0) {
    if (mb > 0)
      rc = dgemm_wy(stream, 1, nr, jb, mb, 1.0, C + (long long)nid * ldc + jb, ldc, Ap + jb, lda, 0.0,
                    W + (long long)nid * jb, jb);
    if (rc) return rc;
    rc = ttb_dgemm(stream, 0, 1, nr, jb, jb, 1.0, C + (long long)nid * ldc, ldc, 0, Vtop, jb, 0, mb > 0 ? 1.0 : 0.0,
                   W + (long long)nid * jb, jb, 0, 1);
    if (rc) return rc;
  }
  rc = ttb_dgemm(stream, 0, 1, nq, jb, jb, 1.0, W, jb, 0, T, jb, 0, 0.0, W2, jb, 0, 1);
  if (rc) return rc;
  rc = ttb_dgemm(stream, 0, 0, nq, jb, jb, -1.0, W2, jb, 0, Vtop, jb, 0, 1.0, C, ldc, 0, 1);
  if (rc || mb <= 0) return rc;
  return dgemm_wy(stream, 0, nq, mb, jb, -1.0, W2, jb, Ap + jb, lda, 1.0, C + jb, ldc);
}

// G = V^T V for the in-place reflectors of apply_wy_panel
int gram_panel(void* stream, int mp, int jb, const double* Ap, long long lda, const double* Vtop, double* G) {
  const int mb = mp - jb;
  int rc = 0;
  if (mb > 0) rc = ttb_dgemm(stream, 0, 1, jb, jb, mb, 1.0, Ap + jb, lda, 0, Ap + jb, lda, 0, 0.0, G, jb, 0, 1);
  if (rc) return rc;
  return ttb_dgemm(stream, 0, 1, jb, jb, jb, 1.0, Vtop, jb, 0, Vtop, jb, 0, mb > 0 ? 1.0 : 0.0, G, jb, 0, 1);
}

}  // namespace

// Householder panel with dgeqr2 + dlarft outputs (single-CTA kernel when it fits shared memory,
// else the cooperative one + Gram + larft); tsqr.cu runs it on the stacked R factors.
// part: kMaxPanelBlocks * (NB * NB + NB + 2) doubles, G: NB * NB doubles.
int householder_panel(int m, int jb, double* P, long long ld, double* tau, double* V, double* T, double* part,
                      double* G, cudaStream_t st) {
  if (panel_is_small(m, jb)) return launch_panel_small(m, jb, P, ld, tau, V, T, st);
  int rc = launch_panel(m, jb, P, ld, tau, V, T, part, st);
  if (rc) return rc;
  rc = launch_gram(m, jb, V, G, part, st);
  if (rc) return rc;
  larft_kernel<<<1, 128, 0, st>>>(jb, G, jb, tau, T); ttb_count();
  return ttb_last_error();
}
long long householder_panel_part() { return (long long)kMaxPanelBlocks * (NB * NB + NB + 2); }

// Workspace sizes (in doubles) for ttb_geqrf / ttb_orgqr.
TTB_API long long ttb_qr_workspace(int m, int n) {
  const int k = m < n ? m : n;
  const long long wn = (long long)(n > k ? n : k);
  long long s = (long long)kMaxPanelBlocks * (NB * NB + NB + 2);
  s += (long long)m * NB + (long long)m * NB2 + 2 * wn * NB2 + (long long)NB2 * NB2;
  s += (long long)((k + NB - 1) / NB) * NB * NB + (long long)((k + NB2 - 1) / NB2) * NB2 * NB2;
  s += tsqr_workspace(m);
  s += 2 * wn * NB2 + 3LL * NB2 * NB2;  // look-ahead: second W, W2, G and two Vtop blocks
  s += cholqr_workspace(m, NB2);
  return s + 64;
}

namespace {

// Panels of outer block [J0, J0 + JB) on stream s (inner WY updates inside the block; a block that
// is a single panel updates the whole trailing matrix), then the block's Vtop, Gram and T.
// TTB_PANEL_CHOLQR=0 keeps the 128-column blocks of tall QRs on the TSQR panels (A/B)
bool cholqr_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TTB_PANEL_CHOLQR");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int factor_block(cudaStream_t s, int m, int n, int J0, int JB, double* A, long long lda, double* tau, QrWs& w,
                 double* Wp, double* W2p, double* Vtop, double* G) {
  void* stream = (void*)s;
  if (JB == NB2 && (long long)(m - J0) >= 65536 && cholqr_enabled()) {
    // well-conditioned tall block: CholeskyQR2 + Householder reconstruction (four GEMM passes)
    // instead of eight TSQR panels; falls through to them when the Cholesky pivots say otherwise
    double* Tb = w.Tout + (long long)(J0 / NB2) * NB2 * NB2;
    const int rc = cholqr_block(s, m - J0, JB, A + (long long)J0 * lda + J0, lda, tau + J0, Vtop, Tb, w.cq);
    TTB_DBG(s, "geqrf cholqr block");
    if (rc != TTB_CHOLQR_FALLBACK) return rc;
  }
  for (int j0 = J0; j0 < J0 + JB; j0 += NB) {
    const int jb = (J0 + JB - j0) < NB ? (J0 + JB - j0) : NB;
    const int mp = m - j0;
    double* P = A + (long long)j0 * lda + j0;
    double* T = w.Tin + (long long)(j0 / NB) * NB * NB;
    int rc;
    if (panel_is_small(mp, jb)) {
      rc = launch_panel_small(mp, jb, P, lda, tau + j0, w.Vp, T, s);
    } else if (tsqr_applies(mp, jb) && !coop_panels()) {
      rc = tsqr_panel(mp, jb, P, lda, tau + j0, w.Vp, T, w.ts, s);
    } else {
      rc = launch_panel(mp, jb, P, lda, tau + j0, w.Vp, T, w.part, s);
      if (!rc) rc = launch_gram(mp, jb, w.Vp, G, w.part, s);
      if (!rc) { larft_kernel<<<1, 128, 0, s>>>(jb, G, jb, tau + j0, T); ttb_count(); }
    }
    TTB_DBG(s, "geqrf panel");
    if (rc) return rc;
    const int n2 = (JB <= NB) ? (n - j0 - jb) : (J0 + JB - j0 - jb);
    if (n2 > 0) {
      rc = apply_wy(stream, mp, n2, jb, w.Vp, T, 1, A + (long long)(j0 + jb) * lda + j0, lda, Wp, W2p);
      TTB_DBG(s, "geqrf inner apply_wy");
      if (rc) return rc;
    }
  }
  double* Tb = w.Tout + (long long)(J0 / NB2) * NB2 * NB2;
  if (JB <= NB) {
    cudaMemcpyAsync(Tb, w.Tin + (long long)(J0 / NB) * NB * NB, sizeof(double) * JB * JB, cudaMemcpyDeviceToDevice, s);
    return ttb_last_error();
  }
  const double* Ap = A + (long long)J0 * lda + J0;
  extract_v_kernel<<<grid_v((long long)JB * JB), 256, 0, s>>>(JB, JB, Ap, lda, Vtop); ttb_count();
  int rc = gram_panel(stream, m - J0, JB, Ap, lda, Vtop, G);
  if (rc) return rc;
  rc = launch_larft_block(JB, G, JB, w.Tin + (long long)(J0 / NB) * NB * NB, Tb, s);
  TTB_DBG(s, "geqrf outer larft");
  return rc;
}

struct LookAhead {
  cudaStream_t sb = nullptr;
  cudaEvent_t* ev = nullptr;
  int nev = 0;
};

LookAhead& look_ahead(int need) {
  static LookAhead la;
  if (!la.sb) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&la.sb, cudaStreamNonBlocking, hi);  // panels first when SMs free up
  }
  if (need > la.nev) {
    cudaEvent_t* ev = new cudaEvent_t[need];
    for (int i = 0; i < la.nev; ++i) ev[i] = la.ev[i];
    for (int i = la.nev; i < need; ++i) cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    delete[] la.ev;
    la.ev = ev;
    la.nev = need;
  }
  return la;
}

// TTB_QR_LOOKAHEAD=0 keeps the serial order (A/B testing)
bool lookahead_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TTB_QR_LOOKAHEAD");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// Right-looking blocked QR with depth-1 look-ahead: the panels of block J+1 (their columns first
// updated by block J) are factored on a second, high-priority stream while the caller's stream
// applies block J to the columns beyond block J+1. Column sets are disjoint; each stream has its
// own WY scratch, Vtop/Gram buffers alternate by block parity.
int geqrf_lookahead(cudaStream_t st, int m, int n, double* A, long long lda, double* tau, QrWs& w) {
  const int k = m < n ? m : n;
  const int nblk = (k + NB2 - 1) / NB2;
  LookAhead& la = look_ahead(2 * nblk + 2);
  cudaStream_t sb = la.sb;
  cudaEvent_t ev_start = la.ev[0], ev_done = la.ev[1];
  cudaEvent_t* ev_fact = la.ev + 2;         // block J factored (T_J ready), on sb
  cudaEvent_t* ev_big = la.ev + 2 + nblk;   // big update of block J applied, on st
  cudaEventRecord(ev_start, st);
  cudaStreamWaitEvent(sb, ev_start, 0);
  auto vtop = [&](int J) { return w.Vt2 + (long long)(J & 1) * NB2 * NB2; };
  auto gbuf = [&](int J) { return (J & 1) ? w.Gb : w.G; };
  int rc = factor_block(sb, m, n, 0, k < NB2 ? k : NB2, A, lda, tau, w, w.W, w.W2, vtop(0), gbuf(0));
  if (rc) return rc;
  cudaEventRecord(ev_fact[0], sb);
  for (int J = 0; J < nblk; ++J) {
    const int J0 = J * NB2;
    const int JB = (k - J0) < NB2 ? (k - J0) : NB2;
    const int J1 = J0 + JB;
    const int JBn = (J + 1 < nblk) ? ((k - J1) < NB2 ? (k - J1) : NB2) : 0;
    const double* Ap = A + (long long)J0 * lda + J0;
    double* Tb = w.Tout + (long long)(J0 / NB2) * NB2 * NB2;
    // the trailing update of block J is enqueued first: the next block's factorization may wait
    // on the host (CholeskyQR2 pivot check) and the main stream must already have its work
    const int nrest = n - (J1 + JBn);
    if (nrest > 0 && JB > NB) {
      cudaStreamWaitEvent(st, ev_fact[J], 0);
      rc = apply_wy_panel((void*)st, m - J0, nrest, JB, Ap, lda, vtop(J), Tb, 1, A + (long long)(J1 + JBn) * lda + J0,
                          lda, w.Wb, w.W2b);
      if (rc) return rc;
    }
    cudaEventRecord(ev_big[J], st);
    if (JBn > 0) {
      if (J >= 1) cudaStreamWaitEvent(sb, ev_big[J - 1], 0);
      if (JB > NB) {  // a single-panel block already updated everything to its right
        rc = apply_wy_panel((void*)sb, m - J0, JBn, JB, Ap, lda, vtop(J), Tb, 1, A + (long long)J1 * lda + J0, lda, w.W,
                            w.W2);
        if (rc) return rc;
      }
      rc = factor_block(sb, m, n, J1, JBn, A, lda, tau, w, w.W, w.W2, vtop(J + 1), gbuf(J + 1));
      if (rc) return rc;
      cudaEventRecord(ev_fact[J + 1], sb);
    }
  }
  cudaEventRecord(ev_done, sb);
  cudaStreamWaitEvent(st, ev_done, 0);
  return ttb_last_error();
}

}  // namespace

// In-place QR of col-major A (m x n, lda). tau: min(m,n). ws: ttb_qr_workspace doubles; the outer
// WY factors stay in ws for a following ttb_orgqr. Two-level blocking: 32-column panels (cooperative
// kernel) inside 128-column blocks whose trailing update is three GEMMs with K = 128.
TTB_API int ttb_geqrf(void* stream, int m, int n, double* A, long long lda, double* tau, double* ws) {
  if (m < 0 || n < 0 || lda < (m > 1 ? m : 1)) return TTB_EARG;
  const int k = m < n ? m : n;
  if (k == 0) return TTB_OK;
  cudaStream_t st = as_stream(stream);
  QrWs w = carve(ws, m, n);
  if (lookahead_enabled() && m >= 65536 && k > NB2) return geqrf_lookahead(st, m, n, A, lda, tau, w);
  for (int J0 = 0; J0 < k; J0 += NB2) {
    const int JB = (k - J0) < NB2 ? (k - J0) : NB2;
    const int MP = m - J0;
    for (int j0 = J0; j0 < J0 + JB; j0 += NB) {
      const int jb = (J0 + JB - j0) < NB ? (J0 + JB - j0) : NB;
      const int mp = m - j0;
      double* P = A + (long long)j0 * lda + j0;
      double* T = w.Tin + (long long)(j0 / NB) * NB * NB;
      int rc;
      if (panel_is_small(mp, jb)) {
        rc = launch_panel_small(mp, jb, P, lda, tau + j0, w.Vp, T, st);
        if (rc) return rc;
      } else if (tsqr_applies(mp, jb) && !coop_panels()) {
        rc = tsqr_panel(mp, jb, P, lda, tau + j0, w.Vp, T, w.ts, st);
        TTB_DBG(st, "geqrf tsqr panel");
        if (rc) return rc;
      } else {
        rc = launch_panel(mp, jb, P, lda, tau + j0, w.Vp, T, w.part, st);
        if (rc) return rc;
        // T from the Gram V^T V (one streaming pass over V) -- dlarft
        rc = launch_gram(mp, jb, w.Vp, w.G, w.part, st);
        if (rc) return rc;
        larft_kernel<<<1, 128, 0, st>>>(jb, w.G, jb, tau + j0, T); ttb_count();
      }
      // inside the outer block, or -- when the block is a single panel -- the whole trailing matrix
      const int n2 = (JB <= NB) ? (n - j0 - jb) : (J0 + JB - j0 - jb);
      if (n2 > 0) {
        rc = apply_wy(stream, mp, n2, jb, w.Vp, T, 1, A + (long long)(j0 + jb) * lda + j0, lda, w.W, w.W2);
        TTB_DBG(st, "geqrf inner apply_wy");
        if (rc) return rc;
      }
    }
    double* Tb = w.Tout + (long long)(J0 / NB2) * NB2 * NB2;
    if (JB <= NB) {
      cudaMemcpyAsync(Tb, w.Tin + (long long)(J0 / NB) * NB * NB, sizeof(double) * JB * JB,
                      cudaMemcpyDeviceToDevice, st);
      continue;
    }
    const double* Ap = A + (long long)J0 * lda + J0;
    extract_v_kernel<<<grid_v((long long)JB * JB), 256, 0, st>>>(JB, JB, Ap, lda, w.Vb); ttb_count();  // Vtop
    int rc = gram_panel(stream, MP, JB, Ap, lda, w.Vb, w.G);
    TTB_DBG(st, "geqrf outer gram");
    if (rc) return rc;
    rc = launch_larft_block(JB, w.G, JB, w.Tin + (long long)(J0 / NB) * NB * NB, Tb, st);
    TTB_DBG(st, "geqrf outer larft");
    if (rc) return rc;
    const int n2 = n - J0 - JB;
    if (n2 > 0) {
      rc = apply_wy_panel(stream, MP, n2, JB, Ap, lda, w.Vb, Tb, 1, A + (long long)(J0 + JB) * lda + J0, lda, w.W,
                          w.W2);
      if (rc) return rc;
    }
  }
  return ttb_last_error();
}

// Explicit Q (m x kq, col-major ld ldq) from a ttb_geqrf result (same ws), kq <= min(m, n_factored).
TTB_API int ttb_orgqr(void* stream, int m, int kq, int kf, const double* A, long long lda, double* Q, long long ldq,
                      double* ws, int n_factored) {
  if (m < 0 || kq < 0 || kq > m) return TTB_EARG;
  cudaStream_t st = as_stream(stream);
  const int k = kf;
  QrWs w = carve(ws, m, n_factored);
  eye_kernel<<<grid_v((long long)m * kq), 256, 0, st>>>(m, kq, Q, ldq); ttb_count();
  const int last = ((k - 1) / NB2) * NB2;
  for (int J0 = last; J0 >= 0; J0 -= NB2) {
    const int JB = (k - J0) < NB2 ? (k - J0) : NB2;
    const int MP = m - J0;
    const int nq = kq - J0;
    if (nq <= 0) continue;
    double* Tb = w.Tout + (long long)(J0 / NB2) * NB2 * NB2;
    const double* Ap = A + (long long)J0 * lda + J0;
    extract_v_kernel<<<grid_v((long long)JB * JB), 256, 0, st>>>(JB, JB, Ap, lda, w.Vb); ttb_count();  // Vtop
    const int nid = JB < nq ? JB : nq;  // columns J0 .. J0+JB-1 of Q are still identity columns here
    int rc = apply_wy_panel_orgqr(stream, MP, nq, JB, nid, Ap, lda, w.Vb, Tb, Q + (long long)J0 * ldq + J0, ldq, w.W,
                                  w.W2);
    if (rc) return rc;
  }
  return ttb_last_error();
}

TTB_API int ttb_extract_r(void* stream, int k, int n, const double* A, long long lda, double* R) {
  long long tot = (long long)k * n;
  if (tot == 0) return TTB_OK;
  int blocks = ceil_div(tot, 256);
  if (blocks > ttb_num_sms() * 8) blocks = ttb_num_sms() * 8;
  extract_r_kernel<<<blocks, 256, 0, as_stream(stream)>>>(k, n, A, lda, R); ttb_count();
  return ttb_last_error();
}

// ---------------------------------------------------------------------------
// Small QR in one CTA: the whole m x n matrix and the explicit Q live in shared memory
// (m*n + m*k <= kSmallQr doubles). This is the shape of almost every TT-rank-sized
// unfolding in the IGA solves (n = TT rank <= 64), where the blocked multi-kernel path
// is launch-latency bound. Same Householder convention as ttb_geqrf/ttb_orgqr.
namespace {

constexpr int SQT = 512;
constexpr int kSmallQr = 24576;  // doubles of shared memory for A and Q (192 KB)

__global__ void __launch_bounds__(SQT) small_qr_kernel(int m, int n, const double* __restrict__ A, long long lda,
                                                        double* Q, long long ldq, double* R, int want_q) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  __shared__ double taus[64];
  __shared__ double betas[64];
  __shared__ double w[64];
  const int k = m < n ? m : n;
  double* S = sm;               // m x n, col-major, ld m
  double* Qs = sm + (long long)m * n;  // m x k
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = SQT / 32;
  for (int e = threadIdx.x; e < m * n; e += SQT) S[e] = A[(long long)(e / m) * lda + (e % m)];
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    double* col = S + (long long)j * m;
    double s = 0.0;
    for (int i = j + 1 + threadIdx.x; i < m; i += SQT) s += col[i] * col[i];
    s = block_sum(s, red);
    const double alpha = col[j];
    double beta, t, scal;
    if (s == 0.0) { beta = alpha; t = 0.0; scal = 0.0; }
    else {
      const double nrm = sqrt(alpha * alpha + s);
      beta = alpha >= 0.0 ? -nrm : nrm;
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    for (int i = j + 1 + threadIdx.x; i < m; i += SQT) col[i] *= scal;
    __syncthreads();
    // w_c = v^T S[j:, c] (one warp per column), then S[j:, c] -= t v w_c
    for (int c = j + 1 + wid; c < n; c += nw) {
      const double* sc = S + (long long)c * m;
      double acc = 0.0;
      for (int i = j + lane; i < m; i += 32) acc += (i == j ? 1.0 : col[i]) * sc[i];
      acc = warp_sum(acc);
      if (lane == 0) w[c] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < (n - j - 1) * (m - j); e += SQT) {
      const int c = j + 1 + e / (m - j), i = j + e % (m - j);
      S[(long long)c * m + i] -= t * (i == j ? 1.0 : col[i]) * w[c];
    }
    if (threadIdx.x == 0) { taus[j] = t; betas[j] = beta; }
    __syncthreads();
  }
  // R (k x n, col-major ld k)
  for (int e = threadIdx.x; e < k * n; e += SQT) {
    const int c = e / k, i = e % k;
    R[e] = (i < c) ? S[(long long)c * m + i] : (i == c ? betas[i] : 0.0);
  }
  if (!want_q) return;
  for (int e = threadIdx.x; e < m * k; e += SQT) Qs[e] = ((e / m) == (e % m)) ? 1.0 : 0.0;
  __syncthreads();
  for (int j = k - 1; j >= 0; --j) {
    const double* v = S + (long long)j * m;
    const double t = taus[j];
    for (int c = j + wid; c < k; c += nw) {
      const double* qc = Qs + (long long)c * m;
      double acc = 0.0;
      for (int i = j + lane; i < m; i += 32) acc += (i == j ? 1.0 : v[i]) * qc[i];
      acc = warp_sum(acc);
      if (lane == 0) w[c] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < (k - j) * (m - j); e += SQT) {
      const int c = j + e / (m - j), i = j + e % (m - j);
      Qs[(long long)c * m + i] -= t * (i == j ? 1.0 : v[i]) * w[c];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * k; e += SQT) Q[(long long)(e / m) * ldq + (e % m)] = Qs[e];
}

}  // namespace

// 1 if (m, n) fits the single-CTA shared-memory QR.
TTB_API int ttb_qr_small_fits(int m, int n) {
  const long long k = m < n ? m : n;
  return (n <= 64 && (long long)m * n + (long long)m * k <= kSmallQr) ? 1 : 0;
}

// Q (m x k col-major, ld ldq; skipped when Q == NULL) and R (k x n col-major, ld k) of col-major A.
TTB_API int ttb_qr_small(void* stream, int m, int n, const double* A, long long lda, double* Q, long long ldq,
                         double* R) {
  if (!ttb_qr_small_fits(m, n) || m < 1 || n < 1) return TTB_EARG;
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(small_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmallQr * 8);
    cfg = true;
  }
  const long long k = m < n ? m : n;
  const size_t smem = (size_t)((long long)m * n + (Q ? (long long)m * k : 0)) * sizeof(double);
  small_qr_kernel<<<1, SQT, smem, as_stream(stream)>>>(m, n, A, lda, Q, ldq, R, Q ? 1 : 0); ttb_count();
  return ttb_last_error();
}
