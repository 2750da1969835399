// TSQR panel factorization for tall Householder panels (m x jb, jb <= 16, m in the millions).
//
// The blocked QR (qr.cu) needs, per NB-column panel, the LAPACK-style outputs of dgeqr2 +
// dlarft: Householder vectors V (unit lower trapezoidal, stored below the diagonal), R (on and
// above it), tau and the compact-WY factor T. A column-by-column panel over 1M rows is bound by
// one grid-wide reduction per column and by re-streaming the panel once per column. Here:
//
//   1. every warp factors one tile of <= 128 rows held in registers (4 rows per lane; one
//      batched warp reduction per column, T built alongside in the dlarft recurrence);
//   2. the jb x jb R factors of all tiles (m/8 rows) are stacked and factored by the ordinary
//      Householder panel (qr.cu), whose WY form gives their explicit Q, X1;
//   3. Householder reconstruction (Ballard, Demmel, Grigori, Jacquelin, Nguyen, Solomonik
//      2014): with the panel's orthonormal Q (Q_tile = H_tile [X1 block; 0]), the LU
//      factorization Y = [I; 0] - Q S = V U with the sign matrix S chosen on the fly (pivots
//      1 + |q_kk| >= 1) gives V (= L on top), T = U L^{-T}, tau = diag(U), R = S R_tsqr;
//   4. one leaf pass forms every tile's Q rows and writes V_below = -Q_below S U^{-1}.
//
// Passes over the panel: read + write in step 1, read + write (P and the explicit V copy) in
// step 4; the stacked level touches jb/8 of the rows.
#include "common.cuh"

namespace {

constexpr int NB = 16;   // max panel width (matches qr.cu)
constexpr int TR = 128;  // rows per tile
constexpr int TS = TR / 32;
constexpr int FW = 8;    // warps per CTA, factor kernel
constexpr int QW = 4;    // warps per CTA, Q-formation kernels
constexpr int LDS = NB + 1;

__device__ __forceinline__ void tile_bounds(long long rows, int nt, int t, long long& r0, int& r) {
  r0 = rows * t / nt;
  r = (int)(rows * (t + 1) / nt - r0);
}

__device__ __forceinline__ void load_tile(double (&a)[TS][NB], const double* M, long long ld, long long r0, int r,
                                          int jb, int lane) {
#pragma unroll
  for (int c = 0; c < NB; ++c)
#pragma unroll
    for (int s = 0; s < TS; ++s) {
      const int i = lane + 32 * s;
      a[s][c] = (c < jb && i < r) ? M[(long long)c * ld + r0 + i] : 0.0;
    }
}

// Householder QR of every tile of an (rows x jb) col-major matrix M (in place: R on/above the
// diagonal, V below), T per tile (NB x NB row-major) and the tile's R into rows [t jb, t jb + jb)
// of S (col-major, ld ldS). JB > 0: compile-time panel width. Columns >= jb are zero.
//
// One batched warp reduction per column: with x = A[j+1:, j] the statistics
// z_c = x^T A[j+1:, c] (c = j: ||x||^2; c > j: trailing columns; c < j: stored reflectors) give
// both the reflector application w_c = A[j, c] + scal z_c and the dlarft column
// v_b^T v_j = V[j, b] + scal z_b, and are accumulated right after column j-1's update.
template <int JB>
__global__ void __launch_bounds__(FW * 32) tsqr_factor_kernel(double* M, long long ld, long long rows, int nt, int jb_rt,
                                                               double* Tt, double* S, long long ldS) {
  __shared__ double Tsh[FW][NB * NB];
  const int jb = JB ? JB : jb_rt;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = blockIdx.x * FW + w;
  if (t >= nt) return;
  long long r0;
  int r;
  tile_bounds(rows, nt, t, r0, r);
  double a[TS][NB];
  load_tile(a, M, ld, r0, r, jb, lane);
  double* T = Tsh[w];
  for (int e = lane; e < NB * NB; e += 32) T[e] = 0.0;
  double z[NB];
  {
    double x[TS];
#pragma unroll
    for (int s = 0; s < TS; ++s) {
      const int i = lane + 32 * s;
      x[s] = (i > 0 && i < r) ? a[s][0] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      z[c] = 0.0;
#pragma unroll
      for (int s = 0; s < TS; ++s) z[c] += x[s] * a[s][c];
    }
  }
  warp_allreduce16(z, lane);
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    if (j < jb) {
      double rowj[NB];  // row j of the tile (lane j, slot 0)
#pragma unroll
      for (int c = 0; c < NB; ++c) rowj[c] = __shfl_sync(0xffffffffu, a[0][c], j);
      const double alpha = rowj[j], s2 = z[j];
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
      for (int c = 0; c < NB; ++c) wv[c] = rowj[c] + scal * z[c];  // c > j: v^T A[:, c]; c < j: v_c^T v
      if (lane < j) {
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < NB; ++b)
          if (b >= lane && b < j) acc += T[lane * NB + b] * wv[b];
        T[lane * NB + j] = -tj * acc;
      }
      if (lane == 0) T[j * NB + j] = tj;
      // v (zero above row j, 1 at row j), then A[:, c] -= tj v w_c for c > j
#pragma unroll
      for (int s = 0; s < TS; ++s) {
        const int i = lane + 32 * s;
        const double vi = (i > j && i < r) ? a[s][j] * scal : (i == j ? 1.0 : 0.0);
        if (i > j) a[s][j] = vi;
        const double tv = tj * vi;
#pragma unroll
        for (int c = j + 1; c < NB; ++c) a[s][c] -= tv * wv[c];
      }
      if (lane == j) a[0][j] = beta;
      if (j + 1 < jb) {  // statistics of column j + 1
        double x[TS];
#pragma unroll
        for (int s = 0; s < TS; ++s) {
          const int i = lane + 32 * s;
          x[s] = (i > j + 1 && i < r) ? a[s][j + 1] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          z[c] = 0.0;
#pragma unroll
          for (int s = 0; s < TS; ++s) z[c] += x[s] * a[s][c];
        }
        warp_allreduce16(z, lane);
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int c = 0; c < NB; ++c)
#pragma unroll
    for (int s = 0; s < TS; ++s) {
      const int i = lane + 32 * s;
      if (c < jb && i < r) M[(long long)c * ld + r0 + i] = a[s][c];
    }
  if (lane < jb)
#pragma unroll
    for (int c = 0; c < NB; ++c)
      if (c < jb) S[(long long)c * ldS + (long long)t * jb + lane] = (c >= lane) ? a[0][c] : 0.0;
  for (int e = lane; e < NB * NB; e += 32) Tt[(long long)t * NB * NB + e] = T[e];
}

// Inner tree level: the explicit Q rows of every tile, Q_tile = [X; 0] - V (T (V_top^T X)), written
// in place over the tile's reflectors (X = the tile's jb x jb block of the parent level's Q).
__global__ void __launch_bounds__(QW * 32) tsqr_form_kernel(double* M, long long ld, long long rows, int nt, int jb,
                                                             const double* __restrict__ Tt, const double* X,
                                                             long long ldX) {
  __shared__ double Bf[QW][3][NB * LDS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = blockIdx.x * QW + w;
  if (t >= nt) return;
  long long r0;
  int r;
  tile_bounds(rows, nt, t, r0, r);
  double* vt = Bf[w][0];
  double* xs = Bf[w][1];
  double* ms = Bf[w][2];
  if (lane < NB)
#pragma unroll
    for (int c = 0; c < NB; ++c)
      vt[lane * LDS + c] = (c < jb && lane < r) ? (lane > c ? M[(long long)c * ld + r0 + lane] : (lane == c ? 1.0 : 0.0))
                                                : 0.0;
  for (int e = lane; e < NB * NB; e += 32) {
    const int i = e % NB, c = e / NB;
    xs[i * LDS + c] = (i < jb && c < jb) ? X[(long long)c * ldX + (long long)t * jb + i] : 0.0;
  }
  __syncwarp();
  const double* Tg = Tt + (long long)t * NB * NB;
  for (int e = lane; e < NB * NB; e += 32) {  // ms = V_top^T X
    const int p = e / NB, c = e % NB;
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < NB; ++i) acc += vt[i * LDS + p] * xs[i * LDS + c];
    ms[p * LDS + c] = acc;
  }
  __syncwarp();
  for (int e = lane; e < NB * NB; e += 32) {  // vt = W = T ms
    const int p = e / NB, c = e % NB;
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < NB; ++b) acc += (b >= p ? Tg[p * NB + b] : 0.0) * ms[b * LDS + c];
    vt[p * LDS + c] = acc;
  }
  __syncwarp();
  for (int s = 0; s < TS; ++s) {
    const int i = lane + 32 * s;
    if (i >= r) continue;
    double v[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) v[c] = (c < jb) ? (i > c ? M[(long long)c * ld + r0 + i] : (i == c ? 1.0 : 0.0)) : 0.0;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      if (c < jb) {
        double acc = (i < NB) ? xs[i * LDS + c] : 0.0;
#pragma unroll
        for (int p = 0; p < NB; ++p) acc -= v[p] * vt[p * LDS + c];
        M[(long long)c * ld + r0 + i] = acc;
      }
    }
  }
}

// Leaf pass: the panel's Householder vectors V = Q Z (Z = -S U^{-1}) for rows >= jb, where the
// tile's orthonormal rows are Q_tile = H_tile [X; 0] = [X; 0] - V_tile (T (V_top^T X)) and X is
// the tile's jb x jb block of X1 (col-major, ld ldX). Folded: V = [X Z; 0] - V_tile (W Z),
// W = T V_top^T X, one 16 x 16 product per row. Written to M (below-diagonal storage) and to
// the explicit copy Vx (col-major, ld rows); the top jb rows of tile 0 (R and L) come from
// the setup kernel through Z + NB*NB.
__global__ void __launch_bounds__(QW * 32) tsqr_leaf_kernel(double* M, long long ld, long long rows, int nt, int jb,
                                                             const double* __restrict__ Tt, const double* X,
                                                             long long ldX, const double* __restrict__ Z,
                                                             double* Vx) {
  __shared__ double Bf[QW][3][NB * LDS];
  __shared__ double Zs[NB * LDS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) Zs[(e / NB) * LDS + (e % NB)] = Z[e];
  __syncthreads();
  const int t = blockIdx.x * QW + w;
  if (t >= nt) return;
  long long r0;
  int r;
  tile_bounds(rows, nt, t, r0, r);
  double* vt = Bf[w][0];
  double* xs = Bf[w][1];
  double* ms = Bf[w][2];
  if (lane < NB)
#pragma unroll
    for (int c = 0; c < NB; ++c)
      vt[lane * LDS + c] = (c < jb && lane < r) ? (lane > c ? M[(long long)c * ld + r0 + lane] : (lane == c ? 1.0 : 0.0))
                                                : 0.0;
  for (int e = lane; e < NB * NB; e += 32) {
    const int i = e % NB, c = e / NB;
    xs[i * LDS + c] = (i < jb && c < jb) ? X[(long long)c * ldX + (long long)t * jb + i] : 0.0;
  }
  __syncwarp();
  const double* Tg = Tt + (long long)t * NB * NB;
  for (int e = lane; e < NB * NB; e += 32) {  // ms = V_top^T X
    const int p = e / NB, c = e % NB;
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < NB; ++i) acc += vt[i * LDS + p] * xs[i * LDS + c];
    ms[p * LDS + c] = acc;
  }
  __syncwarp();
  for (int e = lane; e < NB * NB; e += 32) {  // vt = W = T ms (T upper)
    const int p = e / NB, c = e % NB;
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < NB; ++b) acc += (b >= p ? Tg[p * NB + b] : 0.0) * ms[b * LDS + c];
    vt[p * LDS + c] = acc;
  }
  __syncwarp();
  for (int e = lane; e < NB * NB; e += 32) {  // ms = W Z, Z upper
    const int p = e / NB, c = e % NB;
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < NB; ++b) acc += (b <= c ? vt[p * LDS + b] * Zs[b * LDS + c] : 0.0);
    ms[p * LDS + c] = acc;
  }
  __syncwarp();
  for (int e = lane; e < NB * NB; e += 32) {  // vt = X Z
    const int p = e / NB, c = e % NB;
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < NB; ++b) acc += (b <= c ? xs[p * LDS + b] * Zs[b * LDS + c] : 0.0);
    vt[p * LDS + c] = acc;
  }
  __syncwarp();
  for (int s = 0; s < TS; ++s) {  // one row per lane at a time (keeps registers low)
    const int i = lane + 32 * s;
    if (i >= r) continue;
    if (r0 + i < jb) {  // top rows (R and L), prepared by the setup kernel behind Z
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c < jb) M[(long long)c * ld + i] = Z[NB * NB + c * NB + i];
      continue;
    }
    double v[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) v[c] = (c < jb) ? (i > c ? M[(long long)c * ld + r0 + i] : (i == c ? 1.0 : 0.0)) : 0.0;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      if (c < jb) {
        double acc = (i < NB) ? vt[i * LDS + c] : 0.0;
#pragma unroll
        for (int p = 0; p < NB; ++p) acc -= v[p] * ms[p * LDS + c];
        M[(long long)c * ld + r0 + i] = acc;
        Vx[(long long)c * rows + r0 + i] = acc;
      }
    }
  }
}

// One warp. Top rows of the leaf Q (from tile 0 of level 0 and X1 = level-1 Q), the sign-chosen
// LU Y = [I;0] - Q S = V U, then: the P top block (R = S R_tsqr on/above, L below the diagonal;
// stored behind Z and written by the leaf pass, which still reads tile 0's reflectors), the
// explicit V top rows, tau = diag(U), T = U L^{-T} (row-major, ld jb), and Z = -S U^{-1} for the
// leaf pass.
__global__ void tsqr_setup_kernel(int jb, double* P, long long ld, long long mp, const double* __restrict__ T0,
                                  const double* __restrict__ X1, long long ldX1, const double* __restrict__ Rt,
                                  long long ldR, double* tau, double* Vx, double* Tout, double* Z) {
  __shared__ double Vt[NB * LDS], Xs[NB * LDS], Ms[NB * LDS], Ws[NB * LDS];
  __shared__ double E[NB * LDS], Q[NB * LDS], L[NB * LDS], U[NB * LDS], Li[NB * LDS];
  __shared__ double sg[NB];
  const int lane = threadIdx.x;
  for (int e = lane; e < NB * NB; e += 32) {
    const int i = e % NB, c = e / NB;
    double v = 0.0, x = 0.0;
    if (i < jb && c < jb) {
      v = i > c ? P[(long long)c * ld + i] : (i == c ? 1.0 : 0.0);
      x = X1[(long long)c * ldX1 + i];
    }
    Vt[i * LDS + c] = v;
    Xs[i * LDS + c] = x;
    E[i * LDS + c] = (i == c) ? 1.0 : 0.0;
    L[i * LDS + c] = (i == c) ? 1.0 : 0.0;
    U[i * LDS + c] = 0.0;
  }
  __syncwarp();
  for (int e = lane; e < NB * NB; e += 32) {
    const int p = e / NB, c = e % NB;
    double acc = 0.0;
    for (int i = 0; i < NB; ++i) acc += Vt[i * LDS + p] * Xs[i * LDS + c];
    Ms[p * LDS + c] = acc;
  }
  __syncwarp();
  for (int e = lane; e < NB * NB; e += 32) {
    const int p = e / NB, c = e % NB;
    double acc = 0.0;
    for (int b = p; b < NB; ++b) acc += T0[p * NB + b] * Ms[b * LDS + c];
    Ws[p * LDS + c] = acc;
  }
  __syncwarp();
  for (int e = lane; e < NB * NB; e += 32) {
    const int i = e / NB, c = e % NB;
    double acc = Xs[i * LDS + c];
    for (int p = 0; p < NB; ++p) acc -= Vt[i * LDS + p] * Ws[p * LDS + c];
    Q[i * LDS + c] = (i < jb && c < jb) ? acc : 0.0;
  }
  __syncwarp();
  // modified LU: column k of Y is E[:,k] - s_k Q[:,k]; row operations act on E and Q alike
  for (int k = 0; k < jb; ++k) {
    const double sk = Q[k * LDS + k] >= 0.0 ? -1.0 : 1.0;
    const double piv = E[k * LDS + k] - sk * Q[k * LDS + k];
    if (lane == 0) sg[k] = sk;
    const int i = lane;
    if (i > k && i < jb) {
      const double l = (E[i * LDS + k] - sk * Q[i * LDS + k]) / piv;
      L[i * LDS + k] = l;
      for (int c = k + 1; c < jb; ++c) {
        E[i * LDS + c] -= l * E[k * LDS + c];
        Q[i * LDS + c] -= l * Q[k * LDS + c];
      }
    }
    __syncwarp();
  }
  for (int e = lane; e < NB * NB; e += 32) {
    const int k = e / NB, c = e % NB;
    if (k < jb && c < jb && c >= k) U[k * LDS + c] = E[k * LDS + c] - sg[c] * Q[k * LDS + c];
  }
  // Li = L^{-1} (unit lower), one column per lane
  if (lane < NB) {
    const int c = lane;
    for (int i = 0; i < NB; ++i) Li[i * LDS + c] = (i == c) ? 1.0 : 0.0;
    for (int i = c + 1; i < jb; ++i) {
      double acc = 0.0;
      for (int b = c; b < i; ++b) acc += L[i * LDS + b] * Li[b * LDS + c];
      Li[i * LDS + c] = -acc;
    }
  }
  __syncwarp();
  for (int e = lane; e < jb * jb; e += 32) {
    const int p = e / jb, c = e % jb;
    double acc = 0.0;  // T = U L^{-T}: sum_b U[p][b] Li[c][b], b in [p, c]
    for (int b = p; b <= c; ++b) acc += U[p * LDS + b] * Li[c * LDS + b];
    Tout[p * jb + c] = (c >= p) ? acc : 0.0;
  }
  for (int e = lane; e < jb * jb; e += 32) {
    const int i = e % jb, c = e / jb;
    Z[NB * NB + c * NB + i] = (i <= c) ? sg[i] * Rt[(long long)c * ldR + i] : L[i * LDS + c];  // P top block
    Vx[(long long)c * mp + i] = (i < c) ? 0.0 : (i == c ? 1.0 : L[i * LDS + c]);
  }
  if (lane < jb) tau[lane] = U[lane * LDS + lane];
  // Z = -S U^{-1} (upper): column c of U^{-1} by back substitution, one column per lane
  if (lane < NB) {
    const int c = lane;
    double ui[NB];
#pragma unroll
    for (int i = NB - 1; i >= 0; --i) {
      double acc = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int b = i + 1; b < NB; ++b) acc -= U[i * LDS + b] * ui[b];
      ui[i] = (i <= c && c < jb) ? acc / U[i * LDS + i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) Z[i * NB + c] = -sg[i] * ui[i];
  }
}

// X = [I; 0] - V (T V_top^T): explicit Q of a WY-factored panel (V col-major, ld rows, unit lower;
// T row-major jb x jb, upper)
__global__ void tsqr_q1_kernel(long long rows, int jb, const double* __restrict__ V, const double* __restrict__ T,
                               double* X) {
  __shared__ double W[NB * NB];
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int p = e / NB, c = e % NB;
    double acc = 0.0;
    if (p < jb && c < jb)
      for (int b = p; b <= c; ++b) acc += T[p * jb + b] * (b == c ? 1.0 : V[(long long)b * rows + c]);
    W[e] = acc;
  }
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows; i += (long long)gridDim.x * blockDim.x) {
    double v[NB];
#pragma unroll
    for (int p = 0; p < NB; ++p) v[p] = (p < jb) ? (i == p ? 1.0 : (i > p ? V[(long long)p * rows + i] : 0.0)) : 0.0;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      if (c >= jb) break;
      double acc = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int p = 0; p < NB; ++p) acc -= v[p] * W[p * NB + c];
      X[(long long)c * rows + i] = acc;
    }
  }
}

int tiles_of(long long rows) { return (int)((rows + TR - 1) / TR); }

}  // namespace

int householder_panel(int m, int jb, double* P, long long ld, double* tau, double* V, double* T, double* part,
                      double* G, cudaStream_t st);
long long householder_panel_part();

// Tree levels: the stacked R factors are factored by warp tiles again until they fit the
// register-resident single-CTA panel (qr.cu), whose WY form gives the top level's Q.
constexpr long long kTopRows = 1280;
constexpr int kMaxLevels = 12;

long long tsqr_top_rows() {
  static const long long v = getenv("TTB_TSQR_TOP") ? atoll(getenv("TTB_TSQR_TOP")) : kTopRows;
  return v;
}

// Workspace (doubles) for tsqr_panel on panels of up to m rows. The level arrays shrink with the
// panel height, but the top level does not (a shorter panel can stop the tree one level earlier
// with a taller top), so the top arrays are reserved for the largest top any height can produce.
long long tsqr_workspace(long long m) {
  long long s = householder_panel_part() + 6 * NB * NB + 2 * NB + 256;
  long long rows = m;
  const long long top = tsqr_top_rows();
  for (int l = 0; l < kMaxLevels && (rows > top || l == 0); ++l) {
    const long long nt = (rows + TR - 1) / TR;
    s += nt * NB * NB;   // T per tile
    rows = nt * NB;
    s += rows * NB;      // stacked R of the next level (becomes its Q in place)
  }
  const long long rows1 = ((m + TR - 1) / TR) * NB;
  const long long top_max = rows1 < top ? rows1 : top;
  return s + 2 * (top_max > rows ? top_max : rows) * NB;  // top level: explicit V and Q
}

bool tsqr_applies(long long m, int jb) { return m > 8LL * TR && jb >= 1 && jb <= NB; }

// Factor the m x jb panel P (col-major, ld) in place with dgeqr2 conventions; tau[0..jb),
// explicit V (m x jb, ld m, unit diagonal, zeros above) and T (jb x jb row-major, upper).
int tsqr_panel(long long m, int jb, double* P, long long ld, double* tau, double* V, double* Tout, double* ws,
               cudaStream_t st) {
  double* part = ws;
  double* G = part + householder_panel_part();
  double* Ttop = G + NB * NB;
  double* Z = Ttop + NB * NB;       // Z = -S U^{-1} | P top block
  double* tautop = Z + 2 * NB * NB;
  double* cur = tautop + 2 * NB + 256;
  double* M[kMaxLevels + 1];
  long long ldm[kMaxLevels + 1], rows[kMaxLevels + 1];
  double* Tt[kMaxLevels];
  int nt[kMaxLevels];
  int L = 0;
  M[0] = P; ldm[0] = ld; rows[0] = m;
  const long long top_rows = tsqr_top_rows();
  while (rows[L] > top_rows || L == 0) {
    if (L >= kMaxLevels) return TTB_EARG;
    nt[L] = tiles_of(rows[L]);
    Tt[L] = cur;
    cur += (long long)nt[L] * NB * NB;
    rows[L + 1] = (long long)nt[L] * jb;
    ldm[L + 1] = rows[L + 1];
    M[L + 1] = cur;
    cur += rows[L + 1] * NB;
    if (jb == NB)
      tsqr_factor_kernel<NB><<<ceil_div(nt[L], FW), FW * 32, 0, st>>>(M[L], ldm[L], rows[L], nt[L], jb, Tt[L], M[L + 1],
                                                                      ldm[L + 1]);
    else
      tsqr_factor_kernel<0><<<ceil_div(nt[L], FW), FW * 32, 0, st>>>(M[L], ldm[L], rows[L], nt[L], jb, Tt[L], M[L + 1],
                                                                     ldm[L + 1]);
    ttb_count();
    TTB_DBG(st, "tsqr factor");
    ++L;
  }
  // top level: ordinary Householder panel (register-resident single CTA), then its explicit Q
  const long long rt = rows[L];
  double* Vtop = cur;
  double* Xtop = Vtop + rt * NB;
  int rc = householder_panel((int)rt, jb, M[L], rt, tautop, Vtop, Ttop, part, G, st);
  TTB_DBG(st, "tsqr top panel");
  if (rc) return rc;
  {
    int blocks = ceil_div(rt, 256);
    if (blocks > ttb_num_sms() * 4) blocks = ttb_num_sms() * 4;
    tsqr_q1_kernel<<<blocks, 256, 0, st>>>(rt, jb, Vtop, Ttop, Xtop); ttb_count();
    TTB_DBG(st, "tsqr q1");
  }
  // explicit Q of the inner levels, top-down (in place over their reflectors)
  const double* X = Xtop;
  long long ldX = rt;
  for (int l = L - 1; l >= 1; --l) {
    tsqr_form_kernel<<<ceil_div(nt[l], QW), QW * 32, 0, st>>>(M[l], ldm[l], rows[l], nt[l], jb, Tt[l], X, ldX);
    ttb_count();
    TTB_DBG(st, "tsqr form");
    X = M[l];
    ldX = ldm[l];
  }
  // R of the whole panel = R of the top level (rows 0..jb-1 of its storage, ld rt)
  tsqr_setup_kernel<<<1, 32, 0, st>>>(jb, P, ld, m, Tt[0], X, ldX, M[L], rt, tau, V, Tout, Z); ttb_count();
  TTB_DBG(st, "tsqr setup");
  tsqr_leaf_kernel<<<ceil_div(nt[0], QW), QW * 32, 0, st>>>(P, ld, m, nt[0], jb, Tt[0], X, ldX, Z, V);
  ttb_count();
  TTB_DBG(st, "tsqr leaf");
  return ttb_last_error();
}
