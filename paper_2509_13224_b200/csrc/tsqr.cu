// TSQR panel factorization for tall Householder panels (m x jb, jb <= 16, m in the millions).
//
// The blocked QR (qr.cu) needs, per NB-column panel, the LAPACK-style outputs of dgeqr2 +
// dlarft: Householder vectors V (unit lower trapezoidal, stored below the diagonal), R (on and
// above it), tau and the compact-WY factor T. A column-by-column panel over 1M rows is bound by
// one grid-wide reduction per column and by re-streaming the panel once per column. Here:
//
//   1. every warp factors one tile of <= 128 rows held in registers (4 rows per lane; the
//      column reductions are warp shuffles, T is built alongside in the dlarft recurrence);
//   2. the jb x jb R factors of all tiles are stacked and factored the same way, level by
//      level (8x fewer rows per level), until one tile is left;
//   3. the explicit orthonormal Q of the panel is formed top-down (Q_tile = H_tile [X; 0],
//      X = the tile's block of its parent's Q, applied in compact-WY form);
//   4. Householder reconstruction (Ballard, Demmel, Grigori, Jacquelin, Nguyen, Solomonik
//      2014): the LU factorization Y = [I; 0] - Q S = V U with the sign matrix S chosen on the
//      fly (pivots 1 + |q_kk| >= 1) gives V (= L), T = U L^{-T}, tau = diag(U), R = S R_tsqr.
//      The leaf pass of step 3 writes V_below = -Q_below S U^{-1} directly.
//
// Passes over the panel: read + write in step 1, read + write (P and the explicit V copy) in
// the leaf pass; everything else touches jb/8 of the rows or less.
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

// Sum each of the first n entries of z over the warp (butterfly; every lane gets the sums).
template <int N>
__device__ __forceinline__ void warp_sum_vec(double (&z)[NB], int n) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < N; ++c)
      if (c < n) z[c] += __shfl_xor_sync(0xffffffffu, z[c], o);
}

// Householder QR of every tile of an (rows x jb) col-major matrix M (in place: R on/above the
// diagonal, V below), T per tile (NB x NB row-major) and the tile's R into rows [t jb, t jb + jb)
// of S (col-major, ld ldS). JB > 0: compile-time panel width.
//
// One batched warp reduction per column: with x = A[j+1:, j] the statistics
// z_c = x^T A[j+1:, c] (c = j: ||x||^2; c > j: trailing columns; c < j: stored reflectors) give
// both the reflector application w_c = A[j, c] + scal z_c and the dlarft column
// v_b^T v_j = V[j, b] + scal z_b, and are accumulated while column j-1's update is applied.
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
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    z[c] = 0.0;
#pragma unroll
    for (int s = 0; s < TS; ++s) {
      const int i = lane + 32 * s;
      if (i > 0 && i < r && c < jb) z[c] += a[s][0] * a[s][c];
    }
  }
  warp_sum_vec<JB ? JB : NB>(z, jb);
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    if (j < jb) {
      double rowj[NB];  // row j of the tile (lane j, slot 0)
#pragma unroll
      for (int c = 0; c < NB; ++c) rowj[c] = (c < jb) ? __shfl_sync(0xffffffffu, a[0][c], j) : 0.0;
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
#pragma unroll
      for (int s = 0; s < TS; ++s) {
        const int i = lane + 32 * s;
        if (i >= j && i < r) {
          double vi = 1.0;
          if (i > j) { vi = a[s][j] * scal; a[s][j] = vi; }
#pragma unroll
          for (int c = 0; c < NB; ++c)
            if (c > j && c < jb) a[s][c] -= tj * vi * wv[c];
        }
      }
      if (lane == j) a[0][j] = beta;
      if (j + 1 < jb) {  // statistics of column j + 1
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          z[c] = 0.0;
#pragma unroll
          for (int s = 0; s < TS; ++s) {
            const int i = lane + 32 * s;
            if (i > j + 1 && i < r && c < jb) z[c] += a[s][j + 1] * a[s][c];
          }
        }
        warp_sum_vec<JB ? JB : NB>(z, jb);
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

// Q_tile = H_tile [X; 0] = [X; 0] - V (T (V_top^T X)) for every tile of a factored level.
// X = rows [t jb, t jb + jb) of the parent's Q (col-major, ld ldX), or the identity (top level).
// LEAF: instead of Q, write the reconstructed Householder vectors V = Q Z, Z = -S U^{-1}, of rows
// >= jb to M (below-diagonal storage) and to the explicit V copy Vx (col-major, ld rows).
template <bool LEAF>
__global__ void __launch_bounds__(QW * 32) tsqr_form_kernel(double* M, long long ld, long long rows, int nt, int jb,
                                                             const double* __restrict__ Tt, const double* X,
                                                             long long ldX, const double* __restrict__ Z,
                                                             double* Vx) {
  __shared__ double Vt[QW][NB * LDS];  // V_top, later W
  __shared__ double Xs[QW][NB * LDS];
  __shared__ double Ms[QW][NB * LDS];
  __shared__ double Zs[NB * LDS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (LEAF) {
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) Zs[(e / NB) * LDS + (e % NB)] = Z[e];
    __syncthreads();
  }
  const int t = blockIdx.x * QW + w;
  if (t >= nt) return;
  long long r0;
  int r;
  tile_bounds(rows, nt, t, r0, r);
  double* vt = Vt[w];
  double* xs = Xs[w];
  double* ms = Ms[w];
  // V_top (rows 0..NB-1 of the tile; explicit: unit diagonal, zeros above; rows >= jb meet X = 0)
  if (lane < NB)
#pragma unroll
    for (int c = 0; c < NB; ++c)
      vt[lane * LDS + c] = (c < jb && lane < r) ? (lane > c ? M[(long long)c * ld + r0 + lane] : (lane == c ? 1.0 : 0.0))
                                                : 0.0;
  for (int e = lane; e < NB * NB; e += 32) {
    const int i = e % NB, c = e / NB;
    double x = 0.0;
    if (i < jb && c < jb) x = X ? X[(long long)c * ldX + (long long)t * jb + i] : (i == c ? 1.0 : 0.0);
    xs[i * LDS + c] = x;
  }
  __syncwarp();
  const double* Tg = Tt + (long long)t * NB * NB;
  for (int e = lane; e < NB * NB; e += 32) {  // M1 = V_top^T X
    const int p = e / NB, c = e % NB;
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < NB; ++i) acc += vt[i * LDS + p] * xs[i * LDS + c];
    ms[p * LDS + c] = acc;
  }
  __syncwarp();
  for (int e = lane; e < NB * NB; e += 32) {  // W = T M1 (T upper)
    const int p = e / NB, c = e % NB;
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < NB; ++b) acc += (b >= p ? Tg[p * NB + b] : 0.0) * ms[b * LDS + c];
    vt[p * LDS + c] = acc;
  }
  __syncwarp();
  double v[TS][NB];
#pragma unroll
  for (int s = 0; s < TS; ++s) {
    const int i = lane + 32 * s;
#pragma unroll
    for (int c = 0; c < NB; ++c)
      v[s][c] = (c < jb && i < r) ? (i > c ? M[(long long)c * ld + r0 + i] : (i == c ? 1.0 : 0.0)) : 0.0;
  }
#pragma unroll
  for (int s = 0; s < TS; ++s) {
    const int i = lane + 32 * s;
    if (i >= r) continue;
    double q[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      double acc = (i < NB) ? xs[i * LDS + c] : 0.0;
#pragma unroll
      for (int p = 0; p < NB; ++p) acc -= v[s][p] * vt[p * LDS + c];
      q[c] = acc;
    }
    if (!LEAF) {
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c < jb) M[(long long)c * ld + r0 + i] = q[c];
    } else {
      if (r0 + i < jb) {  // top rows (R and L), prepared by the setup kernel behind Z
#pragma unroll
        for (int c = 0; c < NB; ++c)
          if (c < jb) M[(long long)c * ld + i] = Z[NB * NB + c * NB + i];
        continue;
      }
      // V row = -(q S) U^{-1} = q Z (Z from the setup kernel)
      double y[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int p = 0; p <= c; ++p) acc += q[p] * Zs[p * LDS + c];
        y[c] = acc;
      }
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c < jb) {
          M[(long long)c * ld + r0 + i] = y[c];
          Vx[(long long)c * rows + r0 + i] = y[c];
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
                                  double* tau, double* Vx, double* Tout, double* Z) {
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
    Z[NB * NB + c * NB + i] = (i <= c) ? sg[i] * Rt[(long long)c * jb + i] : L[i * LDS + c];  // P top block
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

int tiles_of(long long rows) { return (int)((rows + TR - 1) / TR); }

}  // namespace

// Workspace (doubles) for tsqr_panel on panels of up to m rows.
long long tsqr_workspace(long long m) {
  long long s = 3 * NB * NB + 128;
  long long rows = m;
  while (rows > TR) {
    const long long nt = (rows + TR - 1) / TR;
    s += nt * NB * NB;          // T per tile
    rows = nt * NB;
    s += rows * NB;             // stacked R of the next level
  }
  return s + NB * NB + 64;      // top level T
}

bool tsqr_applies(long long m, int jb) { return m > 8LL * TR && jb >= 1 && jb <= NB; }

// Factor the m x jb panel P (col-major, ld) in place with dgeqr2 conventions; tau[0..jb),
// explicit V (m x jb, ld m, unit diagonal, zeros above) and T (jb x jb row-major, upper).
int tsqr_panel(long long m, int jb, double* P, long long ld, double* tau, double* V, double* Tout, double* ws,
               cudaStream_t st) {
  constexpr int kMaxLevels = 16;
  double* US = ws;                  // Z = -S U^{-1} (NB x NB) | P top block (NB x NB, col-major)
  double* Rt = US + 2 * NB * NB;    // top-level R (jb x jb, ld jb)
  double* cur = Rt + NB * NB + 64;
  double* M[kMaxLevels];
  long long ldm[kMaxLevels], rows[kMaxLevels];
  double* Tt[kMaxLevels];
  int nt[kMaxLevels];
  int L = 0;
  M[0] = P; ldm[0] = ld; rows[0] = m;
  for (;;) {
    if (L + 1 >= kMaxLevels) return TTB_EARG;
    nt[L] = tiles_of(rows[L]);
    Tt[L] = cur;
    cur += (long long)nt[L] * NB * NB;
    if (nt[L] == 1) break;
    rows[L + 1] = (long long)nt[L] * jb;
    ldm[L + 1] = rows[L + 1];
    M[L + 1] = cur;
    cur += rows[L + 1] * NB;
    ++L;
  }
  for (int l = 0; l <= L; ++l) {
    double* S = (l == L) ? Rt : M[l + 1];
    const long long ldS = (l == L) ? jb : ldm[l + 1];
    if (jb == NB)
      tsqr_factor_kernel<NB><<<ceil_div(nt[l], FW), FW * 32, 0, st>>>(M[l], ldm[l], rows[l], nt[l], jb, Tt[l], S, ldS);
    else
      tsqr_factor_kernel<0><<<ceil_div(nt[l], FW), FW * 32, 0, st>>>(M[l], ldm[l], rows[l], nt[l], jb, Tt[l], S, ldS);
    ttb_count();
  }
  for (int l = L; l >= 1; --l) {
    const double* X = (l == L) ? nullptr : M[l + 1];
    const long long ldX = (l == L) ? 0 : ldm[l + 1];
    tsqr_form_kernel<false><<<ceil_div(nt[l], QW), QW * 32, 0, st>>>(M[l], ldm[l], rows[l], nt[l], jb, Tt[l], X, ldX,
                                                                     nullptr, nullptr);
    ttb_count();
  }
  tsqr_setup_kernel<<<1, 32, 0, st>>>(jb, P, ld, m, Tt[0], M[1], ldm[1], Rt, tau, V, Tout, US); ttb_count();
  tsqr_form_kernel<true><<<ceil_div(nt[0], QW), QW * 32, 0, st>>>(P, ld, m, nt[0], jb, Tt[0], M[1], ldm[1], US, V);
  ttb_count();
  return ttb_last_error();
}
