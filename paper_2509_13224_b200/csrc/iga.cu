// IGA kernels: B-spline/NURBS basis windows at Gauss points, the rational
// geometry map with its Jacobian / det J / metric factor R = J^-1 J^-T det J at
// cross-fiber multi-indices, the per-direction weighted mass/stiffness
// quadrature that turns a quadrature-grid TT core into a banded operator core,
// and the volume error integral.
#include "common.cuh"

namespace {

constexpr int PMAX = 8;

// ---------------------------------------------------------------------------
// Cox-de Boor (NURBS Book A2.2/A2.3) for one parameter; reference splines.py:146-221.
// One thread per quadrature point; the (p+1)-long value / derivative records of the CTA's 128 points are
// staged in shared memory and written as one contiguous, coalesced range per table (a thread-strided
// store of (p+1)-records would touch p+1 times the sectors per instruction).
constexpr int BASIS_T = 128;
__global__ void __launch_bounds__(BASIS_T) basis_kernel(int nq, const double* __restrict__ x, const double* __restrict__ t,
                                                        int nk, int p, const double* __restrict__ w, int* first,
                                                        double* V, double* D, int* bad) {
  __shared__ double sV[BASIS_T * (PMAX + 1)], sD[BASIS_T * (PMAX + 1)];
  const int q0 = blockIdx.x * BASIS_T;
  const int q = q0 + threadIdx.x;
  const int cnt = min(BASIS_T, nq - q0) * (p + 1);
  const long long base = (long long)q0 * (p + 1);
  auto flush = [&]() {
    __syncthreads();
    for (int e = threadIdx.x; e < cnt; e += BASIS_T) {
      V[base + e] = sV[e];
      D[base + e] = sD[e];
    }
  };
  const double xq = q < nq ? x[q] : t[0];
  const bool ok = q < nq && xq >= t[0] && xq <= t[nk - 1];
  if (q < nq && !ok) atomicMin(bad, q);
  const double xv = ok ? xq : t[0];   // out-of-range points: evaluated at t[0], records zeroed below
  const int nb = nk - p - 1;
  int k;
  if (xv >= t[nb]) {
    k = nb - 1;
    while (t[k] == t[k + 1]) --k;
  } else {  // last i with t[i] <= x
    int lo = 0, hi = nk - 1;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (t[mid] <= xv) lo = mid; else hi = mid;
    }
    k = lo;
  }
  double N[PMAX + 1], low[PMAX + 1];
  N[0] = 1.0;
  low[0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    if (j == p)
      for (int r = 0; r < p; ++r) low[r] = N[r];
    double carry = 0.0;
    for (int r = 0; r < j; ++r) {
      const double a = xv - t[k + 1 - j + r];
      const double b = t[k + 1 + r] - xv;
      const double den = a + b;
      const double qq = den != 0.0 ? N[r] / den : 0.0;
      N[r] = carry + b * qq;
      carry = a * qq;
    }
    N[j] = carry;
  }
  double dN[PMAX + 1];
  for (int j = 0; j <= p; ++j) {
    double acc = 0.0;
    if (p > 0) {
      const int i = k - p + j;
      if (j > 0) {
        double den = t[i + p] - t[i];
        if (den != 0.0) acc += p / den * low[j - 1];
      }
      if (j < p) {
        double den = t[i + p + 1] - t[i + 1];
        if (den != 0.0) acc -= p / den * low[j];
      }
    }
    dN[j] = acc;
  }
  if (w) {
    double W = 0.0, dW = 0.0;
    for (int j = 0; j <= p; ++j) { W += N[j] * w[k - p + j]; dW += dN[j] * w[k - p + j]; }
    for (int j = 0; j <= p; ++j) {
      const double wj = w[k - p + j];
      const double v = N[j] * wj / W;
      const double d = (dN[j] * wj * W - N[j] * wj * dW) / (W * W);
      N[j] = v;
      dN[j] = d;
    }
  }
  if (q < nq) first[q] = k - p;
  for (int j = 0; j <= p; ++j) {
    sV[threadIdx.x * (p + 1) + j] = ok ? N[j] : 0.0;
    sD[threadIdx.x * (p + 1) + j] = ok ? dN[j] : 0.0;
  }
  flush();
}

// ---------------------------------------------------------------------------
struct GeoArgs {
  const int* first[3];
  const double* V[3];
  const double* D[3];
  int p[3];
  int n[3];
  const double* cw;  // (n0, n1, n2, 4): w*x, w*y, w*z, w
  double sing_tol;
};

struct GeoOut {
  double J[3][3];
  double x[3];
  double det;
};

__device__ __forceinline__ void geo_point(const GeoArgs& g, int q0, int q1, int q2, GeoOut& o) {
  const int f0 = g.first[0][q0], f1 = g.first[1][q1], f2 = g.first[2][q2];
  const int p0 = g.p[0] + 1, p1 = g.p[1] + 1, p2 = g.p[2] + 1;
  const double* V0 = g.V[0] + (long long)q0 * p0;
  const double* D0 = g.D[0] + (long long)q0 * p0;
  const double* V1 = g.V[1] + (long long)q1 * p1;
  const double* D1 = g.D[1] + (long long)q1 * p1;
  const double* V2 = g.V[2] + (long long)q2 * p2;
  const double* D2 = g.D[2] + (long long)q2 * p2;
  // sums over the window: value, d/dxi0, d/dxi1, d/dxi2 of (wx, wy, wz, w)
  double S[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) S[a][b] = 0.0;
  for (int a = 0; a < p0; ++a) {
    const double va = V0[a], da = D0[a];
    double T[3][4];  // after contracting b,c: [v2v1, v2d1, d2v1] x 4 comps... accumulate directly
#pragma unroll
    for (int u = 0; u < 3; ++u)
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) T[u][cc] = 0.0;
    for (int b = 0; b < p1; ++b) {
      const double vb = V1[b], db = D1[b];
      double R0[4] = {0, 0, 0, 0}, R2[4] = {0, 0, 0, 0};
      const double* row = g.cw + (((long long)(f0 + a) * g.n[1] + (f1 + b)) * g.n[2] + f2) * 4;
      for (int c = 0; c < p2; ++c) {
        const double2 lo = *reinterpret_cast<const double2*>(row + 4 * c);
        const double2 hi = *reinterpret_cast<const double2*>(row + 4 * c + 2);
        const double vc = V2[c], dc = D2[c];
        R0[0] += vc * lo.x; R0[1] += vc * lo.y; R0[2] += vc * hi.x; R0[3] += vc * hi.y;
        R2[0] += dc * lo.x; R2[1] += dc * lo.y; R2[2] += dc * hi.x; R2[3] += dc * hi.y;
      }
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        T[0][cc] += vb * R0[cc];
        T[1][cc] += db * R0[cc];
        T[2][cc] += vb * R2[cc];
      }
    }
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      S[0][cc] += va * T[0][cc];
      S[1][cc] += da * T[0][cc];
      S[2][cc] += va * T[1][cc];
      S[3][cc] += va * T[2][cc];
    }
  }
  const double den = S[0][3];
  const double inv2 = 1.0 / (den * den);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    o.x[c] = S[0][c] / den;
#pragma unroll
    for (int e = 0; e < 3; ++e) o.J[c][e] = (S[1 + e][c] * den - S[0][c] * S[1 + e][3]) * inv2;
  }
  const double(*J)[3] = o.J;
  o.det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
          J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
}

__device__ __forceinline__ void metric_from(const GeoOut& o, double R[3][3]) {
  const double(*J)[3] = o.J;
  double A[3][3];  // adjugate: inv = A / det
  A[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  A[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
  A[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
  A[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  A[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
  A[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
  A[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  A[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
  A[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  const double id = 1.0 / o.det;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) R[i][j] = (A[i][0] * A[j][0] + A[i][1] * A[j][1] + A[i][2] * A[j][2]) * id;
}

__device__ __forceinline__ double source_fn(int id, const double* x) {
  const double PI = 3.141592653589793;
  switch (id) {
    case 0: return 0.0;
    case 1: return 1.0;
    case 2: return sin(PI * x[0]) * sin(PI * x[1]);
    case 3: return sin(PI * x[0]) * sin(PI * x[1]) * sin(PI * x[2]);
    case 4: return 3.0 * PI * PI * sin(PI * x[0]) * sin(PI * x[1]) * sin(PI * x[2]);
    case 5: {
      const double e = exp(x[0] + x[1] + x[2]);
      const double s0 = sin(PI * x[0]), s1 = sin(PI * x[1]), s2 = sin(PI * x[2]);
      const double c0 = cos(PI * x[0]), c1 = cos(PI * x[1]), c2 = cos(PI * x[2]);
      const double S = s0 * s1 * s2, mix = c0 * s1 * s2 + s0 * c1 * s2 + s0 * s1 * c2;
      return -e * ((3.0 - 3.0 * PI * PI) * S + 2.0 * PI * mix);
    }
  }
  return 0.0;
}

// analytic solutions: 0 lshape_exact, 1 cube_sines, 2 ring_radial(prm: u_in,u_out,r_in,r_out), 3 exp_sines
__device__ __forceinline__ double exact_fn(int id, const double* x, const double* prm) {
  const double PI = 3.141592653589793;
  switch (id) {
    case 0: return sin(PI * x[0]) * sin(PI * x[1]) / (2.0 * PI * PI);
    case 1: return sin(PI * x[0]) * sin(PI * x[1]) * sin(PI * x[2]);
    case 2: {
      const double r = hypot(x[0], x[1]);
      return (prm[0] * log(prm[3] / r) + prm[1] * log(r / prm[2])) / log(prm[3] / prm[2]);
    }
    case 3: return exp(x[0] + x[1] + x[2]) * sin(PI * x[0]) * sin(PI * x[1]) * sin(PI * x[2]);
  }
  return 0.0;
}

// mode 0: R[ri][rj]; 1: f(x) det; 2: full record (J9, x3, det, R9) stride 22; 3: x only (stride 3)
__global__ void geo_kernel(GeoArgs g, long long N, const long long* __restrict__ idx, int mode, int ri, int rj, int src,
                           double* out, long long* bad) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < N; k += (long long)gridDim.x * blockDim.x) {
    const int q0 = (int)idx[3 * k], q1 = (int)idx[3 * k + 1], q2 = (int)idx[3 * k + 2];
    GeoOut o;
    geo_point(g, q0, q1, q2, o);
    if (mode == 3) {
      out[3 * k] = o.x[0]; out[3 * k + 1] = o.x[1]; out[3 * k + 2] = o.x[2];
      continue;
    }
    if (mode != 1 && fabs(o.det) < g.sing_tol) {
      atomicMin((unsigned long long*)bad, (unsigned long long)k);
      if (mode == 0) { out[k] = 0.0; continue; }
    }
    if (mode == 1) {
      out[k] = source_fn(src, o.x) * o.det;
    } else if (mode == 0) {
      double R[3][3];
      metric_from(o, R);
      out[k] = R[ri][rj];
    } else {
      double* r = out + 22 * k;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) r[3 * a + b] = o.J[a][b];
      r[9] = o.x[0]; r[10] = o.x[1]; r[11] = o.x[2];
      r[12] = o.det;
      double R[3][3];
      metric_from(o, R);
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) r[13 + 3 * a + b] = R[a][b];
    }
  }
}

// ---------------------------------------------------------------------------
// Per-direction 1D weighted quadrature of a quadrature-grid TT core (reference assembly.py:208-233):
//   operator core (banded): out[a, i, t, b] = sum_{q: f_q <= min(i,j), f_q >= max(i,j) - p} G[a,q,b] w[q] X[q,i-f_q] Y[q,j-f_q],
//                           j = i + t - h;
//   load core:              out[a, i, b]    = sum_{q: i - p <= f_q <= i} G[a,q,b] w[q] V[q,i-f_q].
// f_q (the first basis index of q's element) is non-decreasing in q, so every sum runs over a contiguous
// q range. One CTA owns one rank index a and a tile of QT_I consecutive basis indices i: it stages the
// tile's quadrature window of G (the contiguous rows G[a, qlo:qhi, :]), the weights, the basis tables
// and the per-index range starts/ends in shared memory, then every output is reduced by a group of
// QT_L lanes (strided over the range, combined with warp shuffles). The outputs of a tile are one
// contiguous run of QT_I (2h+1) s doubles.
constexpr int QT_T = 256;   // threads per CTA
constexpr int QT_L = 4;     // lanes per output (shuffle-reduced)
constexpr int QT_SMEM = 96 * 1024;

__device__ __forceinline__ int lower_bound_first(const int* f, int lo, int hi, int v) {  // first q with f[q] >= v
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (f[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Stages the tile's window (q in [qlo, qlo + nw)) in shared memory, or -- when nw exceeds the staging
// capacity `cap` (a knot vector with very uneven elements) -- points the same views at global memory.
// rb/re (per basis index k = i0 - h + e of the extended tile): the window-relative q range whose
// first index satisfies k - p <= f_q <= k.
__device__ __forceinline__ void qt_stage(int s, int p, int h, int i0, int ni, int cap, const int* __restrict__ first,
                                         const double* __restrict__ Ga, const double* __restrict__ w,
                                         const double* __restrict__ X, const double* __restrict__ Y, char* sm,
                                         int qlo, int nw, const double*& Gs, const double*& ws, const double*& Xs,
                                         const double*& Ys, const int*& fs, int*& rb, int*& re) {
  const int P1 = p + 1;
  const int next = ni + 2 * h;
  rb = reinterpret_cast<int*>(sm);
  re = rb + next;
  if (nw <= cap) {
    double* g = reinterpret_cast<double*>(sm + (((2 * next * 4) + 15) & ~15));
    double* wv = g + (long long)nw * s;
    double* xv = wv + nw;
    double* yv = xv + nw * P1;
    int* fv = reinterpret_cast<int*>(yv + (Y ? nw * P1 : 0));
    // G rows qlo..qlo+nw-1 of rank a: one contiguous run (16-byte vector loads when aligned)
    const long long tot = (long long)nw * s;
    const double* src = Ga + (long long)qlo * s;
    if ((((uintptr_t)src) & 15) == 0) {
      const double2* s2 = reinterpret_cast<const double2*>(src);
      double2* d2 = reinterpret_cast<double2*>(g);
      for (long long e = threadIdx.x; e < tot / 2; e += QT_T) d2[e] = __ldg(s2 + e);
      if ((tot & 1) && threadIdx.x == 0) g[tot - 1] = __ldg(src + tot - 1);
    } else {
      for (long long e = threadIdx.x; e < tot; e += QT_T) g[e] = __ldg(src + e);
    }
    for (int e = threadIdx.x; e < nw; e += QT_T) {
      wv[e] = w[qlo + e];
      fv[e] = first[qlo + e];
    }
    for (int e = threadIdx.x; e < nw * P1; e += QT_T) {
      xv[e] = X[(long long)qlo * P1 + e];
      if (Y) yv[e] = Y[(long long)qlo * P1 + e];
    }
    Gs = g; ws = wv; Xs = xv; Ys = yv; fs = fv;
  } else {
    Gs = Ga + (long long)qlo * s;
    ws = w + qlo;
    Xs = X + (long long)qlo * P1;
    Ys = Y ? Y + (long long)qlo * P1 : nullptr;
    fs = first + qlo;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < next; e += QT_T) {
    const int k = i0 - h + e;
    rb[e] = lower_bound_first(fs, 0, nw, k - p);
    re[e] = lower_bound_first(fs, 0, nw, k + 1);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(QT_T) op_core_kernel(int r, int nq, int s, const double* __restrict__ G,
                                                       const double* __restrict__ w, const int* __restrict__ first,
                                                       const double* __restrict__ X, const double* __restrict__ Y,
                                                       int p, int n, int h, int ti, int cap, double* out) {
  extern __shared__ __align__(16) char qsm[];
  const int a = blockIdx.y;
  const int i0 = blockIdx.x * ti, ni = min(ti, n - i0);
  const int B = 2 * h + 1, P1 = p + 1;
  // quadrature window of the tile: q with f_q in [i0 - p, i0 + ni - 1]
  const int qlo = lower_bound_first(first, 0, nq, i0 - p);
  const int qhi = lower_bound_first(first, qlo, nq, i0 + ni);
  const int nw = qhi - qlo;
  const double *Gs, *ws, *Xs, *Ys;
  const int* fs;
  int *rb, *re;
  qt_stage(s, p, h, i0, ni, cap, first, G + (long long)a * nq * s, w, X, Y, qsm, qlo, nw, Gs, ws, Xs, Ys, fs, rb, re);
  const int lane = threadIdx.x & (QT_L - 1);
  const long long nout = (long long)ni * B * s;
  double* o = out + (((long long)a * n + i0) * B) * s;
  // one output per group of QT_L lanes; all lanes of a warp stay in the loop (shuffles)
  for (long long g0 = threadIdx.x / QT_L; g0 < (nout + QT_T / QT_L - 1) / (QT_T / QT_L) * (QT_T / QT_L);
       g0 += QT_T / QT_L) {
    double acc = 0.0;
    if (g0 < nout) {
      const int b = (int)(g0 % s);
      const long long rest = g0 / s;
      const int t = (int)(rest % B), ii = (int)(rest / B);
      const int i = i0 + ii, j = i + t - h;
      if (j >= 0 && j < n) {
        const int lo = rb[max(i, j) - i0 + h], hi = re[min(i, j) - i0 + h];
        for (int q = lo + lane; q < hi; q += QT_L) {
          const int f = fs[q];
          acc += Gs[(long long)q * s + b] * ws[q] * Xs[q * P1 + (i - f)] * Ys[q * P1 + (j - f)];
        }
      }
    }
#pragma unroll
    for (int m = QT_L / 2; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m, QT_L);
    if (lane == 0 && g0 < nout) o[g0] = acc;
  }
}

__global__ void __launch_bounds__(QT_T) vec_core_kernel(int r, int nq, int s, const double* __restrict__ G,
                                                        const double* __restrict__ w, const int* __restrict__ first,
                                                        const double* __restrict__ V, int p, int n, int ti,
                                                        int cap, double* out) {
  extern __shared__ __align__(16) char qsm[];
  const int a = blockIdx.y;
  const int i0 = blockIdx.x * ti, ni = min(ti, n - i0);
  const int P1 = p + 1;
  const int qlo = lower_bound_first(first, 0, nq, i0 - p);
  const int qhi = lower_bound_first(first, qlo, nq, i0 + ni);
  const int nw = qhi - qlo;
  const double *Gs, *ws, *Xs, *Ys;
  const int* fs;
  int *rb, *re;
  qt_stage(s, p, 0, i0, ni, cap, first, G + (long long)a * nq * s, w, V, nullptr, qsm, qlo, nw, Gs, ws, Xs, Ys, fs, rb,
           re);
  const int lane = threadIdx.x & (QT_L - 1);
  const long long nout = (long long)ni * s;
  double* o = out + ((long long)a * n + i0) * s;
  for (long long g0 = threadIdx.x / QT_L; g0 < (nout + QT_T / QT_L - 1) / (QT_T / QT_L) * (QT_T / QT_L);
       g0 += QT_T / QT_L) {
    double acc = 0.0;
    if (g0 < nout) {
      const int b = (int)(g0 % s), ii = (int)(g0 / s);
      const int i = i0 + ii;
      const int lo = rb[ii], hi = re[ii];
      for (int q = lo + lane; q < hi; q += QT_L) acc += Gs[(long long)q * s + b] * ws[q] * Xs[q * P1 + (i - fs[q])];
    }
#pragma unroll
    for (int m = QT_L / 2; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m, QT_L);
    if (lane == 0 && g0 < nout) o[g0] = acc;
  }
}

// Launch geometry: tile width ti from the mean points per element g = ceil(nq / (n - p)) (exact for
// knot vectors without repeated interior knots), so a tile's window of <= (ti + p) elements fits the
// staging budget; cap = window rows the dynamic shared memory actually holds (larger windows read G
// from global memory in place).
struct QtLaunch {
  int ti, cap;
  size_t smem;
};

__host__ QtLaunch qt_launch(int nq, int s, int p, int n, int h, bool two_tables) {
  const int nel = n - p > 0 ? n - p : 1;
  const int g = (nq + nel - 1) / nel;
  const long long row = 8LL * s + 8 + 8LL * (p + 1) * (two_tables ? 2 : 1) + 4;
  QtLaunch L{1, 0, 0};
  for (int ti = 64; ti >= 1; ti >>= 1) {
    const long long rows = (long long)(ti + p) * g;
    const long long bytes = 16 + 8LL * (ti + 2 * h) + rows * row + 64;
    if (bytes <= QT_SMEM || ti == 1) {
      L.ti = ti;
      L.cap = (int)((QT_SMEM - 16 - 8LL * (ti + 2 * h) - 64) / row);
      if (L.cap < 0) L.cap = 0;
      L.smem = (size_t)QT_SMEM;
      break;
    }
  }
  return L;
}

// previous thread-per-output kernels (any layout of `first`; used when one element holds more points
// than the staging budget allows)
__global__ void op_core_flat_kernel(int r, int nq, int s, const double* __restrict__ G, const double* __restrict__ w,
                                    const int* __restrict__ first, const double* __restrict__ X,
                                    const double* __restrict__ Y, int p, int n, int h, double* out) {
  const int B = 2 * h + 1;
  const long long tot = (long long)r * n * B * s;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e % s);
    long long rest = e / s;
    const int t = (int)(rest % B);
    rest /= B;
    const int i = (int)(rest % n);
    const int a = (int)(rest / n);
    const int j = i + t - h;
    double acc = 0.0;
    if (j >= 0 && j < n) {
      const int lo = lower_bound_first(first, 0, nq, max(i, j) - p);
      for (int q = lo; q < nq; ++q) {
        const int f = first[q];
        if (f > min(i, j)) break;
        acc += G[((long long)a * nq + q) * s + b] * w[q] * X[(long long)q * (p + 1) + (i - f)] *
               Y[(long long)q * (p + 1) + (j - f)];
      }
    }
    out[e] = acc;
  }
}

__global__ void vec_core_flat_kernel(int r, int nq, int s, const double* __restrict__ G, const double* __restrict__ w,
                                     const int* __restrict__ first, const double* __restrict__ V, int p, int n,
                                     double* out) {
  const long long tot = (long long)r * n * s;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e % s);
    const int i = (int)((e / s) % n);
    const int a = (int)(e / ((long long)s * n));
    double acc = 0.0;
    const int lo = lower_bound_first(first, 0, nq, i - p);
    for (int q = lo; q < nq; ++q) {
      const int f = first[q];
      if (f > i) break;
      acc += G[((long long)a * nq + q) * s + b] * w[q] * V[(long long)q * (p + 1) + (i - f)];
    }
    out[e] = acc;
  }
}

// field tables: T[a, q, b] = sum_k u[a, first[q]+k, b] V[q, k]
__global__ void field_table_kernel(int r, int n, int s, const double* __restrict__ u, int nq,
                                   const int* __restrict__ first, const double* __restrict__ V, int p, double* T) {
  const long long tot = (long long)r * nq * s;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e % s);
    const int q = (int)((e / s) % nq);
    const int a = (int)(e / ((long long)s * nq));
    double acc = 0.0;
    for (int k = 0; k <= p; ++k) acc += u[((long long)a * n + first[q] + k) * s + b] * V[(long long)q * (p + 1) + k];
    T[e] = acc;
  }
}

// error integral: one CTA per (q0, q1); partial (num, den) per CTA
__global__ void l1err_kernel(GeoArgs g, int nq0, int nq1, int nq2, const double* __restrict__ U0, int r1,
                             const double* __restrict__ U1, int r2, const double* __restrict__ U2,
                             const double* __restrict__ w0, const double* __restrict__ w1,
                             const double* __restrict__ w2, int exact_id, const double* __restrict__ prm,
                             double* part) {
  extern __shared__ double Tsh[];  // r2
  __shared__ double red[32];
  const int q0 = blockIdx.x / nq1, q1 = blockIdx.x % nq1;
  for (int c = threadIdx.x; c < r2; c += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < r1; ++b) s += U0[(long long)q0 * r1 + b] * U1[((long long)b * nq1 + q1) * r2 + c];
    Tsh[c] = s;
  }
  __syncthreads();
  double num = 0.0, den = 0.0;
  const double w01 = w0[q0] * w1[q1];
  for (int q2 = threadIdx.x; q2 < nq2; q2 += blockDim.x) {
    double u = 0.0;
    for (int c = 0; c < r2; ++c) u += Tsh[c] * U2[(long long)c * nq2 + q2];
    GeoOut o;
    geo_point(g, q0, q1, q2, o);
    const double ue = exact_id < 0 ? prm[((long long)q0 * nq1 + q1) * nq2 + q2] : exact_fn(exact_id, o.x, prm);
    const double wd = w01 * w2[q2] * o.det;
    num += wd * fabs(u - ue);
    den += wd * fabs(ue);
  }
  num = block_sum(num, red);
  den = block_sum(den, red);
  if (threadIdx.x == 0) {
    part[2 * (long long)blockIdx.x] = num;
    part[2 * (long long)blockIdx.x + 1] = den;
  }
}

__global__ void pair_sum_kernel(long long np, const double* part, double* out) {
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  for (long long i = threadIdx.x; i < np; i += blockDim.x) { a += part[2 * i]; b += part[2 * i + 1]; }
  a = block_sum(a, red);
  b = block_sum(b, red);
  if (threadIdx.x == 0) { out[0] = a; out[1] = b; }
}

int grid_for(long long tot, int threads = 256) {
  long long b = (tot + threads - 1) / threads;
  if (b > (long long)ttb_num_sms() * 16) b = (long long)ttb_num_sms() * 16;
  if (b < 1) b = 1;
  return (int)b;
}

GeoArgs make_geo(const int* const* first, const double* const* V, const double* const* D, const int* p, const int* n,
                 const double* cw, double sing_tol) {
  GeoArgs g;
  for (int d = 0; d < 3; ++d) {
    g.first[d] = first[d];
    g.V[d] = V[d];
    g.D[d] = D[d];
    g.p[d] = p[d];
    g.n[d] = n[d];
  }
  g.cw = cw;
  g.sing_tol = sing_tol;
  return g;
}

}  // namespace

// Basis windows at nq parameters. bad: device int (init INT_MAX) receives the first out-of-range index.
TTB_API int ttb_basis_eval(void* stream, int nq, const double* x, const double* knots, int nk, int p,
                           const double* weights, int* first, double* V, double* D, int* bad) {
  if (p < 0 || p > PMAX || nk < 2 * p + 2) return TTB_EARG;
  if (nq == 0) return TTB_OK;
  basis_kernel<<<ceil_div(nq, BASIS_T), BASIS_T, 0, as_stream(stream)>>>(nq, x, knots, nk, p, weights, first, V, D, bad);
  ttb_count();
  return ttb_last_error();
}

// Geometry evaluation at N grid multi-indices (int64 N x 3). tables: per-direction first/V/D of the
// geometry bases at the grid axes. bad: device int64 (init INT64_MAX) <- first singular row.
TTB_API int ttb_geo_eval(void* stream, long long N, const long long* idx, const int* f0, const int* f1, const int* f2,
                         const double* V0, const double* V1, const double* V2, const double* D0, const double* D1,
                         const double* D2, int p0, int p1, int p2, int n0, int n1, int n2, const double* cw,
                         double sing_tol, int mode, int ri, int rj, int src, double* out, long long* bad) {
  if (N == 0) return TTB_OK;
  const int* f[3] = {f0, f1, f2};
  const double* V[3] = {V0, V1, V2};
  const double* D[3] = {D0, D1, D2};
  int p[3] = {p0, p1, p2}, n[3] = {n0, n1, n2};
  GeoArgs g = make_geo(f, V, D, p, n, cw, sing_tol);
  geo_kernel<<<grid_for(N, 128), 128, 0, as_stream(stream)>>>(g, N, idx, mode, ri, rj, src, out, bad); ttb_count();
  return ttb_last_error();
}

// min det J over the full tensor grid n0 x n1 x n2 (and the count of det J <= 0): the admissibility
// check of seeded random geometries at every Gauss point of the solve (8.4e9 points at configs[3]).
// One thread per point, grid-stride; min as an order-preserving 64-bit key.
__device__ __forceinline__ unsigned long long dkey(double d) {
  const long long b = __double_as_longlong(d);
  return b >= 0 ? ((unsigned long long)b ^ 0x8000000000000000ULL) : ~(unsigned long long)b;
}
__global__ void __launch_bounds__(256) min_det_kernel(GeoArgs g, int n0, int n1, int n2, unsigned long long* minkey,
                                                      unsigned long long* count) {
  const long long N = (long long)n0 * n1 * n2;
  double mn = 1.0e308;
  unsigned long long cnt = 0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < N; k += (long long)gridDim.x * blockDim.x) {
    const int q2 = (int)(k % n2);
    const long long t = k / n2;
    const int q1 = (int)(t % n1), q0 = (int)(t / n1);
    GeoOut o;
    geo_point(g, q0, q1, q2, o);
    mn = fmin(mn, o.det);
    cnt += (o.det <= 0.0);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, off));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(minkey, dkey(mn));
    if (cnt) atomicAdd(count, cnt);
  }
}

// Sum-factorized variant (n2 <= 64 control points in the last direction): one warp per (q0, q1) line
// contracts the first two directions once -- W_v[c][comp] = sum_{a,b} X0_a X1_b cw[f0+a][f1+b][c][comp]
// for (X0, X1) = (N0, N1), (D0, N1), (N0, D1) over every c -- and then every point of the line needs
// only (p2 + 1) terms per quantity: ~90 FMA per point instead of the ~1000 FMA and 2 KB of window loads
// of geo_point (1.47 s -> ~0.1 s for the 8.4e9-point configs[3] grid).
constexpr int MD_MAXC = 64;
__global__ void __launch_bounds__(256) min_det_sf_kernel(GeoArgs g, int n0q, int n1q, int n2q, unsigned long long* minkey,
                                                         unsigned long long* count) {
  __shared__ double Wsh[8][3][MD_MAXC * 4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long lines = (long long)n0q * n1q;
  const int nc = g.n[2];
  const int p0 = g.p[0] + 1, p1 = g.p[1] + 1, p2 = g.p[2] + 1;
  double mn = 1.0e308;
  unsigned long long cnt = 0;
  double (*W)[MD_MAXC * 4] = Wsh[w];
  for (long long line = blockIdx.x * 8LL + w; line < lines; line += (long long)gridDim.x * 8) {
    const int q0 = (int)(line / n1q), q1 = (int)(line % n1q);
    const int f0 = g.first[0][q0], f1 = g.first[1][q1];
    const double* V0 = g.V[0] + (long long)q0 * p0;
    const double* D0 = g.D[0] + (long long)q0 * p0;
    const double* V1 = g.V[1] + (long long)q1 * p1;
    const double* D1 = g.D[1] + (long long)q1 * p1;
    for (int e = lane; e < nc * 4; e += 32) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int a = 0; a < p0; ++a) {
        const double va = V0[a], da = D0[a];
        double t0 = 0.0, t1 = 0.0;
        for (int b = 0; b < p1; ++b) {
          const double x = g.cw[((long long)(f0 + a) * g.n[1] + (f1 + b)) * nc * 4 + e];
          t0 += V1[b] * x;
          t1 += D1[b] * x;
        }
        s0 += va * t0;
        s1 += da * t0;
        s2 += va * t1;
      }
      W[0][e] = s0;
      W[1][e] = s1;
      W[2][e] = s2;
    }
    __syncwarp();
    for (int q2 = lane; q2 < n2q; q2 += 32) {
      const int f2 = g.first[2][q2];
      const double* V2 = g.V[2] + (long long)q2 * p2;
      const double* D2 = g.D[2] + (long long)q2 * p2;
      double S[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) S[u][cc] = 0.0;
      for (int c = 0; c < p2; ++c) {
        const double vc = V2[c], dc = D2[c];
        const double* w0 = W[0] + (f2 + c) * 4;
        const double* w1 = W[1] + (f2 + c) * 4;
        const double* w2 = W[2] + (f2 + c) * 4;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          S[0][cc] += vc * w0[cc];
          S[1][cc] += vc * w1[cc];
          S[2][cc] += vc * w2[cc];
          S[3][cc] += dc * w0[cc];
        }
      }
      const double den = S[0][3];
      const double inv2 = 1.0 / (den * den);
      double J[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int e = 0; e < 3; ++e) J[c][e] = (S[1 + e][c] * den - S[0][c] * S[1 + e][3]) * inv2;
      const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      mn = fmin(mn, det);
      cnt += (det <= 0.0);
    }
    __syncwarp();
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, off));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  }
  if (lane == 0) {
    atomicMin(minkey, dkey(mn));
    if (cnt) atomicAdd(count, cnt);
  }
}

TTB_API int ttb_geo_min_det(void* stream, int nq0, int nq1, int nq2, const int* f0, const int* f1, const int* f2,
                            const double* V0, const double* V1, const double* V2, const double* D0, const double* D1,
                            const double* D2, int p0, int p1, int p2, int n0, int n1, int n2, const double* cw,
                            unsigned long long* out) {
  if (nq0 < 1 || nq1 < 1 || nq2 < 1 || !out) return TTB_EARG;
  const int* f[3] = {f0, f1, f2};
  const double* V[3] = {V0, V1, V2};
  const double* D[3] = {D0, D1, D2};
  int p[3] = {p0, p1, p2}, n[3] = {n0, n1, n2};
  GeoArgs g = make_geo(f, V, D, p, n, cw, 0.0);
  cudaStream_t st = as_stream(stream);
  const unsigned long long init[2] = {~0ULL, 0ULL};
  cudaMemcpyAsync(out, init, sizeof(init), cudaMemcpyHostToDevice, st);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long N = (long long)nq0 * nq1 * nq2;
  if (n2 <= MD_MAXC) {
    long long blocks = ((long long)nq0 * nq1 + 7) / 8;
    if (blocks > 16LL * sms) blocks = 16LL * sms;
    min_det_sf_kernel<<<(unsigned)blocks, 256, 0, st>>>(g, nq0, nq1, nq2, out, out + 1); ttb_count();
    return ttb_last_error();
  }
  long long blocks = (N + 255) / 256;
  if (blocks > 8LL * sms) blocks = 8LL * sms;
  min_det_kernel<<<(unsigned)blocks, 256, 0, st>>>(g, nq0, nq1, nq2, out, out + 1); ttb_count();
  return ttb_last_error();
}

TTB_API int ttb_op_core(void* stream, int r, int nq, int s, const double* G, const double* w, const int* first,
                        const double* X, const double* Y, int p, int n, int h, double* out) {
  long long tot = (long long)r * n * (2 * h + 1) * s;
  if (tot == 0) return TTB_OK;
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(op_core_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, QT_SMEM);
    cudaFuncSetAttribute(vec_core_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, QT_SMEM);
    cfg = true;
  }
  const QtLaunch L = qt_launch(nq, s, p, n, h, true);
  op_core_kernel<<<dim3(ceil_div(n, L.ti), r), QT_T, L.smem, as_stream(stream)>>>(r, nq, s, G, w, first, X, Y, p, n, h,
                                                                                  L.ti, L.cap, out); ttb_count();
  return ttb_last_error();
}

TTB_API int ttb_vec_core(void* stream, int r, int nq, int s, const double* G, const double* w, const int* first,
                         const double* V, int p, int n, double* out) {
  long long tot = (long long)r * n * s;
  if (tot == 0) return TTB_OK;
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(vec_core_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, QT_SMEM);
    cfg = true;
  }
  const QtLaunch L = qt_launch(nq, s, p, n, 0, false);
  vec_core_kernel<<<dim3(ceil_div(n, L.ti), r), QT_T, L.smem, as_stream(stream)>>>(r, nq, s, G, w, first, V, p, n, L.ti,
                                                                                   L.cap, out); ttb_count();
  return ttb_last_error();
}

// Previous thread-per-output kernels (tools/bench comparisons only).
TTB_API int ttb_op_core_flat(void* stream, int r, int nq, int s, const double* G, const double* w, const int* first,
                             const double* X, const double* Y, int p, int n, int h, double* out) {
  long long tot = (long long)r * n * (2 * h + 1) * s;
  if (tot == 0) return TTB_OK;
  op_core_flat_kernel<<<grid_for(tot), 256, 0, as_stream(stream)>>>(r, nq, s, G, w, first, X, Y, p, n, h, out); ttb_count();
  return ttb_last_error();
}

TTB_API int ttb_vec_core_flat(void* stream, int r, int nq, int s, const double* G, const double* w, const int* first,
                              const double* V, int p, int n, double* out) {
  long long tot = (long long)r * n * s;
  if (tot == 0) return TTB_OK;
  vec_core_flat_kernel<<<grid_for(tot), 256, 0, as_stream(stream)>>>(r, nq, s, G, w, first, V, p, n, out); ttb_count();
  return ttb_last_error();
}

TTB_API int ttb_field_table(void* stream, int r, int n, int s, const double* u, int nq, const int* first,
                            const double* V, int p, double* T) {
  long long tot = (long long)r * nq * s;
  if (tot == 0) return TTB_OK;
  field_table_kernel<<<grid_for(tot), 256, 0, as_stream(stream)>>>(r, n, s, u, nq, first, V, p, T); ttb_count();
  return ttb_last_error();
}

// out[0] = sum w det |u - u*|, out[1] = sum w det |u*| over the tensor quadrature grid.
TTB_API int ttb_l1_error(void* stream, const int* f0, const int* f1, const int* f2, const double* V0, const double* V1,
                         const double* V2, const double* D0, const double* D1, const double* D2, int p0, int p1,
                         int p2, int n0, int n1, int n2, const double* cw, int nq0, int nq1, int nq2,
                         const double* U0, int r1, const double* U1, int r2, const double* U2, const double* w0,
                         const double* w1, const double* w2, int exact_id, const double* prm, double* part,
                         double* out) {
  const int* f[3] = {f0, f1, f2};
  const double* V[3] = {V0, V1, V2};
  const double* D[3] = {D0, D1, D2};
  int p[3] = {p0, p1, p2}, n[3] = {n0, n1, n2};
  GeoArgs g = make_geo(f, V, D, p, n, cw, 0.0);
  long long blocks = (long long)nq0 * nq1;
  cudaStream_t st = as_stream(stream);
  l1err_kernel<<<(unsigned)blocks, 128, r2 * sizeof(double), st>>>(g, nq0, nq1, nq2, U0, r1, U1, r2, U2, w0, w1, w2,
                                                                     exact_id, prm, part); ttb_count();
  pair_sum_kernel<<<1, 1024, 0, st>>>(blocks, part, out); ttb_count();
  return ttb_last_error();
}
