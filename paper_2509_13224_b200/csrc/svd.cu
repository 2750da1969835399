// One-sided (Hestenes) Jacobi SVD of small square FP64 matrices.
//
// Used on the R factor of a Householder QR (so only n x n, n = TT rank, is
// rotated). Round-robin (tournament) ordering: every round is n/2 disjoint
// column pairs, one warp per pair, warp-shuffle reductions for the 2x2 Gram
// entries. n <= 64 runs entirely in shared memory; larger n keeps A and V in
// global memory (L2 resident) with the same schedule.
#include "common.cuh"
#include <stdlib.h>

namespace {

constexpr int JT = 1024;  // threads per CTA

__device__ __forceinline__ int rr_index(int k, int r, int N) {
  return k == 0 ? 0 : ((k - 1 + r) % (N - 1)) + 1;
}

__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// Rotation of jrot, branch-free, with the tangent from approximate (MUFU) reciprocal square root and
// reciprocal on power-of-two-scaled operands: t only chooses the angle -- any t gives an exactly
// orthogonal (c, s) below, and a t off by ~1e-6 relative leaves ~1e-6 of g_pq for the next visit --
// while c = (1 + t^2)^(-1/2) is the FP64 rsqrt, so (c, s) are orthogonal to rounding. Replaces jrot's
// FP64 square root and division.
__device__ __forceinline__ void jrot_fast(double al, double be, double ga, double thr2, double& c, double& s) {
  const double d = be - al, g2 = 2.0 * ga;
  const double m = fmax(fabs(d), fabs(g2));
  const long long ex = (__double_as_longlong(m) >> 52) & 0x7ff;
  const double sc = __longlong_as_double((2046LL - min(ex, 2045LL)) << 52);   // 2^(1023 - ex): m sc in [1, 2)
  const double ds = fabs(d) * sc, gs = fabs(g2) * sc;
  const double h = fma(ds, ds, gs * gs);
  const double den = fma(h, rsqrt_approx(h), ds);          // |d| + sqrt(d^2 + g^2), scaled, >= 1
  double t = gs * rcp_approx(den);
  const bool pos = (d == 0.0) || ((d > 0.0) == (g2 > 0.0));
  t = pos ? t : -t;
  // c from the library rsqrt (unbiased rounding): a hand-rolled Newton step from the approximate
  // rsqrt lands ~2e-17 high on average, and 1e4 rotation visits per column turn that into a 3e-13
  // drift of the column norms
  const double r = rsqrt(fma(t, t, 1.0));
  const bool act = ga != 0.0 && ga * ga > thr2 * al * be;
  c = act ? r : 1.0;
  s = act ? r * t : 0.0;
}

// A (n x n col-major, ld n) -> columns mutually orthogonal; V accumulates rotations.
// Returns number of sweeps in *sweeps_out (thread 0).
__device__ void jacobi_core(int n, double* A, double* V, int* flag, int max_sweeps, double tol, int* sweeps_out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int N = (n + 1) & ~1;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int r = 0; r < N - 1; ++r) {
      for (int pr = wid; pr < N / 2; pr += nw) {
        int p = rr_index(pr, r, N), q = rr_index(N - 1 - pr, r, N);
        if (p > q) { int t = p; p = q; q = t; }
        if (q >= n) continue;
        double* ap = A + (long long)p * n;
        double* aq = A + (long long)q * n;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < n; i += 32) {
          double x = ap[i], y = aq[i];
          al += x * x; be += y * y; ga += x * y;
        }
        al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
        if (ga == 0.0 || fabs(ga) <= tol * sqrt(al * be)) continue;
        if (lane == 0) *flag = 1;
        double c, s;
        jrot_fast(al, be, ga, 0.0, c, s);
        for (int i = lane; i < n; i += 32) {
          double x = ap[i], y = aq[i];
          ap[i] = c * x - s * y;
          aq[i] = s * x + c * y;
        }
        if (V) {
          double* vp = V + (long long)p * n;
          double* vq = V + (long long)q * n;
          for (int i = lane; i < n; i += 32) {
            double x = vp[i], y = vq[i];
            vp[i] = c * x - s * y;
            vq[i] = s * x + c * y;
          }
        }
      }
      __syncthreads();
    }
    int f = *flag;
    __syncthreads();
    if (!f) break;
  }
  if (threadIdx.x == 0) *sweeps_out = sweep;
}

// batch of matrices along blockIdx.x; A overwritten with U (col-major), S descending.
template <bool SMEM>
__global__ void __launch_bounds__(JT) jacobi_kernel(int n, double* Ag, long long strideA, double* Sg, long long strideS,
                                                    double* Ug, double* Vg, long long strideUV, double* work,
                                                    int max_sweeps, double tol, int* info) {
  extern __shared__ double dyn[];
  __shared__ int flag, nsweep;
  const long long b = blockIdx.x;
  double* Ain = Ag + b * strideA;
  double* U = Ug + b * strideUV;
  double* Vout = Vg ? Vg + b * strideUV : nullptr;
  double* S = Sg + b * strideS;
  const long long nn = (long long)n * n;
  double *A, *V;
  if (SMEM) {
    A = dyn;
    V = dyn + nn;
  } else {
    A = work + b * (2 * nn + n);
    V = A + nn;
  }
  if (!Vg) V = nullptr;
  for (long long e = threadIdx.x; e < nn; e += blockDim.x) {
    A[e] = Ain[e];
    if (V) V[e] = ((e / n) == (e % n)) ? 1.0 : 0.0;
  }
  __syncthreads();
  jacobi_core(n, A, V, &flag, max_sweeps, tol, &nsweep);
  __syncthreads();
  // column norms, descending order rank (stable by index)
  double* sig = SMEM ? (dyn + (Vg ? 2 : 1) * nn) : (work + b * (2 * nn + n) + 2 * nn);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = wid; j < n; j += nw) {
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += A[(long long)j * n + i] * A[(long long)j * n + i];
    s = warp_sum(s);
    if (lane == 0) sig[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double sj = sig[j];
    int rank = 0;
    for (int k = 0; k < n; ++k) {
      double sk = sig[k];
      rank += (sk > sj) || (sk == sj && k < j);
    }
    S[rank] = sj;
    double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    for (int i = 0; i < n; ++i) {
      U[(long long)rank * n + i] = A[(long long)j * n + i] * inv;
      if (Vout) Vout[(long long)rank * n + i] = V[(long long)j * n + i];
    }
  }
  if (threadIdx.x == 0 && info) info[b] = nsweep;
}

// Multi-CTA variant for one large matrix: every warp of the grid takes disjoint pairs of a
// round, rounds separated by grid-wide barriers; a per-sweep rotation counter (double
// buffered by sweep parity) gives a uniform convergence decision.
constexpr int CT = 256;

__global__ void __launch_bounds__(CT) jacobi_coop_kernel(int n, double* A, double* V, int* cnt, int max_sweeps,
                                                          double tol, int* sweeps_out) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int N = (n + 1) & ~1;
  int sweep = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) { cnt[0] = 0; cnt[1] = 0; }
  grid.sync();
  for (; sweep < max_sweeps; ++sweep) {
    int* c = cnt + (sweep & 1);
    for (int r = 0; r < N - 1; ++r) {
      for (int pr = gw; pr < N / 2; pr += nwarps) {
        int p = rr_index(pr, r, N), q = rr_index(N - 1 - pr, r, N);
        if (p > q) { int t = p; p = q; q = t; }
        if (q >= n) continue;
        double* ap = A + (long long)p * n;
        double* aq = A + (long long)q * n;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < n; i += 32) {
          double x = ap[i], y = aq[i];
          al += x * x; be += y * y; ga += x * y;
        }
        al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
        if (ga == 0.0 || fabs(ga) <= tol * sqrt(al * be)) continue;
        if (lane == 0) atomicAdd(c, 1);
        double cs, sn;
        jrot_fast(al, be, ga, 0.0, cs, sn);
        for (int i = lane; i < n; i += 32) {
          double x = ap[i], y = aq[i];
          ap[i] = cs * x - sn * y;
          aq[i] = sn * x + cs * y;
        }
        if (V) {
          double* vp = V + (long long)p * n;
          double* vq = V + (long long)q * n;
          for (int i = lane; i < n; i += 32) {
            double x = vp[i], y = vq[i];
            vp[i] = cs * x - sn * y;
            vq[i] = sn * x + cs * y;
          }
        }
      }
      grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[(sweep + 1) & 1] = 0;
    const int done = (*(volatile int*)c) == 0;
    grid.sync();
    if (done) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = sweep;
}

// Block one-sided Jacobi: the n columns are split into blocks of b; in every round each CTA
// takes one pair of blocks (tournament order over blocks), stages their 2b columns (and V's)
// in shared memory and runs a full local sweep over all their column pairs there, so a
// grid-wide barrier is paid once per block round (nb-1 per sweep) instead of once per
// column round (n-1 per sweep).
constexpr int BT = 256;

__global__ void __launch_bounds__(BT) jacobi_block_kernel(int n, int b, double* A, double* V, int* cnt,
                                                           int max_sweeps, double tol, int* sweeps_out) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  __shared__ int rot;
  __shared__ int cols[64];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = BT / 32;
  const int nb = (n + b - 1) / b;
  const int NB2 = (nb + 1) & ~1;
  double* As = sm;
  double* Vs = sm + (long long)2 * b * n;
  if (blockIdx.x == 0 && threadIdx.x == 0) { cnt[0] = 0; cnt[1] = 0; }
  grid.sync();
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int* c = cnt + (sweep & 1);
    for (int r = 0; r < NB2 - 1; ++r) {
      for (int pr = blockIdx.x; pr < NB2 / 2; pr += gridDim.x) {
        int bp = rr_index(pr, r, NB2), bq = rr_index(NB2 - 1 - pr, r, NB2);
        if (bp > bq) { int t = bp; bp = bq; bq = t; }
        if (bq >= nb) continue;  // dummy block (uniform per CTA)
        int L = 0;
        for (int j = bp * b; j < min(n, bp * b + b); ++j) cols[L++] = j;
        for (int j = bq * b; j < min(n, bq * b + b); ++j) cols[L++] = j;
        for (int lc = 0; lc < L; ++lc) {
          const double* src = A + (long long)cols[lc] * n;
          double* dst = As + (long long)lc * n;
          for (int i = threadIdx.x; i < n; i += BT) dst[i] = src[i];
          if (V) {
            const double* vs = V + (long long)cols[lc] * n;
            double* vd = Vs + (long long)lc * n;
            for (int i = threadIdx.x; i < n; i += BT) vd[i] = vs[i];
          }
        }
        if (threadIdx.x == 0) rot = 0;
        __syncthreads();
        const int Lp = (L + 1) & ~1;
        for (int ir = 0; ir < Lp - 1; ++ir) {
          for (int ip = wid; ip < Lp / 2; ip += nw) {
            int p = rr_index(ip, ir, Lp), q = rr_index(Lp - 1 - ip, ir, Lp);
            if (p > q) { int t = p; p = q; q = t; }
            if (q >= L) continue;
            double* ap = As + (long long)p * n;
            double* aq = As + (long long)q * n;
            double al = 0.0, be = 0.0, ga = 0.0;
            for (int i = lane; i < n; i += 32) {
              const double x = ap[i], y = aq[i];
              al += x * x; be += y * y; ga += x * y;
            }
            al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
            if (ga == 0.0 || fabs(ga) <= tol * sqrt(al * be)) continue;
            if (lane == 0) rot = 1;
            double cs, sn;
            jrot_fast(al, be, ga, 0.0, cs, sn);
            for (int i = lane; i < n; i += 32) {
              const double x = ap[i], y = aq[i];
              ap[i] = cs * x - sn * y;
              aq[i] = sn * x + cs * y;
            }
            if (V) {
              double* vp = Vs + (long long)p * n;
              double* vq = Vs + (long long)q * n;
              for (int i = lane; i < n; i += 32) {
                const double x = vp[i], y = vq[i];
                vp[i] = cs * x - sn * y;
                vq[i] = sn * x + cs * y;
              }
            }
          }
          __syncthreads();
        }
        for (int lc = 0; lc < L; ++lc) {
          double* dst = A + (long long)cols[lc] * n;
          const double* src = As + (long long)lc * n;
          for (int i = threadIdx.x; i < n; i += BT) dst[i] = src[i];
          if (V) {
            double* vd = V + (long long)cols[lc] * n;
            const double* vs = Vs + (long long)lc * n;
            for (int i = threadIdx.x; i < n; i += BT) vd[i] = vs[i];
          }
        }
        if (threadIdx.x == 0 && rot) atomicAdd(c, 1);
        __syncthreads();
      }
      grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[(sweep + 1) & 1] = 0;
    const int done = (*(volatile int*)c) == 0;
    grid.sync();
    if (done) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = sweep;
}

// Gram block one-sided Jacobi (n >= 128, one matrix). The n columns form blocks of GB/2; each
// round (tournament order over blocks, one grid-wide barrier) every CTA owns one pair of blocks
// = GB columns, staged in shared memory, and orthogonalizes them completely:
//   repeat { G = A_loc^T A_loc (DMMA, fresh from the columns);
//            stop if every pair passes |g_pq| <= tol sqrt(g_pp g_qq)  (the scalar test);
//            eigen-decompose G by a cyclic two-sided Jacobi in one warp (rotations J);
//            A_loc <- A_loc J (DMMA) }
// The pass/fail test always uses a Gram recomputed from the columns, so the stopping rule
// and the attainable orthogonality are those of the scalar one-sided method (relative
// accuracy); only the rotation angles come from the 8 x 8 eigen-solve. A sweep in which no
// CTA rotates ends the iteration.
constexpr int GT = 256;     // threads per CTA
constexpr int GW = GT / 32;
constexpr int kLocalIters = 1;   // Gram -> rotate -> apply rounds per block pair and visit
constexpr int kEigenSweeps = 1;  // cyclic sweeps of the 8 x 8 eigen-solve per local round
int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

__device__ __forceinline__ void dmma8(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Rotation (c, s) annihilating g_pq of the symmetric 2 x 2 [[al, ga], [ga, be]] (one-sided
// convention: a_p' = c a_p - s a_q, a_q' = s a_p + c a_q); identity when inactive or when
// ga^2 <= thr2 al be. t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (be - al) / (2 ga),
// evaluated as |2ga| / (|d| + sqrt(d^2 + 4ga^2)) with one division and one rsqrt.
__device__ __forceinline__ void jrot(double al, double be, double ga, double thr2, bool active, double& c, double& s) {
  c = 1.0;
  s = 0.0;
  if (active && ga != 0.0 && ga * ga > thr2 * al * be) {
    const double d = be - al, g2 = 2.0 * ga;
    const double mag = fabs(g2) / (fabs(d) + sqrt(d * d + g2 * g2));
    const bool pos = (d == 0.0) || ((d > 0.0) == (g2 > 0.0));
    const double t = pos ? mag : -mag;
    c = rsqrt(1.0 + t * t);
    s = c * t;
  }
}

// Rounds are ordered by per-block version counters instead of grid-wide barriers: a CTA starts
// its pair in round R as soon as both blocks have finished round R - 1 (ver[b] == R), and
// publishes them with a release store; one grid barrier per sweep takes the stop decision.
template <int GB>
__global__ void __launch_bounds__(GT) jacobi_gram_kernel(int n, double* A, double* V, int* cnt, int* ver,
                                                          int max_sweeps, double tol, int* sweeps_out,
                                                          int local_iters, int eigen_sweeps) {
  constexpr int NTL = GB / 8;  // 8-column tiles
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  __shared__ double Gp[GW][GB * GB];
  __shared__ double G[GB * GB];
  __shared__ double J[GB * GB];
  __shared__ double rc[GB / 2], rs[GB / 2];
  __shared__ int rp[GB / 2], rq[GB / 2];
  __shared__ int cols[GB];
  __shared__ int ncols, need, rotated;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int hb = GB / 2;
  const int nb = (n + hb - 1) / hb;
  const int NBL = (nb + 1) & ~1;
  const int NR = (n + 31) & ~31;      // padded rows (zeros)
  const int LD = NR + 4;
  double* As = sm;
  double* Vs = sm + (long long)GB * LD;
  if (blockIdx.x == 0 && threadIdx.x == 0) { cnt[0] = 0; cnt[1] = 0; }
  if (blockIdx.x == 0)
    for (int b = threadIdx.x; b < nb; b += GT) ver[b] = 0;
  for (int e = threadIdx.x; e < GB * LD; e += GT) { As[e] = 0.0; if (V) Vs[e] = 0.0; }
  grid.sync();
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int* c = cnt + (sweep & 1);
    for (int r = 0; r < NBL - 1; ++r) {
      const int R = sweep * (NBL - 1) + r;
      for (int pr = blockIdx.x; pr < NBL / 2; pr += gridDim.x) {
        int bp = rr_index(pr, r, NBL), bq = rr_index(NBL - 1 - pr, r, NBL);
        if (bp > bq) { int t = bp; bp = bq; bq = t; }
        if (bq >= nb) {  // paired with the dummy block: just pass the round
          if (threadIdx.x == 0 && bp < nb) {
            while (ld_acquire(ver + bp) < R) {}
            st_release(ver + bp, R + 1);
          }
          continue;
        }
        if (threadIdx.x == 0) {
          while (ld_acquire(ver + bp) < R || ld_acquire(ver + bq) < R) {}
          int L = 0;
          for (int j = bp * hb; j < min(n, bp * hb + hb); ++j) cols[L++] = j;
          for (int j = bq * hb; j < min(n, bq * hb + hb); ++j) cols[L++] = j;
          ncols = L;
          rotated = 0;
        }
        __syncthreads();
        const int L = ncols;
        for (int i0 = 0; i0 < n; i0 += 4 * GT) {  // 4 x GB independent loads in flight per thread
          double buf[GB][4];
#pragma unroll
          for (int lc = 0; lc < GB; ++lc)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = i0 + u * GT + threadIdx.x;
              buf[lc][u] = (lc < L && i < n) ? __ldcg(A + (long long)cols[lc] * n + i) : 0.0;
            }
#pragma unroll
          for (int lc = 0; lc < GB; ++lc)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = i0 + u * GT + threadIdx.x;
              if (i < n) As[lc * LD + i] = buf[lc][u];
            }
          if (V) {
#pragma unroll
            for (int lc = 0; lc < GB; ++lc)
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * GT + threadIdx.x;
                buf[lc][u] = (lc < L && i < n) ? __ldcg(V + (long long)cols[lc] * n + i) : 0.0;
              }
#pragma unroll
            for (int lc = 0; lc < GB; ++lc)
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * GT + threadIdx.x;
                if (i < n) Vs[lc * LD + i] = buf[lc][u];
              }
          }
        }
        __syncthreads();
        for (int it = 0; it < local_iters; ++it) {
          // fresh Gram: warp w sums rows [w NR/GW, (w+1) NR/GW) with DMMA (A operand tiles = B tiles)
          {
            double d[NTL][NTL][2];
#pragma unroll
            for (int ti = 0; ti < NTL; ++ti)
#pragma unroll
              for (int tj = 0; tj < NTL; ++tj) d[ti][tj][0] = d[ti][tj][1] = 0.0;
            const int k0 = wid * (NR / GW), k1 = k0 + NR / GW;
            const double* col = As + (lane >> 2) * LD + (lane & 3);
            for (int k = k0; k < k1; k += 4) {
              double x[NTL];
#pragma unroll
              for (int ti = 0; ti < NTL; ++ti) x[ti] = col[ti * 8 * LD + k];
#pragma unroll
              for (int ti = 0; ti < NTL; ++ti)
#pragma unroll
                for (int tj = 0; tj < NTL; ++tj) dmma8(d[ti][tj][0], d[ti][tj][1], x[ti], x[tj]);
            }
#pragma unroll
            for (int ti = 0; ti < NTL; ++ti)
#pragma unroll
              for (int tj = 0; tj < NTL; ++tj) {
                Gp[wid][(ti * 8 + (lane >> 2)) * GB + tj * 8 + 2 * (lane & 3)] = d[ti][tj][0];
                Gp[wid][(ti * 8 + (lane >> 2)) * GB + tj * 8 + 2 * (lane & 3) + 1] = d[ti][tj][1];
              }
          }
          __syncthreads();
          for (int e = threadIdx.x; e < GB * GB; e += GT) {
            double g = 0.0;
            for (int w = 0; w < GW; ++w) g += Gp[w][e];
            G[e] = g;
          }
          if (threadIdx.x == 0) need = 0;
          __syncthreads();
          for (int e = threadIdx.x; e < GB * GB; e += GT) {
            const int p = e / GB, q = e % GB;
            if (p < q && q < L) {
              const double ga = G[p * GB + q];
              if (!(ga == 0.0 || fabs(ga) <= tol * sqrt(G[p * GB + p] * G[q * GB + q]))) need = 1;
            }
          }
          __syncthreads();
          if (!need) break;
          if (wid == 0) {
            // cyclic two-sided Jacobi on G (one warp), rotations accumulated in J. Per round the
            // GB/2 disjoint rotations go to shared memory, then G <- J_r^T G J_r is formed block-wise
            // (item = row pair k1, col pair k2, row r of the pair) and J <- J J_r column-pair-wise.
            for (int e = lane; e < GB * GB; e += 32) J[e] = (e / GB == e % GB) ? 1.0 : 0.0;
            __syncwarp();
            const double thr2 = 0.0625 * tol * tol;
            constexpr int HB = GB / 2;
            for (int es = 0; es < eigen_sweeps; ++es) {
              bool any = false;
              for (int rd = 0; rd < GB - 1; ++rd) {
                if (lane < HB) {
                  int p = rr_index(lane, rd, GB), q = rr_index(GB - 1 - lane, rd, GB);
                  if (p > q) { int t = p; p = q; q = t; }
                  double cs, sn;
                  jrot(G[p * GB + p], G[q * GB + q], G[p * GB + q], thr2, q < L, cs, sn);
                  rp[lane] = p; rq[lane] = q; rc[lane] = cs; rs[lane] = sn;
                  any |= (sn != 0.0);
                }
                __syncwarp();
                constexpr int ITEMS = HB * HB * 2;
                double nv[ITEMS / 32 > 0 ? ITEMS / 32 : 1][2];
#pragma unroll
                for (int u = 0; u < ITEMS / 32; ++u) {
                  const int item = lane + 32 * u;
                  const int k1 = item / (2 * HB), k2 = (item >> 1) % HB, r = item & 1;
                  const int p1 = rp[k1], q1 = rq[k1], p2 = rp[k2], q2 = rq[k2];
                  const double c1 = rc[k1], s1 = rs[k1], c2 = rc[k2], s2 = rs[k2];
                  const double gpp = G[p1 * GB + p2], gpq = G[p1 * GB + q2], gqp = G[q1 * GB + p2], gqq = G[q1 * GB + q2];
                  const double up = r ? (s1 * gpp + c1 * gqp) : (c1 * gpp - s1 * gqp);
                  const double uq = r ? (s1 * gpq + c1 * gqq) : (c1 * gpq - s1 * gqq);
                  nv[u][0] = c2 * up - s2 * uq;
                  nv[u][1] = s2 * up + c2 * uq;
                }
                constexpr int JITEMS = HB * GB;
                double jv[JITEMS / 32][2];
#pragma unroll
                for (int u = 0; u < JITEMS / 32; ++u) {
                  const int item = lane + 32 * u;
                  const int k = item / GB, i = item % GB;
                  const double jp = J[i * GB + rp[k]], jq = J[i * GB + rq[k]];
                  jv[u][0] = rc[k] * jp - rs[k] * jq;
                  jv[u][1] = rs[k] * jp + rc[k] * jq;
                }
                __syncwarp();
#pragma unroll
                for (int u = 0; u < ITEMS / 32; ++u) {
                  const int item = lane + 32 * u;
                  const int k1 = item / (2 * HB), k2 = (item >> 1) % HB, r = item & 1;
                  const int x = r ? rq[k1] : rp[k1];
                  G[x * GB + rp[k2]] = nv[u][0];
                  G[x * GB + rq[k2]] = nv[u][1];
                }
#pragma unroll
                for (int u = 0; u < JITEMS / 32; ++u) {
                  const int item = lane + 32 * u;
                  const int k = item / GB, i = item % GB;
                  J[i * GB + rp[k]] = jv[u][0];
                  J[i * GB + rq[k]] = jv[u][1];
                }
                __syncwarp();
              }
              if (!__any_sync(0xffffffffu, any)) break;
            }
          }
          __syncthreads();
          // A_loc <- A_loc J (and V_loc): warp w takes row tiles of 8, GB/4 k-steps of 4 columns
          for (int rt = wid; rt < NR / 8; rt += GW) {
            const int r0 = rt * 8;
            for (int mat = 0; mat < (V ? 2 : 1); ++mat) {
              double* X = mat ? Vs : As;
              double a[GB / 4];
#pragma unroll
              for (int ks = 0; ks < GB / 4; ++ks) a[ks] = X[(4 * ks + (lane & 3)) * LD + r0 + (lane >> 2)];
              double d[NTL][2];
#pragma unroll
              for (int tj = 0; tj < NTL; ++tj) {
                d[tj][0] = d[tj][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < GB / 4; ++ks)
                  dmma8(d[tj][0], d[tj][1], a[ks], J[(4 * ks + (lane & 3)) * GB + tj * 8 + (lane >> 2)]);
              }
              __syncwarp();
#pragma unroll
              for (int tj = 0; tj < NTL; ++tj) {
                X[(tj * 8 + 2 * (lane & 3)) * LD + r0 + (lane >> 2)] = d[tj][0];
                X[(tj * 8 + 2 * (lane & 3) + 1) * LD + r0 + (lane >> 2)] = d[tj][1];
              }
            }
          }
          if (threadIdx.x == 0) rotated = 1;
          __syncthreads();
        }
        if (rotated) {
          for (int i0 = 0; i0 < n; i0 += 4 * GT) {
#pragma unroll
            for (int lc = 0; lc < GB; ++lc)
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * GT + threadIdx.x;
                if (lc < L && i < n) {
                  A[(long long)cols[lc] * n + i] = As[lc * LD + i];
                  if (V) V[(long long)cols[lc] * n + i] = Vs[lc * LD + i];
                }
              }
          }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          if (rotated) atomicAdd(c, 1);
          __threadfence();
          st_release(ver + bp, R + 1);
          st_release(ver + bq, R + 1);
        }
      }
    }
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[(sweep + 1) & 1] = 0;
    const int done = (*(volatile int*)c) == 0;
    grid.sync();
    if (done) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = sweep;
}

// Warp-sliced Gram block one-sided Jacobi (n even, n <= 1024, one matrix). Same pairing, rotation
// rule and stopping test as jacobi_gram_kernel<8> (tournament order over blocks of 4 columns, each
// CTA orthogonalizes one pair = 8 columns per round), but the rows are split across the 8 warps
// (warp w owns rows [w RW, (w+1) RW) of every column for the whole run) so that a round has a
// single CTA barrier:
//   per warp: wait until the previous owners' warp w published these rows (ver[b][w], acquire),
//             cp.async its 8 x RW slab into shared memory, partial Gram by DMMA;
//   CTA:      barrier, every warp sums the 8 partial Grams (same order: identical G in all warps);
//   per warp: convergence test + one cyclic sweep of the 8 x 8 two-sided Jacobi (redundantly in
//             every warp: no broadcast barrier), A_slab J by DMMA straight to global, fence,
//             publish ver[b][w] (release).
// Rows never move between warps, so a warp depends only on the same warp index of the CTAs that
// held its two blocks in the previous round; the per-round critical path is one L2 round trip,
// one 8 KB slab load, ~70 DMMA and the 8 x 8 rotation sweep instead of eight barriers around
// single-warp and single-thread sections (jacobi_gram_kernel: 11 us per round, 46% barrier stall).
constexpr int WS_W = 8;          // warps per CTA
constexpr int WS_T = WS_W * 32;

__device__ __forceinline__ uint32_t sm_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_wait_parity(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}\n" ::"r"(mbar),
      "r"(phase)
      : "memory");
}

// 1-D bulk copy global -> shared (TMA engine), completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   sm_u32(dst)),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

__device__ __forceinline__ void st_relaxed(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// CROSS: only the 16 pairs between the two blocks (4 rounds of 4 disjoint rotations instead of the
// 7-round sweep over all 28 pairs): used for every visit but the first of a sweep, so that over a sweep
// every column pair is rotated exactly once (a block's own pairs at its round-0 visit, every cross pair
// when its two blocks meet) -- a cyclic-by-blocks ordering -- instead of the intra-block pairs at every
// one of the 255 visits.
template <bool CROSS = false>
__device__ __forceinline__ bool jw_eigen8(double* G, double* J, double tol, int lane) {
  // absent columns (n % 4 != 0) are zero: they pass the test and never rotate
  bool nd = false;
  for (int e = lane; e < 64; e += 32) {
    const int p = e >> 3, q = e & 7;
    if (p < q && (!CROSS || (p < 4 && q >= 4))) {
      const double ga = G[e];
      if (!(ga == 0.0 || fabs(ga) <= tol * sqrt(G[p * 9] * G[q * 9]))) nd = true;
    }
  }
  nd = __any_sync(0xffffffffu, nd);
  if (nd) {
    // every lane computes the two rotations it needs itself (pairs k1 = lane / 8 and k2),
    // so a round is one shared-memory read / update / write with no parameter broadcast
    const double thr2 = 0.0625 * tol * tol;
    const int k1 = lane >> 3, k2 = (lane >> 1) & 3, rr = lane & 1, ji = lane & 7;
#pragma unroll
    for (int rd = 0; rd < (CROSS ? 4 : 7); ++rd) {
      int p1 = CROSS ? k1 : rr_index(k1, rd, 8), q1 = CROSS ? 4 + ((k1 + rd) & 3) : rr_index(7 - k1, rd, 8);
      int p2 = CROSS ? k2 : rr_index(k2, rd, 8), q2 = CROSS ? 4 + ((k2 + rd) & 3) : rr_index(7 - k2, rd, 8);
      if (p1 > q1) { int t = p1; p1 = q1; q1 = t; }
      if (p2 > q2) { int t = p2; p2 = q2; q2 = t; }
      const double a1 = G[p1 * 9], b1 = G[q1 * 9], g1 = G[p1 * 8 + q1];
      const double a2 = G[p2 * 9], b2 = G[q2 * 9], g2 = G[p2 * 8 + q2];
      const double gpp = G[p1 * 8 + p2], gpq = G[p1 * 8 + q2], gqp = G[q1 * 8 + p2], gqq = G[q1 * 8 + q2];
      const double jp = J[ji * 8 + p1], jq = J[ji * 8 + q1];
      double c1, s1, c2, s2;
      jrot_fast(a1, b1, g1, thr2, c1, s1);
      jrot_fast(a2, b2, g2, thr2, c2, s2);
      const double up = rr ? (s1 * gpp + c1 * gqp) : (c1 * gpp - s1 * gqp);
      const double uq = rr ? (s1 * gpq + c1 * gqq) : (c1 * gpq - s1 * gqq);
      const double nv0 = c2 * up - s2 * uq, nv1 = s2 * up + c2 * uq;
      const double jv0 = c1 * jp - s1 * jq, jv1 = s1 * jp + c1 * jq;
      const int gx = rr ? q1 : p1;
      __syncwarp();
      G[gx * 8 + p2] = nv0;
      G[gx * 8 + q2] = nv1;
      J[ji * 8 + p1] = jv0;
      J[ji * 8 + q1] = jv1;
      __syncwarp();
    }
  }
  return nd;
}

__global__ void __launch_bounds__(WS_T) jacobi_wslice_kernel(int n, int RW, double* A, double* V, int* cnt, int* ver,
                                                              int max_sweeps, double tol, int* sweeps_out,
                                                              long long* prof = nullptr, int cross = 1) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  __shared__ double Gp[2][WS_W][64];
  __shared__ double G[64], J[64];
  __shared__ int need_s;
  __shared__ __align__(8) unsigned long long mbar[WS_W];
#define JW_STAMP(k)                                                                                          \
  if (prof && lane == 0 && w == 0 && R >= 64 && R < 80) {                                                 \
    long long t_;                                                                                            \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                                 \
    prof[((long long)blockIdx.x * 16 + (R - 64)) * 8 + (k)] = t_;                                          \
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nb = (n + 3) / 4;
  const int NBL = (nb + 1) & ~1;
  const int LDW = RW + 4;
  const int nmat = V ? 2 : 1;
  double* slab = sm + (size_t)w * nmat * 8 * LDW;  // [mat][col][row] for this warp
  const int row0 = w * RW;
  const int vrows = max(0, min(RW, n - row0));     // rows of this warp's slab inside the matrix
  const uint32_t bar = sm_u32(&mbar[w]);
  if (blockIdx.x == 0 && threadIdx.x == 0) { cnt[0] = 0; cnt[1] = 0; }
  if (blockIdx.x == 0)
    for (int b = threadIdx.x; b < nb * WS_W; b += WS_T) ver[b] = 0;
  for (int e = lane; e < nmat * 8 * LDW; e += 32) slab[e] = 0.0;   // rows >= n stay zero
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  grid.sync();
  uint32_t phase = 0;
  int sweep = 0, gpar = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int* c = cnt + (sweep & 1);
    for (int r = 0; r < NBL - 1; ++r) {
      const int R = sweep * (NBL - 1) + r;
      for (int pr = blockIdx.x; pr < NBL / 2; pr += gridDim.x) {
        int bp = rr_index(pr, r, NBL), bq = rr_index(NBL - 1 - pr, r, NBL);
        if (bp > bq) { int t = bp; bp = bq; bq = t; }
        if (bq >= nb) {  // paired with the dummy block: pass the round
          if (lane == 0 && bp < nb) {
            while (ld_acquire(ver + bp * WS_W + w) < R) {}
            st_release(ver + bp * WS_W + w, R + 1);
          }
          __syncwarp();
          continue;
        }
        JW_STAMP(0);
        // slab load: block bp's 4 columns as soon as bp is published, then bq's (bulk copies of
        // this warp's rows; absent columns zeroed)
        const int cp_ = min(4, n - bp * 4), cq_ = min(4, n - bq * 4);
        if (lane == 0 && vrows > 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                       "r"((uint32_t)(nmat * (cp_ + cq_) * vrows * 8))
                       : "memory");
          while (ld_acquire(ver + bp * WS_W + w) < R) {}
          for (int mat = 0; mat < nmat; ++mat)
            for (int lc = 0; lc < cp_; ++lc)
              bulk_g2s(slab + (mat * 8 + lc) * LDW, (mat ? V : A) + (long long)(bp * 4 + lc) * n + row0, vrows * 8, bar);
          while (ld_acquire(ver + bq * WS_W + w) < R) {}
          for (int mat = 0; mat < nmat; ++mat)
            for (int lc = 0; lc < cq_; ++lc)
              bulk_g2s(slab + (mat * 8 + 4 + lc) * LDW, (mat ? V : A) + (long long)(bq * 4 + lc) * n + row0, vrows * 8,
                       bar);
        } else if (lane == 0) {
          while (ld_acquire(ver + bp * WS_W + w) < R || ld_acquire(ver + bq * WS_W + w) < R) {}
        }
        if (cp_ < 4 || cq_ < 4) {
          for (int mat = 0; mat < nmat; ++mat)
            for (int lc = 0; lc < 8; ++lc)
              if ((lc < 4 && lc >= cp_) || (lc >= 4 && lc - 4 >= cq_))
                for (int e = lane; e < RW; e += 32) slab[(mat * 8 + lc) * LDW + e] = 0.0;
        }
        JW_STAMP(1);
        if (vrows > 0) {
          mbar_wait_parity(bar, phase);
          phase ^= 1;
        }
        __syncwarp();
        JW_STAMP(2);
        // partial Gram of this warp's rows: 4 independent DMMA chains over k-steps of 4 rows
        {
          const double* col = slab + (lane >> 2) * LDW + (lane & 3);
          double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
          for (int k = 0; k < RW; k += 16) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double x = col[k + 4 * u];
              dmma8(d[u][0], d[u][1], x, x);
            }
          }
          const int e0 = (lane >> 2) * 8 + 2 * (lane & 3);
          Gp[gpar][w][e0] = (d[0][0] + d[1][0]) + (d[2][0] + d[3][0]);
          Gp[gpar][w][e0 + 1] = (d[0][1] + d[1][1]) + (d[2][1] + d[3][1]);
        }
        __syncthreads();
        JW_STAMP(3);
        // warp 0: full Gram, convergence test, one cyclic sweep of the 8 x 8 two-sided Jacobi
        // (rotations accumulated in J); the other warps wait at the broadcast barrier
        if (w == 0) {
          for (int e = lane; e < 64; e += 32) {
            double g = 0.0;
#pragma unroll
            for (int v = 0; v < WS_W; ++v) g += Gp[gpar][v][e];
            G[e] = g;
            J[e] = ((e >> 3) == (e & 7)) ? 1.0 : 0.0;
          }
          __syncwarp();
          // full visits at round 0 (and round 1 when a dummy block pads an odd block count: the block
          // paired with the dummy at round 0 gets its own pairs at round 1)
          const bool nd = (cross && r >= (NBL != nb ? 2 : 1)) ? jw_eigen8<true>(G, J, tol, lane)
                                                              : jw_eigen8<false>(G, J, tol, lane);
          if (lane == 0) need_s = nd;
        }
        gpar ^= 1;
        __syncthreads();
        const bool need = need_s;
        if (need) {
          JW_STAMP(4);
          // A_slab <- A_slab J (and V_slab), straight to global, as (A_slab J)^T = J^T A_slab^T so that
          // each lane holds two consecutive rows of one column (16-byte stores, 64-byte segments)
          const double j0 = J[(lane & 3) * 8 + (lane >> 2)], j1 = J[(4 + (lane & 3)) * 8 + (lane >> 2)];
          const int oc = lane >> 2;
          const int gco = (oc < 4 ? bp * 4 : bq * 4) + (oc & 3);
          const bool oko = oc < 4 ? oc < cp_ : oc - 4 < cq_;
          for (int mat = 0; mat < nmat; ++mat) {
            double* X = mat ? V : A;
            const double* src = slab + mat * 8 * LDW + (lane & 3) * LDW + (lane >> 2);
            double2* dst = reinterpret_cast<double2*>(X + (long long)gco * n + row0 + 2 * (lane & 3));
#pragma unroll 4
            for (int s = 0; s < RW; s += 8) {
              const double a0 = src[s], a1 = src[4 * LDW + s];
              double d0 = 0.0, d1 = 0.0;
              dmma8(d0, d1, j0, a0);
              dmma8(d0, d1, j1, a1);
              if (oko && row0 + s + 2 * (lane & 3) < n) dst[s / 2] = make_double2(d0, d1);
            }
          }
          JW_STAMP(5);
        }
        // generic-proxy slab accesses of this round before the next round's bulk writes
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        JW_STAMP(6);
        // publish: the warp barrier orders every lane's stores before lane 0's release fence, which
        // is cumulative over them (and over the acquires that admitted this round)
        if (lane == 0) {
          if (need && w == 0) atomicAdd(c, 1);
          asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
          st_relaxed(ver + bp * WS_W + w, R + 1);
          st_relaxed(ver + bq * WS_W + w, R + 1);
        }
        JW_STAMP(7);
      }
    }
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[(sweep + 1) & 1] = 0;
    const int done = (*(volatile int*)c) == 0;
    grid.sync();
    if (done) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = sweep;
}

__global__ void init_av_kernel(int n, const double* Ain, double* A, double* V) {
  const long long nn = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nn; e += (long long)gridDim.x * blockDim.x) {
    A[e] = Ain[e];
    if (V) V[e] = ((e / n) == (e % n)) ? 1.0 : 0.0;
  }
}

// column norms -> descending ranks -> U = A / sigma, V permuted (one warp per column)
__global__ void jacobi_finish_kernel(int n, const double* A, const double* V, double* sig, double* S, double* U,
                                     double* Vout) {
  const int lane = threadIdx.x & 31;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= n) return;
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s += A[(long long)j * n + i] * A[(long long)j * n + i];
  s = warp_sum(s);
  if (lane == 0) sig[j] = sqrt(s);
}

__global__ void jacobi_scatter_kernel(int n, const double* A, const double* V, const double* sig, double* S, double* U,
                                      double* Vout) {
  const int lane = threadIdx.x & 31;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= n) return;
  const double sj = sig[j];
  int rank = 0;
  for (int k = lane; k < n; k += 32) {
    const double sk = sig[k];
    rank += (sk > sj) || (sk == sj && k < j);
  }
  for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
  if (lane == 0) S[rank] = sj;
  const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
  for (int i = lane; i < n; i += 32) {
    U[(long long)rank * n + i] = A[(long long)j * n + i] * inv;
    if (Vout) Vout[(long long)rank * n + i] = V[(long long)j * n + i];
  }
}

}  // namespace

// SVD of `batch` square n x n col-major matrices A (= U diag(S) V^T).
// U, V: n x n col-major per matrix; S descending. work: batch*(2n^2+n) doubles when n > 64.
TTB_API int ttb_svd_jacobi(void* stream, int n, double* A, long long strideA, double* S, long long strideS, double* U,
                           double* V, long long strideUV, int batch, double* work, int* info) {
  if (n < 1 || batch < 1) return TTB_EARG;
  cudaStream_t st = as_stream(stream);
  const int max_sweeps = 60;
  const double tol = 4.0e-16 * (n > 16 ? sqrt((double)n) : 4.0);
  int threads = n >= 64 ? JT : ((n + 1) / 2 * 32 > 1024 ? 1024 : ((n + 1) / 2) * 32);
  if (threads < 32) threads = 32;
  const size_t smem = ((size_t)(V ? 2 : 1) * n * n + n) * sizeof(double);
  // single matrices with n >= 72 (even) take the multi-CTA warp-sliced kernel below: 2-3x faster than the
  // one-CTA shared-memory sweep from there on (n = 100: 4.3 -> ~1.5 ms; tools/jacobi_wslice_check.py)
  const bool wslice_ok = batch == 1 && n >= 72 && n % 2 == 0 && work != nullptr;
  if (smem <= 200 * 1024 && !wslice_ok) {
    static bool cfg = false;
    if (!cfg) {
      cudaFuncSetAttribute(jacobi_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cfg = true;
    }
    jacobi_kernel<true><<<batch, threads, smem, st>>>(n, A, strideA, S, strideS, U, V, strideUV, nullptr, max_sweeps,
                                                      tol, info); ttb_count();
  } else if (batch > 1 || (n <= 128 && !wslice_ok)) {
    if (!work) return TTB_EARG;
    jacobi_kernel<false><<<batch, JT, 0, st>>>(n, A, strideA, S, strideS, U, V, strideUV, work, max_sweeps, tol, info); ttb_count();
  } else {
    if (!work) return TTB_EARG;
    const long long nn = (long long)n * n;
    double* Aw = work;
    double* Vw = V ? work + nn : nullptr;
    double* sig = work + 2 * nn;
    static int* cnt = nullptr;
    static int* sw = nullptr;
    static int max_blocks = 0;
    if (!cnt) {
      cudaMalloc(&cnt, 4 * sizeof(int));
      sw = cnt + 2;
      int dev = 0, sms = 0, per = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, jacobi_coop_kernel, CT, 0);
      max_blocks = sms * (per > 0 ? (per > 2 ? 2 : per) : 1);
    }
    init_av_kernel<<<ceil_div(nn, 256) < 2048 ? ceil_div(nn, 256) : 2048, 256, 0, st>>>(n, A, Aw, Vw); ttb_count();
    int ms = max_sweeps;
    double tl = tol;
    // block size: 2b columns of A (and V) must fit in ~200 KB of shared memory
    int bsz = (int)(200 * 1024 / (16LL * n * (V ? 2 : 1)));
    if (bsz > 8) bsz = 8;
    cudaError_t e;
    static int jalg = -1;
    if (jalg < 0) {
      const char* ev = getenv("TTB_JACOBI");
      jalg = (ev && ev[0] == 'b') ? 1 : (ev && ev[0] == '1') ? 2 : (ev && ev[0] == 'g') ? 3 : 0;  // block | 16-column | gram | default
    }
    const size_t rows_pad = (size_t)(((n + 31) & ~31) + 4);
    const size_t gsmem16 = (size_t)16 * rows_pad * (V ? 2 : 1) * sizeof(double);
    const size_t gsmem8 = (size_t)8 * rows_pad * (V ? 2 : 1) * sizeof(double);
    // 8 columns per CTA: measured 38 ms vs 57 ms (16 columns) for n = 1024 at equal sweep counts
    const bool use16 = jalg == 2 && gsmem16 <= 200 * 1024;
    // warp-sliced kernel (default): n even, <= 1024 (rows per warp <= 128)
    const int wrw = ((((n + WS_W - 1) / WS_W) + 15) / 16) * 16;
    const size_t wsmem = (size_t)WS_W * (V ? 2 : 1) * 8 * (wrw + 4) * sizeof(double);
    if (jalg == 0 && n % 2 == 0 && n <= 1024 && wsmem <= 200 * 1024) {
      static int wmax = 0;
      if (!wmax) {
        cudaFuncSetAttribute(jacobi_wslice_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, jacobi_wslice_kernel, WS_T, 200 * 1024);
        wmax = sms * (per > 0 ? per : 1);
      }
      const int nbk = (n + 3) / 4;
      int nblk = ((nbk + 1) / 2) < wmax ? ((nbk + 1) / 2) : wmax;
      static int* wver = nullptr;
      static int wver_cap = 0;
      if (nbk * WS_W > wver_cap) {
        if (wver) { cudaStreamSynchronize(st); cudaFree(wver); }
        wver_cap = nbk * WS_W + 1024;
        if (cudaMalloc(&wver, sizeof(int) * wver_cap) != cudaSuccess) { wver = nullptr; wver_cap = 0; return (int)cudaErrorMemoryAllocation; }
      }
      int rw = wrw;
      long long* noprof = nullptr;
      static int cross = env_int("TTB_JACOBI_CROSS", 1);   // 0: every visit sweeps all 28 pairs
      void* args[] = {&n, &rw, &Aw, &Vw, &cnt, &wver, &ms, &tl, &sw, &noprof, &cross};
      e = cudaLaunchCooperativeKernel((const void*)jacobi_wslice_kernel, dim3(nblk), dim3(WS_T), args, wsmem, st); ttb_count();
    } else if (jalg != 1 && gsmem8 <= 200 * 1024) {
      const int GBsel = use16 ? 16 : 8;
      const void* kfn = use16 ? (const void*)jacobi_gram_kernel<16> : (const void*)jacobi_gram_kernel<8>;
      static int gmax[2] = {0, 0};
      int& gm = gmax[use16 ? 1 : 0];
      if (!gm) {
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kfn, GT, 200 * 1024);
        gm = sms * (per > 0 ? per : 1);
      }
      const int nbk = (n + GBsel / 2 - 1) / (GBsel / 2);
      int nblk = ((nbk + 1) / 2) < gm ? ((nbk + 1) / 2) : gm;
      static int li = env_int("TTB_JACOBI_LI", kLocalIters), es = env_int("TTB_JACOBI_ES", kEigenSweeps);
      static int* ver = nullptr;
      static int ver_cap = 0;
      if (nbk > ver_cap) {
        if (ver) { cudaStreamSynchronize(st); cudaFree(ver); }
        ver_cap = nbk + 1024;
        if (cudaMalloc(&ver, sizeof(int) * ver_cap) != cudaSuccess) { ver = nullptr; ver_cap = 0; return (int)cudaErrorMemoryAllocation; }
      }
      void* args[] = {&n, &Aw, &Vw, &cnt, &ver, &ms, &tl, &sw, &li, &es};
      e = cudaLaunchCooperativeKernel(kfn, dim3(nblk), dim3(GT), args, use16 ? gsmem16 : gsmem8, st); ttb_count();
    } else if (bsz >= 2) {
      static int bmax = 0;
      if (!bmax) {
        cudaFuncSetAttribute(jacobi_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, jacobi_block_kernel, BT, 200 * 1024);
        bmax = sms * (per > 0 ? per : 1);
      }
      const int nbk = (n + bsz - 1) / bsz;
      int nblk = ((nbk + 1) / 2) < bmax ? ((nbk + 1) / 2) : bmax;
      const size_t smem = (size_t)2 * bsz * n * (V ? 2 : 1) * sizeof(double);
      void* args[] = {&n, &bsz, &Aw, &Vw, &cnt, &ms, &tl, &sw};
      e = cudaLaunchCooperativeKernel((void*)jacobi_block_kernel, dim3(nblk), dim3(BT), args, smem, st); ttb_count();
    } else {
      int want = ceil_div((n + 1) / 2, CT / 32);  // one warp per pair
      int nblk = want < max_blocks ? want : max_blocks;
      if (nblk < 1) nblk = 1;
      void* args[] = {&n, &Aw, &Vw, &cnt, &ms, &tl, &sw};
      e = cudaLaunchCooperativeKernel((void*)jacobi_coop_kernel, dim3(nblk), dim3(CT), args, 0, st); ttb_count();
    }
    if (e != cudaSuccess) return (int)e;
    jacobi_finish_kernel<<<ceil_div((long long)n * 32, 256), 256, 0, st>>>(n, Aw, Vw, sig, S, U, V); ttb_count();
    jacobi_scatter_kernel<<<ceil_div((long long)n * 32, 256), 256, 0, st>>>(n, Aw, Vw, sig, S, U, V); ttb_count();
    if (info) cudaMemcpyAsync(info, sw, sizeof(int), cudaMemcpyDeviceToDevice, st);
  }
  return ttb_last_error();
}
