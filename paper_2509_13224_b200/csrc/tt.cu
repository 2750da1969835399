// TT operator kernels: banded operator-core x vector-core contraction (TT-matvec),
// the banded contractions inside AMEn (environment updates and the projected
// local operator), the projected dense local matrix, its Jacobi diagonal, TT
// entry gather, and a Jacobi-preconditioned CG that runs on the device with
// convergence flags (no per-iteration host round trip).
//
// Banded operator core layout: M[a, i, t, b] = A_k[a, i, i + t - h, b], shape
// (Ra, n, 2h+1, Rb); out-of-range (i+t-h outside [0,n)) slots are zero.
#include "common.cuh"

TTB_API int ttb_dgemm(void* stream, int tA, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
                      long long sA, const double* B, long long ldb, long long sB, double beta, double* C,
                      long long ldc, long long sC, int batch);

namespace {

int grid_for(long long tot, int threads = 256) {
  long long b = (tot + threads - 1) / threads;
  if (b > (long long)ttb_num_sms() * 16) b = (long long)ttb_num_sms() * 16;
  if (b < 1) b = 1;
  return (int)b;
}

// Y[(a,c), i, (b,d)] = sum_t M[a,i,t,b] X[c, i+t-h, d]
__global__ void band_matvec_kernel(int Ra, int Rb, int n, int h, int rc, int rd, const double* __restrict__ M,
                                   const double* __restrict__ X, double* __restrict__ Y) {
  const int B = 2 * h + 1;
  const long long tot = (long long)Ra * rc * n * Rb * rd;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int d = (int)(e % rd);
    long long rest = e / rd;
    const int b = (int)(rest % Rb);
    rest /= Rb;
    const int i = (int)(rest % n);
    rest /= n;
    const int c = (int)(rest % rc);
    const int a = (int)(rest / rc);
    double acc = 0.0;
    for (int t = 0; t < B; ++t) {
      const int j = i + t - h;
      if (j < 0 || j >= n) continue;
      acc += M[(((long long)a * n + i) * B + t) * Rb + b] * X[((long long)c * n + j) * rd + d];
    }
    Y[e] = acc;
  }
}

// fwd: out[x,i,b,w] = sum_{a,t} M[a,i,t,b] T[x,a,i+t-h,w]
// rev: out[x,i,a,w] = sum_{b,t} M[a,i,t,b] T[x,b,i+t-h,w]
__global__ void band_apply_kernel(int X, int Ra, int Rb, int n, int h, int W, const double* __restrict__ M,
                                  const double* __restrict__ T, double* __restrict__ out, int rev) {
  const int B = 2 * h + 1;
  const int Rin = rev ? Rb : Ra, Rout = rev ? Ra : Rb;
  const long long tot = (long long)X * n * Rout * W;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int w = (int)(e % W);
    long long rest = e / W;
    const int o = (int)(rest % Rout);
    rest /= Rout;
    const int i = (int)(rest % n);
    const int x = (int)(rest / n);
    double acc = 0.0;
    for (int t = 0; t < B; ++t) {
      const int j = i + t - h;
      if (j < 0 || j >= n) continue;
      for (int k = 0; k < Rin; ++k) {
        const int a = rev ? o : k, b = rev ? k : o;
        acc += M[(((long long)a * n + i) * B + t) * Rb + b] * T[(((long long)x * Rin + k) * n + j) * W + w];
      }
    }
    out[e] = acc;
  }
}

// dense projected matrix B[(x,i,z),(y,j,w)] = sum_b T1[x,y,i,t,b] phiR[z,b,w], j = i+t-h
// T1[x,y,i,t,b] = sum_a phiL[x,a,y] M[a,i,t,b]  (precomputed by GEMM)
__global__ void local_dense_kernel(int r0, int n, int r1, int h, int Rb, const double* __restrict__ T1,
                                   const double* __restrict__ phiR, double* __restrict__ Bm) {
  const int B = 2 * h + 1;
  const long long N = (long long)r0 * n * r1;
  const long long tot = (long long)r0 * n * r1 * r0 * B * r1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int w = (int)(e % r1);
    long long rest = e / r1;
    const int y = (int)(rest % r0);
    rest /= r0;
    const int t = (int)(rest % B);
    rest /= B;
    const int z = (int)(rest % r1);
    rest /= r1;
    const int i = (int)(rest % n);
    const int x = (int)(rest / n);
    const int j = i + t - h;
    if (j < 0 || j >= n) continue;
    double acc = 0.0;
    const double* tp = T1 + ((((long long)x * r0 + y) * n + i) * B + t) * Rb;
    const double* pp = phiR + (long long)z * Rb * r1 + w;
    for (int b = 0; b < Rb; ++b) acc += tp[b] * pp[(long long)b * r1];
    const long long row = ((long long)x * n + i) * r1 + z;
    const long long col = ((long long)y * n + j) * r1 + w;
    Bm[row * N + col] = acc;
  }
}

// d[x,i,z] = sum_{a,b} phiL[x,a,x] M[a,i,h,b] phiR[z,b,z]
__global__ void jacobi_diag_kernel(int r0, int n, int r1, int Ra, int Rb, int h, const double* __restrict__ phiL,
                                   const double* __restrict__ M, const double* __restrict__ phiR, double* d) {
  const int B = 2 * h + 1;
  const long long tot = (long long)r0 * n * r1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int z = (int)(e % r1);
    const int i = (int)((e / r1) % n);
    const int x = (int)(e / ((long long)r1 * n));
    double acc = 0.0;
    for (int a = 0; a < Ra; ++a) {
      const double l = phiL[((long long)x * Ra + a) * r0 + x];
      for (int b = 0; b < Rb; ++b)
        acc += l * M[(((long long)a * n + i) * B + h) * Rb + b] * phiR[((long long)z * Rb + b) * r1 + z];
    }
    d[e] = acc;
  }
}

// floor |d| at max|d| * 1e-14 (reference amen.py:179-181): d <- max(|d|, floor)
__global__ void abs_floor_kernel(long long n, double* d, const double* dmax) {
  const double fl = fmax(*dmax, 1e-300) * 1e-14;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double v = fabs(d[i]);
    d[i] = v < fl ? fl : v;
  }
}

__global__ void absmax_partial(long long n, const double* x, double* part) {
  __shared__ double sm[32];
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(x[i]));
  // block max via warp shuffles
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

__global__ void max_final(int np, const double* part, double* out) {
  double m = 0.0;
  for (int i = threadIdx.x; i < np; i += 32) m = fmax(m, part[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (threadIdx.x == 0) *out = m;
}

// ---------------------------------------------------------------------------
// PCG (scipy.sparse.linalg.cg semantics, reference amen.py:175-193)
// device scalars S: [0] rho, [1] rho_prev, [2] pq, [3] rr(||r||^2), [4] atol^2, [5] done flag, [6] iterations
constexpr int PB = 296;

__global__ void pcg_dot_partial(long long n, const double* __restrict__ x, const double* __restrict__ y,
                                const double* __restrict__ S, double* part) {
  if (S[5] != 0.0) return;
  __shared__ double sm[32];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += x[i] * y[i];
  s = block_sum(s, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void pcg_dot_final(int np, const double* part, double* S, int slot) {
  if (S[5] != 0.0) return;
  __shared__ double sm[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = block_sum(s, sm);
  if (threadIdx.x == 0) S[slot] = s;
}

// top of an iteration: if ||r|| < atol -> done. else z = r/d ; rho partials
__global__ void pcg_check_z(long long n, const double* __restrict__ r, const double* __restrict__ d, double* z,
                            double* S, double* part, int maxiter) {
  if (S[5] != 0.0) return;
  if (sqrt(S[3]) < sqrt(S[4]) || S[6] >= maxiter) {
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) S[7] = 1.0;  // request done (committed by pcg_commit)
    return;
  }
  __shared__ double sm[32];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double v = r[i] / d[i];
    z[i] = v;
    s += r[i] * v;
  }
  s = block_sum(s, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void pcg_commit(double* S) {
  if (S[7] != 0.0) S[5] = 1.0;
}

// p = z + beta p (beta = rho/rho_prev; first iteration p = z)
__global__ void pcg_update_p(long long n, const double* __restrict__ z, double* p, const double* S) {
  if (S[5] != 0.0) return;
  const bool first = S[6] == 0.0;
  const double beta = first ? 0.0 : S[0] / S[1];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = first ? z[i] : z[i] + beta * p[i];
}

// x += alpha p ; r -= alpha q ; rr partials
__global__ void pcg_update_xr(long long n, double* x, double* r, const double* __restrict__ p,
                              const double* __restrict__ q, const double* S, double* part) {
  if (S[5] != 0.0) return;
  __shared__ double sm[32];
  const double alpha = S[0] / S[2];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    double rv = r[i] - alpha * q[i];
    r[i] = rv;
    s += rv * rv;
  }
  s = block_sum(s, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void pcg_finish_iter(int np, const double* part, double* S) {
  if (S[5] != 0.0) return;
  __shared__ double sm[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = block_sum(s, sm);
  if (threadIdx.x == 0) {
    S[3] = s;
    S[1] = S[0];
    S[6] += 1.0;
  }
}

// r = b - r (r holds A x0), rr
__global__ void sub_from_kernel(long long n, const double* b, double* r, double* part) {
  __shared__ double sm[32];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double v = b[i] - r[i];
    r[i] = v;
    s += v * v;
  }
  s = block_sum(s, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void set_scalars(double* S, double atol2) {
  S[0] = S[1] = S[2] = 0.0;
  S[4] = atol2;
  S[5] = 0.0;
  S[6] = 0.0;
  S[7] = 0.0;
}

__global__ void gather_kernel(int N, int r1, int r2, const long long* __restrict__ idx, const double* __restrict__ G0,
                              int n0, const double* __restrict__ G1, int n1, const double* __restrict__ G2, int n2,
                              double* out) {
  // d = 3 chain: out[q] = G0[0,i0,:] G1[:,i1,:] G2[:,i2,0]; one warp per entry
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= N) return;
  const long long i0 = idx[3 * (long long)q], i1 = idx[3 * (long long)q + 1], i2 = idx[3 * (long long)q + 2];
  double acc = 0.0;
  for (int c = lane; c < r2; c += 32) {
    double s = 0.0;
    for (int b = 0; b < r1; ++b) s += G0[i0 * r1 + b] * G1[((long long)b * n1 + i1) * r2 + c];
    acc += s * G2[(long long)c * n2 + i2];
  }
  acc = warp_sum(acc);
  if (lane == 0) out[q] = acc;
}

// TT-cross index bookkeeping on the device (reference tensor_train/cross.py:88-100, 150-152, 178-180).
// Fiber multi-indices of the unfolding C[(l, i), r]: row (l nk + i) nr + r of out (d wide) is
// (left[l, 0..k), i, right[r, 0..w)), k + 1 + w = d.
__global__ void fiber_index_kernel(long long tot, int nk, int nr, int k, int w, const long long* __restrict__ left,
                                   const long long* __restrict__ right, long long* __restrict__ out) {
  const int d = k + 1 + w;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot * d; e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / d;
    const int c = (int)(e - row * d);
    const long long rr = row % nr, li = row / nr;
    const long long i = li % nk, l = li / nk;
    out[e] = c < k ? left[l * k + c] : (c == k ? i : right[rr * w + (c - k - 1)]);
  }
}
// Nested index sets from the maxvol rows sel of an unfolding with inner size q:
// side 0 (left set after a left-to-right step, rows ordered (l, i), q = n_k): out[s] = (src[sel[s] / q], sel[s] % q);
// side 1 (right set after a right-to-left step, rows ordered (i, r), q = n_r): out[s] = (sel[s] / q, src[sel[s] % q]).
__global__ void nested_index_kernel(int r, int q, int w, int side, const int* __restrict__ sel,
                                    const long long* __restrict__ src, long long* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= r * (w + 1)) return;
  const int s = e / (w + 1), c = e % (w + 1);
  const int v = sel[s];
  if (side == 0)
    out[e] = c < w ? src[(long long)(v / q) * w + c] : (long long)(v % q);
  else
    out[e] = c == 0 ? (long long)(v / q) : src[(long long)(v % q) * w + (c - 1)];
}

}  // namespace

TTB_API int ttb_fiber_index(void* stream, int nl, int nk, int nr, int k, int w, const long long* left,
                            const long long* right, long long* out) {
  const long long tot = (long long)nl * nk * nr;
  if (tot == 0) return TTB_OK;
  fiber_index_kernel<<<grid_for(tot * (k + 1 + w)), 256, 0, as_stream(stream)>>>(tot, nk, nr, k, w, left, right, out);
  ttb_count();
  return ttb_last_error();
}

TTB_API int ttb_nested_index(void* stream, int r, int q, int w, int side, const int* sel, const long long* src,
                             long long* out) {
  if (r == 0) return TTB_OK;
  nested_index_kernel<<<ceil_div(r * (w + 1), 256), 256, 0, as_stream(stream)>>>(r, q, w, side, sel, src, out);
  ttb_count();
  return ttb_last_error();
}

TTB_API int ttb_band_matvec(void* stream, int Ra, int Rb, int n, int h, int rc, int rd, const double* M,
                            const double* X, double* Y) {
  long long tot = (long long)Ra * rc * n * Rb * rd;
  if (tot == 0) return TTB_OK;
  band_matvec_kernel<<<grid_for(tot), 256, 0, as_stream(stream)>>>(Ra, Rb, n, h, rc, rd, M, X, Y); ttb_count();
  return ttb_last_error();
}

TTB_API int ttb_band_apply(void* stream, int X, int Ra, int Rb, int n, int h, int W, const double* M, const double* T,
                           double* out, int rev) {
  long long tot = (long long)X * n * (rev ? Ra : Rb) * W;
  if (tot == 0) return TTB_OK;
  band_apply_kernel<<<grid_for(tot), 256, 0, as_stream(stream)>>>(X, Ra, Rb, n, h, W, M, T, out, rev); ttb_count();
  return ttb_last_error();
}

// Bm must be zeroed by the caller (only band entries are written)
TTB_API int ttb_local_dense(void* stream, int r0, int n, int r1, int h, int Rb, const double* T1, const double* phiR,
                            double* Bm) {
  long long tot = (long long)r0 * n * r1 * r0 * (2 * h + 1) * r1;
  if (tot == 0) return TTB_OK;
  local_dense_kernel<<<grid_for(tot), 256, 0, as_stream(stream)>>>(r0, n, r1, h, Rb, T1, phiR, Bm); ttb_count();
  return ttb_last_error();
}

TTB_API int ttb_jacobi_diag(void* stream, int r0, int n, int r1, int Ra, int Rb, int h, const double* phiL,
                            const double* M, const double* phiR, double* d, double* part) {
  long long tot = (long long)r0 * n * r1;
  cudaStream_t st = as_stream(stream);
  jacobi_diag_kernel<<<grid_for(tot), 256, 0, st>>>(r0, n, r1, Ra, Rb, h, phiL, M, phiR, d); ttb_count();
  int nb = grid_for(tot) < PB ? grid_for(tot) : PB;
  absmax_partial<<<nb, 256, 0, st>>>(tot, d, part); ttb_count();
  max_final<<<1, 32, 0, st>>>(nb, part, part + PB); ttb_count();
  abs_floor_kernel<<<grid_for(tot), 256, 0, st>>>(tot, d, part + PB); ttb_count();
  return ttb_last_error();
}

// d = max(|d|, 1e-14 max|d|) in place (the reference's Jacobi floor, amen.py:179-181); part >= 320 doubles
TTB_API int ttb_abs_floor(void* stream, long long tot, double* d, double* part) {
  cudaStream_t st = as_stream(stream);
  int nb = grid_for(tot) < PB ? grid_for(tot) : PB;
  absmax_partial<<<nb, 256, 0, st>>>(tot, d, part); ttb_count();
  max_final<<<1, 32, 0, st>>>(nb, part, part + PB); ttb_count();
  abs_floor_kernel<<<grid_for(tot), 256, 0, st>>>(tot, d, part + PB); ttb_count();
  return ttb_last_error();
}

TTB_API int ttb_tt_gather3(void* stream, int N, const long long* idx, const double* G0, int n0, int r1,
                           const double* G1, int n1, int r2, const double* G2, int n2, double* out) {
  if (N == 0) return TTB_OK;
  gather_kernel<<<ceil_div(N, 8), 256, 0, as_stream(stream)>>>(N, r1, r2, idx, G0, n0, G1, n1, G2, n2, out); ttb_count();
  return ttb_last_error();
}

// Local projected operator y = phiL * A_k * phiR applied to v (reference _LocalSystem.matvec3):
//   t1[x,a,j,w] = sum_y phiL[x,a,y] v[y,j,w]; t2 = band_apply(M, t1); y[x,i,z] = sum_{b,w} t2[x,i,b,w] phiR[z,b,w]
// ws: r0*Ra*n*r1 + r0*n*Rb*r1 doubles
TTB_API int ttb_local_matvec(void* stream, int r0, int n, int r1, int Ra, int Rb, int h, const double* phiL,
                             const double* M, const double* phiR, const double* v, double* y, double* ws) {
  double* t1 = ws;
  double* t2 = ws + (long long)r0 * Ra * n * r1;
  int rc = ttb_dgemm(stream, 0, 0, r0 * Ra, n * r1, r0, 1.0, phiL, r0, 0, v, (long long)n * r1, 0, 0.0, t1,
                     (long long)n * r1, 0, 1);
  if (rc) return rc;
  rc = ttb_band_apply(stream, r0, Ra, Rb, n, h, r1, M, t1, t2, 0);
  if (rc) return rc;
  return ttb_dgemm(stream, 0, 1, r0 * n, r1, Rb * r1, 1.0, t2, (long long)Rb * r1, 0, phiR, (long long)Rb * r1, 0,
                   0.0, y, r1, 0, 1);
}

TTB_API long long ttb_pcg_workspace(int r0, int n, int r1, int Ra, int Rb) {
  long long N = (long long)r0 * n * r1;
  return 4 * N + (long long)r0 * Ra * n * r1 + (long long)r0 * n * Rb * r1 + 2 * PB + 16;
}

// ---------------------------------------------------------------------------
// Banded operator contractions as batched DMMA GEMMs (large operator ranks).
//
// With the operator core re-laid out as Mf[i, t, a, b] = M[a, i, t, b] (or Mr[i, t, b, a] for the
// reverse direction) and the vector-side operand as Tp[j + h, a, X] (j-major, h zero blocks of
// padding on both ends), the banded contraction
//     out[i, X, b] = sum_{t, a} Tp[i + t, a, X] Mf[i, t, a, b]
// is, for every mode index i, one GEMM whose K = (2h+1) Ra operand is the contiguous window of
// Tp rows starting at block i: C_i (X x Rb) = Tp_window_i^T (X x K) * Mf_i (K x Rb).
// The padding blocks of Tp must be zero (they meet the zero out-of-band slots of Mf).
TTB_API long long ttb_band_gemm_ozaki_workspace(int n, int h, int Rin, int Rout, int X, int G);
TTB_API int ttb_band_gemm_ozaki(void* stream, int n, int h, int Rin, int Rout, int X, const double* Tp,
                                const double* Mt, double* out, void* ws, int G);
double* ttb_scratch(size_t bytes, cudaStream_t st);

// Large band contractions (>= 2e10 flop, X >= 128, K <= 4096) run as Ozaki-scheme FP64 on the int8
// tensor cores (ozaki.cu ttb_band_gemm_ozaki: 1.9x the DMMA batch at the configs[3] local shape, 1.2-1.4x
// from 2-3e10 flop, break-even below; tools/bench_band_ozaki.py);
// TTB_BAND_OZAKI=0 keeps every band GEMM on DMMA, TTB_BAND_OZ_G sets the A slice group size (32).
static int band_oz_group() {
  static int g = -1;
  if (g < 0) {
    const char* e = getenv("TTB_BAND_OZAKI");
    const char* eg = getenv("TTB_BAND_OZ_G");
    g = (e && e[0] == '0') ? 0 : (eg ? atoi(eg) : 32);
    if (g < 0) g = 0;
  }
  return g;
}

TTB_API int ttb_band_gemm(void* stream, int n, int h, int Rin, int Rout, int X, const double* Tp, const double* Mt,
                          double* out) {
  const int B = 2 * h + 1;
  const int G = band_oz_group();
  const double flop = 2.0 * n * (double)X * Rout * B * Rin;
  if (G > 0 && flop >= 2.0e10 && X >= 128 && B * Rin <= 4096) {
    cudaStream_t st = as_stream(stream);
    void* ws = ttb_scratch((size_t)ttb_band_gemm_ozaki_workspace(n, h, Rin, Rout, X, G), st);
    if (ws) return ttb_band_gemm_ozaki(stream, n, h, Rin, Rout, X, Tp, Mt, out, ws, G);
  }
  return ttb_dgemm(stream, 1, 0, X, Rout, B * Rin, 1.0, Tp, X, (long long)Rin * X, Mt, Rout,
                   (long long)B * Rin * Rout, 0.0, out, Rout, (long long)X * Rout, n);
}

// The staged operand's column count X = r0 r1p is kept even (r1p = r1 + 1 when r0 and r1 are
// both odd, the extra w column staying zero) so both band-GEMM operands take the 16-byte path.
static inline int local_r1p(int r0, int r1) { return r1 + (r0 & r1 & 1); }

TTB_API long long ttb_local_gemm_workspace(int r0, int n, int r1, int Ra, int Rb, int h) {
  const int r1p = local_r1p(r0, r1);
  return (long long)(n + 2 * h) * Ra * r0 * r1p + (long long)n * r0 * r1p * Rb;
}

// Local projected operator in the mode-major (i, x, z) vector layout, three GEMM stages:
//   Tp[j+h, a, x, w] = sum_y phiLp[a, x, y] v[j, y, w]           (batched over j)
//   t2[i, x, w, b]   = band_gemm(Tp, Mf)                           (batched over i)
//   y[i, x, z]       = sum_{w, b} t2[i, x, w, b] phiRp[z, w, b]    (one GEMM)
// phiLp = phiL permuted to (a, x, y); phiRp = phiR permuted to (z, w, b) and zero-padded to
// (r1, r1p, Rb) with r1p = r1 + (r0 & r1 & 1); Mf (n, 2h+1, Ra, Rb) (Rb may carry zero padding).
// ws (ttb_local_gemm_workspace doubles) must be initialised once by ttb_local_gemm_ws_init (zero
// padding blocks / columns of the staged operand); the rest is overwritten every call.
TTB_API int ttb_local_gemm_ws_init(void* stream, int r0, int n, int r1, int Ra, int h, double* ws) {
  const int r1p = local_r1p(r0, r1);
  const long long blk = (long long)Ra * r0 * r1p;
  cudaStream_t st = as_stream(stream);
  if (r1p != r1) {
    cudaMemsetAsync(ws, 0, (size_t)(n + 2 * h) * blk * sizeof(double), st);
  } else if (h > 0) {
    cudaMemsetAsync(ws, 0, (size_t)h * blk * sizeof(double), st);
    cudaMemsetAsync(ws + (long long)(n + h) * blk, 0, (size_t)h * blk * sizeof(double), st);
  }
  return ttb_last_error();
}

TTB_API int ttb_local_matvec_gemm(void* stream, int r0, int n, int r1, int Ra, int Rb, int h, const double* phiLp,
                                  const double* Mf, const double* phiRp, const double* v, double* y, double* ws) {
  const int r1p = local_r1p(r0, r1);
  const long long blk = (long long)Ra * r0 * r1p;
  double* Tp = ws;
  double* t2 = ws + (long long)(n + 2 * h) * blk;
  int rc = ttb_dgemm(stream, 0, 0, Ra * r0, r1, r0, 1.0, phiLp, r0, 0, v, r1, (long long)r0 * r1, 0.0,
                     Tp + (long long)h * blk, r1p, blk, n);
  if (rc) return rc;
  rc = ttb_band_gemm(stream, n, h, Ra, Rb, r0 * r1p, Tp, Mf, t2);
  if (rc) return rc;
  return ttb_dgemm(stream, 0, 1, n * r0, r1, r1p * Rb, 1.0, t2, (long long)r1p * Rb, 0, phiRp, (long long)r1p * Rb, 0,
                   0.0, y, r1, 0, 1);
}

namespace {

// Jacobi-PCG on the local system with scipy.sparse.linalg.cg stopping semantics; MV(p, q) applies
// the local operator. ws: 4N (+ matvec workspace owned by MV) + 2 PB + 16 doubles after it.
template <class MV>
int pcg_run(cudaStream_t st, long long N, const MV& mv, const double* b, double* x, const double* d, double atol,
            int maxiter, int x0_nonzero, double* ws, double* part, double* S, int* iters, int chunk) {
  double* r = ws;
  double* z = r + N;
  double* p = z + N;
  double* q = p + N;
  const int nb = grid_for(N) < PB ? grid_for(N) : PB;
  set_scalars<<<1, 1, 0, st>>>(S, atol * atol); ttb_count();
  int rc;
  if (x0_nonzero) {
    rc = mv(x, r);
    if (rc) return rc;
    sub_from_kernel<<<nb, 256, 0, st>>>(N, b, r, part); ttb_count();
  } else {
    cudaMemsetAsync(x, 0, N * sizeof(double), st);
    cudaMemcpyAsync(r, b, N * sizeof(double), cudaMemcpyDeviceToDevice, st);
    pcg_dot_partial<<<nb, 256, 0, st>>>(N, r, r, S, part); ttb_count();
  }
  pcg_dot_final<<<1, 256, 0, st>>>(nb, part, S, 3); ttb_count();
  // iterations are enqueued `chunk` at a time between host checks of the device done-flag (the
  // kernels of a finished solve still run, as no-ops on x); chunk = 1 when one matvec costs far more
  // than a host round trip
  double host[8];
  for (int it0 = 0; it0 <= maxiter; it0 += chunk) {
    for (int k = 0; k < chunk; ++k) {
      pcg_check_z<<<nb, 256, 0, st>>>(N, r, d, z, S, part, maxiter); ttb_count();
      pcg_commit<<<1, 1, 0, st>>>(S); ttb_count();
      pcg_dot_final<<<1, 256, 0, st>>>(nb, part, S, 0); ttb_count();
      pcg_update_p<<<grid_for(N), 256, 0, st>>>(N, z, p, S); ttb_count();
      // q = A p   (skipped work when done: kernels still run but results unused)
      rc = mv(p, q);
      if (rc) return rc;
      pcg_dot_partial<<<nb, 256, 0, st>>>(N, p, q, S, part); ttb_count();
      pcg_dot_final<<<1, 256, 0, st>>>(nb, part, S, 2); ttb_count();
      pcg_update_xr<<<nb, 256, 0, st>>>(N, x, r, p, q, S, part); ttb_count();
      pcg_finish_iter<<<1, 256, 0, st>>>(nb, part, S); ttb_count();
    }
    cudaMemcpyAsync(host, S, 8 * sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (host[5] != 0.0) break;
  }
  if (iters) *iters = (int)host[6];
  return ttb_last_error();
}

}  // namespace

// Jacobi-PCG on the local system; x holds x0 on entry (x0_nonzero says whether to form b - A x0).
// d: preconditioner diagonal (already floored). Returns iterations in *iters.
TTB_API int ttb_local_pcg(void* stream, int r0, int n, int r1, int Ra, int Rb, int h, const double* phiL,
                          const double* M, const double* phiR, const double* b, double* x, const double* d,
                          double atol, int maxiter, int x0_nonzero, double* ws, double* S, int* iters) {
  const long long N = (long long)r0 * n * r1;
  double* mvws = ws + 4 * N;
  double* part = mvws + (long long)r0 * Ra * n * r1 + (long long)r0 * n * Rb * r1;
  auto mv = [&](const double* in, double* out) {
    return ttb_local_matvec(stream, r0, n, r1, Ra, Rb, h, phiL, M, phiR, in, out, mvws);
  };
  return pcg_run(as_stream(stream), N, mv, b, x, d, atol, maxiter, x0_nonzero, ws, part, S, iters, 8);
}

TTB_API long long ttb_pcg_gemm_workspace(int r0, int n, int r1, int Ra, int Rb, int h) {
  return 4LL * r0 * n * r1 + ttb_local_gemm_workspace(r0, n, r1, Ra, Rb, h) + 2 * PB + 16;
}

// Same PCG with vectors in the (i, x, z) layout and the GEMM-staged local operator
// (ttb_local_matvec_gemm); ws: ttb_pcg_gemm_workspace doubles, its matvec part initialised by
// ttb_local_gemm_ws_init at offset 4 r0 n r1.
TTB_API int ttb_local_pcg_gemm(void* stream, int r0, int n, int r1, int Ra, int Rb, int h, const double* phiLp,
                               const double* Mf, const double* phiRp, const double* b, double* x, const double* d,
                               double atol, int maxiter, int x0_nonzero, double* ws, double* S, int* iters) {
  const long long N = (long long)r0 * n * r1;
  double* mvws = ws + 4 * N;
  double* part = mvws + ttb_local_gemm_workspace(r0, n, r1, Ra, Rb, h);
  auto mv = [&](const double* in, double* out) {
    return ttb_local_matvec_gemm(stream, r0, n, r1, Ra, Rb, h, phiLp, Mf, phiRp, in, out, mvws);
  };
  const double mv_flops = 2.0 * N * (2 * h + 1) * Ra * Rb;
  return pcg_run(as_stream(stream), N, mv, b, x, d, atol, maxiter, x0_nonzero, ws, part, S, iters,
                 mv_flops > 2e9 ? 1 : mv_flops > 2e8 ? 2 : 8);
}

// ---------------------------------------------------------------------------
// Banded direct solve of the projected AMEn system. In the (i, x, z) ordering
// (mode index outermost) the local matrix B = phiL (x) A_k (x) phiR is banded with
// half-bandwidth bw = (h+1) r0 r1 - 1, so its Cholesky costs N bw^2 instead of N^3.
// The solution of the permuted system is the reference's (amen.py:164-172) up to roundoff.
namespace {

// LB[row * (bw+1) + d] = B[row, row - d] (lower band), rows/cols in (i, x, z) order
__global__ void local_band_build_kernel(int r0, int n, int r1, int h, int Rb, int bw, const double* __restrict__ T1,
                                        const double* __restrict__ phiR, double* __restrict__ LB) {
  const int B = 2 * h + 1;
  const long long N = (long long)r0 * n * r1;
  const long long tot = N * (bw + 1);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int d = (int)(e % (bw + 1));
    const long long row = e / (bw + 1);
    const long long col = row - d;
    double acc = 0.0;
    if (col >= 0) {
      const int z = (int)(row % r1), x = (int)((row / r1) % r0), i = (int)(row / ((long long)r1 * r0));
      const int w = (int)(col % r1), y = (int)((col / r1) % r0), j = (int)(col / ((long long)r1 * r0));
      const int t = j - i + h;
      if (t >= 0 && t < B) {
        const double* tp = T1 + ((((long long)x * r0 + y) * n + i) * B + t) * Rb;
        const double* pp = phiR + (long long)z * Rb * r1 + w;
        for (int b = 0; b < Rb; ++b) acc += tp[b] * pp[(long long)b * r1];
      }
    }
    LB[e] = acc;
  }
}

// in-place banded Cholesky (lower) + forward/backward solve of b; one CTA
__global__ void __launch_bounds__(256) band_chol_solve_kernel(long long N, int bw, double* LB, double* b, int* info) {
  __shared__ int bad;
  const int W = bw + 1;
  if (threadIdx.x == 0) { bad = 0; *info = 0; }
  __syncthreads();
  for (long long k = 0; k < N; ++k) {
    const double dkk = LB[k * W];
    if (!(dkk > 0.0) || !isfinite(dkk)) {
      if (threadIdx.x == 0) { bad = 1; *info = (int)(k + 1); }
      __syncthreads();
      return;
    }
    const double lkk = sqrt(dkk);
    const int m = (int)min((long long)bw, N - 1 - k);
    // column k below the diagonal: L[k+q, k] = A[k+q, k] / lkk, stored at LB[(k+q)*W + q]
    for (int q = 1 + threadIdx.x; q <= m; q += blockDim.x) LB[(k + q) * W + q] /= lkk;
    __syncthreads();
    if (threadIdx.x == 0) LB[k * W] = lkk;
    // trailing update inside the band: A[k+q, k+s] -= L[k+q,k] L[k+s,k], 1 <= s <= q <= m
    const int pairs = m * (m + 1) / 2;
    for (int e = threadIdx.x; e < pairs; e += blockDim.x) {
      int q = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while ((q + 1) * (q + 2) / 2 <= e) ++q;
      while (q * (q + 1) / 2 > e) --q;
      const int s = e - q * (q + 1) / 2;  // 0..q
      const int qq = q + 1, ss = s + 1;   // 1-based offsets
      LB[(k + qq) * W + (qq - ss)] -= LB[(k + qq) * W + qq] * LB[(k + ss) * W + ss];
    }
    __syncthreads();
  }
  // forward: L y = b (one warp)
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (long long k = 0; k < N; ++k) {
      double s = 0.0;
      for (int q = 1 + lane; q <= bw && q <= k; q += 32) s += LB[k * W + q] * b[k - q];
      s = warp_sum(s);
      if (lane == 0) b[k] = (b[k] - s) / LB[k * W];
      __syncwarp();
    }
    // backward: L^T x = y
    for (long long k = N - 1; k >= 0; --k) {
      double s = 0.0;
      for (int q = 1 + lane; q <= bw && k + q < N; q += 32) s += LB[(k + q) * W + q] * b[k + q];
      s = warp_sum(s);
      if (lane == 0) b[k] = (b[k] - s) / LB[k * W];
      __syncwarp();
    }
  }
}

// Blocked banded Cholesky + solves in one CTA with a shared-memory window (bw <= 127, N <= 8192).
// Storage as band_chol_solve_kernel: LB[i*W + q] = A[i][i-q], W = bw + 1. The window holds rows
// [k0, k0 + NBB + bw) plus the NBB rows of the next block, prefetched while the current block is
// processed (circular, WRC = 2 NBB + bw slots); per block of NBB columns: warp 0 factors the panel,
// all warps apply the rank-NBB update of the band triangle, finished rows stream out. Solves
// stream rows through staged chunks; b lives in shared memory; the forward solve takes blocks of
// NBB rows (band dots in parallel over warps, then the NBB x NBB triangle).
#ifndef TTB_BAND_NBB
#define TTB_BAND_NBB 8
#endif
constexpr int BCT = 256, NBB = TTB_BAND_NBB, BCH = 64;

__global__ void __launch_bounds__(BCT) band_chol_blocked_kernel(int N, int bw, double* LB, double* b, int* info) {
  extern __shared__ double sm[];
  const int W = bw + 1;
  const int WRC = 2 * NBB + bw;
  const int WROWS = max(WRC, BCH);
  double* win = sm;                               // WRC x W (factorization) / BCH x W (solves)
  double* bs = sm + (long long)WROWS * W;         // N
  __shared__ int bad;
  __shared__ double dot[NBB], rinv[BCH];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) { bad = 0; *info = 0; }
  auto row = [&](int i) { return win + (long long)(i % WRC) * W; };
  // rows [0, NBB + bw) now, rows [NBB + bw, 2 NBB + bw) as the prefetch of block 1
  const int r0n = min(N, WRC);
  for (int e = tid; e < r0n * W; e += BCT) win[e] = LB[e];
  __syncthreads();
  for (int k0 = 0; k0 < N; k0 += NBB) {
    const int nb = min(NBB, N - k0);
    asm volatile("cp.async.wait_group 1;\n" ::);  // rows prefetched two blocks ago have landed
    __syncthreads();
    if (warp == 0) {
      for (int c = k0; c < k0 + nb; ++c) {
        double* rc = row(c);
        const double d = rc[0];
        if (!(d > 0.0) || !isfinite(d)) {
          if (lane == 0) { bad = 1; *info = c + 1; }
          break;
        }
        const double l = sqrt(d), il = 1.0 / l;
        const int iend = min(N - 1, c + bw);
        for (int i = c + 1 + lane; i <= iend; i += 32) row(i)[i - c] *= il;
        __syncwarp();
        if (lane == 0) rc[0] = l;
        for (int c2 = c + 1; c2 < k0 + nb; ++c2) {
          const double lc2 = row(c2)[c2 - c];
          for (int i = c2 + lane; i <= iend; i += 32) row(i)[i - c2] -= row(i)[i - c] * lc2;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (bad) return;
    const int ib = k0 + nb, ie = min(N - 1, k0 + nb - 1 + bw);
    for (int i = ib + warp; i <= ie; i += BCT / 32) {
      double* ri = row(i);
      double li[NBB];
      const int cmin = max(k0, i - bw);
#pragma unroll
      for (int t = 0; t < NBB; ++t) {
        const int c = k0 + t;
        li[t] = (t < nb && c >= cmin) ? ri[i - c] : 0.0;
      }
      for (int j = max(ib, i - bw) + lane; j <= i; j += 32) {
        const double* rj = row(j);
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < NBB; ++t) {
          const int c = k0 + t;
          if (t < nb && c >= cmin) acc += li[t] * rj[j - c];
        }
        ri[i - j] -= acc;
      }
    }
    __syncthreads();
    // finished rows out; their slots take the rows of block + 2 (prefetch one block ahead)
    for (int e = tid; e < nb * W; e += BCT) {
      const int t = e / W, q = e % W;
      const int i = k0 + t;
      double* slot = row(i);
      LB[(long long)i * W + q] = slot[q];
      const int inew = i + WRC;
      if (inew < N) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(slot + q);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(LB + (long long)inew * W + q));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  for (int e = tid; e < N; e += BCT) bs[e] = b[e];
  __syncthreads();
  // forward L y = b in blocks of NBB rows
  for (int c0 = 0; c0 < N; c0 += BCH) {
    const int cn = min(BCH, N - c0);
    for (int e = tid; e < cn * W; e += BCT) win[e] = LB[(long long)c0 * W + e];
    __syncthreads();
    for (int e = tid; e < cn; e += BCT) rinv[e] = 1.0 / win[(long long)e * W];
    for (int k = c0; k < c0 + cn; k += NBB) {
      const int kn = min(NBB, c0 + cn - k);
      // contributions of rows before the block: one warp per row
      if (warp < kn) {
        const int r = k + warp;
        const double* rr = win + (long long)(r - c0) * W;
        double s = 0.0;
        for (int q = (r - k) + 1 + lane; q <= bw && q <= r; q += 32) s += rr[q] * bs[r - q];
        s = warp_sum(s);
        if (lane == 0) dot[warp] = s;
      }
      __syncthreads();
      if (tid == 0) {
        for (int t = 0; t < kn; ++t) {
          const int r = k + t;
          const double* rr = win + (long long)(r - c0) * W;
          double v = bs[r] - dot[t];
          for (int u = 0; u < t; ++u)
            if (t - u <= bw) v -= rr[t - u] * bs[k + u];
          bs[r] = v * rinv[r - c0];
        }
      }
      __syncthreads();
    }
  }
  // backward L^T x = y, row-oriented: x_k = y_k / L_kk, then y_{k-q} -= L[k][k-q] x_k
  for (int c1 = N; c1 > 0; c1 -= BCH) {
    const int c0 = max(0, c1 - BCH);
    const int cn = c1 - c0;
    for (int e = tid; e < cn * W; e += BCT) win[e] = LB[(long long)c0 * W + e];
    __syncthreads();
    for (int e = tid; e < cn; e += BCT) rinv[e] = 1.0 / win[(long long)e * W];
    __syncthreads();
    if (warp == 0) {
      for (int k = c1 - 1; k >= c0; --k) {
        const double* rk = win + (long long)(k - c0) * W;
        const double xk = bs[k] * rinv[k - c0];
        __syncwarp();
        if (lane == 0) bs[k] = xk;
        for (int q = 1 + lane; q <= bw && q <= k; q += 32) bs[k - q] -= rk[q] * xk;
        __syncwarp();
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < N; e += BCT) b[e] = bs[e];
}

}  // namespace

TTB_API int ttb_local_band_build(void* stream, int r0, int n, int r1, int h, int Rb, const double* T1,
                                 const double* phiR, double* LB) {
  const int bw = (h + 1) * r0 * r1 - 1;
  const long long tot = (long long)r0 * n * r1 * (bw + 1);
  if (tot == 0) return TTB_OK;
  local_band_build_kernel<<<grid_for(tot), 256, 0, as_stream(stream)>>>(r0, n, r1, h, Rb, bw, T1, phiR, LB); ttb_count();
  return ttb_last_error();
}

TTB_API int ttb_band_chol_solve(void* stream, long long N, int bw, double* LB, double* b, int* info) {
  if (N < 1 || bw < 0) return TTB_EARG;
  const size_t rows = (size_t)((2 * NBB + bw) > BCH ? (2 * NBB + bw) : BCH);
  const size_t smem = (rows * (bw + 1) + (size_t)N) * sizeof(double);
  if (bw <= 127 && N <= 8192 && smem <= 200 * 1024) {
    static bool cfg = false;
    if (!cfg) {
      cudaFuncSetAttribute(band_chol_blocked_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cfg = true;
    }
    band_chol_blocked_kernel<<<1, BCT, smem, as_stream(stream)>>>((int)N, bw, LB, b, info); ttb_count();
    return ttb_last_error();
  }
  band_chol_solve_kernel<<<1, 256, 0, as_stream(stream)>>>(N, bw, LB, b, info); ttb_count();
  return ttb_last_error();
}
