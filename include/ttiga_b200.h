/*
 * ttiga_b200.h -- C ABI of libttiga_b200.so, the sm_100a TT-IGA hot path.
 *
 * Plain pointers and sizes only (no torch types). Every pointer argument is a
 * DEVICE pointer unless noted; `stream` is a cudaStream_t passed as void*.
 * Matrices are FP64; "col-major" follows LAPACK, otherwise row-major (C order,
 * the layout of numpy/torch TT cores). Return value: 0 ok, >0 CUDA error code,
 * <0 argument/numerical status (see TTB_E* below).
 *
 * Each entry point names the reference interface it replaces
 * (reference tree: arxiv/paper_2509_13224, pkg/src/ttiga/...).
 */
#ifndef TTIGA_B200_H
#define TTIGA_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define TTB_OK 0
#define TTB_EARG (-1)
#define TTB_ENOTPD (-2)
#define TTB_ESINGULAR (-3)

/* Number of kernels this library launched since the last reset (host counter; bench.py evidence). */
long long ttb_launch_count(int reset);

/* ---- dense FP64 building blocks ------------------------------------------------------------ */

/* C[b] = alpha * op(A[b]) op(B[b]) + beta * C[b], row-major, strided batch.
 * Replaces the np.einsum / np.tensordot contractions of tensor_train/core.py:300,335,373,388
 * and tensor_train/amen.py:106-123,147-150,152-156. DMMA (mma.sync m8n8k4 f64) tiles, split-K when the
 * output is too small to fill the 148 SMs. */
int ttb_dgemm(void* stream, int tA, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
              long long sA, const double* B, long long ldb, long long sB, double beta, double* C, long long ldc,
              long long sC, int batch);

/* dst = src.transpose(perm) for a row-major nd-array (nd <= 8); in_dims is a HOST array. */
int ttb_permute(void* stream, int nd, const long long* in_dims, const int* perm, const double* src, double* dst);

/* out[0] = x.y (y == NULL: ||x||^2; take_sqrt: ||x||). part: >= 296 doubles scratch. Deterministic. */
int ttb_dot(void* stream, long long n, const double* x, const double* y, double* out, double* part, int take_sqrt);

/* ---- Householder QR / SVD / solvers (np.linalg.qr, np.linalg.svd, np.linalg.solve,
 *      scipy.linalg.cho_factor/cho_solve as used by tensor_train/core.py:316,371,384,
 *      tensor_train/cross.py:170,188,190, tensor_train/amen.py:168-171, assembly.py:412-413) -- */

long long ttb_qr_workspace(int m, int n); /* doubles */
/* In-place blocked Householder QR of col-major A (m x n, lda); tau: min(m,n). */
int ttb_geqrf(void* stream, int m, int n, double* A, long long lda, double* tau, double* ws);
/* Explicit Q (m x kq, col-major) from ttb_geqrf (same ws); kf = reflector count, n_factored = n of geqrf. */
int ttb_orgqr(void* stream, int m, int kq, int kf, const double* A, long long lda, double* Q, long long ldq, double* ws,
              int n_factored);
/* Single-CTA shared-memory QR for TT-rank-sized unfoldings (n <= 64, m*n + m*min(m,n) <= 24576):
 * ttb_qr_small_fits(m, n) says whether it applies; Q (nullable) m x k col-major, R k x n col-major. */
int ttb_qr_small_fits(int m, int n);
int ttb_qr_small(void* stream, int m, int n, const double* A, long long lda, double* Q, long long ldq, double* R);
/* R (k x n col-major) = upper triangle of the geqrf result. */
int ttb_extract_r(void* stream, int k, int n, const double* A, long long lda, double* R);

/* One-sided Jacobi SVD of `batch` n x n col-major matrices: A = U diag(S) V^T, S descending.
 * work: batch*(2n^2+n) doubles when n > 64 (shared memory otherwise); info: sweeps per matrix (nullable). */
int ttb_svd_jacobi(void* stream, int n, double* A, long long strideA, double* S, long long strideS, double* U,
                   double* V, long long strideUV, int batch, double* work, int* info);

/* LU with partial pivoting (in place, col-major) and solve of op(A) X = B (B col-major n x nrhs). */
int ttb_lu_solve(void* stream, int n, double* A, long long lda, int* piv, int nrhs, double* B, long long ldb,
                 int trans, int* info);
/* Banded LU WITHOUT pivoting (totally positive matrices, e.g. B-spline collocation at Greville
 * points, assembly.py:409-413) and solve of A X = B for nrhs columns (in place). */
int ttb_band_lu_solve(void* stream, int n, int kl, int ku, double* A, long long lda, int nrhs, double* B,
                      long long ldb);
/* Blocked Cholesky (lower, col-major) ; *info > 0 on a non-positive pivot (device int). */
int ttb_potrf(void* stream, int n, double* A, long long lda, int* info);
/* Solve L L^T x = b in place (n <= 25600). */
int ttb_potrs(void* stream, int n, const double* L, long long lda, double* b);

/* ---- maxvol (tensor_train/maxvol.py:37-62) --------------------------------------------------- */
long long ttb_maxvol_workspace(int n, int r); /* doubles */
/* rows_out: r sorted row indices of a tol-dominant r x r submatrix of Q (n x r col-major), n > r.
 * iws: n + 1 ints; iws[n] = 1 on a rank-deficient input (reference MaxvolError). Cooperative launch. */
int ttb_maxvol(void* stream, int n, int r, const double* Q, double tol, int max_iters, int* rows_out, double* ws,
               int* iws);

/* ---- IGA kernels (splines.py:146-221, geometry.py:150-261, assembly.py:208-233, driver.py:388-422) */

/* Nonzero basis values/derivatives at nq parameters (Cox-de Boor; NURBS when weights != NULL).
 * first: int[nq]; V, D: nq x (p+1). bad: device int, min'ed with the first out-of-range index. */
int ttb_basis_eval(void* stream, int nq, const double* x, const double* knots, int nk, int p, const double* weights,
                   int* first, double* V, double* D, int* bad);

/* min det J over the full nq0 x nq1 x nq2 tensor grid of the windows (f_d, V_d, D_d) (admissibility of the
 * seeded random geometry at every Gauss point of the solve, BASELINE configs[3]). out (device, 2 x u64):
 * out[0] = order-preserving key of min det J (decode: k >> 63 ? bits k ^ 2^63 : bits ~k), out[1] = number of
 * points with det J <= 0. No reference counterpart (configs[3]'s geometry is a BASELINE extension). */
int ttb_geo_min_det(void* stream, int nq0, int nq1, int nq2, const int* f0, const int* f1, const int* f2,
                    const double* V0, const double* V1, const double* V2, const double* D0, const double* D1,
                    const double* D2, int p0, int p1, int p2, int n0, int n1, int n2, const double* cw,
                    unsigned long long* out);

/* Rational geometry map at N grid multi-indices idx (int64, N x 3) of a tensor grid whose per-direction
 * basis windows are (f_d, V_d, D_d). cw: control grid (n0, n1, n2, 4) = (w x, w y, w z, w).
 * mode 0: out[k] = R[ri][rj], R = J^-1 J^-T det J       (assembly.metric_oracle)
 * mode 1: out[k] = f(x) det J, f = source id `src`      (assembly.load_oracle)
 * mode 2: out[22 k ...] = J (9), x (3), det, R (9)        (GridEvaluator.jacobians/metric)
 * mode 3: out[3 k ...] = x                                (GridEvaluator.points)
 * bad: device int64, min'ed with the first index where |det J| < sing_tol (SingularMapError). */
int ttb_geo_eval(void* stream, long long N, const long long* idx, const int* f0, const int* f1, const int* f2,
                 const double* V0, const double* V1, const double* V2, const double* D0, const double* D1,
                 const double* D2, int p0, int p1, int p2, int n0, int n1, int n2, const double* cw, double sing_tol,
                 int mode, int ri, int rj, int src, double* out, long long* bad);

/* Banded operator core from a quadrature-grid TT core G (r, nq, s) (reference assembly.py:208-222):
 * out[a, i, t, b] = sum_q G[a,q,b] w[q] X[q, i-first[q]] Y[q, j-first[q]], j = i+t-h, out (r, n, 2h+1, s).
 * first[] must be non-decreasing in q (Gauss points ordered by element). One CTA per (a, tile of basis
 * indices): the tile's quadrature window of G, w, X, Y staged in shared memory, each output reduced by
 * 4 lanes with warp shuffles. */
int ttb_op_core(void* stream, int r, int nq, int s, const double* G, const double* w, const int* first,
                const double* X, const double* Y, int p, int n, int h, double* out);
/* Load core (reference assembly.py:225-233): out[a, i, b] = sum_q G[a,q,b] w[q] V[q, i-first[q]] (same scheme). */
int ttb_vec_core(void* stream, int r, int nq, int s, const double* G, const double* w, const int* first,
                 const double* V, int p, int n, double* out);
/* The previous one-thread-per-output forms of ttb_op_core / ttb_vec_core (A/B comparisons and tests). */
int ttb_op_core_flat(void* stream, int r, int nq, int s, const double* G, const double* w, const int* first,
                     const double* X, const double* Y, int p, int n, int h, double* out);
int ttb_vec_core_flat(void* stream, int r, int nq, int s, const double* G, const double* w, const int* first,
                      const double* V, int p, int n, double* out);
/* Solution core at quadrature points: T[a,q,b] = sum_k u[a, first[q]+k, b] V[q,k]. */
int ttb_field_table(void* stream, int r, int n, int s, const double* u, int nq, const int* first, const double* V,
                    int p, double* T);
/* driver.l2_error integrals: out[0] = sum w det|u-u*|, out[1] = sum w det|u*| (part: 2*nq0*nq1 doubles).
 * exact_id >= 0: u* in-kernel (iga.cu exact_fn, parameters prm); exact_id = -1: prm is the table of u* at
 * every quadrature point (nq0 x nq1 x nq2, row-major) for a user-supplied analytic function. */
int ttb_l1_error(void* stream, const int* f0, const int* f1, const int* f2, const double* V0, const double* V1,
                 const double* V2, const double* D0, const double* D1, const double* D2, int p0, int p1, int p2,
                 int n0, int n1, int n2, const double* cw, int nq0, int nq1, int nq2, const double* U0, int r1,
                 const double* U1, int r2, const double* U2, const double* w0, const double* w1, const double* w2,
                 int exact_id, const double* prm, double* part, double* out);

/* ---- classical full-grid system (reference driver.py:561-703, full_grid_reference) -------------- */

/* Element-by-element stiffness and load of the tensor-product B-spline space on the device: one CTA per
 * element accumulates the local (p+1)^3 x (p+1)^3 matrix over the element's g0 g1 g2 Gauss points and adds
 * it into the stencil storage K (n0 n1 n2 x prod(2 p_d + 1), slot ((o0 (2p1+1) + o1)(2p2+1) + o2) for the
 * column with per-direction offsets o_d - p_d), and the local load into f (n0 n1 n2). ne, g, p, n: host
 * int[3] (elements, Gauss points per element, degree, basis functions per direction); s_d, V_d, D_d: the
 * per-quadrature-point basis windows; Rw: (nq0 nq1 nq2, 9) weighted metric w R_ij; Fw: weighted f det J.
 * K and f must be zeroed by the caller. Replaces the reference's numpy einsum + scipy COO assembly. */
int ttb_fullgrid_assemble(void* stream, const int* ne, const int* g, const int* p, const int* n, const int* s0,
                          const int* s1, const int* s2, const double* V0, const double* V1, const double* V2,
                          const double* D0, const double* D1, const double* D2, const double* Rw, const double* Fw,
                          double* K, double* f);
/* y = M K M x on the stencil storage (M = diag(mask) selects the interior dofs; mask NULL: y = K x). */
int ttb_stencil_spmv(void* stream, int n0, int n1, int n2, int p0, int p1, int p2, const double* K, const double* x,
                     const unsigned char* mask, double* y);

/* ---- TT operator kernels (tensor_train/core.py:327-338, tensor_train/amen.py:51-193) ----------- */

/* TT-matvec of a banded operator core M (Ra, n, 2h+1, Rb) with a vector core X (rc, n, rd):
 * Y[(a,c), i, (b,d)] = sum_t M[a,i,t,b] X[c, i+t-h, d]. */
int ttb_band_matvec(void* stream, int Ra, int Rb, int n, int h, int rc, int rd, const double* M, const double* X,
                    double* Y);
/* rev=0: out[x,i,b,w] = sum_{a,t} M[a,i,t,b] T[x,a,i+t-h,w];  rev=1: out[x,i,a,w] = sum_{b,t} M[a,i,t,b] T[x,b,j,w]. */
int ttb_band_apply(void* stream, int X, int Ra, int Rb, int n, int h, int W, const double* M, const double* T,
                   double* out, int rev);
/* Dense projected local matrix (band entries only; Bm pre-zeroed), T1[x,y,i,t,b] = sum_a phiL[x,a,y] M[a,i,t,b]. */
int ttb_local_dense(void* stream, int r0, int n, int r1, int h, int Rb, const double* T1, const double* phiR,
                    double* Bm);
/* Banded form of the projected local matrix in (i, x, z) ordering: LB[row*(bw+1)+d] = B[row,row-d],
 * bw = (h+1) r0 r1 - 1 (same T1 as ttb_local_dense). */
int ttb_local_band_build(void* stream, int r0, int n, int r1, int h, int Rb, const double* T1, const double* phiR,
                         double* LB);
/* In-place banded Cholesky + solve (one CTA); *info > 0 on a non-positive pivot (caller falls back to LU). */
int ttb_band_chol_solve(void* stream, long long N, int bw, double* LB, double* b, int* info);
/* Jacobi diagonal of the local operator, floored at 1e-14 max|d| (amen.py:158-161,179-181). part: >= 297 doubles. */
int ttb_jacobi_diag(void* stream, int r0, int n, int r1, int Ra, int Rb, int h, const double* phiL, const double* M,
                    const double* phiR, double* d, double* part);
/* Entries of a 3-core TT at N multi-indices (TtTensor.gather, core.py:118-124). */
/* d = max(|d|, 1e-14 max|d|) elementwise (Jacobi preconditioner floor, amen.py:179-181); part >= 320 doubles. */
int ttb_abs_floor(void* stream, long long tot, double* d, double* part);
int ttb_tt_gather3(void* stream, int N, const long long* idx, const double* G0, int n0, int r1, const double* G1,
                   int n1, int r2, const double* G2, int n2, double* out);
/* TT-cross index bookkeeping on the device (reference tensor_train/cross.py:88-100): out ((nl nk nr) x d int64,
   d = k + 1 + w) row (l nk + i) nr + r = (left[l, 0..k), i, right[r, 0..w)). */
int ttb_fiber_index(void* stream, int nl, int nk, int nr, int k, int w, const long long* left, const long long* right,
                    long long* out);
/* Nested index set from maxvol rows sel (r int32) of an unfolding with inner size q (cross.py:150-152, 178-180):
   side 0: out[s] = (src[sel[s] / q, 0..w), sel[s] % q); side 1: out[s] = (sel[s] / q, src[sel[s] % q, 0..w)). */
int ttb_nested_index(void* stream, int r, int q, int w, int side, const int* sel, const long long* src, long long* out);
/* y = local projected operator applied to v (amen._LocalSystem.matvec3). ws: r0*Ra*n*r1 + r0*n*Rb*r1 doubles. */
int ttb_local_matvec(void* stream, int r0, int n, int r1, int Ra, int Rb, int h, const double* phiL, const double* M,
                     const double* phiR, const double* v, double* y, double* ws);
long long ttb_pcg_workspace(int r0, int n, int r1, int Ra, int Rb); /* doubles */
/* Jacobi-preconditioned CG with scipy.sparse.linalg.cg stopping semantics (||r|| < atol, maxiter),
 * x: x0 in / solution out; S: >= 8 device doubles; iters: HOST int (nullable). */
int ttb_local_pcg(void* stream, int r0, int n, int r1, int Ra, int Rb, int h, const double* phiL, const double* M,
                  const double* phiR, const double* b, double* x, const double* d, double atol, int maxiter,
                  int x0_nonzero, double* ws, double* S, int* iters);

/* Banded contraction as one batched DMMA GEMM (large operator ranks; replaces the inner loops of
 * amen.py:77-99 _OpCore.apply/apply_rev): out[i, X, o] = sum_{t, r} Tp[i + t, r, X] Mt[i, t, r, o],
 * Tp (n + 2h, Rin, X) with h zero blocks at both ends, Mt (n, 2h+1, Rin, Rout) = the banded core
 * M[a, i, t, b] permuted to (i, t, a, b) (forward) or (i, t, b, a) (reverse). */
int ttb_band_gemm(void* stream, int n, int h, int Rin, int Rout, int X, const double* Tp, const double* Mt,
                  double* out);
/* The same contraction as Ozaki-scheme FP64 on the int8 tensor cores (ttb_band_gemm dispatches to it for
 * >= 2e10 flop, X >= 128, (2h+1) Rin <= 4096; TTB_BAND_OZAKI=0 disables): Tp sliced once per group of G
 * batches (one exponent per row over the group's G + 2h blocks), Mt per batch; ws:
 * ttb_band_gemm_ozaki_workspace bytes. */
/* TT-matvec core (tensor_train/core.py tt_matvec, reference core.py:327-338) as ONE Ozaki-scheme FP64 GEMM:
 * Y (Ra rc, n, Rb rd) [(a,c), i, (b,d)] = sum_j M (Ra, n, m, Rb)[a,i,j,b] G (rc, m, rd)[c,j,d], both operands
 * sliced from their core layouts, Y written in its core layout (no regrouping passes). Shapes: Ra n Rb % 128,
 * rc rd % 64, m % 64, rd % 16, Rb, rd <= 64 dividing 256, no split-K (TTB_EARG otherwise). */
long long ttb_matvec_core_ozaki_workspace(int Ra, int n, int m, int Rb, int rc, int rd);
int ttb_matvec_core_ozaki(void* stream, int Ra, int n, int m, int Rb, int rc, int rd, const double* M, const double* G,
                          double* Y, void* ws);
long long ttb_band_gemm_ozaki_workspace(int n, int h, int Rin, int Rout, int X, int G);
int ttb_band_gemm_ozaki(void* stream, int n, int h, int Rin, int Rout, int X, const double* Tp, const double* Mt,
                        double* out, void* ws, int G);
/* Local projected operator (amen.py:147-150 matvec3) with vectors in the mode-major (i, x, z) layout:
 * phiLp = phiL permuted (a, x, y), Mf = (n, 2h+1, Ra, Rb), phiRp = phiR permuted (z, w, b) and
 * zero-padded to (r1, r1 + (r0 & r1 & 1), Rb) (the staged operand keeps an even column count).
 * ws: ttb_local_gemm_workspace doubles, padding zeroed once by ttb_local_gemm_ws_init. */
long long ttb_local_gemm_workspace(int r0, int n, int r1, int Ra, int Rb, int h); /* doubles */
int ttb_local_gemm_ws_init(void* stream, int r0, int n, int r1, int Ra, int h, double* ws);
int ttb_local_matvec_gemm(void* stream, int r0, int n, int r1, int Ra, int Rb, int h, const double* phiLp,
                          const double* Mf, const double* phiRp, const double* v, double* y, double* ws);
/* ttb_local_pcg over ttb_local_matvec_gemm, vectors in (i, x, z) layout; ws: ttb_pcg_gemm_workspace
 * doubles, ttb_local_gemm_ws_init applied at offset 4 r0 n r1. */
long long ttb_pcg_gemm_workspace(int r0, int n, int r1, int Ra, int Rb, int h); /* doubles */
int ttb_local_pcg_gemm(void* stream, int r0, int n, int r1, int Ra, int Rb, int h, const double* phiLp,
                       const double* Mf, const double* phiRp, const double* b, double* x, const double* d,
                       double atol, int maxiter, int x0_nonzero, double* ws, double* S, int* iters);

/* INT8 tensor-core GEMM (tcgen05.mma kind::i8, TMEM accumulators): C (int32 M x N row-major) =
 * A (int8 M x K row-major) B (int8 N x K row-major)^T; M, N, K multiples of 128. Building block of the
 * Ozaki-scheme FP64 emulation. */
int ttb_i8gemm(void* stream, int M, int N, int K, const void* A, const void* B, int* C);
/* Per-launch timing of the Ozaki GEMM kernel (bench.py's roofline record): enable = 1 drops earlier records and
   times every oz_gemm_kernel launch from now on (two CUDA events on its stream), 0 stops; returns the records
   held. _read: up to cap records in launch order, ms[i] = kernel duration, shape[4i..] = M, N, K, kind
   (0 general, 1 Gram, 2 A lower-triangular, 3 B upper-triangular, 4 TT-matvec core); returns the count. */
int ttb_ozaki_kernel_events(int enable);
int ttb_ozaki_kernel_events_read(int cap, double* ms, int* shape);
/* FP64 GEMM emulated on the INT8 tensor cores (Ozaki scheme, 7 balanced 8-bit slices per operand,
 * 54-bit operands, exact int32 level sums): C (M x N, ldc) = A (M x K row-major, lda) op(B), op(B) = B
 * (K x N, ldb) for tB = 0 or B^T (B: N x K) for tB = 1. Replaces ttb_dgemm for large tcgen05-tileable
 * shapes (ttb_ozaki_applies: M % 128, N % 64, K % 64); ws: ttb_ozaki_workspace bytes. */
long long ttb_ozaki_workspace(int M, int N, int K); /* bytes */
int ttb_ozaki_applies(int M, int N, int K);
int ttb_dgemm_ozaki(void* stream, int tB, int M, int N, int K, const double* A, long long lda, const double* B,
                    long long ldb, double* C, long long ldc, void* ws);
/* General form C = alpha A op(B) + beta C (same workspace). Any K % 64 == 0: K ranges of 4096 are summed
 * exactly in TMEM and combined in int64; with fewer output tiles than SMs the K dimension is split across
 * CTAs (partials reduced in a fixed order). */
int ttb_dgemm_ozaki_ex(void* stream, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
                       const double* B, long long ldb, double beta, double* C, long long ldc, void* ws);
/* C = A B with A (M x M) lower triangular (strict upper triangle zero): each 128-row block of C runs
 * only the k steps below its diagonal block (half the work). B row-major M x N; ws as ttb_ozaki_workspace(M, N, M). */
int ttb_dgemm_ozaki_trilA(void* stream, int M, int N, const double* A, long long lda, const double* B, long long ldb,
                          double* C, long long ldc, void* ws);
/* C = A B with B (N x N) upper triangular (strict lower triangle zero): each 64-column block of C runs only
 * the k steps above its diagonal block (~half the work). A row-major M x N; ws as ttb_ozaki_workspace(M, N, N).
 * Q = X R^-1 of a rounding step certified full rank (reference tensor_train/core.py:377-386 with keep == r1). */
int ttb_dgemm_ozaki_triuB(void* stream, int M, int N, const double* A, long long lda, const double* B, long long ldb,
                          double* C, long long ldc, void* ws);
/* Gram matrix G (n x n) = X^T X of a row-major m x n X, FP64 via the Ozaki scheme (columns sliced once,
 * upper block triangle computed, mirrored); n % 128 == 0, m % 64 == 0 (else workspace 0 / TTB_EARG). */
long long ttb_ozaki_gram_workspace(int m, int n); /* bytes */
int ttb_ozaki_gram(void* stream, int m, int n, const double* X, long long ldx, double* G, long long ldg, void* ws);
/* Gram matrix of the rows, G (n x n) = T T^T of a row-major n x m T (same conditions and workspace). */
long long ttb_ozaki_gram_rows_workspace(int n, int m); /* bytes */
int ttb_ozaki_gram_rows(void* stream, int n, int m, const double* T, long long ldt, double* G, long long ldg, void* ws);
/* Linv = L^{-1} of a lower-triangular row-major n x n L (strict upper triangle ignored), n % 128 == 0;
 * ws: n * n doubles. */
int ttb_trtri_lower(void* stream, int n, const double* L, long long ldl, double* Li, long long ldi, double* ws);
/* Row-major lower L (ldl) from the buffer ttb_potrf left (col-major lower factor; its row-major view holds
 * L^T above the diagonal and the untouched Gram entries below); offmax (device double, nullable) receives
 * max |G_ij| over the strict lower part (CholeskyQR2's second-Gram test). Replaces triu().t() / tril().abs().max(). */
int ttb_tri_from_potrf(void* stream, int n, const double* G, long long ldg, double* L, long long ldl, double* offmax);
/* ||A||_2 estimate of a square row-major matrix by `iters` power-iteration steps on B = A^T A (one DMMA GEMM,
 * then one cooperative launch; ws: n^2 + 2n + 2 doubles; out: device double). CholeskyQR's one-pass test
 * cond(L1) <= 4. */
int ttb_norm2_est(void* stream, int n, const double* A, long long lda, int iters, double* ws, double* out);

#ifdef __cplusplus
}
#endif
#endif
