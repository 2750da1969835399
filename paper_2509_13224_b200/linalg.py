"""Device FP64 linear algebra on torch CUDA tensors, computed by libttiga_b200.so.

Layout notes: torch tensors are row-major. A "col-major m x n" matrix is held
as a contiguous torch tensor of shape (n, m) (its transpose), which is what the
LAPACK-convention kernels (QR, Jacobi SVD, LU, Cholesky, maxvol) consume.
"""

from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np
import torch

from ._lib import call, call_raw, device, ptr

F64 = torch.float64
I32 = torch.int32


class LinAlgError(np.linalg.LinAlgError):
    """Device counterpart of numpy's LinAlgError."""


def empty(*shape, dtype=F64):
    return torch.empty(*shape, dtype=dtype, device=device())


def zeros(*shape, dtype=F64):
    return torch.zeros(*shape, dtype=dtype, device=device())


def _rows(A):
    """Row-major 2-D operand with unit column stride."""
    if A.dim() != 2:
        raise ValueError("expected a matrix")
    if A.stride(1) != 1 or (A.shape[0] > 1 and A.stride(0) < A.shape[1]):
        A = A.contiguous()
    return A


_GEMM_PROFILE = None  # when a list: (start_event, end_event, flops) per GEMM launch


def gemm_profile(enable: bool):
    """Start/stop recording CUDA events around every GEMM (bench.py roofline); returns the records
    (start_event, end_event, flops, "ozaki"|"dmma", (M, N, K))."""
    global _GEMM_PROFILE
    rec = _GEMM_PROFILE
    _GEMM_PROFILE = [] if enable else None
    return rec


_OZAKI = os.environ.get("TTB_OZAKI", "1") != "0"
_OZAKI_MIN_WORK = 1 << 33          # M N K: only the rounding-sized products (>= 8.6 GFMA)
_OZAKI_CHECK = os.environ.get("TTB_OZAKI_CHECK", "0") == "1"   # debug: compare every emulated product with DMMA


_OZAKI_MAX_PAD = 1.6    # padded shapes (M to 128, N and K to 64) run emulated while padded work <= 1.6x


def _ozaki_padding_ok(M, N, K):
    r = lambda v, m: -(-v // m) * m   # noqa: E731
    return r(M, 128) * r(N, 64) * r(K, 64) <= _OZAKI_MAX_PAD * M * N * K


def gemm(A, B, tA=False, tB=False, alpha=1.0, beta=0.0, out=None, emulate=False):
    """out = alpha op(A) op(B) + beta out (row-major, FP64 DMMA kernel).

    emulate: large products (M N K >= 2^33, padding to M % 128, N % 64, K % 64 costing <= 1.6x, alpha = 1,
    beta = 0, A not transposed) run as the Ozaki-scheme FP64 GEMM on the INT8 tensor cores (ttb_dgemm_ozaki: 54-bit
    operands in 7 balanced 8-bit slices, 8 exact int32 level sums; agrees with DGEMM to ~1e-15
    normwise). TTB_OZAKI=0 keeps every product on DMMA."""
    A = _rows(A)
    B = _rows(B)
    M, K = (A.shape[1], A.shape[0]) if tA else (A.shape[0], A.shape[1])
    K2, N = (B.shape[1], B.shape[0]) if tB else (B.shape[0], B.shape[1])
    if K != K2:
        raise ValueError(f"gemm inner dims {K} != {K2}")
    if out is None:
        out = empty(M, N)
        beta = 0.0
    elif out.shape != (M, N) or out.stride(1) != 1:
        raise ValueError("bad gemm output")
    if (emulate and _OZAKI and not tA and alpha == 1.0 and beta == 0.0 and M * N * K >= _OZAKI_MIN_WORK
            and _ozaki_padding_ok(M, N, K)):
        ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, K)), dtype=torch.uint8, device=device())
        prof = _GEMM_PROFILE
        if prof is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
        call("ttb_dgemm_ozaki", int(tB), M, N, K, ptr(A), max(A.stride(0), 1), ptr(B), max(B.stride(0), 1), ptr(out),
             max(out.stride(0), 1), ptr(ws))
        if prof is not None:
            e1.record()
            prof.append((e0, e1, 2.0 * M * N * K, "ozaki", (M, N, K)))
        if _OZAKI_CHECK:
            ref = empty(M, N)
            call("ttb_dgemm", int(tA), int(tB), M, N, K, 1.0, ptr(A), max(A.stride(0), 1), 0, ptr(B),
                 max(B.stride(0), 1), 0, 0.0, ptr(ref), N, 0, 1)
            print(f"ozaki check M={M} N={N} K={K} tB={int(tB)}: rel {float((out - ref).norm() / ref.norm()):.3e} "
                  f"|A| {float(A.norm()):.3e} |B| {float(B.norm()):.3e}", flush=True)
        return out
    if M and N:
        prof = _GEMM_PROFILE
        if prof is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
        call("ttb_dgemm", int(tA), int(tB), M, N, K, float(alpha), ptr(A), max(A.stride(0), 1), 0, ptr(B),
             max(B.stride(0), 1), 0, float(beta), ptr(out), max(out.stride(0), 1), 0, 1)
        if prof is not None:
            e1.record()
            prof.append((e0, e1, 2.0 * M * N * K, "dmma", (M, N, K)))
    return out


def gemm_triu(A, W, out=None):
    """out = A W for a row-major A (M x N) and an upper-triangular W (N x N, strict lower triangle zero):
    the Ozaki GEMM that skips the zero k steps of every column block (ttb_dgemm_ozaki_triuB) when the
    shape takes it, else the general product."""
    A = _rows(A)
    W = _rows(W)
    M, N = A.shape
    if W.shape != (N, N):
        raise ValueError("gemm_triu: W must be N x N")
    if not (_OZAKI and M * N * N >= _OZAKI_MIN_WORK and call_raw("ttb_ozaki_applies", M, N, N)):
        return gemm(A, W, out=out, emulate=True)
    if out is None:
        out = empty(M, N)
    elif out.shape != (M, N) or out.stride(1) != 1:
        raise ValueError("bad gemm output")
    ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, N)), dtype=torch.uint8, device=device())
    prof = _GEMM_PROFILE
    if prof is not None:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
    call("ttb_dgemm_ozaki_triuB", M, N, ptr(A), max(A.stride(0), 1), ptr(W), N, ptr(out), max(out.stride(0), 1), ptr(ws))
    if prof is not None:
        e1.record()
        prof.append((e0, e1, 1.0 * M * N * (N + 64), "ozaki-triu", (M, N, N)))
    return out


def gemm_strided(tA, tB, M, N, K, A, lda, sA, B, ldb, sB, C, ldc, sC, batch, alpha=1.0, beta=0.0):
    """Strided-batched C_b = alpha op(A_b) op(B_b) + beta C_b on raw device tensors (row-major views;
    A, B, C are tensors whose data_ptr is the first batch's first element)."""
    if M and N and batch:
        call("ttb_dgemm", int(tA), int(tB), int(M), int(N), int(K), float(alpha), ptr(A), int(lda), int(sA), ptr(B),
             int(ldb), int(sB), float(beta), ptr(C), int(ldc), int(sC), int(batch))
    return C


def permute(X, perm, out=None):
    """Materialized X.permute(perm) (row-major), by the native transpose kernel (into ``out`` if given)."""
    perm = tuple(int(p) for p in perm)
    if perm == tuple(range(X.dim())) and out is None:
        return X.contiguous()
    X = X.contiguous()
    shape = [X.shape[p] for p in perm]
    if out is None:
        out = empty(*shape)
    elif list(out.shape) != shape or not out.is_contiguous():
        raise ValueError("bad permute output")
    if X.numel():
        dims = (C.c_longlong * X.dim())(*X.shape)
        pm = (C.c_int * X.dim())(*perm)
        call("ttb_permute", X.dim(), dims, pm, ptr(X), ptr(out))
    return out


def tdot(A, B, axes, emulate=False):
    """np.tensordot(A, B, axes) on the device: permute to matrix form + one GEMM."""
    ia, ib = axes
    ia = [a % A.dim() for a in (ia if isinstance(ia, (list, tuple)) else [ia])]
    ib = [b % B.dim() for b in (ib if isinstance(ib, (list, tuple)) else [ib])]
    fa = [k for k in range(A.dim()) if k not in ia]
    fb = [k for k in range(B.dim()) if k not in ib]
    M = int(np.prod([A.shape[k] for k in fa], dtype=np.int64))
    K = int(np.prod([A.shape[k] for k in ia], dtype=np.int64))
    N = int(np.prod([B.shape[k] for k in fb], dtype=np.int64))
    if ia == list(range(len(ia))):
        Am, tA = A.contiguous().reshape(K, M), True
    else:
        Am, tA = permute(A, fa + ia).reshape(M, K), False
    if ib == list(range(B.dim() - len(ib), B.dim())) and fb == list(range(len(fb))):
        Bm, tB = B.contiguous().reshape(N, K), True
    else:
        Bm, tB = permute(B, ib + fb).reshape(K, N), False
    out = gemm(Am, Bm, tA=tA, tB=tB, emulate=emulate)
    return out.reshape([A.shape[k] for k in fa] + [B.shape[k] for k in fb])


def dot(x, y=None, sqrt=False):
    """Deterministic device dot product / squared norm; returns a 0-d device tensor."""
    x = x.contiguous().reshape(-1)
    out = empty(1)
    part = empty(320)
    call("ttb_dot", x.numel(), ptr(x), None if y is None else ptr(y.contiguous().reshape(-1)), ptr(out), ptr(part),
         int(sqrt))
    return out[0]


def nrm2(x):
    return dot(x, None, sqrt=True)


# ---------------------------------------------------------------------------
# QR

def qr_colmajor(Acm, m, n, want_q=True, want_r=True, overlap_r=None):
    """Householder QR of a col-major m x n matrix held as torch (n, m) (consumed).

    Returns (Qt, Rt): Qt = torch (k, m) == col-major Q (m x k); Rt = torch (n, k) == col-major R (k x n).
    ``overlap_r(Rt)``, if given, is called on a side stream as soon as R is available and runs
    concurrently with the formation of Q (the two are independent); its result is returned third.
    """
    k = min(m, n)
    if k == 0:
        return (empty(0, m), empty(n, 0)) if overlap_r is None else (empty(0, m), empty(n, 0), overlap_r(empty(n, 0)))
    if call_raw("ttb_qr_small_fits", m, n):
        Qt = empty(k, m) if want_q else None
        Rt = empty(n, k)
        call("ttb_qr_small", m, n, ptr(Acm), m, ptr(Qt), m, ptr(Rt))
        if overlap_r is not None:
            return Qt, Rt, overlap_r(Rt)
        return Qt, (Rt if want_r else None)
    ws = empty(int(call_raw("ttb_qr_workspace", m, n)))
    tau = empty(k)
    call("ttb_geqrf", m, n, ptr(Acm), m, ptr(tau), ptr(ws))
    Qt = Rt = None
    if want_r or overlap_r is not None:
        Rt = empty(n, k)
        call("ttb_extract_r", k, n, ptr(Acm), m, ptr(Rt))
    side = None
    if overlap_r is not None:
        main = torch.cuda.current_stream()
        side = _side_stream()
        side.wait_stream(main)
        with torch.cuda.stream(side):
            res = overlap_r(Rt)
    if want_q:
        Qt = empty(k, m)
        call("ttb_orgqr", m, k, k, ptr(Acm), m, ptr(Qt), m, ptr(ws), n)
    if side is not None:
        main.wait_stream(side)
        for t in (Rt,) + tuple(x for x in (res if isinstance(res, tuple) else (res,)) if isinstance(x, torch.Tensor)):
            t.record_stream(main)
        return Qt, Rt, res
    return Qt, Rt


_CHOLQR2 = os.environ.get("TTB_RL_CHOLQR2", "1") != "0"
_CHOLQR2_MIN_M = int(os.environ.get("TTB_RL_CHOLQR2_MIN_M", str(1 << 19)))


class _profiled:
    """Records (start, end, flops, kind, shape) of the enclosed launches when gemm_profile is on."""

    def __init__(self, kind, shape, flops):
        self.rec = (kind, shape, flops)

    def __enter__(self):
        if _GEMM_PROFILE is not None:
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e0.record()

    def __exit__(self, *exc):
        if _GEMM_PROFILE is not None and exc[0] is None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            kind, shape, flops = self.rec
            _GEMM_PROFILE.append((self.e0, e1, flops, kind, shape))
        return False


def _chol_rows(T, n, m, offdiag=False):
    """Row-major lower Cholesky factor L of G = T T^T (T: n x m row-major, Ozaki-scheme Gram), or None;
    offdiag: also max |G_ij| over i != j (read from the triangle potrf leaves untouched)."""
    ws = torch.empty(int(call_raw("ttb_ozaki_gram_rows_workspace", n, m)), dtype=torch.uint8, device=device())
    G = empty(n, n)
    with _profiled("ozaki-gram", (n, n, m), 1.0 * n * (n + 128) * m):     # the lower-triangle tiles only
        call("ttb_ozaki_gram_rows", n, m, ptr(T), max(T.stride(0), 1), ptr(G), n, ptr(ws))
    del ws
    info = empty(1, dtype=I32)
    call("ttb_potrf", n, ptr(G), n, ptr(info))   # col-major lower L: row-major view of the buffer = L^T
    if int(info.item()) != 0:
        return None
    Lr = empty(n, n)
    if offdiag:
        off = empty(1)
        call("ttb_tri_from_potrf", n, ptr(G), n, ptr(Lr), n, ptr(off))
        return Lr, float(off.item())
    call("ttb_tri_from_potrf", n, ptr(G), n, ptr(Lr), n, None)
    return Lr


def _trtri(Lr, n):
    Li = empty(n, n)
    ws = empty(n * n)
    call("ttb_trtri_lower", n, ptr(Lr), n, ptr(Li), n, ptr(ws))
    return Li


_CHOLQR1_KAPPA = float(os.environ.get("TTB_CHOLQR_ONEPASS_KAPPA", "4"))


def _norm2_est(A, iters=24):
    """||A||_2 of a square device matrix by power iteration on A^T A (seeded start; a lower estimate
    that is within a few percent after 24 steps for the clustered spectra it is used on)."""
    return float(_norm2_est_dev(A, iters).item())


def _norm2_est_dev(A, iters=24):
    """_norm2_est as a 1-element device tensor (no host sync)."""
    n = A.shape[0]
    ws = empty(n * n + 2 * n + 2)
    out = empty(1)
    call("ttb_norm2_est", n, ptr(A.contiguous()), n, int(iters), ptr(ws), ptr(out))   # one cooperative launch
    return out


def _trmm_oz(Li, X, n, m):
    """Li (n x n lower) @ X (n x m) as the Ozaki GEMM that skips the zero upper triangle."""
    out = empty(n, m)
    ws = torch.empty(int(call_raw("ttb_ozaki_workspace", n, m, n)), dtype=torch.uint8, device=device())
    with _profiled("ozaki-tril", (n, m, n), 1.0 * n * (n + 128) * m):
        call("ttb_dgemm_ozaki_trilA", n, m, ptr(Li), n, ptr(X), max(X.stride(0), 1), ptr(out), m, ptr(ws))
    return out


_LAZY_Q = os.environ.get("TTB_ROUND_LAZY_Q", "1") != "0"


class LazyQt:
    """The transposed orthonormal factor Q^T = Li @ X (n x m) of a one-pass CholeskyQR, held as its
    factors: Li = L1^-1 (n x n row-major lower) and the factored rows X (torch (n, m), not copied).
    The rounding's left-to-right pass only ever needs carry @ Q^T, which is (carry @ Li) @ X: one small
    product and ONE large one, instead of forming Q^T (a large triangular product) and then carrying
    into it (a second large product)."""

    def __init__(self, Li, X):
        self.Li, self.X = Li, X
        self.shape = X.shape

    def carried(self, carry):
        """carry @ Q^T for a row-major carry (k x n)."""
        return gemm(gemm(carry, self.Li), self.X, emulate=True)

    def dense(self):
        n, m = self.X.shape
        return _trmm_oz(self.Li, self.X, n, m)


def cholqr2_colmajor(Acm, m, n, lazy=False):
    """Q R of a very tall col-major m x n matrix held as torch (n, m), by CholeskyQR2 with Ozaki-scheme
    FP64 Gram matrices and products on the int8 tensor cores:
        G1 = X^T X = L1 L1^T,  Q1 = X L1^-T,  G2 = Q1^T Q1 = L2 L2^T,  Q = Q1 L2^-T,  R = L2^T L1^T.
    Q spans the same space as the Householder Q and differs from it only by column signs (R has a
    positive diagonal) and rounding, so the orthogonalized TT represents the same tensor. CholeskyQR2
    needs cond(X) well below eps^-1/2: the Cholesky factorizations must succeed and the second Gram
    must be within 0.1 of I (else the first pass lost orthogonality beyond what one repeat restores).
    When the power-iteration estimate of cond(L1) is <= 4 (TTB_CHOLQR_ONEPASS_KAPPA) the first pass
    is kept as is (orthogonality error ~ eps cond^2 <= 16 eps), and with ``lazy`` its Q^T is returned
    unformed (LazyQt: the caller multiplies through the factors; TTB_ROUND_LAZY_Q=0 forms it);
    returns (Qt, Rt) in qr_colmajor's layout, or None (the caller takes the Householder path).
    Used for the rounding's right-to-left sweep (core.py _rl_orthogonalize)."""
    if not (_CHOLQR2 and _OZAKI and m >= _CHOLQR2_MIN_M and n >= 256 and n % 128 == 0 and m % 64 == 0):
        return None
    L1 = _chol_rows(Acm, n, m)
    if L1 is None:
        return None
    Li1 = _trtri(L1, n)
    onepass = False
    if _CHOLQR1_KAPPA > 0.0:
        est = torch.cat([_norm2_est_dev(L1), _norm2_est_dev(Li1)]).cpu().numpy()   # one host sync
        onepass = bool(np.isfinite(est).all() and est[0] * est[1] <= _CHOLQR1_KAPPA)
    if onepass and lazy and _LAZY_Q:
        return LazyQt(Li1, Acm), L1
    Q1 = _trmm_oz(Li1, Acm, n, m)                        # (n, m) = L1^-1 X^T = Q1^T
    if onepass:
        # cond(X) = cond(L1) <= 4: one CholeskyQR pass is already orthogonal to ~eps cond^2
        return Q1, L1
    got = _chol_rows(Q1, n, m, offdiag=True)
    if got is None:
        return None
    L2, off = got
    if off > 0.1 or float((L2.diagonal() - 1.0).abs().max()) > 0.1:
        return None
    Qt = _trmm_oz(_trtri(L2, n), Q1, n, m)               # Q^T
    del Q1
    return Qt, gemm(L1, L2)                              # R^T = L1 L2 (row-major) == col-major R


_SIDE = None


def _side_stream():
    global _SIDE
    if _SIDE is None:
        _SIDE = torch.cuda.Stream(priority=-1)
    return _SIDE


def qr(X):
    """np.linalg.qr(X) (reduced) for a row-major matrix: returns (Q (m x k), R (k x n)) views."""
    m, n = X.shape
    Qt, Rt = qr_colmajor(permute(X, (1, 0)), m, n)
    return Qt.t(), Rt.t()


# ---------------------------------------------------------------------------
# SVD

def _jacobi(Rcm, n, want_v=False, info=None):
    """SVD of a col-major n x n matrix held as torch (n, n): returns (U_mem, S, V_mem|None) col-major.

    ``info`` (optional int32 device tensor) receives the number of Jacobi sweeps.
    """
    S = empty(n)
    U = empty(n, n)
    V = empty(n, n) if want_v else None
    work = empty(2 * n * n + n) if n > 64 else None
    call("ttb_svd_jacobi", n, ptr(Rcm), n * n, ptr(S), n, ptr(U), ptr(V), n * n, 1, ptr(work), ptr(info))
    return U, S, V


_JACOBI_RT_MAX = int(os.environ.get("TTB_JACOBI_RT_MAX", "64"))
_PRECOND = os.environ.get("TTB_JACOBI_PRECOND", "1") != "0"
_PRECOND_RATIO = 100.0
_PRECOND_MAX_N = int(os.environ.get("TTB_JACOBI_PRECOND_MAX_N", "160"))   # the assembly sums; larger: no sweep gain


def _graded(norms):
    """Whether a matrix whose row/column norms (or |diag R|) are ``norms`` is graded enough for the QR
    preconditioner to pay (max/min > 100; zero entries count as graded)."""
    if not _PRECOND or norms.numel() < 2 or norms.numel() > _PRECOND_MAX_N:
        return False
    mn, mx = torch.aminmax(norms.abs())
    return bool(mn * _PRECOND_RATIO < mx)


def _jacobi_r(Rt, n, want_v):
    """U_R, S (and V_R if want_v) of the n x n triangular factor R of a tall QR; Rt is torch (n, n) ==
    col-major R. Graded R (the rounding's unfoldings of sums of TTs: row norms spanning 1e9-1e15) is
    preconditioned by a second QR, R^T = Q2 R2 (Drmac-Veselic): R = R2^T Q2^T, so one-sided Jacobi on the
    columns of R2^T yields R's left singular vectors and singular values directly, in 5-7 sweeps instead
    of the 15-29 Jacobi needs on R itself (tools/jacobi_sweeps.py); the right vectors would need Q2, so
    want_v keeps the plain form."""
    if not want_v and _graded(Rt.diagonal()):
        _, Rt2 = qr_colmajor(Rt.t().contiguous(), n, n, want_q=False)
        return _jacobi(Rt2.t().contiguous(), n, False)
    return _jacobi(Rt.contiguous(), n, want_v)


def _jacobi_rt(Rt, n, want_v=False):
    """One-sided Jacobi on the columns of R^T (R's right singular vectors = R^T's left ones, and S); Rt is
    torch (n, n) == col-major R. Graded R: R = Q3 R3 (QR of R itself), R3 has R's right singular vectors
    and values, and Jacobi runs on R3^T instead (the same Drmac-Veselic preconditioning as _jacobi_r)."""
    if not want_v and _graded(Rt.diagonal()):
        _, Rt3 = qr_colmajor(Rt.clone(), n, n, want_q=False)
        return _jacobi(Rt3.t().contiguous(), n, False)
    return _jacobi(permute(Rt, (1, 0)), n, want_v)
_IMPLICIT_U = os.environ.get("TTB_SVD_IMPLICIT_U", "1") != "0"
_IMPLICIT_U_MIN_M = int(os.environ.get("TTB_SVD_IMPLICIT_U_MIN_M", "65536"))
_IMPLICIT_U_MIN_RATIO = 1e-7   # U orthogonality error ~ eps s_max / s_k <= ~1e-9


_GRAM = os.environ.get("TTB_SVD_GRAM", "1") != "0"
_GRAM_MIN_M = int(os.environ.get("TTB_SVD_GRAM_MIN_M", str(1 << 19)))
_GRAM_MIN_RATIO = 1e-4   # s_min / s_max: singular values from X^T X carry relative error ~ eps (s_max / s)^2


# Full-rank certificate of a rounding step (reference tensor_train/core.py:377-386). _chop keeps every
# singular value of the unfolding X when the smallest one exceeds delta (the tail of dropping even one is
# s_min > delta), and then U[:, :keep] diag(s) Vt = X = Q R: the step's output core may be the QR factor Q
# and its carry R -- the same tensor, the same ranks, the same left-orthogonality, without the SVD. The
# certificate is rigorous: for the triangular factor L (X^T X = L L^T, so X and L share singular values)
#   s_min(X) = 1 / ||L^-1||_2 >= 1 / ||L^-1||_F,
# with a factor 2 of margin over delta for the rounding of L and L^-1. Only taken for the large factors
# (n >= 256, n % 128 == 0) where the Jacobi SVD costs milliseconds; TTB_ROUND_FULLRANK_QR=0 disables it.
_FULLRANK = os.environ.get("TTB_ROUND_FULLRANK_QR", "1") != "0"
_FULLRANK_MIN_N = 256
_FULLRANK_MARGIN = 2.0
# square steps: U = I, carry = X when certified (SVDFactors._direct_fullrank); and the right-to-left sweep's
# square / wide unfoldings take Q = I, R = X with no factorization at all (core.py _rl_orthogonalize)
_FULLRANK_IDENTITY = os.environ.get("TTB_ROUND_IDENTITY_Q", "1") != "0"
_IDENTITY_Q_MIN = 256


def _fullrank_wanted(delta, m, n, want_v):
    return (_FULLRANK and delta is not None and delta > 0.0 and not want_v and m >= n >= _FULLRANK_MIN_N
            and n % 128 == 0)


def _fullrank_inverse(Lr, n, delta, cond_max=None, info=None):
    """L^-1 (row-major lower) of the row-major lower-triangular Lr when 1 / ||L^-1||_F > 2 delta (and,
    with cond_max, the power-iteration estimate of cond_2(L) is <= cond_max), else None. One host sync.
    ``info``: the Cholesky status word that produced Lr, read in the same copy (non-zero -> None)."""
    Li = _trtri(Lr, n)
    vals = [nrm2(Li).reshape(1)]
    if cond_max is not None:
        vals += [_norm2_est_dev(Lr), _norm2_est_dev(Li)]
    if info is not None:
        vals.append(info.to(F64).reshape(1))
    v = torch.cat(vals).cpu().numpy()
    if info is not None:
        if v[-1] != 0.0:
            return None
        v = v[:-1]
    if not (np.isfinite(v).all() and v[0] > 0.0 and 1.0 / v[0] > _FULLRANK_MARGIN * delta):
        return None
    if cond_max is not None and not (1.1 * v[1] * v[2] <= cond_max):
        return None
    return Li


def _gram_jacobi(X, m, n, fullrank_delta=None):
    """Right singular vectors and singular values of a very tall X (m x n) without its QR: R from the
    Cholesky factor of G = X^T X (Ozaki-scheme FP64 Gram on the int8 tensor cores), then the same
    one-sided Jacobi on R^T as the QR path (R^T R = G, so R differs from the Householder R only by row
    signs and rounding). Used only when X is well conditioned (s_min >= 1e-4 s_max over ALL singular
    values, so eps (s_max / s)^2 <= 1e-8 relative and <= 1e-12 s_max absolute); returns
    (Rt, Vr, S) or None (the caller takes the Householder QR path). With ``fullrank_delta`` the
    full-rank certificate is tried first on the Cholesky factor (same conditioning limit, by estimate):
    certified, returns (Rt, L^-1, None) and no SVD is computed."""
    if not (_GRAM and _OZAKI and m >= _GRAM_MIN_M and n >= 256 and n % 128 == 0 and m % 64 == 0):
        return None
    ws = torch.empty(int(call_raw("ttb_ozaki_gram_workspace", m, n)), dtype=torch.uint8, device=device())
    G = empty(n, n)
    with _profiled("ozaki-gram", (n, n, m), 1.0 * n * (n + 128) * m):
        call("ttb_ozaki_gram", m, n, ptr(X), max(X.stride(0), 1), ptr(G), n, ptr(ws))
    del ws
    info = empty(1, dtype=I32)
    call("ttb_potrf", n, ptr(G), n, ptr(info))   # col-major lower L: row-major view of the buffer = L^T = R
    if int(info.item()) != 0:
        return None
    Rt = empty(n, n)                             # col-major R (the QR path's layout) = row-major L
    call("ttb_tri_from_potrf", n, ptr(G), n, ptr(Rt), n, None)
    if fullrank_delta is not None:
        Li = _fullrank_inverse(Rt, n, fullrank_delta, cond_max=1.0 / _GRAM_MIN_RATIO)
        if Li is not None:
            return Rt, Li, None
    Vr, S, _ = _jacobi_rt(Rt, n)                 # Jacobi on R^T: its U = X's right singular vectors
    s = S.cpu().numpy()
    if not (s.max() > 0.0 and s.min() >= _GRAM_MIN_RATIO * s.max()):
        return None
    return Rt, Vr, S


class SVDFactors:
    """Thin SVD X = U diag(S) Vt by Householder QR + one-sided Jacobi on the triangular factor.

    Only the left vectors are rotated; the "carry" S Vt needed by rounding is the
    backward-stable product U^T X (formed from the triangular factor), so the
    right vectors are accumulated only when explicitly requested (want_v).
    Tall X = Q R: Jacobi on R.  Wide X (X^T = Q R): Jacobi on R^T.
    """

    def __init__(self, X, want_v=False, fullrank_delta=None):
        """fullrank_delta: the rounding step's truncation threshold; when the full-rank certificate
        (see _fullrank_inverse) holds, ``fullrank`` is set, no SVD is computed, U(n) is the QR factor Q
        and SVt(n) is R (keep == n: the caller must not truncate)."""
        X = X.contiguous()
        m, n = X.shape
        self.m, self.n = m, n
        fr = fullrank_delta if _fullrank_wanted(fullrank_delta, m, n, want_v) else None
        # square: one-sided Jacobi straight on X (its column Gram equals R's, so the rotation
        # sequence and sweep count are those of Jacobi on R, and the QR is saved)
        self.direct = m == n and n > 64
        self.tall = m >= n and not self.direct
        if self.direct and fr is not None and self._direct_fullrank(X, n, fr):
            pass
        elif self.direct:
            self.X = X
            if not want_v and _graded(torch.linalg.vector_norm(X, dim=0)):
                # X^T = Q2 R2, X = R2^T Q2^T: Jacobi on the columns of R2^T gives U and S of X directly
                _, Rt2 = qr_colmajor(X.clone(), n, n, want_q=False)
                self.UJ, self.S, self.VJ = _jacobi(Rt2.t().contiguous(), n, False)
            else:
                self.UJ, self.S, self.VJ = _jacobi(permute(X, (1, 0)), n, want_v)
        elif self.tall and m >= _IMPLICIT_U_MIN_M and n > _JACOBI_RT_MAX and _IMPLICIT_U:
            # very tall X (the rounding's (r n) x r unfoldings): X = Q R without forming Q; Jacobi
            # on R^T, R^T = U' S V'^T, so the right singular vectors of X are U' (no rotations
            # accumulated) and U = X U' S^-1 (one GEMM, chunkable, no orgqr). A kept column whose
            # singular value is below _IMPLICIT_U_MIN_RATIO s_max would lose orthogonality
            # (error ~ eps s_max / s_k), so U() then falls back to the explicit-Q path.
            self.implicit = True
            self.X = X
            self._want_v = want_v
            got = _gram_jacobi(X, m, n, fr)
            if got is None:
                _, Rt = qr_colmajor(permute(X, (1, 0)), m, n, want_q=False)
                got = (Rt,) + _jacobi_rt(Rt, n)[:2]   # rows: right singular vectors
            self.Rt, self.Vr, self.S = got
            self.UJ = self.VJ = self.Qt = None
            self._W = None
            if self.S is None:          # certified full rank: Vr holds L^-1, U = X L^-T, carry = R = L^T
                self.fullrank = True
                self._W = self.Vr.t().contiguous()
        elif self.tall:
            # small R: one-sided Jacobi on R^T (rows of R, graded by the QR) converges in fewer
            # rounds; R = V' S U'^T, so U_R is the accumulated rotation V' and V_R = U'
            self.rt = n <= _JACOBI_RT_MAX
            if self.rt:
                job = lambda R: _jacobi(permute(R, (1, 0)), n, True)    # noqa: E731
            else:
                job = lambda R: _jacobi_r(R, n, want_v)                 # noqa: E731
            # the Jacobi SVD of R runs on a side stream while Q is formed (independent work)
            Qt, Rt, (UJ, self.S, VJ) = qr_colmajor(permute(X, (1, 0)), m, n, overlap_r=job)
            self.UJ, self.VJ = (VJ, UJ) if self.rt else (UJ, VJ)
            self.Qt = Qt                      # (n, m) == col-major Q (m x n)
            self.Rt = Rt                      # (n, n) == col-major R == row-major R^T
        else:
            Qt, Rt = qr_colmajor(X.clone(), n, m)  # X^T = Q R, Q (n x m), R (m x m)
            self.Qt = Qt                      # (m, n) == col-major Q == row-major Q^T
            self.Rt = Rt                      # row-major R^T
            self.UJ, self.S, self.VJ = _jacobi_rt(Rt, m, want_v)  # Jacobi on R^T

    implicit = False
    fullrank = False
    _s = None

    @classmethod
    def certified(cls, X, Rt, Li):
        """Factors of a tall X already certified full rank: U = X L^-T (implicit, chunkable), carry = R = L^T;
        Rt row-major L (X^T X = L L^T), Li = L^-1."""
        f = cls.__new__(cls)
        f.m, f.n = X.shape
        f.direct, f.tall, f.implicit, f.fullrank = False, True, True, True
        f.X, f._want_v = X, False
        f.Rt, f.Vr, f.S = Rt, Li, None
        f.UJ = f.VJ = f.Qt = None
        f._W = Li.t().contiguous()
        return f

    def _direct_fullrank(self, X, n, delta):
        """Square X. First the factorization-free form: X = I X is an orthogonal-times-carry split as good
        as Q R (the output core only has to be left-orthonormal), so when X is certified full rank the step
        returns U = I and the carry X. The certificate comes from the Cholesky factor of X^T X (same
        singular values as X; its estimate of s_min is off by ~n eps cond^2 relative, so the route is
        limited to an estimated cond <= 1e5, where that is <= 1e-3 against the factor-2 margin):
        one n^3 GEMM + Cholesky + triangular inverse instead of a Householder QR with explicit Q.
        Otherwise: Householder X = Q R, the certificate on R^T (its L^-1 and norm on a side stream
        while Q is formed); certified -> full-rank mode with the explicit Q, else nothing is kept."""
        if _FULLRANK_IDENTITY:
            G = gemm(X, X, tA=True)
            info = empty(1, dtype=I32)
            call("ttb_potrf", n, ptr(G), n, ptr(info))
            Lr = empty(n, n)
            call("ttb_tri_from_potrf", n, ptr(G), n, ptr(Lr), n, None)
            # a failed Cholesky leaves non-finite / garbage factors: the norms below then fail the test
            Li = _fullrank_inverse(Lr, n, delta, cond_max=1e5, info=info)
            if Li is not None:
                self.fullrank = True
                self.direct = False
                self.tall = True
                self.Qt = torch.eye(n, dtype=F64, device=device())
                self.Rt = X.t().contiguous()      # SVt() returns Rt^T = X
                self.S = self.UJ = self.VJ = None
                return True

        def cert(Rt):
            Li = _trtri(Rt, n)        # Rt row-major = R^T, lower triangular
            return nrm2(Li).reshape(1)
        Qt, Rt, nrm = qr_colmajor(permute(X, (1, 0)), n, n, overlap_r=cert)
        v = float(nrm.item())
        if not (np.isfinite(v) and v > 0.0 and 1.0 / v > _FULLRANK_MARGIN * delta):
            return False
        self.fullrank = True
        self.direct = False
        self.tall = True
        self.Qt, self.Rt = Qt, Rt
        self.S = self.UJ = self.VJ = None
        return True

    def record_stream(self, stream):
        """Mark every device tensor held here as used on ``stream`` (factors made on a side stream)."""
        for v in vars(self).values():
            if isinstance(v, torch.Tensor) and v.is_cuda:
                v.record_stream(stream)

    def s_host(self):
        if self.fullrank:
            raise ValueError("certified full-rank factors hold no singular values (keep == n)")
        if self._s is None:
            self._s = self.S.cpu().numpy()
        return self._s

    def _implicit_w(self, r):
        """W = U'[:r]^T S[:r]^-1 (n x r) when every kept singular value is well separated from 0,
        else switch to the explicit-Q path (returns None)."""
        if self.fullrank:
            return self._W
        s = self.s_host()
        if s[0] > 0.0 and s[r - 1] >= _IMPLICIT_U_MIN_RATIO * s[0]:
            if self._W is None or self._W.shape[1] != r:
                self._W = (self.Vr[:r] / self.S[:r, None]).t().contiguous()
            return self._W
        self._explicit()
        return None

    def _explicit(self):
        """Fall back to Q R with explicit Q and Jacobi on R (the default tall path)."""
        X, n, m = self.X, self.n, self.m
        self.implicit = False
        self.rt = False
        Qt, Rt, (UJ, S, VJ) = qr_colmajor(permute(X, (1, 0)), m, n,
                                          overlap_r=lambda R: _jacobi_r(R, n, self._want_v))
        self.Qt, self.Rt, self.UJ, self.S, self.VJ = Qt, Rt, UJ, S, VJ
        self._s = None

    def U(self, r):
        """First r left singular vectors, row-major (m x r)."""
        if self.fullrank:
            self._full(r)
            if self.implicit:
                return gemm_triu(self.X, self._W)
            return self.Qt.t().contiguous()
        if self.implicit and self._implicit_w(r) is not None:
            return gemm(self.X, self._W, emulate=True)
        if self.tall:
            return gemm(self.Qt, self.UJ[:r], tA=True, tB=True)
        return self.UJ[:r].t().contiguous()

    def U_rows(self, r, i0, i1, out):
        """Rows [i0, i1) of U(r) into ``out`` ((i1 - i0) x r, row-major) -- chunked formation."""
        if self.fullrank:
            self._full(r)
            if self.implicit:
                return gemm_triu(self.X[i0:i1], self._W, out=out)
            out.copy_(self.Qt[:, i0:i1].t())
            return out
        if self.implicit and self._implicit_w(r) is not None:
            return gemm(self.X[i0:i1], self._W, out=out, emulate=True)
        if self.tall:
            return gemm(self.Qt[:, i0:i1], self.UJ[:r], tA=True, tB=True, out=out)
        out.copy_(self.UJ[:r, i0:i1].t())
        return out

    def SVt(self, r):
        """diag(S[:r]) Vt[:r] = U[:, :r]^T X  (r x n)."""
        if self.fullrank:
            self._full(r)
            return self.Rt.t().contiguous()      # R (n x n, row-major): U(n) R = X
        if self.implicit:
            return (self.S[:r, None] * self.Vr[:r]).contiguous()
        if self.direct:
            return gemm(self.UJ[:r], self.X)                    # U^T X
        if self.tall:
            return gemm(self.UJ[:r], self.Rt, tB=True)          # U_R^T R
        W = gemm(self.UJ[:r], self.Rt)                          # U'^T R^T  (r x m)
        return gemm(W, self.Qt)                                 # ... Q^T   (r x n)

    def _full(self, r):
        if r != self.n:
            raise ValueError("certified full-rank factors cannot be truncated")

    def Vt(self, r):
        """First r right singular vectors as rows (r x n); needs want_v=True."""
        if self.implicit:
            return self.Vr[:r].contiguous()
        if self.VJ is None:
            raise ValueError("right singular vectors were not accumulated (want_v=False)")
        if self.tall or self.direct:
            return self.VJ[:r].contiguous()
        return gemm(self.VJ[:r], self.Qt)


# ---------------------------------------------------------------------------
# leading singular triplets only (rank-capped rounding)

_TOPK = os.environ.get("TTB_TOPK_SVD", "1") != "0"
_TOPK_MAX = 8          # largest rank cap served
_TOPK_MIN_N = 200      # smaller factors: the full Jacobi SVD is already cheap
_TOPK_BLOCK = 16       # iteration block (rank cap + oversampling)
_TOPK_CHECK = 6        # iterations between Rayleigh-Ritz convergence checks
_TOPK_MAX_ITERS = 60
_TOPK_TOL = 1e-13      # Ritz residual ||R^T u - theta v|| <= tol theta_max for every kept triplet
_topk_start = {}


def _topk_start_block(n, b):
    """Fixed (seeded) b x n start block, cached per shape: the iteration is deterministic."""
    key = (n, b)
    if key not in _topk_start:
        g = torch.Generator(device="cpu").manual_seed(20250913)
        _topk_start[key] = torch.randn(b, n, generator=g, dtype=F64).to(device())
    return _topk_start[key]


def topk_svd(X, kmax, delta):
    """Leading part of the truncated SVD a rank-capped rounding step needs (reference tensor_train/core.py
    :341-350, 377-386 with max_rank): returns (U (m x keep), carry = U^T X (keep x n)) with
    keep = min(kmax, _chop(s, delta)), or None when the route does not apply or did not converge (the
    caller then takes the full SVD). With a cap of a few ranks only the leading kmax singular triplets and
    ||X||_F matter: _chop's tails are tail_j^2 = ||X||_F^2 - sum_{i<j} s_i^2 for j <= kmax, so they are
    computed by a block power iteration on the triangular factor R of X (block 16, re-orthonormalized every
    step, Rayleigh-Ritz every 6 steps, deterministic start) until every kept triplet's residual is
    <= 1e-13 s_max -- instead of a one-sided Jacobi SVD of all n columns (21 ms at n = 510, twice per
    AMEn residual rounding). Used only for loose thresholds (delta >= 1e-3 ||X||_F, where the tails are
    free of cancellation); TTB_TOPK_SVD=0 disables it."""
    m, n = X.shape
    if not (_TOPK and kmax is not None and 1 <= kmax <= _TOPK_MAX and m >= n >= _TOPK_MIN_N):
        return None
    X = X.contiguous()
    fro2 = dot(X)
    if m > n:
        Qt, Rt = qr_colmajor(permute(X, (1, 0)), m, n)       # Qt (n, m) == col-major Q, Rt == row-major R^T
        R = Rt.t().contiguous()
    else:
        Qt, R = None, X
    b = _TOPK_BLOCK
    Vt = gemm(_topk_start_block(n, b), R)                     # rows: start vectors pulled through R once
    theta = None
    for it in range(0, _TOPK_MAX_ITERS, _TOPK_CHECK):
        for _ in range(_TOPK_CHECK):
            Vt, _ = qr_colmajor(Vt, n, b, want_r=False)       # orthonormal rows
            Wt = gemm(Vt, R, tB=True)                         # (R V)^T
            Vt = gemm(Wt, R)                                  # (R^T R V)^T
        Vt, _ = qr_colmajor(Vt, n, b, want_r=False)
        Wt = gemm(Vt, R, tB=True)                             # (b, n): columns of R V as rows
        Qwt, Rwt = qr_colmajor(Wt.clone(), n, b)              # R V = Qw Rw
        Us, S, Vst = svd(Rwt.t().contiguous())                # Rw = Us diag(S) Vst (b x b)
        order = torch.argsort(S, descending=True)
        S, Us, Vst = S[order], Us[:, order], Vst[order]
        Ut = gemm(Us, Qwt, tA=True)                           # left Ritz vectors of R as rows (b, n)
        Vr = gemm(Vst, Vt)                                    # right Ritz vectors as rows
        E = gemm(Ut[:kmax], R) - S[:kmax, None] * Vr[:kmax]   # rows: R^T u_i - theta_i v_i
        stats = torch.cat([S, torch.linalg.vector_norm(E, dim=1), fro2.reshape(1)]).cpu().numpy()
        theta, res, f2 = stats[:b], stats[b:b + kmax], float(stats[-1])
        if not np.isfinite(stats).all() or theta[0] <= 0.0:
            return None
        if delta < 1e-3 * np.sqrt(f2):
            return None                                       # tight threshold: tails would cancel
        if (res <= _TOPK_TOL * theta[0]).all():
            break
    else:
        return None
    head = np.concatenate([[0.0], np.cumsum(theta[:kmax] ** 2)])
    tails = np.sqrt(np.maximum(f2 - head, 0.0))               # tails[j]: after keeping j values, j = 0..kmax
    hit = np.flatnonzero(tails <= delta)
    keep = max(1, int(hit[0])) if hit.size else kmax
    keep = min(keep, kmax, n)
    UXt = Ut[:keep] if Qt is None else gemm(Ut[:keep], Qt)    # (keep, m): left singular vectors of X as rows
    carry = gemm(UXt, X)                                      # diag(S) Vt = U^T X
    return UXt.t().contiguous(), carry


_SPECULATIVE = os.environ.get("TTB_ROUND_SPECULATIVE", "1") != "0"
_SPEC_SUBSET = 8        # the step-0 certificate uses the Gram over 1 / 8 of the middle core's columns


def speculative_applies(n0, r1, n1, n2, d):
    """Shapes fullrank_speculative_3core serves: square first unfolding (n0 == r1), large tile-aligned factors."""
    return bool(_SPECULATIVE and _FULLRANK and _FULLRANK_IDENTITY and _GRAM and _OZAKI and d == 3 and n0 == r1
                and r1 >= _FULLRANK_MIN_N and r1 % 128 == 0 and n2 >= _IDENTITY_Q_MIN and n2 % 128 == 0
                and r1 * n1 >= _GRAM_MIN_M and (r1 * n1) % 64 == 0 and n1 % _SPEC_SUBSET == 0
                and (n1 // _SPEC_SUBSET) * n2 >= 4 * r1 and ((n1 // _SPEC_SUBSET) * n2) % 64 == 0)


def fullrank_speculative_3core(Y0, Y1p, eps, d):
    """Certified full-rank rounding of a 3-core TT whose last core is already the identity, in one pass.

    Y0 (n0 x r1, square, r1 = n0): the first core's unfolding; Y1p (r1, n1, n2): the middle core after the
    carry of the last one. When BOTH left-to-right steps keep every singular value the rounded TT is
        core 0 = I,   core 1 = Q of (Y0 x_1 Y1p) = Z L^-T,   core 2 = L^T      (Z = Y0 x_1 Y1p, Z^T Z = L L^T),
    and the right-to-left orthogonalization of the middle core (a 1024 x 1M Gram, its Cholesky factor L1
    and the carry through it) only ever served two numbers: the tensor norm (for delta) and the step-0
    certificate s_min(Y0 L1) > 2 delta. Both are had more cheaply, and rigorously:
      * ||Y||_F^2 = trace(Z^T Z) -- the Gram the second step needs anyway (cores 0 and 2 are identities);
      * s_min(Y0 L1) >= s_min(Y0 L_S) for the Cholesky factor L_S of the Gram over ANY subset S of the
        middle core's columns, since B B^T - B_S B_S^T is positive semidefinite: 1 / 8 of the columns here.
    So Z is formed speculatively (the carry Y0, no L1 in it: Y0 L1 L1^-1 = Y0), one host synchronization
    reads both certificates, and on any failure None is returned and the caller runs the ordinary sweeps.
    Returns (factors of the middle step, total norm) with factors.U(n) the middle core and factors.SVt(n) the
    carry into the last."""
    r1, n1, n2 = Y1p.shape
    if not (speculative_applies(Y0.shape[0], r1, n1, n2, d) and Y0.shape == (r1, r1)):
        return None
    B = Y1p.reshape(r1, n1 * n2)
    sub = (n1 // _SPEC_SUBSET) * n2
    # ---- step-0 certificate from the column subset S: the Gram G_S = B_S B_S^T, then H = Y0 G_S Y0^T
    ws = torch.empty(int(call_raw("ttb_ozaki_gram_rows_workspace", r1, sub)), dtype=torch.uint8, device=device())
    Gs = empty(r1, r1)
    with _profiled("ozaki-gram", (r1, r1, sub), 1.0 * r1 * (r1 + 128) * sub):
        call("ttb_ozaki_gram_rows", r1, sub, ptr(B), B.stride(0), ptr(Gs), r1, ptr(ws))
    del ws
    # s_min(Y0 L_S)^2 = lambda_min(Y0 G_S Y0^T): one Cholesky factorization of H = Y0 G_S Y0^T (L_S itself is
    # not needed); the Gram's upper block triangle is mirrored, so G_S is symmetric to the bit and so is H's
    # lower triangle that potrf reads
    info_s = torch.zeros(1, dtype=I32, device=device())
    G0 = gemm(gemm(Y0, Gs), Y0, tB=True)
    info0 = empty(1, dtype=I32)
    call("ttb_potrf", r1, ptr(G0), r1, ptr(info0))
    L0 = empty(r1, r1)
    call("ttb_tri_from_potrf", r1, ptr(G0), r1, ptr(L0), r1, None)
    Li0 = _trtri(L0, r1)
    # ---- speculative middle unfolding Z = Y0 x_1 Y1p and its Gram
    Z = gemm(Y0, B, emulate=True).reshape(r1 * n1, n2)
    m = r1 * n1
    ws = torch.empty(int(call_raw("ttb_ozaki_gram_workspace", m, n2)), dtype=torch.uint8, device=device())
    G = empty(n2, n2)
    with _profiled("ozaki-gram", (n2, n2, m), 1.0 * n2 * (n2 + 128) * m):
        call("ttb_ozaki_gram", m, n2, ptr(Z), n2, ptr(G), n2, ptr(ws))
    del ws
    trace = G.diagonal().sum().reshape(1)
    info1 = empty(1, dtype=I32)
    call("ttb_potrf", n2, ptr(G), n2, ptr(info1))
    Rt = empty(n2, n2)
    call("ttb_tri_from_potrf", n2, ptr(G), n2, ptr(Rt), n2, None)
    Li = _trtri(Rt, n2)
    v = torch.cat([trace, nrm2(Li0).reshape(1), _norm2_est_dev(L0), _norm2_est_dev(Li0), nrm2(Li).reshape(1),
                   _norm2_est_dev(Rt), _norm2_est_dev(Li), info_s.to(F64), info0.to(F64), info1.to(F64)]).cpu().numpy()
    if not np.isfinite(v).all() or v[7] != 0.0 or v[8] != 0.0 or v[9] != 0.0 or v[0] <= 0.0:
        return None
    total = float(np.sqrt(v[0]))
    delta = eps * total / np.sqrt(d - 1)
    ok0 = v[1] > 0.0 and 1.0 / v[1] > _FULLRANK_MARGIN * delta and 1.1 * v[2] * v[3] <= 1e5
    ok1 = v[4] > 0.0 and 1.0 / v[4] > _FULLRANK_MARGIN * delta and 1.1 * v[5] * v[6] <= 1.0 / _GRAM_MIN_RATIO
    if not (ok0 and ok1):
        return None
    return SVDFactors.certified(Z, Rt, Li), total


def svd(X):
    """np.linalg.svd(X, full_matrices=False) on the device: (U, S, Vt)."""
    f = SVDFactors(X, want_v=True)
    k = min(f.m, f.n)
    return f.U(k), f.S, f.Vt(k)


# ---------------------------------------------------------------------------
# solvers

def solve(A, B, status=None):
    """np.linalg.solve(A, B) with LU + partial pivoting on the device. ``status`` (an object with
    add(kind, status_tensor)): the singularity flag is handed to it instead of being read here (the caller
    raises LinAlgError at its next synchronization)."""
    n = A.shape[0]
    if A.shape != (n, n):
        raise ValueError("square matrix expected")
    vec = B.dim() == 1
    Bm = B.reshape(n, 1) if vec else B
    LU = A.contiguous().clone()          # col-major memory of A^T
    Bcm = permute(Bm, (1, 0))            # col-major B
    piv = empty(n, dtype=I32)
    info = empty(1, dtype=I32)
    call("ttb_lu_solve", n, ptr(LU), n, ptr(piv), Bm.shape[1], ptr(Bcm), n, 1, ptr(info))
    if status is not None:
        status.add("solve", info)
    elif int(info.item()) != 0:
        raise LinAlgError("Singular matrix")
    X = Bcm.t()
    return X.reshape(n) if vec else X


def cho_solve_or_lu(Bm, b):
    """scipy cho_factor/cho_solve with fallback to a pivoted LU solve (reference amen.py:166-171)."""
    n = Bm.shape[0]
    L = Bm.contiguous().clone()
    info = empty(1, dtype=I32)
    call("ttb_potrf", n, ptr(L), n, ptr(info))
    if int(info.item()) == 0 and n * 8 <= 200 * 1024:
        x = b.contiguous().clone().reshape(-1)
        call("ttb_potrs", n, ptr(L), n, ptr(x))
        return x
    return solve(Bm, b.reshape(-1))


class MaxvolError(np.linalg.LinAlgError):
    """Mirror of reference MaxvolError (tensor_train/maxvol.py:15)."""


def maxvol_colmajor(Qcm, n, r, tol=1.01, max_iters=200):
    """Sorted maxvol rows of a col-major n x r matrix (torch (r, n)); host int64 array."""
    if n <= r:
        return np.arange(n)
    ws = empty(int(call_raw("ttb_maxvol_workspace", n, r)))
    iws = empty(n + 1, dtype=I32)
    rows = empty(r, dtype=I32)
    call("ttb_maxvol", n, r, ptr(Qcm.contiguous()), float(tol), int(max_iters), ptr(rows), ptr(ws), ptr(iws))
    if int(iws[n].item()) != 0:
        raise MaxvolError("degenerate pivot: matrix has deficient column rank")
    return rows.cpu().numpy().astype(np.int64)


def maxvol_colmajor_dev(Qcm, n, r, pending, tol=1.01, max_iters=200):
    """maxvol_colmajor without the host round trip: the sorted rows stay on the device (int32 CUDA tensor)
    and the degeneracy flag is appended to ``pending`` (an object with add(kind, status_tensor); the caller
    checks it at its next synchronization and raises MaxvolError then). On failure the rows are 0..r-1."""
    if n <= r:
        return torch.arange(n, dtype=I32, device=device())
    ws = empty(int(call_raw("ttb_maxvol_workspace", n, r)))
    iws = empty(n + 1, dtype=I32)
    rows = torch.arange(r, dtype=I32, device=device())
    call("ttb_maxvol", n, r, ptr(Qcm.contiguous()), float(tol), int(max_iters), ptr(rows), ptr(ws), ptr(iws))
    pending.add("maxvol", iws[n:n + 1])
    return rows


def maxvol(M, tol=1.01, max_iters=200):
    """Reference maxvol(M) (tensor_train/maxvol.py:37-62): sorted row indices (host int64 array) of a
    row-major (n x r) matrix -- a CUDA tensor, or a numpy array / nested list as in the reference (copied
    to the device once)."""
    if not isinstance(M, torch.Tensor):
        M = np.asarray(M, dtype=float)
        if M.ndim != 2:
            raise ValueError("maxvol expects a matrix")
        M = torch.as_tensor(M, device=device())
    if M.dim() != 2:
        raise ValueError("maxvol expects a matrix")
    n, r = M.shape
    if tol < 1.0:
        raise ValueError("tol must be at least 1")
    return maxvol_colmajor(permute(M.to(F64).contiguous(), (1, 0)), n, r, tol, max_iters)
