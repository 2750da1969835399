"""Banded TT-operator contractions staged as batched FP64 DMMA GEMMs, and the AMEn residual
``f - A u`` in compressed form.

The reference contracts a banded operator core M[a, i, j, b] (half-bandwidth h) with a
vector-side tensor through 2h+1 shifted einsums (``_OpCore.apply``/``apply_rev``,
amen.py:77-99). With operator ranks ~100 (non-separable geometries, configs[2..4]) those
contractions are the flops of the whole solve, so here they are GEMMs: with the core re-laid
out once per solve as Mf[i, t, a, b] (forward) / Mr[i, t, b, a] (reverse) and the vector-side
operand as Tp[j + h, a, X] (mode-major, h zero blocks at each end), output row block i is
    out[i] (X x Rb) = Tp[i : i + 2h + 1]^T (X x (2h+1) Ra)  @  Mf[i] ((2h+1) Ra x Rb)
i.e. one strided-batched GEMM over the n mode indices (``ttb_band_gemm``).

The residual f - A u of the reference AMEn (amen.py:262-264) is a TT whose middle cores have
rank R_A r_u + r_f (6.9e3 for configs[2]: a 97 GB core at n = 256). Its norm and its rank-
``kick_rank`` rounding depend only on the tensor, not on the representation, so here it is
built directly in a representation whose ranks are at most the mode-size products: the first
cores are left-orthogonalised and the last ones right-orthogonalised *structurally* (the
block-diagonal f (+) A u cores are never formed, only their products with the running
triangular factor), and the middle core is contracted from both sides. The resulting TT has
orthonormal outer cores, so its norm is the middle core's norm, and rounding it with the
reference's tt_round gives the reference's z (exact arithmetic; roundoff differs).
"""

from __future__ import annotations

import os

import torch

from .. import linalg as L
from .._lib import call, call_raw, ptr

_BAND_MODE = os.environ.get("TTB_BAND", "auto")          # gemm | naive | auto
_RES_MODE = os.environ.get("TTB_AMEN_RESIDUAL", "auto")  # compressed | explicit | auto


def use_gemm(Ra: int, Rb: int) -> bool:
    """GEMM-staged banded contractions once the operator rank product makes them dense enough."""
    if _BAND_MODE == "gemm":
        return True
    if _BAND_MODE == "naive":
        return False
    return Ra * Rb >= 64


def use_compressed_residual(Ms, u, F) -> bool:
    """Compressed residual when the explicit f - A u cores would be large (> 8M doubles in total)."""
    if _RES_MODE == "compressed":
        return True
    if _RES_MODE == "explicit":
        return False
    tot = 0
    for M, U, G in zip(Ms, u, F):
        tot += (M.shape[0] * U.shape[0] + G.shape[0]) * U.shape[1] * (M.shape[3] * U.shape[2] + G.shape[2])
    return tot > (1 << 23)


def _even(r):
    return r + (r & 1)


def pad_last(T, P):
    """T with its last axis zero-padded to P entries (T itself when already P)."""
    if T.shape[-1] == P:
        return T
    out = L.zeros(*T.shape[:-1], P)
    out[..., : T.shape[-1]] = T
    return out


class GemmLayouts:
    """Per-core GEMM layouts of a banded operator: Mf = (n, 2h+1, Ra, Rb'), Mr = (n, 2h+1, Rb, Ra').

    The output rank of each layout is zero-padded to even (Rb' = Rb + Rb % 2): the band GEMM's
    B operand and output rows then keep 16-byte alignment (16-byte cp.async path; measured
    29.0 -> 31.7 TF/s at configs[3] shapes). Consumers either carry the zero columns through
    (the PCG matvec, whose phiR operand is padded the same way) or drop them (trim).
    """

    def __init__(self, Ms, h):
        self.Ms, self.h = Ms, h
        self._f = [None] * len(Ms)
        self._r = [None] * len(Ms)

    def fwd(self, k):
        if self._f[k] is None:
            self._f[k] = pad_last(L.permute(self.Ms[k], (1, 2, 0, 3)), _even(self.Ms[k].shape[3]))
        return self._f[k]

    def rev(self, k):
        if self._r[k] is None:
            self._r[k] = pad_last(L.permute(self.Ms[k], (1, 2, 3, 0)), _even(self.Ms[k].shape[0]))
        return self._r[k]


def _padded(n, h, Rin, X):
    blk = Rin * X
    Tp = L.empty((n + 2 * h) * blk)
    if h:
        Tp[: h * blk].zero_()
        Tp[(n + h) * blk:].zero_()
    return Tp


def band_gemm(Tp, Mt, n, h, Rin, X):
    """out[i, X, o] = sum_{t, r} Tp[i + t, r, X] Mt[i, t, r, o]  ->  (n, X, Mt.shape[3]) (padded rank)."""
    Rout = Mt.shape[3]
    out = L.empty(n, X, Rout)
    call("ttb_band_gemm", n, h, Rin, Rout, X, ptr(Tp), ptr(Mt), ptr(out))
    return out


def left_stage(Lp, U, h):
    """Tp[j + h, a, (k, y)] = sum_x Lp[a, k, x] U[x, j, y]   (Lp (Ra, K, x), U (x, n, y))."""
    Ra, Kd, x = Lp.shape
    _, n, y = U.shape
    blk = Ra * Kd * y
    Tp = _padded(n, h, Ra, Kd * y)
    L.gemm_strided(0, 0, Ra * Kd, y, x, Lp.contiguous(), x, 0, U.contiguous(), n * y, y, Tp[h * blk:], y, blk, n)
    return Tp


def right_stage(Rp, U, h):
    """Tp[j + h, b, (k, x)] = sum_y Rp[b, k, y] U[x, j, y]   (Rp (Rb, K, y), U (x, n, y))."""
    Rb, Kd, y = Rp.shape
    x, n, _ = U.shape
    blk = Rb * Kd * x
    Tp = _padded(n, h, Rb, Kd * x)
    L.gemm_strided(0, 1, Rb * Kd, x, y, Rp.contiguous(), y, 0, U.contiguous(), n * y, y, Tp[h * blk:], x, blk, n)
    return Tp


def env_left_A(phi, U, lay, k):
    """Reference _env_left_A (amen.py:106-109) in GEMM form: (x,a,y),(y,j,v) -> (u,b,v)."""
    h = lay.h
    x, Ra, y = phi.shape
    _, n, v = U.shape
    Mf = lay.fwd(k)
    Rb, Rbp = lay.Ms[k].shape[3], Mf.shape[3]
    Tp = left_stage(L.permute(phi, (1, 0, 2)), U, h)                 # (j, a, (x, v))
    out = band_gemm(Tp, Mf, n, h, Ra, x * v)                          # (i, x, v, b')
    Up = L.permute(U, (1, 0, 2)).reshape(n * x, v)                   # (i, x, u)
    res = L.gemm(Up, out.reshape(n * x, v * Rbp), tA=True)           # (u, v, b')
    return L.permute(res.reshape(v, v, Rbp)[:, :, :Rb], (0, 2, 1))


def env_right_A(phi, U, lay, k):
    """Reference _env_right_A (amen.py:112-115) in GEMM form: (s,b,v),(w,j,v) -> (z,a,w)."""
    h = lay.h
    s, Rb, v = phi.shape
    w, n, _ = U.shape
    Mr = lay.rev(k)
    Ra, Rap = lay.Ms[k].shape[0], Mr.shape[3]
    Tp = right_stage(L.permute(phi, (1, 0, 2)), U, h)                # (j, b, (s, w))
    out = band_gemm(Tp, Mr, n, h, Rb, s * w)                         # (i, s, w, a')
    res = L.gemm(U.reshape(w, n * s), out.reshape(n * s, w * Rap))  # (z, w, a')
    return L.permute(res.reshape(w, w, Rap)[:, :, :Ra], (0, 2, 1))


# ---------------------------------------------------------------------------
# compressed residual

def _ones(*shape):
    return torch.ones(*shape, dtype=torch.float64, device=L.device())


def _a_left(LA, U, lay, k):
    """sum_{a,x} LA[k', x, a] (A_k (x) u_k)[(a,x), i, (b,y)] -> (n, K, y, b) (row order i, k')."""
    Kd, x, Ra = LA.shape
    n = U.shape[1]
    y = U.shape[2]
    Mf = lay.fwd(k)
    Rb = lay.Ms[k].shape[3]
    Tp = left_stage(L.permute(LA, (2, 0, 1)), U, lay.h)              # (j, a, (k', y))
    return band_gemm(Tp, Mf, n, lay.h, Ra, Kd * y).reshape(n, Kd, y, Mf.shape[3])[..., :Rb]


def _a_right(RA, U, lay, k):
    """sum_{b,y} (A_k (x) u_k)[(a,x), i, (b,y)] RA[y, b, k'] -> (n, K, x, a)."""
    y, Rb, Kd = RA.shape
    x, n, _ = U.shape
    Mr = lay.rev(k)
    Ra = lay.Ms[k].shape[0]
    Tp = right_stage(L.permute(RA, (1, 2, 0)), U, lay.h)             # (j, b, (k', x))
    return band_gemm(Tp, Mr, n, lay.h, Rb, Kd * x).reshape(n, Kd, x, Mr.shape[3])[..., :Ra]


def compressed_residual(lay, u, F):
    """Cores of f - A u with ranks bounded by the mode-size products, and its norm (device 0-d).

    A-part rank index order inside the running factors is (x, a) (u rank, operator rank)."""
    d = len(u)
    m = (d - 1) // 2
    Lf, LA = _ones(1, 1), -_ones(1, 1, 1)           # (kL, r_f), (kL, r_u, R_A)
    left = []
    for k in range(m):
        Fk, Uk = F[k], u[k]
        c, n, fr = Fk.shape
        kL = Lf.shape[0]
        Zf = L.gemm(Lf, Fk.reshape(c, n * fr)).reshape(kL, n, fr)
        Za = L.permute(_a_left(LA, Uk, lay, k), (1, 0, 2, 3)).reshape(kL, n, -1)
        Z = torch.cat([Zf, Za], dim=2)
        cols = Z.shape[2]
        Qt, Rt = L.qr_colmajor(L.permute(Z.reshape(kL * n, cols), (1, 0)), kL * n, cols)
        kk = Qt.shape[0]
        left.append(L.permute(Qt, (1, 0)).reshape(kL, n, kk))
        R = L.permute(Rt, (1, 0))                                     # (kk, cols)
        Lf = R[:, :fr].contiguous()
        LA = R[:, fr:].contiguous().reshape(kk, Uk.shape[2], lay.Ms[k].shape[3])
    Rf, RA = _ones(1, 1), _ones(1, 1, 1)            # (r_f, kR), (r_u, R_A, kR)
    right = []
    for k in range(d - 1, m, -1):
        Fk, Uk = F[k], u[k]
        c, n, fr = Fk.shape
        kR = Rf.shape[1]
        Zf = L.gemm(Fk.reshape(c * n, fr), Rf).reshape(c, n * kR)
        Za = L.permute(_a_right(RA, Uk, lay, k), (2, 3, 0, 1))       # (x, a, i, k')
        Z = torch.cat([Zf, Za.reshape(-1, n * kR)], dim=0)
        rows = Z.shape[0]
        Qt, Rt = L.qr_colmajor(Z.contiguous(), n * kR, rows)
        kk = Qt.shape[0]
        right.insert(0, Qt.reshape(kk, n, kR))
        Rf = Rt[:c].contiguous()
        RA = Rt[c:].contiguous().reshape(Uk.shape[0], lay.Ms[k].shape[0], kk)
    Fm, Um = F[m], u[m]
    c, n, fr = Fm.shape
    kL, kR = Lf.shape[0], Rf.shape[1]
    Zm = L.gemm(L.gemm(Lf, Fm.reshape(c, n * fr)).reshape(kL * n, fr), Rf).reshape(kL, n, kR)
    out = _a_left(LA, Um, lay, m)                                     # (i, k', y, b)
    ZA = L.gemm(out.reshape(n * kL, -1), RA.reshape(-1, kR), emulate=True)   # (i, k', kR)
    Zm = Zm + L.permute(ZA.reshape(n, kL, kR), (1, 0, 2))
    return left + [Zm] + right, L.nrm2(Zm)
