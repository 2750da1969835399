"""Tensor-train vectors and operators resident in HBM (reference tensor_train/core.py).

Cores are FP64 torch CUDA tensors. ``TtTensor`` cores are (r0, n, r1).
``TtMatrix`` cores are either dense (r0, n, m, r1) or BANDED
(r0, n, 2h+1, r1) with entry [a, i, t, b] = A[a, i, i+t-h, b] -- the IGA
stiffness operator has half-bandwidth h = p, so a banded core stores
(2p+1)/n of the dense one and every kernel reads only the band.

Arithmetic follows the reference exactly (block-diagonal add, core-wise
matvec, right-to-left QR then left-to-right truncated SVD rounding with the
eps*||t||/sqrt(d-1) budget) but each step runs on libttiga_b200.so kernels.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import linalg as L
from .._lib import call_raw, call, device, ptr

__all__ = [
    "TtShapeError", "TtTensor", "TtMatrix", "tt_add", "tt_sub", "tt_scale", "tt_dot", "tt_norm", "tt_matvec",
    "tt_round", "tt_from_full", "tt_matrix_from_full", "to_device",
]


class TtShapeError(ValueError):
    """Mode sizes or bond ranks do not conform (reference core.py:34)."""


def to_device(x):
    if isinstance(x, torch.Tensor):
        return x.to(device=device(), dtype=torch.float64)
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=device())


class DeviceCore(torch.Tensor):
    """A TT core in device memory that numpy can read: ``np.asarray(core)`` copies it to the host, so
    reference-style code that compares cores with numpy (np.array_equal / np.allclose on ``t.cores[k]``,
    the reference's cores being numpy arrays) keeps working. Torch operations see a plain CUDA tensor
    (``__torch_function__`` disabled: no dispatch overhead, results are ordinary tensors)."""

    __torch_function__ = torch._C._disabled_torch_function_impl

    def __array__(self, dtype=None, copy=None):
        a = torch.Tensor.cpu(self).numpy()
        return a if dtype is None else a.astype(dtype, copy=False)


def _core(G):
    return to_device(G).contiguous().as_subclass(DeviceCore)


def _check_chain(cores, order):
    if not cores:
        raise TtShapeError("empty core list")
    for k, G in enumerate(cores):
        if G.dim() != order:
            raise TtShapeError(f"core {k} must have {order} axes, got {G.dim()}")
    if cores[0].shape[0] != 1 or cores[-1].shape[-1] != 1:
        raise TtShapeError("boundary ranks must be 1")
    for k in range(len(cores) - 1):
        if cores[k].shape[-1] != cores[k + 1].shape[0]:
            raise TtShapeError(f"rank mismatch between cores {k} and {k + 1}")


class TtTensor:
    """Chain of (r_{k-1}, n_k, r_k) device cores (reference core.py:54-146)."""

    def __init__(self, cores):
        self.cores = [_core(G) for G in cores]
        _check_chain(self.cores, 3)

    d = property(lambda s: len(s.cores))
    mode_sizes = property(lambda s: tuple(int(G.shape[1]) for G in s.cores))
    ranks = property(lambda s: (1,) + tuple(int(G.shape[2]) for G in s.cores))
    n_params = property(lambda s: int(sum(G.numel() for G in s.cores)))

    def copy(self):
        return TtTensor([G.clone() for G in self.cores])

    @staticmethod
    def zeros(mode_sizes):
        return TtTensor([L.zeros(1, int(n), 1) for n in mode_sizes])

    @staticmethod
    def ones(mode_sizes):
        return TtTensor([torch.ones(1, int(n), 1, dtype=torch.float64, device=device()) for n in mode_sizes])

    @staticmethod
    def rank_one(vectors):
        return TtTensor([to_device(v).reshape(1, -1, 1) for v in vectors])

    @staticmethod
    def random(mode_sizes, ranks, rng):
        """Same draws as the reference (numpy Generator), moved to the device."""
        full = (1,) + tuple(int(r) for r in ranks) + (1,)
        if len(full) != len(mode_sizes) + 1:
            raise TtShapeError("need len(ranks) == d - 1")
        return TtTensor([rng.standard_normal((full[k], n, full[k + 1])) for k, n in enumerate(mode_sizes)])

    def full_device(self):
        X = self.cores[0][0]
        for G in self.cores[1:]:
            X = L.tdot(X, G, ([X.dim() - 1], [0]))
        return X[..., 0]

    def full(self):
        """Densify (small instances); returns a host numpy array like the reference."""
        return self.full_device().cpu().numpy()

    def gather(self, idx):
        """Entries at multi-indices idx (N, d) (reference core.py:118-124): a CUDA index tensor gives a CUDA
        (N,) tensor, numpy / list indices a numpy array (the reference's types)."""
        if not isinstance(idx, torch.Tensor):
            return self.gather(torch.as_tensor(np.asarray(idx), dtype=torch.int64, device=device())).cpu().numpy()
        idx = idx.to(device=device(), dtype=torch.int64).contiguous()
        if self.d != 3:
            v = self.cores[0][0, idx[:, 0], :]
            for k in range(1, self.d):
                v = torch.einsum("nr,rns->ns", v, self.cores[k][:, idx[:, k], :])
            return v[:, 0]
        out = L.empty(idx.shape[0])
        G0, G1, G2 = self.cores
        call("ttb_tt_gather3", int(idx.shape[0]), ptr(idx), ptr(G0), G0.shape[1], G0.shape[2], ptr(G1), G1.shape[1],
             G1.shape[2], ptr(G2), G2.shape[1], ptr(out))
        return out

    __add__ = lambda s, o: tt_add(s, o)
    __sub__ = lambda s, o: tt_sub(s, o)
    __mul__ = lambda s, c: tt_scale(s, c)
    __rmul__ = __mul__
    __neg__ = lambda s: tt_scale(s, -1.0)

    def norm(self):
        return tt_norm(self)

    def round(self, eps, max_rank=None):
        return tt_round(self, eps, max_rank)


class TtMatrix:
    """Chain of operator cores (reference core.py:149-221), dense or banded (``band`` = h)."""

    def __init__(self, cores, band=None, col_sizes=None):
        self.cores = [_core(G) for G in cores]
        self.band = None if band is None else int(band)
        _check_chain(self.cores, 4)
        if self.band is not None:
            for G in self.cores:
                if G.shape[2] != 2 * self.band + 1:
                    raise TtShapeError("banded core width must be 2h+1")

    d = property(lambda s: len(s.cores))
    row_sizes = property(lambda s: tuple(int(G.shape[1]) for G in s.cores))
    ranks = property(lambda s: (1,) + tuple(int(G.shape[3]) for G in s.cores))

    @property
    def col_sizes(self):
        if self.band is not None:
            return self.row_sizes
        return tuple(int(G.shape[2]) for G in self.cores)

    @property
    def n_params(self):
        """Parameter count of the DENSE cores (the reference's compression-ratio convention)."""
        return int(sum(G.shape[0] * G.shape[1] * n * G.shape[3] for G, n in zip(self.cores, self.col_sizes)))

    @property
    def stored_params(self):
        return int(sum(G.numel() for G in self.cores))

    def copy(self):
        return TtMatrix([G.clone() for G in self.cores], self.band)

    @staticmethod
    def identity(mode_sizes):
        return TtMatrix([torch.ones(1, int(n), 1, 1, dtype=torch.float64, device=device()) for n in mode_sizes],
                        band=0)

    @staticmethod
    def rank_one(factors):
        return TtMatrix([to_device(A).reshape(1, A.shape[0], A.shape[1], 1) for A in factors])

    @staticmethod
    def banded_from_dense_cores(cores, h):
        """Pack dense (r0, n, n, r1) cores with |i-j| <= h into the banded layout."""
        out = []
        for G in cores:
            G = to_device(G)
            r0, n, m, r1 = G.shape
            B = L.zeros(r0, n, 2 * h + 1, r1)
            for t in range(2 * h + 1):
                o = t - h
                i0, i1 = max(0, -o), min(n, n - o)
                if i1 > i0:
                    ii = torch.arange(i0, i1, device=G.device)
                    B[:, i0:i1, t, :] = G[:, ii, ii + o, :]
            out.append(B)
        return TtMatrix(out, band=h)

    def dense_cores(self):
        if self.band is None:
            return list(self.cores)
        h = self.band
        out = []
        for G in self.cores:
            r0, n, B, r1 = G.shape
            D = L.zeros(r0, n, n, r1)
            for t in range(B):
                o = t - h
                i0, i1 = max(0, -o), min(n, n - o)
                if i1 > i0:
                    ii = torch.arange(i0, i1, device=G.device)
                    D[:, ii, ii + o, :] = G[:, i0:i1, t, :]
            out.append(D)
        return out

    def to_dense(self):
        return TtMatrix(self.dense_cores())

    def transpose(self):
        if self.band is None:
            return TtMatrix([L.permute(G, (0, 2, 1, 3)) for G in self.cores])
        h = self.band
        out = []
        for G in self.cores:
            r0, n, B, r1 = G.shape
            T = L.zeros(r0, n, B, r1)
            for t in range(B):  # A^T[i, i+o] = A[i+o, i] -> band slot 2h - t at row i+o
                o = t - h
                i0, i1 = max(0, -o), min(n, n - o)
                if i1 > i0:
                    T[:, i0:i1, t, :] = G[:, i0 + o:i1 + o, 2 * h - t, :]
            out.append(T)
        return TtMatrix(out, band=h)

    def full(self):
        """Dense (prod rows) x (prod cols) host matrix (small instances)."""
        cores = self.dense_cores()
        X = cores[0][0]
        for G in cores[1:]:
            X = L.tdot(X, G, ([X.dim() - 1], [0]))
        X = X[..., 0]
        d = self.d
        perm = [2 * k for k in range(d)] + [2 * k + 1 for k in range(d)]
        X = L.permute(X, perm)
        return X.reshape(int(np.prod(self.row_sizes)), int(np.prod(self.col_sizes))).cpu().numpy()

    __add__ = lambda s, o: tt_add(s, o)
    __sub__ = lambda s, o: tt_sub(s, o)
    __mul__ = lambda s, c: tt_scale(s, c)
    __rmul__ = __mul__
    __matmul__ = lambda s, x: tt_matvec(s, x)

    def round(self, eps, max_rank=None):
        return tt_round(self, eps, max_rank)


# ---------------------------------------------------------------------------
# fused ("vector") view: operator cores as (r0, n*m, r1) or (r0, n*(2h+1), r1)

def _fused(t):
    if isinstance(t, TtMatrix):
        return [G.reshape(G.shape[0], -1, G.shape[3]) for G in t.cores], ("matrix", t)
    return list(t.cores), ("tensor", None)


def _unfused(cores, tag):
    kind, proto = tag
    if kind == "tensor":
        return TtTensor(cores)
    out = [G.reshape(G.shape[0], P.shape[1], P.shape[2], G.shape[2]) for G, P in zip(cores, proto.cores)]
    M = TtMatrix(out, proto.band)
    if proto.band is not None:
        _zero_band_padding(M)
    return M


def _zero_band_padding(M):
    h = M.band
    for G in M.cores:
        n = G.shape[1]
        for t in range(2 * h + 1):
            o = t - h
            if o < 0:
                G[:, : min(n, -o), t, :] = 0.0
            elif o > 0:
                G[:, max(0, n - o):, t, :] = 0.0


def _same_kind(a, b):
    if isinstance(a, TtMatrix) != isinstance(b, TtMatrix):
        raise TtShapeError("cannot combine a TT tensor with a TT operator")
    if isinstance(a, TtMatrix):
        if a.row_sizes != b.row_sizes or a.col_sizes != b.col_sizes:
            raise TtShapeError("operator mode sizes differ")
        if a.band != b.band:
            ha = a.band if a.band is not None else max(a.col_sizes)
            hb = b.band if b.band is not None else max(b.col_sizes)
            if a.band is None or b.band is None:
                return a.to_dense() if a.band is not None else a, b.to_dense() if b.band is not None else b
            h = max(ha, hb)
            return _widen(a, h), _widen(b, h)
    elif a.mode_sizes != b.mode_sizes:
        raise TtShapeError("tensor mode sizes differ")
    return a, b


def _widen(M, h):
    if M.band == h:
        return M
    out = []
    for G in M.cores:
        r0, n, B, r1 = G.shape
        W = L.zeros(r0, n, 2 * h + 1, r1)
        W[:, :, h - M.band: h + M.band + 1, :] = G
        out.append(W)
    return TtMatrix(out, h)


def tt_add(a, b):
    """Block-diagonal core concatenation, ranks add (reference core.py:260-279)."""
    a, b = _same_kind(a, b)
    ca, tag = _fused(a)
    cb, _ = _fused(b)
    d = len(ca)
    out = []
    for k, (Ga, Gb) in enumerate(zip(ca, cb)):
        ra0, n, ra1 = Ga.shape
        rb0, _, rb1 = Gb.shape
        if d == 1:
            G = Ga + Gb
        elif k == 0:
            G = torch.cat([Ga, Gb], dim=2)
        elif k == d - 1:
            G = torch.cat([Ga, Gb], dim=0)
        else:
            G = L.zeros(ra0 + rb0, n, ra1 + rb1)
            G[:ra0, :, :ra1] = Ga
            G[ra0:, :, ra1:] = Gb
        out.append(G)
    return _unfused(out, tag)


def tt_scale(a, c):
    """Scalar multiple absorbed into the first core (reference core.py:286-291)."""
    cores, tag = _fused(a)
    cores = [G.clone() for G in cores]
    cores[0] = cores[0] * float(c)
    return _unfused(cores, tag)


def tt_sub(a, b):
    return tt_add(a, tt_scale(b, -1.0))


def tt_dot(a, b):
    """Exact chain contraction (reference core.py:294-301); returns a Python float."""
    if a.mode_sizes != b.mode_sizes:
        raise TtShapeError("tensor mode sizes differ")
    return float(_dot_dev(a, b).item())


def _dot_dev(a, b):
    v = torch.ones(1, 1, dtype=torch.float64, device=device())
    for Ga, Gb in zip(a.cores, b.cores):
        ra, n, rc = Ga.shape
        rb, _, rd = Gb.shape
        W = L.gemm(v, Ga.reshape(ra, n * rc), tA=True)            # (rb, n*rc)
        W = L.permute(W.reshape(rb, n, rc), (0, 1, 2)).reshape(rb * n, rc)
        v = L.gemm(W, Gb.reshape(rb * n, rd), tA=True)            # (rc, rd)
    return v[0, 0]


def _carry_into(carry, nxt):
    """carry @ (the next core's left unfolding); nxt: a core, or the unformed Q^T of a one-pass CholeskyQR
    (linalg.LazyQt over the core's (r0, n r1) unfolding, its ``shape`` set to the core's)."""
    if isinstance(nxt, L.LazyQt):
        _, n, r1 = nxt.shape
        return nxt.carried(carry).reshape(carry.shape[0], n, r1)
    return L.gemm(carry, nxt.reshape(nxt.shape[0], -1), emulate=True).reshape(carry.shape[0], nxt.shape[1],
                                                                             nxt.shape[2])


def _rl_orthogonalize(cores, renorm=False, svd0=False, fullrank_eps=None, lazy_q=False):
    """Right-to-left Householder sweep: cores[1:] right-orthonormal (reference core.py:368-373).

    svd0: also return the SVD factors of the final cores[0] (the first step of the rounding's
    left-to-right pass); its carry and SVD run on a side stream while the explicit Q of core 1 is
    formed, since neither needs the other. fullrank_eps (eps / sqrt(d - 1) of the rounding, or None):
    the first step's threshold delta = fullrank_eps ||cores[0]|| is known here, so its factors may take
    the certified full-rank QR route (linalg._fullrank_inverse). lazy_q: cores orthogonalized by a
    one-pass CholeskyQR stay unformed (linalg.LazyQt in place of the core; the caller's left-to-right
    pass multiplies through the factors with _carry_into), since this sweep itself never reads Q."""
    cores = list(cores)

    def as_core(Qt, n, r1):
        if isinstance(Qt, L.LazyQt):
            Qt.shape = (Qt.shape[0], n, r1)
            return Qt
        return Qt.reshape(Qt.shape[0], n, r1)

    scale = None
    f0 = None
    for k in range(len(cores) - 1, 0, -1):
        r0, n, r1 = cores[k].shape
        a, m, _ = cores[k - 1].shape
        if svd0 and k == 1 and not renorm:
            prev = cores[0]

            def first_svd(Rt):
                c0 = L.gemm(prev.reshape(a * m, r0), Rt)
                dl = None if fullrank_eps is None else fullrank_eps * float(L.nrm2(c0).item())
                return c0, L.SVDFactors(c0, fullrank_delta=dl)

            got = L.cholqr2_colmajor(cores[k].reshape(r0, n * r1), n * r1, r0, lazy=lazy_q)
            if got is not None:
                Qt, Rt = got
                c0, f0 = first_svd(Rt)
            else:
                Qt, Rt, (c0, f0) = L.qr_colmajor(cores[k].reshape(r0, n * r1).clone(), n * r1, r0,
                                                 overlap_r=first_svd)
                f0.record_stream(torch.cuda.current_stream())
            kk = Qt.shape[0]
            cores[k] = as_core(Qt, n, r1)
            cores[0] = c0.reshape(a, m, kk)
            continue
        if L._FULLRANK_IDENTITY and r0 >= n * r1 >= L._IDENTITY_Q_MIN:
            # square or wide unfolding X^T (n r1 x r0): X^T = I X^T is an orthogonal-times-carry split like
            # Q R (the sweep only needs orthonormal rows in the core and the carry into the previous one,
            # not a triangular factor): the core becomes the identity, the carry is X itself, the bond
            # rank n r1 is what the Householder QR returns too. No factorization, no rounding.
            mk = n * r1
            Qt = torch.eye(mk, dtype=torch.float64, device=device())
            Rt = cores[k].reshape(r0, mk)
        else:
            got = L.cholqr2_colmajor(cores[k].reshape(r0, n * r1), n * r1, r0, lazy=lazy_q and not renorm)
            Qt, Rt = got if got is not None else L.qr_colmajor(cores[k].reshape(r0, n * r1).clone(), n * r1, r0)
        kk = Qt.shape[0]
        cores[k] = as_core(Qt, n, r1)
        cores[k - 1] = L.gemm(cores[k - 1].reshape(a * m, r0), Rt, emulate=True).reshape(a, m, kk)
        if renorm:
            s = L.nrm2(cores[k - 1])
            ok = s > 0
            div = torch.where(ok, s, torch.ones_like(s))
            cores[k - 1] = cores[k - 1] / div
            scale = div if scale is None else scale * div
    if svd0:
        return cores, scale, f0
    return cores, scale


def tt_norm(a):
    """Frobenius norm through an orthogonalization sweep (reference core.py:304-324)."""
    cores, _ = _fused(a)
    cores, scale = _rl_orthogonalize(cores, renorm=True)
    n0 = L.nrm2(cores[0])
    if scale is not None:
        n0 = n0 * scale
    return float(n0.item())


def _matvec_core_fused(Ra, n, m, Rb, rc, rd):
    """Whether a dense core contraction takes ttb_matvec_core_ozaki (large, tile-aligned, rd % 16 == 0)."""
    M, N = Ra * n * Rb, rc * rd
    return (L._OZAKI and M * N * m >= L._OZAKI_MIN_WORK and M % 128 == 0 and N % 64 == 0 and m % 64 == 0
            and rd % 16 == 0 and Rb <= 64 and rd <= 64 and 256 % Rb == 0 and 256 % rd == 0
            and M * m < 2 ** 31 * 64)


def tt_matvec(A, x):
    """Operator application, ranks multiply (reference core.py:327-338)."""
    if A.col_sizes != x.mode_sizes:
        raise TtShapeError(f"operator column sizes {A.col_sizes} != vector sizes {x.mode_sizes}")
    out = []
    for M, G in zip(A.cores, x.cores):
        if A.band is not None:
            Ra, n, B, Rb = M.shape
            rc, _, rd = G.shape
            Y = L.empty(Ra * rc, n, Rb * rd)
            call("ttb_band_matvec", Ra, Rb, n, A.band, rc, rd, ptr(M), ptr(G), ptr(Y))
        else:
            Ra, n, m, Rb = M.shape
            rc, _, rd = G.shape
            if _matvec_core_fused(Ra, n, m, Rb, rc, rd):
                # one Ozaki GEMM slicing M and G in their core layouts and writing Y in its own
                # (ttb_matvec_core_ozaki): no operand / output regrouping passes
                Y = L.empty(Ra * rc, n, Rb * rd)
                ws = torch.empty(int(call_raw("ttb_matvec_core_ozaki_workspace", Ra, n, m, Rb, rc, rd)),
                                 dtype=torch.uint8, device=device())
                prof = L._GEMM_PROFILE
                if prof is not None:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                call("ttb_matvec_core_ozaki", Ra, n, m, Rb, rc, rd, ptr(M.contiguous()), ptr(G.contiguous()), ptr(Y),
                     ptr(ws))
                if prof is not None:
                    e1.record()
                    prof.append((e0, e1, 2.0 * Ra * n * Rb * rc * rd * m, "ozaki", (Ra * n * Rb, rc * rd, m)))
            else:
                T = L.tdot(M, G, ([2], [1]), emulate=True)       # (a, i, b, c, d)
                Y = L.permute(T, (0, 3, 1, 2, 4)).reshape(Ra * rc, n, Rb * rd)
        out.append(Y)
    return TtTensor(out)


def _chop(s, delta, max_rank=None):
    """Reference _chop (core.py:341-350) on host singular values."""
    if s.size == 0:
        return 1
    tails = np.sqrt(np.cumsum(s[::-1] ** 2))[::-1]
    keep = max(1, int(np.searchsorted(tails <= delta, True)))
    if max_rank is not None:
        keep = min(keep, max_rank)
    return min(keep, s.size)


def _speculative_fullrank(cores, eps, carried=None):
    """The one-pass certified full-rank rounding of linalg.fullrank_speculative_3core for a 3-core TT
    (1, n0, r1), (r1, n1, r2), (r2, n2, 1) with n0 == r1 and a square or wide last unfolding (r2 >= n2).
    Returns None when the shapes do not apply (nothing computed); else (cores, factors): cores has the
    last core carried into the middle one and replaced by the identity, cores[0] replaced by the
    identity when factors is not None (success); factors None = not certified, the caller runs the
    ordinary sweeps on the returned cores (same tensor). ``carried``: the middle core with the last one
    already carried in (tt_matvec_round_host does it under the uploads); only valid when the shapes apply."""
    if len(cores) != 3:
        return None
    G0, G1, G2 = cores
    (a, n0, r1), (r1b, n1, r2), (r2b, n2, one) = G0.shape, G1.shape, G2.shape
    if not (a == 1 and one == 1 and r2 >= n2 and L.speculative_applies(n0, r1, n1, n2, 3)):
        return None
    eye2 = torch.eye(n2, dtype=torch.float64, device=device()).reshape(n2, n2, 1)
    if carried is not None:       # the host path already carried the last core in, slab by slab
        Y1p = carried.reshape(r1, n1, n2)
    else:
        Y1p = L.gemm(G1.reshape(r1 * n1, r2), G2.reshape(r2, n2), emulate=True).reshape(r1, n1, n2)
    got = L.fullrank_speculative_3core(G0.reshape(n0, r1), Y1p, eps, 3)
    if got is None:
        return [G0, Y1p, eye2], None
    f1, _ = got
    eye0 = torch.eye(r1, dtype=torch.float64, device=device()).reshape(1, n0, r1)
    return [eye0, Y1p, eye2], f1


def tt_round(t, eps, max_rank=None):
    """Right-to-left QR then left-to-right truncated SVD (reference core.py:353-389)."""
    if eps <= 0:
        raise ValueError("eps must be positive")
    cores, tag = _fused(t)
    d = len(cores)
    if d == 1:
        return _unfused([G.clone() for G in cores], tag)
    if max_rank is None:
        sp = _speculative_fullrank(cores, eps)
        if sp is not None:
            cores, f1 = sp
            if f1 is not None:      # both steps certified full rank: I, Z L^-T, L^T
                n = f1.n
                r1, n1 = cores[1].shape[0], cores[1].shape[1]
                return _unfused([cores[0], f1.U(n).reshape(r1, n1, n), f1.SVt(n).reshape(n, cores[2].shape[1], 1)], tag)
    fr_eps = eps / np.sqrt(d - 1) if max_rank is None else None
    # rank-capped rounding with a small cap (the AMEn residual's kick rank): only the leading singular
    # triplets are computed (linalg.topk_svd); the first step's SVD is then not started during the sweep
    topk = max_rank is not None and max_rank <= L._TOPK_MAX and L._TOPK
    got = _rl_orthogonalize(cores, svd0=not topk, fullrank_eps=fr_eps, lazy_q=True)
    cores, f0 = got[0], (got[2] if not topk else None)
    total = float(L.nrm2(cores[0]).item())
    if total == 0.0:
        return _unfused([L.zeros(1, G.shape[1], 1) for G in cores], tag)
    delta = eps * total / np.sqrt(d - 1)
    for k in range(d - 1):
        r0, n, r1 = cores[k].shape
        if topk:
            top = L.topk_svd(cores[k].reshape(r0 * n, r1), max_rank, delta)
            if top is not None:
                U, carry = top
                cores[k] = U.reshape(r0, n, U.shape[1])
                cores[k + 1] = _carry_into(carry, cores[k + 1])
                continue
        f = f0 if (k == 0 and f0 is not None) else L.SVDFactors(
            cores[k].reshape(r0 * n, r1), fullrank_delta=delta if max_rank is None else None)
        # certified full rank (s_min > delta): _chop would keep every singular value, U S Vt = Q R
        keep = f.n if f.fullrank else _chop(f.s_host(), delta, max_rank)
        cores[k] = f.U(keep).reshape(r0, n, keep)
        cores[k + 1] = _carry_into(f.SVt(keep), cores[k + 1])
    return _unfused(cores, tag)


def tt_from_full(X, eps=1e-14, max_rank=None):
    """Sequential TT-SVD of a dense array (reference core.py:392-410)."""
    X = to_device(X)
    d = X.dim()
    sizes = tuple(X.shape)
    total = float(L.nrm2(X).item())
    delta = eps * total / np.sqrt(max(d - 1, 1))
    cores = []
    Cm = X.reshape(1, -1)
    r = 1
    for k in range(d - 1):
        Cm = Cm.reshape(r * sizes[k], -1)
        f = L.SVDFactors(Cm)
        keep = _chop(f.s_host(), delta, max_rank) if total > 0 else 1
        cores.append(f.U(keep).reshape(r, sizes[k], keep))
        Cm = f.SVt(keep)
        r = keep
    cores.append(Cm.reshape(r, sizes[-1], 1))
    return TtTensor(cores)


def tt_matrix_from_full(X, eps=1e-14):
    """TT-SVD of a dense operator given as (n1, m1, n2, m2, ...) (reference core.py:413-429)."""
    X = to_device(X)
    if X.dim() % 2:
        raise TtShapeError("operator array needs paired row/col axes")
    d = X.dim() // 2
    rows = X.shape[0::2]
    cols = X.shape[1::2]
    fused = tt_from_full(X.reshape([rows[k] * cols[k] for k in range(d)]), eps)
    return TtMatrix([G.reshape(G.shape[0], rows[k], cols[k], G.shape[2]) for k, G in enumerate(fused.cores)])
