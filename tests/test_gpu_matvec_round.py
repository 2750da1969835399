"""The benchmarked workload against the oracle at benchmark scale (reference tensor_train/core.py:327-389).

The configs[4] microbenchmark is round(A x, 1e-8) for a 3-core TT-matrix with n x n modes,
operator ranks 16 and a TT-vector with ranks 64 (bench.py). Its large products run on the
Ozaki-scheme GEMM and its tall factorizations on CholeskyQR2 / Gram-Cholesky R / implicit U, routes
that only switch on for unfoldings with >= 2^19 rows (linalg.py). Two checks:

* n = 512, oracle run live on the host: the thresholds are lowered to 2^18 rows so every large-scale
  route runs (the test asserts that each did), and the rounded tensors are compared in full
  (||Y - Y_oracle|| / ||Y_oracle||, computed by the oracle on host copies) at 1e-12, ranks equal;
* n = 1024 (the benchmarked size, default thresholds), against the committed oracle fixture
  ``tests/golden/matvec_round_oracle.npz`` (tests/golden/make_matvec_round_fixture.py): ranks equal,
  the singular values of both unfoldings, 4096 sampled entries and the norm.

Achieved errors are printed (pytest -s) and recorded as test properties.
"""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "matvec_round_oracle.npz")


def _instance(n):
    from paper_2509_13224_b200.tensor_train import TtMatrix, TtTensor
    from paper_2509_13224_b200.workloads import matvec_round_instance_np
    A, X = matvec_round_instance_np(n, 16, 64, 3, 0)
    return A, X, TtMatrix([torch.as_tensor(G, device="cuda") for G in A]), \
        TtTensor([torch.as_tensor(G, device="cuda") for G in X])


def _route_spy(monkeypatch):
    """Record which large-scale routes returned a result (None = fell back to Householder)."""
    from paper_2509_13224_b200 import linalg as L
    used = {"cholqr2": 0, "gram": 0, "ozaki": 0, "fullrank": 0, "lazyq": 0}
    chol, gram, oz = L.cholqr2_colmajor, L._gram_jacobi, L.call

    def chol_spy(*a, **k):
        r = chol(*a, **k)
        used["cholqr2"] += r is not None
        used["lazyq"] += r is not None and isinstance(r[0], L.LazyQt)     # Q^T left unformed (one large GEMM less)
        return r

    def gram_spy(*a, **k):
        r = gram(*a, **k)
        used["gram"] += r is not None
        used["fullrank"] += r is not None and r[2] is None      # certified full rank: no SVD
        return r

    def call_spy(name, *a, **k):
        if name in ("ttb_dgemm_ozaki", "ttb_dgemm_ozaki_triuB"):
            used["ozaki"] += 1
        return oz(name, *a, **k)

    monkeypatch.setattr(L, "cholqr2_colmajor", chol_spy)
    monkeypatch.setattr(L, "_gram_jacobi", gram_spy)
    monkeypatch.setattr(L, "call", call_spy)
    return used


def _bond_singular_values(Y):
    """Singular values of both unfoldings of a 3-core device TT in the rounding's output gauge (first two
    cores left-orthonormal), computed with the library's own QR/SVD (the fixture holds the oracle's)."""
    from paper_2509_13224_b200 import linalg as L
    G0, G1, G2 = Y.cores
    r2, n2, _ = G2.shape
    M2 = G2.reshape(r2, n2)
    s2 = L.svd(M2)[1].cpu().numpy()
    Q, R = L.qr(M2.t().contiguous())                     # M2^T = Q R
    r1, n1, _ = G1.shape
    G1r = L.gemm(G1.reshape(r1 * n1, r2), R, tB=True)     # G1 x R^T
    k = G1r.shape[1]
    Q1, R1 = L.qr(G1r.reshape(r1, n1 * k).t().contiguous())
    G0r = L.gemm(G0.reshape(-1, r1), R1, tB=True)
    s1 = L.svd(G0r)[1].cpu().numpy()
    return s1, s2


_ORACLE_N512 = {}


@pytest.mark.parametrize("fullrank,lazy", [(True, True), (False, True), (True, False)],
                         ids=["certified-qr", "svd", "formed-q"])
def test_matvec_round_n512_all_routes_vs_oracle(monkeypatch, record_property, fullrank, lazy):
    """fullrank: the rounding's certified full-rank QR steps on (default) / off (every step a Jacobi SVD);
    lazy: the one-pass CholeskyQR's Q^T left unformed (default) / formed explicitly."""
    from oracle import tt as OT
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200.tensor_train import tt_matvec, tt_round
    n = 512
    monkeypatch.setattr(L, "_CHOLQR2_MIN_M", 1 << 18)
    monkeypatch.setattr(L, "_GRAM_MIN_M", 1 << 18)
    monkeypatch.setattr(L, "_FULLRANK", fullrank)
    monkeypatch.setattr(L, "_LAZY_Q", lazy)
    used = _route_spy(monkeypatch)
    A, X, Ad, Xd = _instance(n)
    Y = tt_round(tt_matvec(Ad, Xd), 1e-8)
    torch.cuda.synchronize()
    assert used["cholqr2"] >= 1 and used["gram"] >= 1 and used["ozaki"] >= 3, used
    assert (used["fullrank"] >= 1) == fullrank, used
    assert (used["lazyq"] >= 1) == lazy, used
    if "Y" not in _ORACLE_N512:
        _ORACLE_N512["Y"] = OT.round_tt(OT.matvec(OT.TTOp(A), OT.TT(X)), 1e-8)
    Yo = _ORACLE_N512["Y"]
    assert tuple(Y.ranks) == tuple(Yo.ranks), (Y.ranks, Yo.ranks)
    Yh = OT.TT([G.cpu().numpy() for G in Y.cores])
    err = OT.norm(OT.sub(Yh, Yo)) / OT.norm(Yo)
    print(f"matvec+round n=512 (all routes, fullrank={fullrank}): rel. error vs oracle {err:.3e}, ranks {Y.ranks}, routes {used}")
    record_property("rel_error", err)
    assert err <= 1e-12, err


@pytest.mark.parametrize("fullrank", [True, False], ids=["certified-qr", "svd"])
def test_matvec_round_n1024_vs_oracle_fixture(monkeypatch, record_property, fullrank):
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200.tensor_train import tt_matvec, tt_norm, tt_round
    monkeypatch.setattr(L, "_FULLRANK", fullrank)
    if not os.path.exists(GOLDEN):
        pytest.fail("tests/golden/matvec_round_oracle.npz missing (tests/golden/make_matvec_round_fixture.py)")
    g = np.load(GOLDEN)
    if "n1024_ranks" not in g:
        pytest.fail("fixture has no n=1024 entry")
    n = 1024
    A, X, Ad, Xd = _instance(n)
    sums = np.array([[float(G.sum()), float((G * G).sum())] for G in list(A) + list(X)])
    assert np.allclose(sums, g["n1024_in_sums"], rtol=1e-12, atol=1e-9), "input generator changed"
    del A, X
    Y = tt_round(tt_matvec(Ad, Xd), 1e-8)
    del Ad, Xd
    assert tuple(Y.ranks) == tuple(int(r) for r in g["n1024_ranks"]), (Y.ranks, g["n1024_ranks"])
    s1, s2 = _bond_singular_values(Y)
    es1 = float(np.abs(s1 - g["n1024_s1"]).max() / g["n1024_s1"].max())
    es2 = float(np.abs(s2 - g["n1024_s2"]).max() / g["n1024_s2"].max())
    vals = Y.gather(torch.as_tensor(g["n1024_idx"].astype(np.int64), device="cuda")).cpu().numpy()
    ev = float(np.abs(vals - g["n1024_vals"]).max() / np.sqrt(np.mean(g["n1024_vals"] ** 2)))
    en = abs(tt_norm(Y) - float(g["n1024_norm"])) / float(g["n1024_norm"])
    print(f"matvec+round n=1024 (fullrank={fullrank}) vs oracle fixture: singular values {es1:.2e} / {es2:.2e} (of s_max), "
          f"sampled entries {ev:.2e} (of rms), norm {en:.2e}")
    for k, v in (("s1", es1), ("s2", es2), ("entries", ev), ("norm", en)):
        record_property(k, v)
    assert es1 <= 1e-12 and es2 <= 1e-12, (es1, es2)
    assert ev <= 1e-11, ev
    assert en <= 1e-12, en
