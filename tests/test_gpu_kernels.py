"""Kernel-level parity: native FP64 kernels vs numpy on seeded inputs (GPU only)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def la():
    from paper_2509_13224_b200 import linalg
    return linalg


def T(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (64, 64, 64), (130, 70, 33), (300, 257, 129),
                                   (1000, 40, 5000), (513, 1024, 96), (40, 32, 70000)])
@pytest.mark.parametrize("tA,tB", [(False, False), (True, False), (False, True), (True, True)])
def test_gemm(la, M, N, K, tA, tB):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.standard_normal((K, M) if tA else (M, K))
    B = rng.standard_normal((N, K) if tB else (K, N))
    C0 = rng.standard_normal((M, N))
    ref = 0.5 * ((A.T if tA else A) @ (B.T if tB else B)) - 2.0 * C0
    out = T(C0)
    la.gemm(T(A), T(B), tA=tA, tB=tB, alpha=0.5, beta=-2.0, out=out)
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()) * np.sqrt(K)


@pytest.mark.parametrize("M,N,K", [(32, 8192, 128), (37, 9001, 16), (128, 20000, 128), (300, 16387, 100),
                                   (896, 40000, 128), (64, 8193, 7)])
@pytest.mark.parametrize("alpha", [-1.0, 1.0])
def test_gemm_short_k_update(la, M, N, K, alpha):
    # C += alpha A B with beta = 1 (the WY trailing-update shape; resident-A persistent kernel)
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K))
    B = rng.standard_normal((K, N))
    C0 = rng.standard_normal((M, N))
    ref = C0 + alpha * (A @ B)
    out = T(C0)
    la.gemm(T(A), T(B), alpha=alpha, beta=1.0, out=out)
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()) * np.sqrt(K)


def test_permute_and_tdot(la):
    rng = np.random.default_rng(1)
    X = rng.standard_normal((3, 4, 5, 6))
    for perm in [(0, 1, 2, 3), (3, 2, 1, 0), (1, 0, 3, 2), (2, 0, 3, 1)]:
        assert np.array_equal(la.permute(T(X), perm).cpu().numpy(), X.transpose(perm))
    Y = rng.standard_normal((6, 5, 7))
    got = la.tdot(T(X), T(Y), ([3, 2], [0, 1])).cpu().numpy()
    assert np.allclose(got, np.tensordot(X, Y, ([3, 2], [0, 1])), atol=1e-12)
    got = la.tdot(T(X), T(rng.standard_normal((3, 2))), ([0], [0])).cpu().numpy()
    assert got.shape == (4, 5, 6, 2)


@pytest.mark.parametrize("m,n", [(1, 1), (5, 3), (3, 5), (64, 64), (200, 37), (1000, 70), (40, 300), (5000, 33),
                                 (20000, 100), (1100, 16), (1500, 17), (200000, 40), (131073, 150), (70001, 300),
                                 (65536, 257)])
def test_qr(la, m, n):
    rng = np.random.default_rng(m + n)
    X = rng.standard_normal((m, n))
    Q, R = la.qr(T(X))
    Q, R = Q.cpu().numpy(), R.cpu().numpy()
    k = min(m, n)
    assert Q.shape == (m, k) and R.shape == (k, n)
    assert np.abs(Q @ R - X).max() <= 1e-12 * np.abs(X).max() * np.sqrt(n)
    assert np.abs(Q.T @ Q - np.eye(k)).max() <= 1e-13 * np.sqrt(m)
    assert np.allclose(np.triu(R), R)
    Rn = np.linalg.qr(X)[1]
    assert np.allclose(np.abs(np.diag(R)), np.abs(np.diag(Rn)), rtol=1e-10)


def test_qr_rank_deficient(la):
    rng = np.random.default_rng(5)
    B = rng.standard_normal((50, 3))
    X = np.hstack([B, B])  # rank 3
    Q, R = la.qr(T(X))
    assert np.abs(Q.cpu().numpy() @ R.cpu().numpy() - X).max() < 1e-12
    Z = np.zeros((20, 4))
    Q, R = la.qr(T(Z))
    assert np.all(R.cpu().numpy() == 0)
    # tall panels (TSQR path): repeated columns, zero columns, an all-zero matrix
    B = rng.standard_normal((60000, 7))
    X = np.hstack([B, B, np.zeros((60000, 3)), B[:, :2] * 1e-9, B])
    Q, R = la.qr(T(X))
    Q, R = Q.cpu().numpy(), R.cpu().numpy()
    assert np.abs(Q @ R - X).max() < 1e-12 * np.abs(X).max() * 10
    assert np.abs(Q.T @ Q - np.eye(X.shape[1])).max() < 1e-12
    Q, R = la.qr(T(np.zeros((30000, 20))))
    assert np.all(R.cpu().numpy() == 0)
    assert np.abs(Q.cpu().numpy().T @ Q.cpu().numpy() - np.eye(20)).max() < 1e-14


@pytest.mark.parametrize("m,n", [(1, 1), (6, 4), (4, 6), (64, 64), (100, 65), (65, 100), (2000, 120), (300, 300),
                                 (257, 257), (3000, 515), (1100, 1024)])
def test_svd(la, m, n):
    rng = np.random.default_rng(10 * m + n)
    X = rng.standard_normal((m, n)) * np.logspace(0, -8, n)[None, :]
    U, S, Vt = la.svd(T(X))
    U, S, Vt = U.cpu().numpy(), S.cpu().numpy(), Vt.cpu().numpy()
    Sn = np.linalg.svd(X, compute_uv=False)
    assert np.allclose(S, Sn, rtol=1e-12, atol=1e-14 * Sn[0])
    assert np.abs((U * S) @ Vt - X).max() <= 1e-13 * Sn[0] * np.sqrt(max(m, n))
    k = min(m, n)
    assert np.abs(U.T @ U - np.eye(k)).max() < 1e-12
    assert np.all(np.diff(S) <= 0)


@pytest.mark.parametrize("M,N,K,alpha,beta", [(50, 5000, 16, -0.7, 1.3), (7, 3001, 20, 2.0, 0.0), (100, 2048, 3, 1.0, -1.0),
                                               (33, 70001, 32, -1.0, 1.0)])
def test_gemm_lowrank_update(la, M, N, K, alpha, beta):
    rng = np.random.default_rng(M * N + K)
    A = rng.standard_normal((M, K))
    B = rng.standard_normal((K, N))
    C0 = rng.standard_normal((M, N))
    ref = beta * C0 + alpha * (A @ B)
    out = T(C0)
    la.gemm(T(A), T(B), alpha=alpha, beta=beta, out=out)
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()) * np.sqrt(K)


@pytest.mark.parametrize("N,bw", [(1, 0), (50, 3), (300, 23), (1792, 55), (3000, 127), (5000, 20), (400, 140)])
def test_band_cholesky_solve(N, bw):
    # banded SPD solve behind AMEn's direct local solves (blocked shared-memory window for bw <= 127)
    from paper_2509_13224_b200._lib import call, ptr
    rng = np.random.default_rng(N + bw)
    A = np.zeros((N, N))
    for q in range(bw + 1):
        v = rng.standard_normal(N - q) * 0.5
        A[np.arange(q, N), np.arange(N - q)] = v
        A[np.arange(N - q), np.arange(q, N)] = v
    A += np.eye(N) * (2.0 * bw + 2.0)
    W = bw + 1
    LB = np.zeros((N, W))
    for q in range(W):
        LB[q:, q] = A[np.arange(q, N), np.arange(N - q)]
    b = rng.standard_normal(N)
    LBd, bd = T(LB), T(b)
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    call("ttb_band_chol_solve", N, bw, ptr(LBd), ptr(bd), ptr(info))
    assert int(info.item()) == 0
    x = np.linalg.solve(A, b)
    assert np.abs(bd.cpu().numpy() - x).max() <= 1e-12 * max(1.0, np.abs(x).max())
    L = np.linalg.cholesky(A)
    Lgot = LBd.cpu().numpy()
    for q in range(W):
        assert np.allclose(Lgot[q:, q], L[np.arange(q, N), np.arange(N - q)], rtol=1e-11, atol=1e-13)
    # indefinite: reported, not silently solved
    A2 = LB.copy()
    A2[N // 2, 0] = -1.0
    LBd2, bd2 = T(A2), T(b)
    call("ttb_band_chol_solve", N, bw, ptr(LBd2), ptr(bd2), ptr(info))
    assert int(info.item()) > 0


def test_svd_graded_and_degenerate(la):
    # graded singular values down to 1e-14 (relative accuracy of the one-sided Jacobi on R),
    # repeated singular values and exact rank deficiency, on the multi-CTA Jacobi sizes
    rng = np.random.default_rng(77)
    for n, spec in ((384, np.logspace(0, -14, 384)), (520, np.repeat([1.0, 1e-3, 1e-7, 0.0], 130))):
        Q1, _ = np.linalg.qr(rng.standard_normal((2 * n, n)))
        Q2, _ = np.linalg.qr(rng.standard_normal((n, n)))
        X = (Q1 * spec) @ Q2.T
        U, S, Vt = la.svd(T(X))
        U, S, Vt = U.cpu().numpy(), S.cpu().numpy(), Vt.cpu().numpy()
        Sn = np.linalg.svd(X, compute_uv=False)
        assert np.abs(S - Sn).max() <= 1e-12 * Sn[0]
        assert np.abs((U * S) @ Vt - X).max() <= 1e-13 * Sn[0] * np.sqrt(n)
        keep = S > 1e-12 * S[0]
        assert np.abs(U[:, keep].T @ U[:, keep] - np.eye(keep.sum())).max() < 1e-12


def test_lu_and_cholesky(la):
    rng = np.random.default_rng(3)
    for n in (1, 5, 64, 300, 1000):
        A = rng.standard_normal((n, n)) + n * np.eye(n) * 0.1
        B = rng.standard_normal((n, 7))
        X = la.solve(T(A), T(B)).cpu().numpy()
        assert np.abs(A @ X - B).max() <= 1e-10 * np.abs(B).max() * n
        S = A @ A.T + n * np.eye(n)
        b = rng.standard_normal(n)
        x = la.cho_solve_or_lu(T(S), T(b)).cpu().numpy()
        assert np.allclose(x, np.linalg.solve(S, b), rtol=1e-10, atol=1e-12)
    S = np.diag([1.0, -2.0, 3.0])
    x = la.cho_solve_or_lu(T(S), T(np.ones(3))).cpu().numpy()
    assert np.allclose(x, [1.0, -0.5, 1.0 / 3.0])


def test_maxvol(la, golden):
    g = golden("tensor_train.npz")
    assert np.array_equal(la.maxvol(T(g["maxvol_M"])), g["maxvol_sel"])
    v = np.array([10.0, 0.0])
    Md = np.vstack([v, v, [0.0, 10.0], [0.1, 0.2], [0.3, 0.1]])
    assert np.array_equal(la.maxvol(T(Md)), g["maxvol_dup_sel"])
    rng = np.random.default_rng(20)
    from oracle.cross import maxvol as omv
    for n, r in [(50, 5), (2000, 20), (30000, 40)]:
        M = rng.standard_normal((n, r))
        assert np.array_equal(la.maxvol(T(M)), omv(M))
    M = np.zeros((10, 3))
    M[:, 0] = np.arange(10)
    M[:, 1] = 2 * np.arange(10)
    M[:, 2] = np.arange(10) + 1
    with pytest.raises(la.MaxvolError):
        la.maxvol(T(M))


@pytest.mark.parametrize("want_v", [False, True])
def test_svd_implicit_u_path(monkeypatch, want_v):
    """Very tall SVD without explicit Q (U = X V S^-1) == the explicit-Q path; ill-conditioned
    kept columns fall back to explicit Q."""
    from paper_2509_13224_b200 import linalg as L
    g = torch.Generator(device="cuda").manual_seed(5)
    m, n = 4096, 96
    X = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
    X[:, -8:] *= 1e-12                                 # tail below the 1e-7 guard
    monkeypatch.setattr(L, "_IMPLICIT_U_MIN_M", 0)
    f = L.SVDFactors(X, want_v=want_v)
    assert f.implicit
    monkeypatch.setattr(L, "_IMPLICIT_U", False)
    ref = L.SVDFactors(X, want_v=want_v)
    assert not ref.implicit
    assert torch.allclose(f.S, ref.S, rtol=1e-12, atol=1e-20 * float(ref.S[0]))
    r = 80                                              # all kept columns above the guard
    U, Ur = f.U(r), ref.U(r)
    assert f.implicit
    eye = torch.eye(r, dtype=torch.float64, device="cuda")
    assert float((U.t() @ U - eye).abs().max()) < 1e-12
    P, Pr = U @ U.t(), Ur @ Ur.t()                     # same subspace (signs may differ)
    assert float((P - Pr).abs().max()) < 1e-11
    assert float((U @ f.SVt(r) - Ur @ ref.SVt(r)).norm() / (Ur @ ref.SVt(r)).norm()) < 1e-12
    if want_v:
        assert float((f.Vt(r).t() @ torch.diag(f.S[:r]) - X.t() @ U).norm() / X.norm()) < 1e-12
    rows = torch.empty(100, r, dtype=torch.float64, device="cuda")
    f.U_rows(r, 50, 150, rows)
    assert torch.allclose(rows, U[50:150], rtol=0, atol=1e-14)
    # keeping the 1e-12 tail violates the guard -> explicit-Q fallback, orthonormal to roundoff
    Uf = f.U(n)
    assert not f.implicit
    assert float((Uf.t() @ Uf - torch.eye(n, dtype=torch.float64, device="cuda")).abs().max()) < 1e-12


@pytest.mark.parametrize("mode", ["near_dependent", "duplicate", "graded"])
def test_qr_tall_blocks_ill_conditioned(la, mode):
    """Tall QR whose 128-column blocks defeat CholeskyQR2 (fallback to the TSQR panels) or stress it."""
    rng = np.random.default_rng(11)
    m, n = 70001, 300
    X = rng.standard_normal((m, n))
    if mode == "near_dependent":
        X[:, 150:160] = X[:, 10:20] + 1e-11 * rng.standard_normal((m, 10))
    elif mode == "duplicate":
        X[:, 200:210] = X[:, 130:140]
    else:
        X *= np.logspace(0, -9, n)[None, :]
    Q, R = la.qr(T(X))
    Q, R = Q.cpu().numpy(), R.cpu().numpy()
    assert np.abs(Q @ R - X).max() <= 1e-12 * np.abs(X).max() * np.sqrt(n)
    assert np.abs(Q.T @ Q - np.eye(n)).max() <= 1e-13 * np.sqrt(m)
    assert np.allclose(np.triu(R), R)


@pytest.mark.parametrize("M,N,K", [(128, 128, 128), (256, 384, 512), (1024, 512, 2048)])
def test_i8gemm_tcgen05_exact(M, N, K):
    """tcgen05 kind::i8 GEMM (TMEM accumulators, 128B-swizzled smem operands): exact int32 result."""
    from paper_2509_13224_b200._lib import call, ptr
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randint(-127, 128, (M, K), generator=g, device="cuda", dtype=torch.int8)
    B = torch.randint(-127, 128, (N, K), generator=g, device="cuda", dtype=torch.int8)
    C = torch.empty(M, N, dtype=torch.int32, device="cuda")
    call("ttb_i8gemm", M, N, K, ptr(A), ptr(B), ptr(C))
    ref = A.double() @ B.double().t()
    assert torch.equal(C.double(), ref)


@pytest.mark.parametrize("tB,graded", [(0, False), (1, False), (0, True)])
def test_dgemm_ozaki_fp64_accuracy(tB, graded):
    """Ozaki-scheme FP64 GEMM on the INT8 tensor cores: normwise agreement with the DMMA DGEMM."""
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200._lib import call, call_raw, ptr
    g = torch.Generator(device="cuda").manual_seed(3 + tB)
    M, N, K = 2048, 512, 1024
    A = torch.randn(M, K, generator=g, device="cuda", dtype=torch.float64)
    B = torch.randn((N, K) if tB else (K, N), generator=g, device="cuda", dtype=torch.float64)
    if graded:
        A *= torch.logspace(0, -8, K, device="cuda", dtype=torch.float64)[None, :]
        A *= torch.logspace(0, 6, M, device="cuda", dtype=torch.float64)[:, None]
    C = torch.empty(M, N, device="cuda", dtype=torch.float64)
    ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, K)), dtype=torch.uint8, device="cuda")
    call("ttb_dgemm_ozaki", tB, M, N, K, ptr(A), K, ptr(B), K if tB else N, ptr(C), N, ptr(ws))
    Cd = L.gemm(A, B, tB=bool(tB))
    scale = A.abs() @ (B.abs().t() if tB else B.abs())
    e_elem = float(((C - Cd).abs() / scale).max())
    e_norm = float((C - Cd).norm() / Cd.norm())
    print(f"ozaki tB={tB} graded={graded}: elementwise {e_elem:.2e} normwise {e_norm:.2e}")
    # measured: ~1.1e-15 Gaussian, 2.9-3.8e-15 graded; bounds ~10x the measured error
    assert e_elem < (3e-14 if graded else 1e-14), e_elem
    assert e_norm < (3e-14 if graded else 1e-14), e_norm
    # operands reproduce exactly through the slices (I x B, incl. tiny negatives next to large entries)
    I = torch.eye(K, dtype=torch.float64, device="cuda")
    Bk = (B.t().contiguous() if tB else B).clone()
    Bk[0, :8] = -2.0 ** -60
    C2 = torch.empty(K, N, device="cuda", dtype=torch.float64)
    ws2 = torch.empty(int(call_raw("ttb_ozaki_workspace", K, N, K)), dtype=torch.uint8, device="cuda")
    call("ttb_dgemm_ozaki", 0, K, N, K, ptr(I), K, ptr(Bk), N, ptr(C2), N, ptr(ws2))
    assert float(((C2 - Bk).abs() / Bk.abs().max(0).values).max()) < 2 ** -54


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K,tB,alpha,beta", [
    (1024, 128, 65536, 1, 1.0, 0.0),    # split-K over 144 CTAs, K ranges > 4096 (int64 level sums)
    (256, 128, 16384, 0, 1.0, 0.0),     # split-K, ranges <= 4096, column-sliced B
    (256, 8192, 128, 0, -1.0, 1.0),     # WY trailing update: C -= W2 V (beta epilogue)
    (384, 4096, 256, 1, 0.5, -2.0),     # general alpha / beta
    (1000, 510, 11011, 0, 1.0, 0.0),    # padded shape (rows, columns, K), split-K partials over the padded tile grid
    (260, 130, 777, 1, 0.5, -2.0),      # padded, row-sliced B, masked beta epilogue
    (4000, 68, 8296, 1, 1.0, 0.0),      # padded narrow N (the AMEn right-stage shape), long K
    (1000, 510, 4099, 0, -1.0, 1.0),    # padded, K ranges > 4096
    (256, 16384, 512, 0, 1.0, 0.0),     # small A, B stack > 32 MB: row-block-fastest unit order
    (384, 20480, 320, 1, 0.5, -2.0),    # the same order with a row-sliced B and the beta epilogue
    (300, 16390, 500, 0, 1.0, 0.0),     # the same order on a padded shape
])
def test_dgemm_ozaki_ex_splitk_beta(M, N, K, tB, alpha, beta):
    """ttb_dgemm_ozaki_ex (split-K, beta) against the DMMA DGEMM: normwise and per element relative to
    |alpha| |A| |B| + |beta C|."""
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200._lib import call, call_raw, ptr
    g = torch.Generator(device="cuda").manual_seed(M + K)
    A = torch.randn(M, K, generator=g, device="cuda", dtype=torch.float64)
    B = torch.randn((N, K) if tB else (K, N), generator=g, device="cuda", dtype=torch.float64)
    C0 = torch.randn(M, N, generator=g, device="cuda", dtype=torch.float64)
    C = C0.clone()
    ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, K)), dtype=torch.uint8, device="cuda")
    call("ttb_dgemm_ozaki_ex", tB, M, N, K, alpha, ptr(A), K, ptr(B), K if tB else N, beta, ptr(C), N, ptr(ws))
    Cd = C0.clone()
    L.gemm(A, B, tB=bool(tB), alpha=alpha, beta=beta, out=Cd)
    scale = abs(alpha) * (A.abs() @ (B.abs().t() if tB else B.abs())) + abs(beta) * C0.abs()
    assert float(((C - Cd).abs() / scale).max()) < 1e-14
    assert float((C - Cd).norm() / Cd.norm()) < 1e-14


@pytest.mark.gpu
def test_ozaki_gram_matches_dgemm():
    """ttb_ozaki_gram (X^T X, symmetric tiles + mirror, split-K) against X^T X on DMMA."""
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200._lib import call, call_raw, ptr
    g = torch.Generator(device="cuda").manual_seed(11)
    for m, n in ((65536, 256), (8192, 640)):
        X = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
        X *= torch.logspace(0, -3, n, device="cuda", dtype=torch.float64)[None, :]
        G = torch.empty(n, n, device="cuda", dtype=torch.float64)
        ws = torch.empty(int(call_raw("ttb_ozaki_gram_workspace", m, n)), dtype=torch.uint8, device="cuda")
        call("ttb_ozaki_gram", m, n, ptr(X), n, ptr(G), n, ptr(ws))
        Gd = L.gemm(X, X, tA=True)
        scale = X.abs().t() @ X.abs()
        assert float(((G - Gd).abs() / scale).max()) < 1e-14
        assert torch.equal(G, G.t())


@pytest.mark.gpu
@pytest.mark.parametrize("graded", [False, True])
def test_svd_gram_path(monkeypatch, graded):
    """Very tall SVDs through the Gram + Cholesky route (well conditioned) and its fallback to the
    Householder QR route (ill conditioned): singular values and U S V^T against torch (cuSOLVER) FP64."""
    from paper_2509_13224_b200 import linalg as L
    monkeypatch.setattr(L, "_GRAM_MIN_M", 65536)
    calls = []
    orig = L._gram_jacobi
    monkeypatch.setattr(L, "_gram_jacobi", lambda *a: calls.append(r := orig(*a)) or r)
    g = torch.Generator(device="cuda").manual_seed(5)
    m, n = 65536, 256
    X = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
    if graded:
        X *= torch.logspace(0, -9, n, device="cuda", dtype=torch.float64)[None, :]
    f = L.SVDFactors(X)
    assert f.implicit and len(calls) == 1 and ((calls[0] is None) == graded)
    S_ref = torch.linalg.svdvals(X)
    S = f.S.sort(descending=True).values
    assert float(((S - S_ref).abs() / S_ref[0]).max()) < 1e-13
    r = n
    Y = L.gemm(f.U(r), f.SVt(r))
    assert float((Y - X).norm() / X.norm()) < 1e-13


@pytest.mark.gpu
def test_dgemm_ozaki_trilA():
    """Lower-triangular A: the k steps above each row block's diagonal are skipped, result == full product."""
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200._lib import call, call_raw, ptr
    g = torch.Generator(device="cuda").manual_seed(4)
    M, N = 384, 4096
    A = torch.tril(torch.randn(M, M, generator=g, device="cuda", dtype=torch.float64))
    B = torch.randn(M, N, generator=g, device="cuda", dtype=torch.float64)
    C = torch.empty(M, N, device="cuda", dtype=torch.float64)
    ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, M)), dtype=torch.uint8, device="cuda")
    call("ttb_dgemm_ozaki_trilA", M, N, ptr(A), M, ptr(B), N, ptr(C), N, ptr(ws))
    Cd = L.gemm(A, B)
    # the Ozaki error model: operands are rounded relative to their row / column maxima (the same
    # 54-bit slicing as the dense product), so the bound scales with K max_k|a_ik| max_k|b_kj|
    scale = M * A.abs().max(1).values[:, None] * B.abs().max(0).values[None, :]
    assert float(((C - Cd).abs() / scale).max()) < 2 ** -52
    assert float((C - Cd).norm() / Cd.norm()) < 1e-14


@pytest.mark.gpu
def test_dgemm_ozaki_triuB():
    """Upper-triangular B: the k steps below each column block's diagonal are skipped, result == full product."""
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200._lib import call, call_raw, ptr
    g = torch.Generator(device="cuda").manual_seed(6)
    M, N = 4096, 384
    A = torch.randn(M, N, generator=g, device="cuda", dtype=torch.float64)
    B = torch.triu(torch.randn(N, N, generator=g, device="cuda", dtype=torch.float64))
    C = torch.empty(M, N, device="cuda", dtype=torch.float64)
    ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, N)), dtype=torch.uint8, device="cuda")
    call("ttb_dgemm_ozaki_triuB", M, N, ptr(A), N, ptr(B), N, ptr(C), N, ptr(ws))
    Cd = L.gemm(A, B)
    scale = N * A.abs().max(1).values[:, None] * B.abs().max(0).values[None, :]
    assert float(((C - Cd).abs() / scale).max()) < 2 ** -52
    assert float((C - Cd).norm() / Cd.norm()) < 1e-14
    # a nonzero strict lower triangle must not be read beyond the diagonal blocks' 64-row granularity:
    # entries below the block diagonal are skipped (documented precondition: they are zero)
    assert L.gemm_triu(A, B).shape == (M, N)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", ["square", "tall"])
def test_svd_fullrank_certificate(monkeypatch, shape):
    """The rounding's certified full-rank route (linalg._fullrank_inverse): a factor whose smallest
    singular value is provably above delta yields Q, R with Q R = X and Q^T Q = I and no SVD; a factor
    with singular values below delta (or a delta too close to s_min) takes the SVD route."""
    from paper_2509_13224_b200 import linalg as L
    monkeypatch.setattr(L, "_GRAM_MIN_M", 65536)
    g = torch.Generator(device="cuda").manual_seed(9)
    m, n = (512, 512) if shape == "square" else (65536 * 2, 256)
    X = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
    s = torch.linalg.svdvals(X)
    eye = torch.eye(n, device="cuda", dtype=torch.float64)
    # certified: delta far below s_min
    f = L.SVDFactors(X, fullrank_delta=1e-8 * float(X.norm()))
    assert f.fullrank and f.S is None
    U, R = f.U(n), f.SVt(n)
    assert float((L.gemm(U, R) - X).norm() / X.norm()) < 1e-14
    assert float((L.gemm(U, U, tA=True) - eye).abs().max()) < 1e-12
    if shape == "tall":
        assert float(torch.tril(R, -1).abs().max()) == 0.0
    else:
        # square: the factorization-free split U = I, carry = X (certificate from the Cholesky factor of X^T X)
        assert torch.equal(U, eye) and torch.equal(R, X)
        monkeypatch.setattr(L, "_FULLRANK_IDENTITY", False)      # the Householder Q R form of the same step
        fh = L.SVDFactors(X, fullrank_delta=1e-8 * float(X.norm()))
        assert fh.fullrank and fh.S is None
        Uh, Rh = fh.U(n), fh.SVt(n)
        assert float((L.gemm(Uh, Rh) - X).norm() / X.norm()) < 1e-14
        assert float((L.gemm(Uh, Uh, tA=True) - eye).abs().max()) < 1e-12
        assert float(torch.tril(Rh, -1).abs().max()) == 0.0
        monkeypatch.setattr(L, "_FULLRANK_IDENTITY", True)
    Uc = L.empty(m, n)
    for i0 in range(0, m, m // 4):
        f.U_rows(n, i0, i0 + m // 4, Uc[i0:i0 + m // 4])
    assert float((Uc - U).abs().max()) < 1e-13     # chunks below the Ozaki size run on DMMA
    with pytest.raises(ValueError):
        f.U(n - 1)
    with pytest.raises(ValueError):
        f.s_host()
    # the certificate is one-sided: a delta above s_min / margin is never certified
    f = L.SVDFactors(X, fullrank_delta=0.6 * float(s[-1]))
    assert not f.fullrank and f.S is not None
    # rank deficient: the last quarter of the columns repeats the first (s_min ~ 1e-16 s_max)
    Xd = X.clone()
    Xd[:, -n // 4:] = Xd[:, :n // 4]
    f = L.SVDFactors(Xd, fullrank_delta=1e-8 * float(Xd.norm()))
    assert not f.fullrank
    S = f.S.sort(descending=True).values
    S_ref = torch.linalg.svdvals(Xd)
    assert float(((S - S_ref).abs() / S_ref[0]).max()) < 5e-13
    # disabled by the switch
    monkeypatch.setattr(L, "_FULLRANK", False)
    assert not L.SVDFactors(X, fullrank_delta=1e-8 * float(X.norm())).fullrank


@pytest.mark.gpu
def test_trtri_lower():
    from paper_2509_13224_b200._lib import call, ptr
    g = torch.Generator(device="cuda").manual_seed(2)
    n = 384
    Lr = torch.tril(torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64)) / n ** 0.5
    Lr += 2.0 * torch.eye(n, device="cuda", dtype=torch.float64)
    Lr_full = Lr + torch.triu(torch.full((n, n), 7.0, device="cuda", dtype=torch.float64), 1)  # ignored
    Li = torch.empty(n, n, device="cuda", dtype=torch.float64)
    ws = torch.empty(n * n, device="cuda", dtype=torch.float64)
    call("ttb_trtri_lower", n, ptr(Lr_full), n, ptr(Li), n, ptr(ws))
    eye = torch.eye(n, device="cuda", dtype=torch.float64)
    assert float((Li @ Lr - eye).abs().max()) < 1e-13
    assert float(torch.triu(Li, 1).abs().max()) == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["gaussian", "gaussian2", "graded", "illcond"])
def test_cholqr2_colmajor(monkeypatch, kind):
    """CholeskyQR2 with Ozaki Grams: Q orthonormal to 1e-14 and Q R = X whenever it returns a result.
    Column scaling alone (graded) does not hurt it (Cholesky and the Ozaki Gram are both invariant to
    it); a matrix whose column-scaled condition number is 1e12 (illcond) is refused."""
    from paper_2509_13224_b200 import linalg as L
    monkeypatch.setattr(L, "_CHOLQR2_MIN_M", 65536)
    if kind == "gaussian2":   # force the second pass on a well-conditioned matrix too
        monkeypatch.setattr(L, "_CHOLQR1_KAPPA", 0.0)
    g = torch.Generator(device="cuda").manual_seed(9)
    n, m = 256, 65536
    Acm = torch.randn(n, m, generator=g, device="cuda", dtype=torch.float64)
    if kind == "graded":
        Acm *= torch.logspace(0, -10, n, device="cuda", dtype=torch.float64)[:, None]
    if kind == "illcond":
        V, _ = torch.linalg.qr(torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64))
        W = torch.linalg.qr(Acm.t())[0]                   # m x n, orthonormal columns
        Acm = ((V * torch.logspace(0, -12, n, device="cuda", dtype=torch.float64)[None, :]) @ W.t()).contiguous()
    got = L.cholqr2_colmajor(Acm, m, n)
    if kind == "illcond":
        assert got is None
        return
    Qt, Rt = got
    eye = torch.eye(n, device="cuda", dtype=torch.float64)
    assert float((Qt @ Qt.t() - eye).abs().max()) < 1e-14
    R = Rt.t()
    assert float(torch.tril(R, -1).abs().max()) < 1e-12 * float(R.abs().max())
    assert float((R.t() @ Qt - Acm).norm() / Acm.norm()) < 1e-14


def test_round_with_emulated_gemms_matches_dmma(monkeypatch):
    """tt_round(tt_matvec) with the large products on the Ozaki path == the all-DMMA result."""
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200.tensor_train import tt_matvec, tt_norm, tt_round, tt_sub
    from paper_2509_13224_b200.workloads import matvec_round_instance
    A, X = matvec_round_instance(512, 16, 64, 3, seed=1)
    launched = []
    orig = L.call

    def spy(name, *a):
        launched.append(name)
        return orig(name, *a)

    monkeypatch.setattr(L, "call", spy)
    Y1 = tt_round(tt_matvec(A, X), 1e-8)
    assert "ttb_dgemm_ozaki" in launched
    monkeypatch.setattr(L, "_OZAKI", False)
    Y2 = tt_round(tt_matvec(A, X), 1e-8)
    assert Y1.ranks == Y2.ranks
    assert tt_norm(tt_sub(Y1, Y2)) <= 1e-12 * tt_norm(Y2)


@pytest.mark.gpu
@pytest.mark.parametrize("tB", [0, 1])
def test_dgemm_ozaki_nonfinite_propagates(tB):
    """A NaN or Inf operand entry makes its whole output row / column NaN (as a DGEMM would make it
    non-finite) instead of being saturated into finite slices; the other outputs are unaffected."""
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200._lib import call, call_raw, ptr
    g = torch.Generator(device="cuda").manual_seed(11)
    M, N, K = 512, 256, 1024
    A = torch.randn(M, K, generator=g, device="cuda", dtype=torch.float64)
    B = torch.randn((N, K) if tB else (K, N), generator=g, device="cuda", dtype=torch.float64)
    A[3, 5] = float("nan")
    A[9, 0] = float("inf")
    if tB:
        B[7, 2] = float("-inf")
    else:
        B[2, 7] = float("-inf")
    C = torch.empty(M, N, device="cuda", dtype=torch.float64)
    ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, K)), dtype=torch.uint8, device="cuda")
    call("ttb_dgemm_ozaki", tB, M, N, K, ptr(A), K, ptr(B), K if tB else N, ptr(C), N, ptr(ws))
    bad_r = torch.zeros(M, dtype=torch.bool, device="cuda")
    bad_r[[3, 9]] = True
    bad_c = torch.zeros(N, dtype=torch.bool, device="cuda")
    bad_c[7] = True
    nan = torch.isnan(C)
    assert bool(nan[bad_r].all()) and bool(nan[:, bad_c].all())
    ok = ~(bad_r[:, None] | bad_c[None, :])
    assert not bool(nan[ok].any())
    Af, Bf = A.clone(), B.clone()
    Af[~torch.isfinite(Af)] = 0.0
    Bf[~torch.isfinite(Bf)] = 0.0
    Cd = L.gemm(Af, Bf, tB=bool(tB))
    assert float(((C - Cd).abs()[ok]).max() / Cd.abs().max()) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("Ra,n,m,Rb,rc,rd", [(16, 256, 256, 16, 16, 64), (1, 512, 128, 16, 4, 64), (4, 128, 192, 8, 2, 32)])
def test_matvec_core_ozaki_layouts(Ra, n, m, Rb, rc, rd):
    """ttb_matvec_core_ozaki (operands sliced in their TT-core layouts, Y scattered in its core layout) against the
    DMMA tensordot + permute of tt_matvec: normwise <= 1e-14."""
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200._lib import call, call_raw, ptr
    g = torch.Generator(device="cuda").manual_seed(Ra + n + rd)
    M = torch.randn(Ra, n, m, Rb, generator=g, dtype=torch.float64, device="cuda")
    G = torch.randn(rc, m, rd, generator=g, dtype=torch.float64, device="cuda")
    T = L.tdot(M, G, ([2], [1]))                               # DMMA
    ref = L.permute(T, (0, 3, 1, 2, 4)).reshape(Ra * rc, n, Rb * rd)
    Y = torch.full((Ra * rc, n, Rb * rd), float("nan"), dtype=torch.float64, device="cuda")
    ws = torch.empty(int(call_raw("ttb_matvec_core_ozaki_workspace", Ra, n, m, Rb, rc, rd)), dtype=torch.uint8,
                     device="cuda")
    call("ttb_matvec_core_ozaki", Ra, n, m, Rb, rc, rd, ptr(M), ptr(G), ptr(Y), ptr(ws))
    assert torch.isfinite(Y).all()
    assert float((Y - ref).norm() / ref.norm()) <= 1e-14


def test_cross_index_kernels_match_numpy():
    """ttb_fiber_index / ttb_nested_index against the reference's list-of-tuples bookkeeping
    (tensor_train/cross.py:88-100, 150-152, 178-180) restated in numpy."""
    from paper_2509_13224_b200.tensor_train import cross as C
    rng = np.random.default_rng(5)
    d = 4
    for k, nl, nk, nr in [(0, 1, 7, 5), (1, 3, 6, 4), (2, 5, 9, 1), (3, 4, 8, 1)]:
        w = d - k - 1
        left = rng.integers(0, 50, size=(nl, k)).astype(np.int64)
        right = rng.integers(0, 50, size=(nr, w)).astype(np.int64)
        got = C._fiber_index(left, nk, right, k, d).cpu().numpy()
        want = np.array([tuple(left[l]) + (i,) + tuple(right[r]) for l in range(nl) for i in range(nk)
                         for r in range(nr)], dtype=np.int64).reshape(nl * nk * nr, d)
        assert np.array_equal(got, want)
        # nested sets from maxvol rows
        sel = np.sort(rng.choice(nl * nk, size=min(3, nl * nk), replace=False)).astype(np.int32)
        got = C._nested(torch.as_tensor(sel, device="cuda"), nk, torch.as_tensor(left, device="cuda"), 0).cpu().numpy()
        want = np.array([tuple(left[s // nk]) + (s % nk,) for s in sel], dtype=np.int64).reshape(len(sel), k + 1)
        assert np.array_equal(got, want)
        sel = np.sort(rng.choice(nk * nr, size=min(3, nk * nr), replace=False)).astype(np.int32)
        got = C._nested(torch.as_tensor(sel, device="cuda"), nr, torch.as_tensor(right, device="cuda"), 1).cpu().numpy()
        want = np.array([(s // nr,) + tuple(right[s % nr]) for s in sel], dtype=np.int64).reshape(len(sel), w + 1)
        assert np.array_equal(got, want)


def test_cross_deferred_status_raises(la):
    """The device-resident maxvol / solve status words raise at the next synchronization what the calls
    themselves raise when they are read at once (MaxvolError, LinAlgError), first failure first."""
    from paper_2509_13224_b200.tensor_train.cross import _Deferred
    M = np.zeros((10, 3))
    M[:, 0] = np.arange(10)
    M[:, 1] = 2 * np.arange(10)
    M[:, 2] = np.arange(10) + 1
    pend = _Deferred()
    rows = la.maxvol_colmajor_dev(T(M.T.copy()), 10, 3, pend)
    assert np.array_equal(rows.cpu().numpy(), np.arange(3))          # untouched on failure: valid indices
    with pytest.raises(la.MaxvolError):
        pend.check(torch.zeros(1, dtype=torch.float64, device="cuda"))
    pend = _Deferred()
    good = np.random.default_rng(0).standard_normal((40, 4))
    rows = la.maxvol_colmajor_dev(T(good.T.copy()), 40, 4, pend)
    assert np.array_equal(rows.cpu().numpy(), la.maxvol(T(good)))
    la.solve(T(np.zeros((3, 3))), T(np.ones((3, 2))), status=pend)
    with pytest.raises(np.linalg.LinAlgError):
        pend.check(torch.zeros(1, dtype=torch.float64, device="cuda"))
    pend = _Deferred()
    la.maxvol_colmajor_dev(T(good.T.copy()), 40, 4, pend)
    assert pend.check(torch.full((1,), 2.5, dtype=torch.float64, device="cuda")) == 2.5 and not pend.items


def test_ozaki_kernel_events_record_launches():
    """ttb_ozaki_kernel_events: one record per oz_gemm_kernel launch with its shape and kind, none when off."""
    from paper_2509_13224_b200._lib import call, call_raw, lib, ptr
    L_ = lib()
    M, N, K = 256, 128, 512
    A = torch.randn(M, K, device="cuda", dtype=torch.float64)
    B = torch.randn(K, N, device="cuda", dtype=torch.float64)
    Cm = torch.empty(M, N, device="cuda", dtype=torch.float64)
    ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, K)), dtype=torch.uint8, device="cuda")
    L_.ttb_ozaki_kernel_events(1)
    for _ in range(3):
        call("ttb_dgemm_ozaki", 0, M, N, K, ptr(A), K, ptr(B), N, ptr(Cm), N, ptr(ws))
    assert L_.ttb_ozaki_kernel_events(0) == 3
    call("ttb_dgemm_ozaki", 0, M, N, K, ptr(A), K, ptr(B), N, ptr(Cm), N, ptr(ws))     # not recorded
    ms = np.zeros(8)
    sh = np.zeros(32, dtype=np.int32)
    n = L_.ttb_ozaki_kernel_events_read(8, ms.ctypes.data, sh.ctypes.data)
    assert n == 3 and (ms[:3] > 0).all() and (ms[:3] < 50).all()
    assert sh[:12].reshape(3, 4).tolist() == [[M, N, K, 0]] * 3
    assert L_.ttb_ozaki_kernel_events(1) == 0 and L_.ttb_ozaki_kernel_events(0) == 0


@pytest.mark.parametrize("r_last", [300, 400], ids=["square", "wide"])
def test_round_identity_q_for_square_and_wide_unfoldings(monkeypatch, r_last):
    """Right-to-left sweep over a last core whose unfolding X^T (n x r) has r >= n >= 256: the core becomes
    the identity and the carry is X (no factorization). Same tensor and ranks as the Householder sweep and
    as the oracle's tt_round (reference tensor_train/core.py:353-389)."""
    from oracle import tt as OT
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200.tensor_train import TtTensor, tt_round
    from paper_2509_13224_b200.tensor_train.core import _rl_orthogonalize
    rng = np.random.default_rng(r_last)
    n = 300
    cores = [rng.standard_normal((1, 6, 5)), rng.standard_normal((5, 7, r_last)) / 5,
             rng.standard_normal((r_last, n, 1)) / np.sqrt(r_last)]
    t = TtTensor([T(G) for G in cores])
    orth, _ = _rl_orthogonalize(list(t.cores))
    k = min(n, r_last)
    assert tuple(orth[2].shape) == (k, n, 1)
    assert torch.equal(orth[2].reshape(k, n), torch.eye(k, dtype=torch.float64, device="cuda"))
    want = OT.TT(cores).full()
    got = TtTensor(orth).full()
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()
    y = tt_round(t, 1e-10)
    monkeypatch.setattr(L, "_FULLRANK_IDENTITY", False)
    yh = tt_round(t, 1e-10)
    yo = OT.round_tt(OT.TT(cores), 1e-10)
    assert tuple(y.ranks) == tuple(yh.ranks) == tuple(yo.ranks)
    assert np.abs(y.full() - yo.full()).max() <= 1e-12 * np.abs(want).max()
    assert np.abs(yh.full() - yo.full()).max() <= 1e-12 * np.abs(want).max()


@pytest.mark.parametrize("shape,decay", [((510, 510), 0.7), ((2040, 510), 0.85), ((300, 300), 0.5), ((510, 510), 1.0)],
                         ids=["square", "tall", "fast-decay", "flat"])
def test_topk_svd_matches_full_svd(la, shape, decay):
    """The rank-capped rounding step from the leading singular triplets only (linalg.topk_svd) against the
    full SVD + _chop (reference tensor_train/core.py:341-350): same keep, same rank-keep approximant. A nearly flat
    spectrum (no gap to converge on) must fall back (None) rather than return an unconverged basis."""
    from paper_2509_13224_b200.tensor_train.core import _chop
    m, n = shape
    rng = np.random.default_rng(m + n)
    Uo, _ = np.linalg.qr(rng.standard_normal((m, n)))
    Vo, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = decay ** np.arange(n) if decay < 1.0 else 1.0 - 1e-3 * np.arange(n) / n     # "flat": no usable gap
    Xh = (Uo * s) @ Vo.T
    X = T(Xh)
    fro = float(np.linalg.norm(Xh))
    for eps, kmax in [(0.5, 4), (0.5, 2), (0.05, 8), (0.9, 4)]:
        delta = eps * fro / np.sqrt(2.0)
        got = la.topk_svd(X, kmax, delta)
        if decay == 1.0:
            assert got is None
            continue
        assert got is not None, (eps, kmax)
        U, carry = got
        f = la.SVDFactors(X)
        sh = np.sort(f.s_host())[::-1]
        keep = _chop(sh, delta, kmax)
        assert U.shape == (m, keep) and carry.shape == (keep, n), (U.shape, keep)
        approx = (U @ carry).cpu().numpy()
        want = (Uo[:, :keep] * s[:keep]) @ Vo[:, :keep].T
        assert np.abs(approx - want).max() <= 1e-11 * s[0]
        assert float((U.t() @ U - torch.eye(keep, dtype=torch.float64, device="cuda")).abs().max()) < 1e-13
    # tight thresholds are left to the full SVD (the tails would cancel)
    assert la.topk_svd(X, 4, 1e-8 * fro) is None


def test_round_rank_capped_topk_matches_full(monkeypatch):
    """tt_round(t, 0.5, max_rank=4) -- the AMEn residual rounding (reference amen.py:262-266) -- through the
    leading-triplet route and through the full SVDs: same ranks, same tensor; also against the oracle."""
    from oracle import tt as OT
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200.tensor_train import TtTensor, tt_round
    rng = np.random.default_rng(12)
    n, r = 320, 300
    dec = 0.8 ** np.arange(r)
    cores = [rng.standard_normal((1, n, r)) * dec[None, None, :], rng.standard_normal((r, 6, r)) * dec[None, None, :] / r,
             rng.standard_normal((r, n, 1)) / np.sqrt(r)]
    t = TtTensor([T(G) for G in cores])
    calls = []
    orig = L.topk_svd
    monkeypatch.setattr(L, "topk_svd", lambda *a, **k: calls.append(orig(*a, **k)) or calls[-1])
    y = tt_round(t, 0.5, max_rank=4)
    assert any(c is not None for c in calls), "the leading-triplet route did not run"
    monkeypatch.setattr(L, "_TOPK", False)
    yf = tt_round(t, 0.5, max_rank=4)
    yo = OT.round_tt(OT.TT(cores), 0.5, 4)
    assert tuple(y.ranks) == tuple(yf.ranks) == tuple(yo.ranks), (y.ranks, yf.ranks, yo.ranks)
    full, fullf, fullo = y.full(), yf.full(), yo.full()
    scale = np.abs(fullo).max()
    assert np.abs(full - fullf).max() <= 1e-10 * scale
    assert np.abs(full - fullo).max() <= 1e-10 * scale
