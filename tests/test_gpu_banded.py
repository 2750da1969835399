"""GEMM-staged banded contractions and the compressed AMEn residual (GPU).

The GEMM forms (tensor_train/banded.py) must equal the reference's shifted-einsum
contractions (amen.py:77-115, 147-150) -- checked against the elementwise banded kernels
and against numpy einsums of the same inputs -- and the compressed residual must
give the same norm and the same rank-kick rounding as the explicit f - A u TT
(amen.py:262-264, 294). FP64 throughout; tolerances are roundoff-level (1e-12
relative) except the rounded z, whose SVD-truncated subspace is compared as a tensor.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rand(rng, *shape):
    return torch.as_tensor(rng.standard_normal(shape), device="cuda")


def _band_layout(M, h):
    """Banded core layout Mb[a, i, t, b] = M[a, i, i + t - h, b] (zero outside the matrix)."""
    Ra, n, _, Rb = M.shape
    Mb = np.zeros((Ra, n, 2 * h + 1, Rb))
    for i in range(n):
        for t in range(2 * h + 1):
            j = i + t - h
            if 0 <= j < n:
                Mb[:, i, t, :] = M[:, i, j, :]
    return torch.as_tensor(Mb, device="cuda")


def _banded_core(rng, Ra, n, h, Rb):
    M = np.zeros((Ra, n, n, Rb))
    for i in range(n):
        for j in range(max(0, i - h), min(n, i + h + 1)):
            M[:, i, j, :] = rng.standard_normal((Ra, Rb))
    return M, _band_layout(M, h)


def _rel(a, b):
    a = a.detach().cpu().numpy() if torch.is_tensor(a) else np.asarray(a)
    b = b.detach().cpu().numpy() if torch.is_tensor(b) else np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("Ra,Rb,n,h,r0,r1", [(9, 11, 37, 3, 5, 7), (16, 12, 64, 2, 8, 6), (3, 1, 20, 1, 4, 1)])
def test_env_and_local_ops_gemm_equal_reference(Ra, Rb, n, h, r0, r1):
    from paper_2509_13224_b200.tensor_train import amen as A
    from paper_2509_13224_b200.tensor_train import banded as BD
    rng = np.random.default_rng(Ra * 100 + n)
    Md, Mb = _banded_core(rng, Ra, n, h, Rb)
    lay = BD.GemmLayouts([Mb], h)
    phiL = _rand(rng, r0, Ra, r0)
    phiR = _rand(rng, r1, Rb, r1)
    U = _rand(rng, r0, n, r1)
    # environments vs numpy einsum of the reference formulas
    pl, pr, Un = phiL.cpu().numpy(), phiR.cpu().numpy(), U.cpu().numpy()
    refL = np.einsum("xiu,xibv->ubv", Un, np.einsum("aijb,xajv->xibv", Md, np.einsum("xay,yjv->xajv", pl, Un)))
    refR = np.einsum("zis,siaw->zaw", Un, np.einsum("aijb,sbjw->siaw", Md, np.einsum("sbv,wjv->sbjw", pr, Un)))
    assert _rel(BD.env_left_A(phiL, U, lay, 0), refL) < 1e-12
    assert _rel(BD.env_right_A(phiR, U, lay, 0), refR) < 1e-12
    assert _rel(A.env_left_A(phiL, U, Mb, h), refL) < 1e-12
    # local operator: GEMM mode vs elementwise kernels vs einsum
    v = _rand(rng, r0, n, r1)
    s_g = A.LocalSystem(phiL, Mb, h, phiR, lay, 0, force_gemm=True)
    s_n = A.LocalSystem(phiL, Mb, h, phiR)
    ref = np.einsum("xibw,zbw->xiz", np.einsum("aijb,xajw->xibw", Md, np.einsum("xay,yjw->xajw", pl, v.cpu().numpy())),
                    pr)
    assert _rel(s_g.matvec3(v), ref) < 1e-12
    assert _rel(s_n.matvec3(v), ref) < 1e-12


def test_pcg_gemm_equals_elementwise_pcg():
    """Jacobi-PCG on an SPD projected system: GEMM-staged (i,x,z) iteration == reference-layout one."""
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200.tensor_train import amen as A
    from paper_2509_13224_b200.tensor_train import banded as BD
    rng = np.random.default_rng(7)
    Ra = Rb = 9
    n, h, r0, r1 = 48, 2, 6, 5
    # SPD banded core: symmetric in (i, j) and (a, b) with a dominant diagonal
    M = np.zeros((Ra, n, n, Rb))
    for i in range(n):
        for j in range(max(0, i - h), min(n, i + h + 1)):
            blk = rng.standard_normal((Ra, Rb)) * 0.05
            M[:, i, j, :] += blk
            M[:, j, i, :] += blk
        M[:, i, i, :] += np.eye(Ra) * 4.0
    Mb = _band_layout(M, h)
    lay = BD.GemmLayouts([Mb], h)

    def spd(r, R):
        out = np.zeros((r, R, r))
        for a in range(R):
            Q = np.linalg.qr(rng.standard_normal((r, r)))[0]
            out[:, a, :] = Q @ np.diag(1.0 + rng.random(r)) @ Q.T
        return torch.as_tensor(out, device="cuda")

    phiL, phiR = spd(r0, Ra), spd(r1, Rb)
    b = _rand(rng, r0, n, r1)
    s_n = A.LocalSystem(phiL, Mb, h, phiR)
    s_g = A.LocalSystem(phiL, Mb, h, phiR, lay, 0, force_gemm=True)
    x_n = s_n.solve(b, None, 1e-12, 0, 500)
    x_g = s_g.solve(b, None, 1e-12, 0, 500)
    assert _rel(s_n.matvec3(x_n), b) < 1e-10
    assert _rel(x_g, x_n) < 1e-9


@pytest.mark.parametrize("d,n,R,ru,rf", [(3, 12, 5, 4, 3), (3, 30, 9, 6, 4), (2, 16, 4, 3, 2), (4, 6, 3, 2, 2),
                                         (1, 10, 1, 1, 1)])
def test_compressed_residual_equals_explicit(d, n, R, ru, rf):
    from paper_2509_13224_b200.tensor_train import TtMatrix, TtTensor, tt_matvec, tt_norm, tt_round, tt_sub
    from paper_2509_13224_b200.tensor_train import banded as BD
    rng = np.random.default_rng(d * 1000 + n)
    h = 2
    Rs = [1] + [R] * (d - 1) + [1]
    us = [1] + [ru] * (d - 1) + [1]
    fs = [1] + [rf] * (d - 1) + [1]
    Ms = [_banded_core(rng, Rs[k], n, h, Rs[k + 1])[1] for k in range(d)]
    A = TtMatrix(Ms, h)
    u = TtTensor([_rand(rng, us[k], n, us[k + 1]) for k in range(d)])
    f = TtTensor([_rand(rng, fs[k], n, fs[k + 1]) for k in range(d)])
    diff = tt_sub(f, tt_matvec(A, u))
    cores, nrm = BD.compressed_residual(BD.GemmLayouts(Ms, h), u.cores, f.cores)
    comp = TtTensor(cores)
    assert abs(float(nrm) - tt_norm(diff)) <= 1e-12 * tt_norm(diff)
    assert _rel(comp.full(), diff.full()) < 1e-12
    # ranks bounded by the mode-size products from each end
    for k in range(1, d):
        assert comp.ranks[k] <= min(n ** k, n ** (d - k))
    # the rank-kick rounding of the enrichment step is the same tensor
    z1 = tt_round(diff, 0.5, max_rank=4)
    z2 = tt_round(comp, 0.5, max_rank=4)
    assert z1.ranks == z2.ranks
    assert _rel(z2.full(), z1.full()) < 1e-9


def test_compressed_residual_cancellation():
    """u solving A u = f to 1e-10: the compressed norm resolves the small residual like the explicit one."""
    from paper_2509_13224_b200.tensor_train import TtMatrix, TtTensor, amen_solve, tt_matvec, tt_norm, tt_sub
    from paper_2509_13224_b200.tensor_train import banded as BD
    n = 24
    lap = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    I = np.eye(n)
    cores = [np.stack([lap, I], axis=-1)[None], np.zeros((2, n, n, 2)), np.stack([I, lap], axis=0)[..., None]]
    cores[1][0, :, :, 0] = I
    cores[1][1, :, :, 1] = I
    cores[1][0, :, :, 1] = lap
    A = TtMatrix([torch.as_tensor(c, device="cuda") for c in cores])
    rng = np.random.default_rng(3)
    f = TtTensor([_rand(rng, a, n, b) for a, b in ((1, 3), (3, 3), (3, 1))])
    res = amen_solve(A, f, 1e-10)
    Ab = TtMatrix.banded_from_dense_cores(A.cores, 1)
    diff = tt_sub(f, tt_matvec(Ab, res.solution))
    _, nrm = BD.compressed_residual(BD.GemmLayouts(Ab.cores, 1), res.solution.cores, f.cores)
    e = tt_norm(diff)
    assert e <= 1e-10 * tt_norm(f)
    assert abs(float(nrm) - e) <= 1e-3 * e


@pytest.mark.parametrize("band,resid", [("gemm", "compressed"), ("naive", "compressed"), ("gemm", "explicit")])
def test_amen_modes_match_oracle(monkeypatch, band, resid):
    """Deformed cube (non-separable, operator ranks ~20-40) at reduced n: every AMEn mode == oracle."""
    from oracle import iga as OI
    from paper_2509_13224_b200 import driver as D
    from paper_2509_13224_b200.tensor_train import banded as BD
    from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
    monkeypatch.setattr(BD, "_BAND_MODE", band)
    monkeypatch.setattr(BD, "_RES_MODE", resid)
    kw = dict(SOLVE_CONFIGS[2])
    kw["n_basis"] = 10
    kw["solver"] = {"direct_solve_max": 200}   # PCG local solves on the larger cores
    rep = D.solve_poisson(D.SolveConfig(seed=0, **kw))
    ref = OI.solve(OI.Config(seed=0, **kw))
    from paper_2509_13224_b200.tensor_train import TtTensor, tt_norm, tt_sub
    uo = TtTensor([torch.as_tensor(G, device="cuda") for G in ref["u"].cores])
    eu = tt_norm(tt_sub(rep.u, uo)) / tt_norm(uo)
    assert eu < 1e-6, eu
    assert all(abs(a - b) <= 2 for a, b in zip(rep.ranks_u, ref["ranks_u"])), (rep.ranks_u, ref["ranks_u"])
    assert abs(rep.l2_error - ref["l2_error"]) <= 0.01 * ref["l2_error"]


@pytest.mark.parametrize("forward", [True, False])
def test_truncation_residuals_basis_form(forward):
    """GEMM-mode trial-rank residuals (operator applied once to the SVD basis) == direct evaluation."""
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200.tensor_train import amen as A
    from paper_2509_13224_b200.tensor_train import banded as BD
    rng = np.random.default_rng(11 if forward else 12)
    Ra, Rb, n, h, r0, r1 = 10, 9, 40, 3, 7, 6
    _, Mb = _banded_core(rng, Ra, n, h, Rb)
    lay = BD.GemmLayouts([Mb], h)
    phiL, phiR = _rand(rng, r0, Ra, r0), _rand(rng, r1, Rb, r1)
    sy = A.LocalSystem(phiL, Mb, h, phiR, lay, 0, force_gemm=True)
    x3 = _rand(rng, r0, n, r1)
    rhs3 = _rand(rng, r0, n, r1)
    mat = x3.reshape(r0 * n, r1) if forward else x3.reshape(r0, n * r1)
    f = L.SVDFactors(mat, want_v=not forward)
    R = int(f.S.shape[0])
    Uf, SVf = f.U(R), f.SVt(R)
    res = sy.truncation_residuals(Uf, SVf, rhs3, forward)
    for q in (1, 2, R // 2, R):
        xq = L.gemm(Uf[:, :q], SVf[:q]).reshape(r0, n, r1)
        direct = float(L.nrm2(sy.matvec3(xq) - rhs3).item())
        assert abs(res(q) - direct) <= 1e-12 * direct


def _band_ref(Tp, Mt, n, h, Rin, Rout, X):
    from paper_2509_13224_b200 import linalg as L
    B = 2 * h + 1
    out = L.empty(n, X, Rout)
    L.gemm_strided(1, 0, X, Rout, B * Rin, Tp, X, Rin * X, Mt, Rout, B * Rin * Rout, out, Rout, X * Rout, n)
    return out


@pytest.mark.parametrize("graded", [False, True])
def test_band_gemm_ozaki_vs_dmma(graded, record_property):
    """The banded batched contraction on the int8 tensor cores (ttb_band_gemm_ozaki; padding of X, Rout and
    K; a partial last slice group) against the DMMA batch at FP64: normwise <= 1e-14. Graded inputs
    (Tp blocks scaled over 1e6 along the mode index, like a solution spanning boundary layers) compare
    the group exponents (G = 8) with per-window ones (G = 1)."""
    from paper_2509_13224_b200._lib import call, call_raw, ptr
    n, h, Rin, Rout, X = 43, 3, 121, 121, 1000
    B = 2 * h + 1
    g = torch.Generator(device="cuda").manual_seed(7)
    Tp = torch.randn(n + 2 * h, Rin, X, generator=g, dtype=torch.float64, device="cuda")
    Tp[:h] = 0
    Tp[n + h:] = 0
    if graded:
        Tp *= torch.logspace(-3, 3, n + 2 * h, dtype=torch.float64, device="cuda")[:, None, None]
    Mt = torch.randn(n, B, Rin, Rout, generator=g, dtype=torch.float64, device="cuda")
    ref = _band_ref(Tp, Mt, n, h, Rin, Rout, X)
    errs = {}
    for G in (1, 8):
        ws = torch.empty(int(call_raw("ttb_band_gemm_ozaki_workspace", n, h, Rin, Rout, X, G)), dtype=torch.uint8,
                         device="cuda")
        out = torch.full((n, X, Rout), float("nan"), dtype=torch.float64, device="cuda")
        call("ttb_band_gemm_ozaki", n, h, Rin, Rout, X, ptr(Tp), ptr(Mt), ptr(out), ptr(ws), G)
        assert torch.isfinite(out).all()
        # per batch (the graded batches differ by 1e6 in scale)
        e = ((out - ref).flatten(1).norm(dim=1) / ref.flatten(1).norm(dim=1)).max().item()
        errs[G] = e
    print(f"band GEMM Ozaki vs DMMA (graded={graded}): max per-batch normwise error G=1 {errs[1]:.2e}, G=8 {errs[8]:.2e}")
    record_property("err_G1", errs[1])
    record_property("err_G8", errs[8])
    assert errs[1] <= 1e-14 and errs[8] <= (1e-14 if not graded else 1e-12), errs
