"""BASELINE configs on the GPU vs the CPU oracle (same seeds), at north_star tolerances.

Parity setting: the solves below run with eps_solve = 1e-12 (PARITY_EPS). At the configs' own
eps_solve = 1e-8 both solvers stop at a relative residual ~1e-8 on operators with cond ~1e3-1e6, so
their solutions may legitimately differ by ~1e-6; at 1e-12 both are converged far below the bar and
the solution is asserted at the north_star's 1e-9 (relative Frobenius norm of the TT difference).

* configs[0] (n=32) and configs[1] (n=128): full size, oracle run live -- K, f, u <= 1e-9, ranks +-2,
  L2 error within 1% (configs[1]: the oracle's error quadrature over 1.25e8 points takes minutes, so
  its solution's error is evaluated with the same device error kernel -- that kernel is itself checked
  against the oracle's error functional on configs[0] and the reference solves, test_gpu_parity.py);
* configs[4] (n=1024, 1.07e9 dofs): full size against the committed oracle fixture
  (tests/golden/make_fullsize_fixtures.py) -- K, f, u <= 1e-9, ranks +-2, L2 error within 1%;
* configs[2] (n=256) assembly: full size against the fixture's load cores (<= 1e-9) and the stiffness
  TT's gauge-invariant summaries (ranks, bond singular values, norm, 4096 sampled entries);
* configs[2]/[3] at reduced n (the oracle's AMEn cannot run at full size: its explicit residual core is
  ~100 GB / ~0.5 TB) and against the n=16 / n=10 fixtures.

Every test prints its achieved errors (pytest -s) and records them as properties.
"""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

PARITY_EPS = 1e-12
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _tt_rel(a, b):
    from paper_2509_13224_b200.tensor_train import tt_norm, tt_sub
    return tt_norm(tt_sub(a, b)) / tt_norm(b)


def _to_gpu(o, band=None):
    from paper_2509_13224_b200.tensor_train import TtMatrix, TtTensor
    if hasattr(o, "row_sizes"):
        M = TtMatrix([torch.as_tensor(G, device="cuda") for G in o.cores])
        return TtMatrix.banded_from_dense_cores(M.cores, band) if band is not None else M
    return TtTensor([torch.as_tensor(G, device="cuda") for G in o.cores])


def _ranks_close(a, b, slack=2):
    return len(a) == len(b) and all(abs(int(x) - int(y)) <= slack for x, y in zip(a, b))


def _report(record_property, tag, **errs):
    print(f"{tag}: " + ", ".join(f"{k} {v:.3e}" if isinstance(v, float) else f"{k} {v}" for k, v in errs.items()))
    for k, v in errs.items():
        record_property(k, v)


def _device_l2(rep, u):
    """The device error functional (reference driver.py:388-422) applied to a given solution TT."""
    from paper_2509_13224_b200 import driver as D
    return D.l2_error(u, D.ANALYTIC[rep.config.analytic](rep.config, rep.patch), rep.patch, rep.disc)


def _run(cfg_kw, opts=None, compare_u=True, want_error=True):
    from oracle import iga as OI
    from paper_2509_13224_b200 import driver as D
    kw = dict(cfg_kw)
    if opts:
        kw["solver"] = opts
    rep = D.solve_poisson(D.SolveConfig(seed=0, **kw), want_error=want_error)
    ref = OI.solve(OI.Config(seed=0, **kw), want_error=want_error)
    p = max(rep.config.degree)
    out = {"eK": _tt_rel(rep.K, _to_gpu(ref["K"], band=p)), "ef": _tt_rel(rep.f, _to_gpu(ref["f"])), "rep": rep,
           "ref": ref}
    assert _ranks_close(rep.ranks_K, ref["ranks_K"]), (rep.ranks_K, ref["ranks_K"])
    assert _ranks_close(rep.ranks_f, ref["ranks_f"]), (rep.ranks_f, ref["ranks_f"])
    if compare_u:
        out["eu"] = _tt_rel(rep.u, _to_gpu(ref["u"]))
        assert _ranks_close(rep.ranks_u, ref["ranks_u"]), (rep.ranks_u, ref["ranks_u"])
    if ref["l2_error"] is not None:
        out["l2"], out["l2_oracle"] = rep.l2_error, ref["l2_error"]
        assert abs(rep.l2_error - ref["l2_error"]) <= 0.01 * ref["l2_error"], (rep.l2_error, ref["l2_error"])
    return out


def _errs(r, *keys):
    return {k: float(r[k]) for k in keys if k in r}


def test_configs0_full_size(record_property):
    from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
    r = _run(dict(SOLVE_CONFIGS[0], eps_solve=PARITY_EPS))
    _report(record_property, "configs[0] n=32", **_errs(r, "eK", "ef", "eu", "l2", "l2_oracle"))
    assert r["eK"] <= 1e-9 and r["ef"] <= 1e-9 and r["eu"] <= 1e-9, (r["eK"], r["ef"], r["eu"])
    assert r["rep"].solver_converged and r["rep"].dofs == 32 ** 3


def test_configs1_full_size(record_property):
    from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
    r = _run(dict(SOLVE_CONFIGS[1], eps_solve=PARITY_EPS), want_error=False)
    from paper_2509_13224_b200.tensor_train import TtTensor
    rep = r["rep"]
    uo = TtTensor([torch.as_tensor(G, device="cuda") for G in r["ref"]["u"].cores])
    l2, l2o = _device_l2(rep, rep.u), _device_l2(rep, uo)
    _report(record_property, "configs[1] n=128", **_errs(r, "eK", "ef", "eu"), l2=l2, l2_oracle_u=l2o)
    assert r["eK"] <= 1e-9 and r["ef"] <= 1e-9 and r["eu"] <= 1e-9, (r["eK"], r["ef"], r["eu"])
    assert abs(l2 - l2o) <= 0.01 * l2o, (l2, l2o)
    assert rep.solver_converged and rep.dofs == 128 ** 3


def test_configs1_default_eps_solve(record_property):
    """configs[1] as specified (eps_solve 1e-8): K/f at 1e-9; u at the solver tolerance."""
    from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
    r = _run(SOLVE_CONFIGS[1], want_error=False)
    _report(record_property, "configs[1] eps_solve=1e-8", **_errs(r, "eK", "ef", "eu"))
    assert r["eK"] <= 1e-9 and r["ef"] <= 1e-9 and r["eu"] <= 1e-6, (r["eK"], r["ef"], r["eu"])


def test_configs2_reduced(record_property):
    from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
    r = _run(dict(SOLVE_CONFIGS[2], n_basis=8, eps_solve=PARITY_EPS))
    _report(record_property, "configs[2] n=8", **_errs(r, "eK", "ef", "eu", "l2", "l2_oracle"))
    assert r["eK"] <= 1e-9 and r["ef"] <= 1e-9 and r["eu"] <= 1e-9, (r["eK"], r["ef"], r["eu"])


def test_configs3_reduced(record_property):
    from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
    r = _run(dict(SOLVE_CONFIGS[3], n_basis=8, eps_solve=PARITY_EPS))
    _report(record_property, "configs[3] n=8", **_errs(r, "eK", "ef", "eu"))
    assert r["eK"] <= 1e-9 and r["ef"] <= 1e-9 and r["eu"] <= 1e-9, (r["eK"], r["ef"], r["eu"])


def test_configs4_family_reduced(record_property):
    from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
    r = _run(dict(SOLVE_CONFIGS[4], n_basis=48, eps_solve=PARITY_EPS))
    _report(record_property, "configs[4] n=48", **_errs(r, "eK", "ef", "eu", "l2", "l2_oracle"))
    assert r["eK"] <= 1e-9 and r["ef"] <= 1e-9 and r["eu"] <= 1e-9, (r["eK"], r["ef"], r["eu"])


def _fullsize():
    path = os.path.join(GOLDEN, "configs_fullsize_oracle.npz")
    if not os.path.exists(path):
        pytest.fail("tests/golden/configs_fullsize_oracle.npz missing (tests/golden/make_fullsize_fixtures.py)")
    return np.load(path)


def test_configs4_full_size_vs_oracle_fixture(record_property):
    """configs[4] at n=1024 (1.07e9 dofs): the reference algorithm's K, f, u (oracle, fixture) vs the device."""
    from paper_2509_13224_b200 import driver as D
    from paper_2509_13224_b200.tensor_train import TtMatrix, TtTensor
    from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
    g = _fullsize()
    if "c4_u0" not in g:
        pytest.fail("fixture has no configs[4] entry")
    eps = float(g["c4_eps_solve"])
    rep = D.solve_poisson(D.SolveConfig(seed=0, **dict(SOLVE_CONFIGS[4], eps_solve=eps)), want_error=True)
    p = max(rep.config.degree)
    Ko = TtMatrix([torch.as_tensor(g[f"c4_K{k}"], device="cuda") for k in range(3)], band=p)
    fo = TtTensor([torch.as_tensor(g[f"c4_f{k}"], device="cuda") for k in range(3)])
    uo = TtTensor([torch.as_tensor(g[f"c4_u{k}"], device="cuda") for k in range(3)])
    eK, ef, eu = _tt_rel(rep.K, Ko), _tt_rel(rep.f, fo), _tt_rel(rep.u, uo)
    l2o = _device_l2(rep, uo)
    _report(record_property, "configs[4] n=1024", eK=eK, ef=ef, eu=eu, l2=rep.l2_error, l2_oracle_u=l2o,
            ranks_u=str(rep.ranks_u), ranks_u_oracle=str(tuple(g["c4_ranks_u"])), residual=rep.residual)
    assert _ranks_close(rep.ranks_K, g["c4_ranks_K"]) and _ranks_close(rep.ranks_f, g["c4_ranks_f"])
    assert _ranks_close(rep.ranks_u, g["c4_ranks_u"]), (rep.ranks_u, g["c4_ranks_u"])
    assert eK <= 1e-9 and ef <= 1e-9 and eu <= 1e-9, (eK, ef, eu)
    assert abs(rep.l2_error - l2o) <= 0.01 * l2o, (rep.l2_error, l2o)
    assert rep.solver_converged and rep.dofs == 1024 ** 3


def _assemble(c, n_basis=None):
    from paper_2509_13224_b200 import driver as D
    from paper_2509_13224_b200.assembly import assemble_load, assemble_stiffness
    from paper_2509_13224_b200.geometry import make_geometry
    from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
    kw = dict(SOLVE_CONFIGS[c])
    if n_basis is not None:
        kw["n_basis"] = n_basis
    cfg = D.SolveConfig(seed=0, **kw)
    patch = make_geometry(cfg.geometry, D.geometry_params(cfg))
    cfg.resolve_bc(patch)
    disc = D.discretize(cfg, patch)
    rK, rf = D._spawn_rngs(cfg.seed, 2)
    K, _ = assemble_stiffness(patch, disc, cfg.eps_round, rank_cap=cfg.rank_cap, rng=rK)
    f, _ = assemble_load(patch, disc, cfg.source, cfg.eps_cross, rank_cap=cfg.rank_cap, rng=rf)
    return K, f, cfg.degree[0]


def _band_bond_singular_values(K):
    """Singular values of both unfoldings of a banded 3-core operator TT (host numpy; zero band slots do not
    change them)."""
    C = [G.reshape(G.shape[0], -1, G.shape[3]).cpu().numpy() for G in K.cores]
    for k in (2, 1):
        r0, n, r1 = C[k].shape
        Q, R = np.linalg.qr(C[k].reshape(r0, n * r1).T)
        C[k] = Q.T.reshape(-1, n, r1)
        C[k - 1] = np.tensordot(C[k - 1], R.T, (2, 0))
    U, s1, Vt = np.linalg.svd(C[0].reshape(-1, C[0].shape[2]), full_matrices=False)
    C1 = np.tensordot(s1[:, None] * Vt, C[1], (1, 0))
    s2 = np.linalg.svd(C1.reshape(-1, C1.shape[2]), compute_uv=False)
    return s1, s2


def _band_entries(K, I, J, h):
    v = None
    for d in range(3):
        i = torch.as_tensor(I[:, d].astype(np.int64), device="cuda")
        t = torch.as_tensor((J[:, d] - I[:, d] + h).astype(np.int64), device="cuda")
        G = K.cores[d][:, i, t, :]                       # (r0, N, r1)
        v = G[0] if v is None else torch.einsum("nr,rns->ns", v, G)
    return v[:, 0].cpu().numpy()


@pytest.mark.parametrize("tag,c,n", [("c2", 2, None), ("c3n128", 3, 128), ("c3", 3, None)])
def test_fullsize_assembly_vs_oracle_fixture(record_property, tag, c, n):
    """TT assembly (reference assembly.py:236-304) against the oracle fixture: configs[2] at its full n=256,
    configs[3] at n=128 (its full n=512 exceeds the oracle's host memory: skipped without a fixture)."""
    from paper_2509_13224_b200.tensor_train import TtTensor, tt_norm
    g = _fullsize()
    if f"{tag}_f0" not in g:
        pytest.skip(f"fixture has no {tag} assembly entry")
    K, f, p = _assemble(c, n)
    fo = TtTensor([torch.as_tensor(g[f"{tag}_f{k}"], device="cuda") for k in range(3)])
    ef = _tt_rel(f, fo)
    s1, s2 = _band_bond_singular_values(K)
    so1, so2 = g[f"{tag}_K_s1"], g[f"{tag}_K_s2"]
    k1, k2 = min(s1.size, so1.size), min(s2.size, so2.size)
    es1 = float(np.abs(s1[:k1] - so1[:k1]).max() / so1[0])
    es2 = float(np.abs(s2[:k2] - so2[:k2]).max() / so2[0])
    vals = _band_entries(K, g[f"{tag}_K_I"], g[f"{tag}_K_J"], p)
    ev = float(np.abs(vals - g[f"{tag}_K_vals"]).max() / np.abs(g[f"{tag}_K_vals"]).max())
    en = abs(tt_norm(K) - float(g[f"{tag}_K_norm"])) / float(g[f"{tag}_K_norm"])
    _report(record_property, f"configs[{c}] assembly ({tag})", ef=ef, K_s1=es1, K_s2=es2, K_entries=ev, K_norm=en,
            ranks_K=str(K.ranks), ranks_K_oracle=str(tuple(g[f"{tag}_ranks_K"])))
    assert _ranks_close(K.ranks, g[f"{tag}_ranks_K"]) and _ranks_close(f.ranks, g[f"{tag}_ranks_f"])
    assert ef <= 1e-9, ef
    assert es1 <= 1e-9 and es2 <= 1e-9 and ev <= 1e-9 and en <= 1e-9, (es1, es2, ev, en)


def _vs_fixture(tag, cfg_idx, n, tol_u, record_property):
    """Device solve vs the committed oracle fixture (tests/golden/make_config_fixtures.py)."""
    from paper_2509_13224_b200 import driver as D
    from paper_2509_13224_b200.tensor_train import TtTensor
    from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
    g = np.load(os.path.join(GOLDEN, "configs_oracle.npz"))
    rep = D.solve_poisson(D.SolveConfig(seed=0, **dict(SOLVE_CONFIGS[cfg_idx], n_basis=n)))
    uo = TtTensor([torch.as_tensor(g[f"{tag}_u{k}"], device="cuda") for k in range(3)])
    fo = TtTensor([torch.as_tensor(g[f"{tag}_f{k}"], device="cuda") for k in range(3)])
    eu, ef = _tt_rel(rep.u, uo), _tt_rel(rep.f, fo)
    _report(record_property, f"{tag} vs fixture", ef=ef, eu=eu, residual=rep.residual)
    assert ef <= 1e-9, ef
    assert eu <= tol_u, eu
    assert _ranks_close(rep.ranks_K, tuple(g[f"{tag}_ranks_K"])), (rep.ranks_K, g[f"{tag}_ranks_K"])
    assert _ranks_close(rep.ranks_u, tuple(g[f"{tag}_ranks_u"])), (rep.ranks_u, g[f"{tag}_ranks_u"])
    # same stopping behaviour: both reach (or stagnate just above) the 1e-8 target
    assert rep.residual <= 2.0 * float(g[f"{tag}_residual"]) + 1e-9, (rep.residual, float(g[f"{tag}_residual"]))
    lo = float(g[f"{tag}_l2_error"])
    if not np.isnan(lo):
        assert abs(rep.l2_error - lo) <= 0.01 * lo, (rep.l2_error, lo)
    return rep


def test_configs2_n16_vs_oracle_fixture(record_property):
    """Deformed cube at n=16 (operator ranks 70): GEMM-staged banded operator and compressed residual. Both
    solves stagnate at a residual of 1-4e-8 after the reference's 50 sweeps (eps_solve 1e-8), so u agrees
    only to the solver tolerance here."""
    _vs_fixture("c2_n16", 2, 16, 1e-5, record_property)


def test_configs3_n10_vs_oracle_fixture(record_property):
    """Random cube at n=10 (operator ranks 53, f = 1, no manufactured solution)."""
    _vs_fixture("c3_n10", 3, 10, 1e-5, record_property)


def test_random_cube_det_check_on_solve_gauss_grid(record_property):
    """configs[3]'s admissibility check covers every Gauss point of the solve: the device min-det kernel
    (ttb_geo_min_det) against the oracle's sum-factorized check at n=64 (244^3 points), and the full
    n=512 grid (2036^3 = 8.4e9 points) timed, with the same draw count as the coarse-grid oracle draw."""
    import time
    from oracle import iga as OI
    from oracle import patch as OP
    from paper_2509_13224_b200 import driver as D
    from paper_2509_13224_b200.geometry import GridEvaluator, make_geometry
    from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
    cfg = D.SolveConfig(seed=0, **dict(SOLVE_CONFIGS[3], n_basis=64))
    prm = D.geometry_params(cfg)
    assert prm["check_gauss"] == [[61, 4]] * 3
    patch = make_geometry("random_cube", prm)
    opt = OP.build_patch("random_cube", OI.geometry_params(OI.Config(seed=0, **dict(SOLVE_CONFIGS[3], n_basis=64))))
    assert patch.metadata["draws"] == opt.meta["draws"]
    assert np.array_equal(patch.control_points, opt.ctrl)
    e_min = abs(patch.metadata["min_det"] - opt.meta["min_det"]) / opt.meta["min_det"]
    axes = [OP.gauss_grid(61, 4)] * 3
    mn, bad = GridEvaluator(patch, axes).min_det()
    assert bad == 0 and abs(mn - patch.metadata["min_det"]) == 0.0
    cfg = D.SolveConfig(seed=0, **SOLVE_CONFIGS[3])
    torch.cuda.synchronize()
    t = time.perf_counter()
    full = make_geometry("random_cube", D.geometry_params(cfg))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    _report(record_property, "random_cube det check", n64_min_det_rel_err=e_min, n512_points=full.metadata["check_points"],
            n512_min_det=full.metadata["min_det"], n512_draws=full.metadata["draws"], n512_check_s=dt)
    assert e_min <= 1e-12
    assert full.metadata["check_points"] == 2036 ** 3 and full.metadata["min_det"] > 0
