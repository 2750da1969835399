"""CPU checks of the oracle's EXTENSION pieces (BASELINE configs beyond the reference) and of
reference properties the parity tests rely on (SPEC acceptance criteria 6a-6h at small sizes)."""

import numpy as np
import pytest

from oracle import bspline as B
from oracle import cross as X
from oracle import iga
from oracle import patch as P
from oracle import tt as T
from oracle.amen import amen


def test_quarter_cylinder_exact_radii():
    pt = P.build_patch("quarter_cylinder")
    rng = np.random.default_rng(0)
    for xi in rng.uniform(0, 1, (300, 3)):
        x = pt.point(xi)
        r = np.hypot(x[0], x[1])
        assert 1.0 - 1e-12 <= r <= 2.0 + 1e-12
        assert x[0] >= -1e-12 and x[1] >= -1e-12 and -1e-12 <= x[2] <= 1 + 1e-12
    # radius is exactly linear in the radial parameter (exact rational arc)
    for t in np.linspace(0, 1, 7):
        x = pt.point(np.array([0.37, t, 0.5]))
        assert abs(np.hypot(x[0], x[1]) - (1.0 + t)) < 1e-13


def test_deformed_cube_interpolates_map():
    pt = P.build_patch("deformed_cube")
    g = pt.sp[0].greville()
    a = 0.1
    for (i, j, k) in [(0, 0, 0), (3, 7, 11), (15, 15, 15), (5, 0, 9)]:
        u, v, s = g[i], g[j], g[k]
        ref = np.array([u + a * np.sin(2 * np.pi * v) * np.sin(np.pi * s),
                        v + a * np.sin(2 * np.pi * s) * np.sin(np.pi * u),
                        s + a * np.sin(2 * np.pi * u) * np.sin(np.pi * v)])
        assert np.allclose(pt.point(np.array([u, v, s])), ref, atol=1e-12)
    # interpolation error of the smooth map is small everywhere
    rng = np.random.default_rng(1)
    xi = rng.uniform(0, 1, 3)
    u, v, s = xi
    ref = np.array([u + a * np.sin(2 * np.pi * v) * np.sin(np.pi * s), v + a * np.sin(2 * np.pi * s) * np.sin(np.pi * u),
                    s + a * np.sin(2 * np.pi * u) * np.sin(np.pi * v)])
    assert np.abs(pt.point(xi) - ref).max() < 1e-3


def test_random_cube_seeded_and_valid():
    a = P.build_patch("random_cube", {"seed": 3})
    b = P.build_patch("random_cube", {"seed": 3})
    c = P.build_patch("random_cube", {"seed": 4})
    assert np.array_equal(a.ctrl, b.ctrl) and not np.array_equal(a.ctrl, c.ctrl)
    # boundary control points untouched -> the patch still covers the unit cube faces
    assert np.allclose(a.ctrl[0, :, :, 0], 0.0) and np.allclose(a.ctrl[-1, :, :, 0], 1.0)
    rng = np.random.default_rng(2)
    for xi in rng.uniform(0, 1, (50, 3)):
        assert a.metric(xi)[1] > 0


def test_random_cube_min_det_sum_factorization_matches_pointwise():
    """The sum-factorized det J grid check (used for the solve's full Gauss grid) against the per-point
    Jacobians of the restated reference evaluator."""
    pt = P.build_patch("random_cube", {"seed": 5, "sigma": 0.05})
    axes = [P.gauss_grid(3, 4), P.gauss_grid(4, 3), P.gauss_grid(5, 2)]
    mn, bad = P.min_det_polynomial_grid(pt, axes, chunk=3)
    ev = P.TensorGridEval(pt, axes)
    idx = np.stack(np.meshgrid(*[np.arange(a.size) for a in axes], indexing="ij"), -1).reshape(-1, 3)
    det = np.linalg.det(ev.jac_points(idx)[0])
    assert bad == int((det <= 0).sum())
    assert abs(mn - det.min()) <= 1e-13 * abs(det).max()


def test_random_cube_checks_the_solve_gauss_grid():
    """configs[3] rejects draws on every Gauss point of the solve: the driver passes (n_basis - p, p + 1)."""
    cfg = iga.Config(geometry="random_cube", degree=3, n_basis=10, source="one")
    prm = iga.geometry_params(cfg)
    assert prm["check_gauss"] == [[7, 4]] * 3
    pt = P.build_patch("random_cube", prm)
    assert pt.meta["check_points"] == 28 ** 3 and pt.meta["min_det"] > 0
    # a draw far off the identity is rejected on the dense grid
    with pytest.raises(P.PatchFault):
        P.build_patch("random_cube", {"sigma": 0.5, "max_draws": 2, "check_gauss": [7, 4]})


def test_exp_sines_source_is_minus_laplacian():
    rng = np.random.default_rng(3)
    x = rng.uniform(0.1, 0.9, (20, 3))
    u = lambda y: np.exp(y.sum(1)) * np.prod(np.sin(np.pi * y), axis=1)
    h = 1e-4
    lap = np.zeros(20)
    for d in range(3):
        e = np.zeros(3)
        e[d] = h
        lap += (u(x + e) - 2 * u(x) + u(x - e)) / h ** 2
    assert np.allclose(iga.SOURCES["exp_sines"](x), -lap, rtol=1e-5, atol=1e-5)


def test_exact_count_solution_space():
    geo = P.build_patch("deformed_cube").sp[0]
    sp = B.solution_space_exact(geo, 3, 40)
    assert sp.n == 40 and sp.p == 3 and np.allclose(np.diff(np.unique(sp.t)), 1 / 37)


def test_lift_adjacent_faces_reproduces_boundary():
    """EXTENSION: Dirichlet data on all faces; the lift interpolates u on every boundary layer."""
    cfg = iga.Config(geometry="deformed_cube", degree=3, n_basis=7, source="exp_sines", analytic="exp_sines",
                     bc_from_analytic=True)
    pt = P.build_patch("deformed_cube")
    cfg.resolve(pt)
    disc = iga.discretize(cfg, pt)
    lift = iga.lift_tt(pt, disc, cfg.bc).full()
    for a in range(3):
        for s in (0, 1):
            ref = iga.face_coeffs(pt, disc, cfg.bc, a, s)
            sl = [slice(None)] * 3
            sl[a] = 0 if s == 0 else -1
            assert np.abs(ref).max() > 1e-3
            assert np.abs(lift[tuple(sl)] - ref).max() < 1e-12 * np.abs(ref).max()
    assert np.abs(lift[1:-1, 1:-1, 1:-1]).max() < 1e-13 * np.abs(lift).max()


def test_config0_small_convergence():
    """configs[0] family (unit cube, p=2, manufactured sines): error decreases ~h^3 (oracle)."""
    errs = []
    for n in (6, 10, 18):
        r = iga.solve(iga.Config(geometry="unit_cube", degree=2, n_basis=n, source="manufactured_sines",
                                 analytic="cube_sines", eps_cross=1e-10, eps_round=1e-10, eps_solve=1e-10))
        assert r["solver_converged"] and r["ranks_K"] == (1, 2, 2, 1)
        errs.append(r["l2_error"])
    assert errs[0] > errs[1] > errs[2]
    assert np.log(errs[1] / errs[2]) / np.log(16 / 8) > 2.5


def test_config1_small_manufactured():
    """configs[1] family at n=10: quarter cylinder, Dirichlet data from u on all faces."""
    r = iga.solve(iga.Config(geometry="quarter_cylinder", degree=3, n_basis=10, source="manufactured_sines",
                             analytic="cube_sines", bc_from_analytic=True, eps_cross=1e-8, eps_round=1e-8,
                             eps_solve=1e-8))
    assert r["solver_converged"] and r["ranks_K"] == (1, 2, 2, 1)
    assert r["l2_error"] < 3e-2
    r2 = iga.solve(iga.Config(geometry="quarter_cylinder", degree=3, n_basis=16, source="manufactured_sines",
                              analytic="cube_sines", bc_from_analytic=True, eps_cross=1e-8, eps_round=1e-8,
                              eps_solve=1e-8))
    assert r2["l2_error"] < 0.25 * r["l2_error"]


def test_round_error_bound_and_zero():
    rng = np.random.default_rng(3)
    for eps in (1e-2, 1e-6, 1e-10):
        Xd = rng.standard_normal((8, 8, 8))
        err = np.linalg.norm(T.round_tt(T.from_full(Xd), eps).full() - Xd)
        assert err <= eps * np.linalg.norm(Xd) + 1e-15
    z = T.round_tt(T.TT.zeros((4, 5, 6)), 1e-8)
    assert z.ranks == (1, 1, 1, 1) and np.all(z.full() == 0)


def test_trilinear_element_and_structure():
    pt = P.build_patch("unit_cube")
    disc = iga.gauss_tables([B.Spline1D.uniform(1, 1)] * 3)
    K, _ = iga.stiffness(pt, disc, 1e-12, rng=np.random.default_rng(5))
    Kd = K.full()
    nodes = [(i, j, k) for i in range(2) for j in range(2) for k in range(2)]
    pat = {0: 1 / 3, 1: 0.0, 2: -1 / 12, 3: -1 / 12}
    for a, na in enumerate(nodes):
        for b, nb in enumerate(nodes):
            assert abs(Kd[a, b] - pat[sum(x != y for x, y in zip(na, nb))]) < 1e-12


def test_cross_rank_one_and_maxvol_dominance():
    f = lambda idx: np.exp(-0.3 * idx[:, 0]) * (idx[:, 1] + 1.0) * np.cos(idx[:, 2])
    t, err, ok, _, _ = X.cross(f, (16, 16, 16), 1e-10, rng=np.random.default_rng(4))
    assert t.ranks == (1, 1, 1, 1) and ok
    M = np.random.default_rng(21).standard_normal((200, 8))
    sel = X.maxvol(M, tol=1.01)
    C = np.linalg.solve(M[sel].T, M.T).T
    assert np.abs(C).max() <= 1.01 + 1e-9
    with pytest.raises(X.MaxvolFault):
        Z = np.zeros((10, 3))
        Z[:, 0] = np.arange(10)
        Z[:, 1] = 2 * np.arange(10)
        X.maxvol(Z)


def test_amen_residual_certificate():
    n = 10
    Lp = (2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)) * (n + 1) ** 2
    I = np.eye(n)
    A = T.round_tt(T.add(T.add(T.TTOp.kron([Lp, I, I]), T.TTOp.kron([I, Lp, I])), T.TTOp.kron([I, I, Lp])), 1e-14)
    f = T.round_tt(T.TT.random((n, n, n), (2, 2), np.random.default_rng(7)), 1e-14)
    u, res, ok, _ = amen(A, f, 1e-8)
    rec = T.norm(T.sub(f, T.matvec(A, u))) / T.norm(f)
    assert ok and res <= 1e-8 and abs(rec - res) <= 1e-12
