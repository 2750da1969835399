"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz)."""

import numpy as np
import pytest

from oracle import bspline as B
from oracle import cross as X
from oracle import iga
from oracle import patch as P
from oracle import tt as T
from oracle.amen import AmenOpts, amen


def test_basis_tables(golden):
    g = golden("splines.npz")
    for c in range(int(g["n_cases"])):
        w = g[f"c{c}_w"]
        sp = B.Spline1D(g[f"c{c}_knots"], int(g[f"c{c}_deg"]), w if w.size else None)
        V, D = B.dense_tables(sp, g[f"c{c}_x"])
        assert np.abs(V - g[f"c{c}_V"]).max() <= 1e-14
        assert np.abs(D - g[f"c{c}_D"]).max() <= 1e-12 * max(1.0, np.abs(g[f"c{c}_D"]).max())


def test_knot_insertion(golden):
    g = golden("splines.npz")
    s = 1 / np.sqrt(2)
    circ = B.Spline1D([0, 0, 0, .25, .25, .5, .5, .75, .75, 1, 1, 1], 2, [1, s, 1, s, 1, s, 1, s, 1])
    Pc = np.array([[1, 0], [1, 1], [0, 1], [-1, 1], [-1, 0], [-1, -1], [0, -1], [1, -1], [1, 0]], float)
    b2, P2 = B.knot_insert(circ, Pc, 0.125)
    assert np.array_equal(b2.t, g["ins_knots"])
    assert np.allclose(b2.w, g["ins_w"], atol=1e-15) and np.allclose(P2, g["ins_P"], atol=1e-14)
    b3, P3 = B.bisect_refine(circ, Pc, 2)
    assert np.array_equal(b3.t, g["ref_knots"])
    assert np.allclose(P3, g["ref_P"], atol=1e-14)
    assert np.allclose(b3.greville(), g["greville"], atol=1e-15)


@pytest.mark.parametrize("name", ["unit_cube", "lshape", "ring", "closed_hemisphere",
                                  "opened_hemisphere", "hyperboloid", "quarter_torus"])
def test_geometry_eval(golden, name):
    g = golden("geometry.npz")
    pt = P.build_patch(name)
    assert np.allclose(pt.ctrl, g[f"{name}_ctrl"], atol=1e-15)
    ev = P.TensorGridEval(pt, list(g[f"{name}_axes"]))
    idx = g[f"{name}_idx"]
    J, x = ev.jac_points(idx)
    det, R = ev.det_metric(idx)
    assert np.abs(J - g[f"{name}_jac"]).max() <= 1e-13
    assert np.abs(x - g[f"{name}_pts"]).max() <= 1e-14
    assert np.abs(det - g[f"{name}_det"]).max() <= 1e-13
    assert np.abs(R - g[f"{name}_R"]).max() <= 1e-12


def test_tt_round_and_matvec(golden):
    g = golden("tensor_train.npz")
    t = T.from_full(g["round_X"])
    for e in (1e-2, 1e-6, 1e-10):
        r = T.round_tt(t, e)
        assert r.ranks == tuple(g[f"round_{e:g}_ranks"])
        assert np.abs(r.full() - g[f"round_{e:g}_full"]).max() <= 1e-12
    A = T.TTOp([g[f"mv_A{k}"] for k in range(3)])
    x = T.TT([g[f"mv_x{k}"] for k in range(3)])
    y = T.matvec(A, x)
    assert np.abs(y.full() - g["mv_y_full"]).max() <= 1e-12 * np.abs(g["mv_y_full"]).max()
    yr = T.round_tt(y, 1e-8)
    assert yr.ranks == tuple(g["mv_round_ranks"])
    assert abs(T.norm(y) - float(g["mv_norm"])) <= 1e-12 * float(g["mv_norm"])


def test_maxvol(golden):
    g = golden("tensor_train.npz")
    assert np.array_equal(X.maxvol(g["maxvol_M"]), g["maxvol_sel"])
    v = np.array([10.0, 0.0])
    Md = np.vstack([v, v, [0.0, 10.0], [0.1, 0.2], [0.3, 0.1]])
    assert np.array_equal(X.maxvol(Md), g["maxvol_dup_sel"])


def test_cross(golden):
    g = golden("tensor_train.npz")
    n = (16, 12, 10)

    def f(idx):
        return (np.sin(idx[:, 0] + 1.0) * np.cos(0.3 * idx[:, 1]) * (idx[:, 2] + 1.0)
                + np.exp(-0.1 * idx[:, 0]) * (idx[:, 1] + 0.5) * np.cos(0.2 * idx[:, 2]))

    t, err, ok, nev, _ = X.cross(f, n, 1e-10, rng=np.random.default_rng(7))
    assert t.ranks == tuple(g["cross_ranks"])
    assert nev == int(g["cross_nevals"])
    assert np.abs(t.full() - g["cross_full"]).max() <= 1e-12 * np.abs(g["cross_full"]).max()


def test_amen(golden):
    g = golden("tensor_train.npz")
    A = T.TTOp([g[f"amen_A{k}"] for k in range(3)])
    f = T.TT([g[f"amen_f{k}"] for k in range(3)])
    u, res, ok, _ = amen(A, f, 1e-10)
    assert ok and u.ranks == tuple(g["amen_ranks"])
    ref = g["amen_u_full"]
    assert np.linalg.norm(u.full() - ref) <= 1e-12 * np.linalg.norm(ref)
    u2, _, _, _ = amen(A, f, 1e-10, AmenOpts(direct_solve_max=16))
    ref2 = g["amen_cg_u_full"]
    assert np.linalg.norm(u2.full() - ref2) <= 1e-10 * np.linalg.norm(ref2)


@pytest.mark.parametrize("name,deg", [("ring", 2), ("lshape", 1), ("hyperboloid", 2), ("quarter_torus", 2)])
def test_assembly(golden, name, deg):
    g = golden("assembly.npz")
    pt = P.build_patch(name)
    bases = tuple(B.solution_space(pt.sp[d], deg, 4) for d in range(3))
    for d in range(3):
        assert np.array_equal(bases[d].t, g[f"{name}_knots{d}"])
    disc = iga.gauss_tables(bases)
    rng = np.random.default_rng(400)
    K, _ = iga.stiffness(pt, disc, 1e-11, rng=rng)
    f, _ = iga.load(pt, disc, iga.SOURCES["sin_pi_xyz"], 1e-11, rng=rng)
    assert K.ranks == tuple(g[f"{name}_Kranks"]) and f.ranks == tuple(g[f"{name}_franks"])
    Kr = g[f"{name}_K"]
    assert np.linalg.norm(K.full() - Kr) <= 1e-12 * np.linalg.norm(Kr)
    fr = g[f"{name}_f"]
    assert np.linalg.norm(f.full() - fr) <= 1e-12 * np.linalg.norm(fr)


SOLVE_CASES = {
    "cube_p2_e8": dict(geometry="unit_cube", degree=2, elements=8, source="manufactured_sines", analytic="cube_sines"),
    "ring_p2_e8": dict(geometry="ring", degree=2, elements=8, source="zero", analytic="ring_radial",
                       bc=iga.Bc({(1, 0): iga.Face("dirichlet", 1.0), (1, 1): iga.Face("dirichlet", 2.0)})),
    "lshape_p1_e8": dict(geometry="lshape", degree=1, elements=8, source="sin_pi_xy", analytic="lshape_exact"),
    "torus_p2_e4": dict(geometry="quarter_torus", degree=2, elements=4, source="sin_pi_xyz"),
    "ohemi_p2_e4": dict(geometry="opened_hemisphere", degree=2, elements=4, source="one"),
}


@pytest.mark.parametrize("tag", list(SOLVE_CASES))
def test_solve_reports(golden, tag):
    g = golden("solves.npz")
    r = iga.solve(iga.Config(seed=0, **SOLVE_CASES[tag]))
    assert r["ranks_K"] == tuple(g[f"{tag}_ranks_K"])
    assert r["ranks_u"] == tuple(g[f"{tag}_ranks_u"])
    ref = g[f"{tag}_u"]
    assert np.linalg.norm(r["u"].full() - ref) <= 1e-10 * np.linalg.norm(ref)
    if not np.isnan(g[f"{tag}_l2"]):
        assert abs(r["l2_error"] - float(g[f"{tag}_l2"])) <= 1e-9 * float(g[f"{tag}_l2"])
