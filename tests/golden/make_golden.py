"""Generate golden vectors from the REAL reference package (build container only).

Run from the repo root with the read-only reference on the path:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``. Nothing on the GPU box reads /root/reference;
the committed fixtures are the reference's outputs on seeded inputs and pin
both the oracle (``tests/test_oracle_golden.py``) and the CUDA path
(``tests/test_gpu_parity.py``).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from ttiga import driver as rdrv  # noqa: E402  (reference)
from ttiga import geometry as rgeo  # noqa: E402
from ttiga import splines as rspl  # noqa: E402
from ttiga import assembly as rasm  # noqa: E402
from ttiga import tensor_train as rtt  # noqa: E402


def save(name, **arrs):
    np.savez_compressed(os.path.join(HERE, name), **arrs)
    print("wrote", name, sum(np.asarray(v).nbytes for v in arrs.values()), "bytes raw")


def splines():
    rng = np.random.default_rng(100)
    rows = []
    out = {}
    cases = []
    for c in range(12):
        p = int(rng.integers(1, 5))
        spans = int(rng.integers(1, 7))
        kv = rspl.KnotVector.open_uniform(p, spans)
        w = rng.uniform(0.2, 3.0, kv.n_basis) if c % 2 else None
        b = rspl.Basis1D(kv, w)
        xs = np.r_[rng.uniform(0, 1, 20), 0.0, 1.0]
        V, D = rspl.tabulate(b, xs)
        out[f"c{c}_knots"] = kv.knots
        out[f"c{c}_deg"] = np.array(p)
        out[f"c{c}_w"] = w if w is not None else np.zeros(0)
        out[f"c{c}_x"] = xs
        out[f"c{c}_V"] = V
        out[f"c{c}_D"] = D
        cases.append(c)
    # knot insertion on the circle
    s = 1 / np.sqrt(2)
    kv = rspl.KnotVector(np.array([0, 0, 0, .25, .25, .5, .5, .75, .75, 1, 1, 1.]), 2)
    circ = rspl.Basis1D(kv, np.array([1, s, 1, s, 1, s, 1, s, 1]))
    P = np.array([[1, 0], [1, 1], [0, 1], [-1, 1], [-1, 0], [-1, -1], [0, -1], [1, -1], [1, 0]], float)
    b2, P2 = rspl.insert_knot(circ, P, 0.125)
    b3, P3 = rspl.h_refine_uniform(circ, P, 2)
    out.update(ins_knots=b2.knot_vector.knots, ins_w=b2.weights, ins_P=P2,
               ref_knots=b3.knot_vector.knots, ref_w=b3.weights, ref_P=P3,
               greville=rspl.greville_points(b3.knot_vector))
    out["n_cases"] = np.array(len(cases))
    save("splines.npz", **out)


def geometry():
    out = {}
    rng = np.random.default_rng(200)
    for name in rgeo.GEOMETRY_NAMES:
        patch = rgeo.make_geometry(name)
        axes = [np.sort(rng.uniform(0.01, 0.99, 7)) for _ in range(3)]
        ev = rgeo.GridEvaluator(patch, axes)
        idx = rng.integers(0, 7, (64, 3))
        jac, pts = ev.jacobians(idx)
        det, R = ev.metric(idx)
        out[f"{name}_axes"] = np.stack(axes)
        out[f"{name}_idx"] = idx
        out[f"{name}_jac"] = jac
        out[f"{name}_pts"] = pts
        out[f"{name}_det"] = det
        out[f"{name}_R"] = R
        out[f"{name}_ctrl"] = patch.control_points
        out[f"{name}_w"] = patch.weights
    save("geometry.npz", **out)


def tensor_train():
    out = {}
    rng = np.random.default_rng(300)
    X = rng.standard_normal((8, 9, 7))
    t = rtt.tt_from_full(X)
    for e in (1e-2, 1e-6, 1e-10):
        r = rtt.tt_round(t, e)
        out[f"round_{e:g}_full"] = r.full()
        out[f"round_{e:g}_ranks"] = np.array(r.ranks)
    out["round_X"] = X
    A = rtt.TtMatrix([rng.standard_normal((1, 4, 4, 3)), rng.standard_normal((3, 5, 5, 2)),
                      rng.standard_normal((2, 6, 6, 1))])
    x = rtt.TtTensor.random((4, 5, 6), (2, 3), rng)
    y = rtt.tt_matvec(A, x)
    for k in range(3):
        out[f"mv_A{k}"] = A.cores[k]
        out[f"mv_x{k}"] = x.cores[k]
    out["mv_y_full"] = y.full()
    yr = rtt.tt_round(y, 1e-8)
    out["mv_round_full"] = yr.full()
    out["mv_round_ranks"] = np.array(yr.ranks)
    out["mv_norm"] = np.array(rtt.tt_norm(y))
    # maxvol
    M = rng.standard_normal((200, 8))
    out["maxvol_M"] = M
    out["maxvol_sel"] = rtt.maxvol(M)
    v = np.array([10.0, 0.0])
    Md = np.vstack([v, v, [0.0, 10.0], [0.1, 0.2], [0.3, 0.1]])
    out["maxvol_dup_sel"] = rtt.maxvol(Md)
    # cross on a two-term function, fixed seed
    n = (16, 12, 10)
    grid = np.indices(n).reshape(3, -1).T

    def f(idx):
        return (np.sin(idx[:, 0] + 1.0) * np.cos(0.3 * idx[:, 1]) * (idx[:, 2] + 1.0)
                + np.exp(-0.1 * idx[:, 0]) * (idx[:, 1] + 0.5) * np.cos(0.2 * idx[:, 2]))

    res = rtt.tt_cross(rtt.CrossOracle(f, n), 1e-10, rng=np.random.default_rng(7))
    out["cross_full"] = res.tensor.full()
    out["cross_ranks"] = np.array(res.ranks)
    out["cross_ref"] = f(grid).reshape(n)
    out["cross_nevals"] = np.array(res.n_evals)
    out["cross_err"] = np.array(res.holdout_error)
    # amen on an 8^3 Laplacian
    nn = 8
    L = (2 * np.eye(nn) - np.eye(nn, k=1) - np.eye(nn, k=-1)) * (nn + 1) ** 2
    I = np.eye(nn)
    Aop = rtt.tt_round(rtt.tt_add(rtt.tt_add(rtt.TtMatrix.rank_one([L, I, I]), rtt.TtMatrix.rank_one([I, L, I])),
                                  rtt.TtMatrix.rank_one([I, I, L])), 1e-14)
    fr = rtt.tt_round(rtt.TtTensor.random((nn, nn, nn), (2, 2), np.random.default_rng(31)), 1e-14)
    sol = rtt.amen_solve(Aop, fr, 1e-10)
    for k in range(3):
        out[f"amen_A{k}"] = Aop.cores[k]
        out[f"amen_f{k}"] = fr.cores[k]
    out["amen_u_full"] = sol.solution.full()
    out["amen_res"] = np.array(sol.residual)
    out["amen_ranks"] = np.array(sol.solution.ranks)
    sol2 = rtt.amen_solve(Aop, fr, 1e-10, rtt.AmenOptions(direct_solve_max=16))
    out["amen_cg_u_full"] = sol2.solution.full()
    save("tensor_train.npz", **out)


def assembly():
    out = {}
    for name, deg in (("ring", 2), ("lshape", 1), ("hyperboloid", 2), ("quarter_torus", 2)):
        patch = rgeo.make_geometry(name)
        bases = tuple(rdrv.solution_basis(patch.bases[d], deg, 4) for d in range(3))
        disc = rasm.build_quadrature(bases)
        rng = np.random.default_rng(400)
        K, info = rasm.assemble_stiffness(patch, disc, 1e-11, rng=rng)
        f, finfo = rasm.assemble_load(patch, disc, rdrv.SOURCES["sin_pi_xyz"], 1e-11, rng=rng)
        out[f"{name}_K"] = K.full()
        out[f"{name}_Kranks"] = np.array(K.ranks)
        out[f"{name}_f"] = f.full()
        out[f"{name}_franks"] = np.array(f.ranks)
        for d in range(3):
            out[f"{name}_knots{d}"] = bases[d].knot_vector.knots
    save("assembly.npz", **out)


def solves():
    out = {}
    ring_bc = rasm.BoundarySpec({(1, 0): rasm.FaceCondition("dirichlet", 1.0),
                                 (1, 1): rasm.FaceCondition("dirichlet", 2.0)})
    cases = [
        ("cube_p2_e8", dict(geometry="unit_cube", degree=2, elements=8, source="manufactured_sines",
                            analytic="cube_sines")),
        ("ring_p2_e8", dict(geometry="ring", degree=2, elements=8, source="zero", analytic="ring_radial",
                            bc=ring_bc)),
        ("lshape_p1_e8", dict(geometry="lshape", degree=1, elements=8, source="sin_pi_xy",
                              analytic="lshape_exact")),
        ("torus_p2_e4", dict(geometry="quarter_torus", degree=2, elements=4, source="sin_pi_xyz")),
        ("ohemi_p2_e4", dict(geometry="opened_hemisphere", degree=2, elements=4, source="one")),
    ]
    for tag, kw in cases:
        rep = rdrv.solve_poisson(rdrv.SolveConfig(seed=0, **kw))
        out[f"{tag}_u"] = rep.u.full()
        out[f"{tag}_ranks_K"] = np.array(rep.ranks_K)
        out[f"{tag}_ranks_f"] = np.array(rep.ranks_f)
        out[f"{tag}_ranks_u"] = np.array(rep.ranks_u)
        out[f"{tag}_l2"] = np.array(np.nan if rep.l2_error is None else rep.l2_error)
        out[f"{tag}_residual"] = np.array(rep.residual)
        out[f"{tag}_sweeps"] = np.array(rep.sweeps)
    save("solves.npz", **out)


if __name__ == "__main__":
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    splines()
    geometry()
    tensor_train()
    assembly()
    solves()
