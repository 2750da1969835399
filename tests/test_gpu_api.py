"""Reference API semantics on the device path: error types, empty/degenerate inputs, the
container format, boundary bookkeeping (mirrors the reference tests' edge cases)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    from paper_2509_13224_b200 import assembly, driver, geometry, splines, tensor_train
    return type("NS", (), dict(tt=tensor_train, asm=assembly, drv=driver, geo=geometry, spl=splines))


def test_shape_errors(M):
    rng = np.random.default_rng(5)
    a = M.tt.TtTensor.random((4, 4, 4), (2, 2), rng)
    b = M.tt.TtTensor.random((4, 5, 4), (2, 2), rng)
    with pytest.raises(M.tt.TtShapeError):
        M.tt.tt_add(a, b)
    with pytest.raises(M.tt.TtShapeError):
        M.tt.tt_matvec(M.tt.TtMatrix.identity((4, 4, 5)), a)
    with pytest.raises(M.tt.TtShapeError):
        M.tt.TtTensor([torch.zeros(2, 3, 1, dtype=torch.float64)])  # boundary rank != 1


def test_zero_tensor_round_and_solve(M):
    z = M.tt.tt_round(M.tt.TtTensor.zeros((4, 5, 6)), 1e-8)
    assert z.ranks == (1, 1, 1, 1) and np.all(z.full() == 0.0)
    res = M.tt.amen_solve(M.tt.TtMatrix.identity((4, 4, 4)), M.tt.TtTensor.zeros((4, 4, 4)), 1e-8)
    assert res.converged and np.all(res.solution.full() == 0.0)
    with pytest.raises(ValueError):
        M.tt.tt_round(z, 0.0)


def test_identity_system_and_nonconvergence_flag(M):
    rng = np.random.default_rng(30)
    f = M.tt.TtTensor.random((6, 7, 8), (3, 2), rng)
    res = M.tt.amen_solve(M.tt.TtMatrix.identity((6, 7, 8)), f, 1e-12)
    assert res.converged and res.residual <= 1e-14
    n = 16
    L = (2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)) * (n + 1) ** 2
    I = np.eye(n)
    R1 = M.tt.TtMatrix.rank_one
    A = M.tt.tt_round(M.tt.tt_add(M.tt.tt_add(R1([L, I, I]), R1([I, L, I])), R1([I, I, L])), 1e-14)
    f = M.tt.tt_round(M.tt.TtTensor.random((n, n, n), (3, 3), np.random.default_rng(34)), 1e-14)
    r = M.tt.amen_solve(A, f, 1e-30, M.tt.AmenOptions(max_sweeps=1))
    assert not r.converged and r.residual > 0


def test_maxvol_validation(M):
    with pytest.raises(ValueError):
        M.tt.maxvol(torch.eye(3, dtype=torch.float64, device="cuda"), tol=0.5)
    assert list(M.tt.maxvol(torch.eye(3, dtype=torch.float64, device="cuda"))) == [0, 1, 2]


def test_cross_constant_and_noise(M):
    res = M.tt.tt_cross(M.tt.CrossOracle(lambda idx: torch.full((idx.shape[0],), 3.5, dtype=torch.float64,
                                                                   device="cuda"), (8, 8, 8), device=True),
                        1e-10, rng=np.random.default_rng(2))
    assert res.ranks == (1, 1, 1, 1) and np.abs(res.tensor.full() - 3.5).max() < 1e-12
    g = torch.Generator(device="cuda").manual_seed(5)
    noisy = M.tt.CrossOracle(lambda idx: 1e-16 * torch.randn(idx.shape[0], dtype=torch.float64, device="cuda",
                                                             generator=g), (12, 12, 12), device=True)
    res = M.tt.tt_cross(noisy, 1e-10, rng=np.random.default_rng(6), scale=1.0)
    assert res.ranks == (1, 1, 1, 1) and np.all(res.tensor.full() == 0.0) and res.converged


def test_container_round_trip(M, tmp_path):
    rng = np.random.default_rng(40)
    t = M.tt.TtTensor.random((5, 6, 7), (3, 4), rng)
    M.tt.save_tt(tmp_path / "t.tt", t)
    back = M.tt.load_tt(tmp_path / "t.tt")
    assert back.ranks == t.ranks and all(torch.equal(a, b) for a, b in zip(back.cores, t.cores))
    # a banded operator is written densified and reads back equal
    n, h = 9, 1
    cores = []
    for r0, r1 in ((1, 2), (2, 2), (2, 1)):
        G = rng.standard_normal((r0, n, n, r1))
        i, j = np.indices((n, n))
        G[:, np.abs(i - j) > h, :] = 0.0
        cores.append(G)
    Kb = M.tt.TtMatrix.banded_from_dense_cores(cores, h)
    M.tt.save_tt(tmp_path / "k.tt", Kb)
    Kd = M.tt.load_tt(tmp_path / "k.tt")
    assert np.array_equal(Kd.full(), Kb.full())
    info = M.tt.tt_info(Kb)
    assert info["kind"] == "operator" and info["full_entries"] == (9 ** 3) ** 2
    (tmp_path / "bad.tt").write_bytes(b"NOPE" + b"\x00" * 32)
    with pytest.raises(ValueError):
        M.tt.load_tt(tmp_path / "bad.tt")


def test_dirichlet_bookkeeping(M):
    patch = M.geo.make_geometry("unit_cube")
    basis = M.spl.Basis1D(M.spl.KnotVector.open_uniform(1, 4))
    disc = M.asm.build_quadrature((basis, basis, basis))
    K, _ = M.asm.assemble_stiffness(patch, disc, 1e-12, rng=np.random.default_rng(15))
    f, _ = M.asm.assemble_load(patch, disc, "one", 1e-12, rng=np.random.default_rng(16))
    bc = M.asm.BoundarySpec({(0, 0): M.asm.FaceCondition("dirichlet", 0.0),
                             (0, 1): M.asm.FaceCondition("dirichlet", 0.0)})
    sysm = M.asm.apply_dirichlet(K, f, bc, disc, patch)
    assert sysm.K.row_sizes == (3, 5, 5)
    with pytest.raises(M.asm.AssemblyError):
        M.asm.apply_dirichlet(K, f, M.asm.BoundarySpec({}), disc, patch)
    adj = M.asm.BoundarySpec({(0, 0): M.asm.FaceCondition("dirichlet", 1.0),
                              (1, 0): M.asm.FaceCondition("dirichlet", 2.0)})
    with pytest.raises(M.asm.AssemblyError):
        M.asm.apply_dirichlet(K, f, adj, disc, patch)


def test_trilinear_element_and_constants_in_kernel(M):
    cube = M.geo.make_geometry("unit_cube")
    basis = M.spl.Basis1D(M.spl.KnotVector.open_uniform(1, 1))
    disc = M.asm.build_quadrature((basis, basis, basis))
    K, _ = M.asm.assemble_stiffness(cube, disc, 1e-12, rng=np.random.default_rng(4))
    dense = K.full()
    nodes = [(i, j, k) for i in range(2) for j in range(2) for k in range(2)]
    pat = {0: 1.0 / 3.0, 1: 0.0, 2: -1.0 / 12.0, 3: -1.0 / 12.0}
    for a, na in enumerate(nodes):
        for b, nb in enumerate(nodes):
            assert abs(dense[a, b] - pat[sum(x != y for x, y in zip(na, nb))]) < 1e-12
    ring = M.geo.make_geometry("ring")
    bases = tuple(M.drv.solution_basis(ring.bases[d], 2, 4) for d in range(3))
    disc = M.asm.build_quadrature(bases)
    K, _ = M.asm.assemble_stiffness(ring, disc, 1e-11, rng=np.random.default_rng(8))
    ones = M.tt.TtTensor.ones(disc.mode_sizes)
    assert M.tt.tt_norm(M.tt.tt_matvec(K, ones)) <= 1e-9 * np.linalg.norm(K.full())
    Kd = K.full()
    assert np.linalg.norm(Kd - K.transpose().full()) <= 1e-10 * np.linalg.norm(Kd)


def test_spline_errors_and_singular_map(M):
    kv = M.spl.KnotVector(np.array([0, 0, 0, 1, 1, 1.0]), 2)
    with pytest.raises(M.spl.SplineError):
        M.spl.find_span(kv, 1.5)
    with pytest.raises(M.spl.SplineError):
        M.spl.KnotVector(np.array([0, 0, 1, 0.5, 1, 1.0]), 2)
    ev = M.spl.eval_basis(M.spl.Basis1D(kv), 0.5)
    assert np.allclose(ev.values, [0.25, 0.5, 0.25]) and np.allclose(ev.derivs, [-1.0, 0.0, 1.0])
    with pytest.raises(M.geo.GeometryError):
        M.geo.make_geometry("ring", {"r_in": 1.5, "r_out": 1.0})
    hemi = M.geo.make_geometry("closed_hemisphere")
    with pytest.raises(M.geo.SingularMapError):
        hemi.eval_metric(np.array([0.3, 1.0, 0.5]))  # pole face: det J = 0


def test_full_grid_reference_anchor():
    """The classical full-grid system (reference driver.py:561-703) on the device: the trilinear element
    stiffness pattern of the reference's own test, and TT solve == full-grid solve on the ring."""
    from paper_2509_13224_b200 import driver as D
    from paper_2509_13224_b200.assembly import BoundarySpec, FaceCondition
    cfg = D.SolveConfig(geometry="unit_cube", degree=1, elements=1, source="one", seed=0,
                        bc=BoundarySpec({(0, 0): FaceCondition("dirichlet", 0.0)}))
    ref = D.full_grid_reference(cfg)
    dense = ref.K.toarray()
    nodes = [(i, j, k) for i in range(2) for j in range(2) for k in range(2)]
    pattern = {0: 1 / 3, 1: 0.0, 2: -1 / 12, 3: -1 / 12}
    for a, na in enumerate(nodes):
        for b, nb in enumerate(nodes):
            assert abs(dense[a, b] - pattern[sum(x != y for x, y in zip(na, nb))]) < 1e-12
    kw = dict(geometry="ring", degree=2, elements=4, source="sin_pi_xyz", seed=0)
    rep = D.solve_poisson(D.SolveConfig(**kw))
    ref = D.full_grid_reference(D.SolveConfig(**kw))
    u = rep.u.full().ravel()
    diff = np.linalg.norm(u - ref.u) / np.linalg.norm(ref.u)
    K = rep.K.full().reshape(ref.K.shape)
    eK = np.linalg.norm(K - ref.K.toarray()) / np.linalg.norm(ref.K.toarray())
    ef = np.linalg.norm(rep.f.full().ravel() - ref.f) / np.linalg.norm(ref.f)
    print(f"full-grid anchor (ring, p=2, 4 el.): K {eK:.2e}, f {ef:.2e}, u {diff:.2e}")
    assert eK <= 1e-9 and ef <= 1e-9 and diff <= 10 * rep.config.eps_solve
    with pytest.raises(D.OracleRefusedError):
        D.full_grid_reference(D.SolveConfig(geometry="unit_cube", degree=1, elements=128, seed=0))
