"""End-to-end TT-IGA solves on one B200 (reference ``pkg/src/ttiga/driver.py``).

``solve_poisson`` runs geometry -> discretization -> TT assembly -> Dirichlet
elimination -> AMEn -> metrics with every numerical step on the device. The
error integral (reference l2_error: int|u-u*| / int|u*| with det J) is one
fused kernel over the whole tensor quadrature grid.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import math
import os
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import linalg as L
from ._lib import call, device, ptr
from .assembly import (BoundarySpec, Discretization, FaceCondition, apply_dirichlet, assemble_load, assemble_stiffness,
                       build_quadrature)
from .geometry import SOURCE_IDS, GeometryPatch, make_geometry
from .pointfn import PointFn, builtin_sources, on_device
from .splines import Basis1D, KnotVector, basis_windows, eval_basis
from .tensor_train import AmenOptions, TtMatrix, TtTensor, amen_solve, tt_add, tt_round

__all__ = ["DriverError", "OracleRefusedError", "FullGridResult", "full_grid_reference", "FULL_GRID_DOF_GUARD",
           "SolveConfig", "SolutionReport", "SOURCES", "ANALYTIC", "solve_poisson", "l2_error",
           "compression_ratio", "evaluate_field", "solution_basis", "fit_slope", "field_on_grid"]


class DriverError(ValueError):
    """Invalid solve configuration (reference driver.py:69)."""


class OracleRefusedError(RuntimeError):
    """Full-grid reference refused: problem exceeds the dof guard (reference driver.py:73)."""


FULL_GRID_DOF_GUARD = 1_000_000


# name -> source term f(x): the reference's numpy lambdas (driver.py:80-98) as PointFn objects that the
# load kernel evaluates in-kernel by id (pointfn.py); SOURCES["one"](numpy points) works as in the reference
SOURCES = builtin_sources(SOURCE_IDS)


def _t_sines(x):
    return torch.sin(math.pi * x[:, 0]) * torch.sin(math.pi * x[:, 1]) * torch.sin(math.pi * x[:, 2])


def _np_sines(x):
    return np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1]) * np.sin(np.pi * x[:, 2])


# analytic solutions (reference driver.py:101-149): factories (cfg, patch) -> u(points), here PointFn
# objects carrying the l1err_kernel id and parameters (exact_fn in iga.cu) and the numpy/torch versions
def _an_lshape(cfg, patch):
    return PointFn(lambda x: np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1]) / (2.0 * np.pi ** 2),
                   lambda x: torch.sin(math.pi * x[:, 0]) * torch.sin(math.pi * x[:, 1]) / (2.0 * math.pi ** 2),
                   name="lshape_exact", analytic_id=0, params=(0.0, 0.0, 1.0, 1.0))


def _an_cube(cfg, patch):
    return PointFn(_np_sines, _t_sines, name="cube_sines", analytic_id=1, params=(0.0, 0.0, 1.0, 1.0))


def _an_exp(cfg, patch):
    return PointFn(lambda x: np.exp(x.sum(1)) * _np_sines(x), lambda x: torch.exp(x.sum(1)) * _t_sines(x),
                   name="exp_sines", analytic_id=3, params=(0.0, 0.0, 1.0, 1.0))


def _an_ring(cfg, patch):
    """Radial harmonic between the cylinder faces (reference driver.py:121-140)."""
    prm = patch.metadata.get("params", {})
    ri, ro = prm.get("r_in", 0.5), prm.get("r_out", 1.0)
    ci, co = cfg.bc.condition(1, 0), cfg.bc.condition(1, 1)
    if ci.kind != "dirichlet" or co.kind != "dirichlet":
        raise DriverError("ring_radial needs Dirichlet data on both radial faces")
    if callable(ci.value) or callable(co.value):
        raise DriverError("ring_radial needs constant radial face values")
    ui, uo = float(ci.value or 0.0), float(co.value or 0.0)

    def u(x):
        r = torch.hypot(x[:, 0], x[:, 1])
        return (ui * torch.log(ro / r) + uo * torch.log(r / ri)) / math.log(ro / ri)

    def u_np(x):
        r = np.hypot(x[:, 0], x[:, 1])
        return (ui * np.log(ro / r) + uo * np.log(r / ri)) / np.log(ro / ri)

    return PointFn(u_np, u, name="ring_radial", analytic_id=2, params=(ui, uo, ri, ro))


ANALYTIC = {"lshape_exact": _an_lshape, "cube_sines": _an_cube, "ring_radial": _an_ring, "exp_sines": _an_exp}


@dataclass
class SolveConfig:
    """Reference SolveConfig (driver.py:153-201) + BASELINE extensions.

    ``n_basis`` (extension): exact basis count per direction on open uniform
    knots instead of the bisection ladder; ``bc_from_analytic`` (extension):
    the geometry's default Dirichlet faces take the analytic solution as data.
    """

    geometry: str
    geometry_params: dict = field(default_factory=dict)
    degree: object = 2
    elements: object = 4
    eps_cross: float = 1e-10
    eps_solve: float = 1e-8
    eps_round: float = 1e-10
    n_gauss: object = None
    rank_cap: int = 64
    bc: BoundarySpec | None = None
    source: str = "zero"
    analytic: str | None = None
    seed: int = 0
    solver: dict = field(default_factory=dict)
    n_basis: object = None
    bc_from_analytic: bool = False

    def __post_init__(self):
        for name in ("eps_cross", "eps_solve", "eps_round"):
            v = getattr(self, name)
            if not 0.0 < v < 1.0:
                raise DriverError(f"{name} must lie in (0, 1), got {v}")
        tri = lambda v: tuple(int(x) for x in (v if not np.isscalar(v) else (v,) * 3))
        self.degree = tri(self.degree)
        self.elements = tri(self.elements)
        if self.n_basis is not None:
            self.n_basis = tri(self.n_basis)
        if any(p < 1 for p in self.degree):
            raise DriverError("degrees must be at least 1")
        if any(e < 1 for e in self.elements):
            raise DriverError("need at least one element per direction")
        if self.source not in SOURCE_IDS:
            raise DriverError(f"unknown source {self.source!r}")
        if self.analytic is not None and self.analytic not in ANALYTIC:
            raise DriverError(f"unknown analytic solution {self.analytic!r}")

    def resolve_bc(self, patch: GeometryPatch) -> "SolveConfig":
        if self.bc is None:
            if self.bc_from_analytic:
                if self.analytic is None:
                    raise DriverError("bc_from_analytic needs an analytic solution")
                fn = ANALYTIC[self.analytic](self, patch)
                self.bc = BoundarySpec({(int(a), int(s)): FaceCondition("dirichlet", fn)
                                        for a, s in patch.metadata.get("default_dirichlet", [])},
                                       allow_adjacent_nonzero=True)
            else:
                self.bc = BoundarySpec({(int(a), int(s)): FaceCondition("dirichlet", 0.0)
                                        for a, s in patch.metadata.get("default_dirichlet", [])})
        return self


@dataclass
class SolutionReport:
    """Reference SolutionReport (driver.py:204-253)."""

    config: SolveConfig
    u: TtTensor
    dofs: int
    mode_sizes: tuple
    l2_error: float | None
    residual: float
    solver_converged: bool
    cross_converged: bool
    ranks_K: tuple
    ranks_f: tuple
    ranks_u: tuple
    compression_K: float
    compression_f: float
    compression_u: float
    timings: dict
    sweeps: int

    def metrics_dict(self):
        return {"geometry": self.config.geometry, "degree": list(self.config.degree),
                "elements": list(self.config.elements), "seed": self.config.seed, "dofs": self.dofs,
                "mode_sizes": list(self.mode_sizes), "l2_error": self.l2_error, "residual": self.residual,
                "solver_converged": self.solver_converged, "cross_converged": self.cross_converged,
                "ranks_K": list(self.ranks_K), "ranks_f": list(self.ranks_f), "ranks_u": list(self.ranks_u),
                "compression_K": self.compression_K, "compression_f": self.compression_f,
                "compression_u": self.compression_u, "sweeps": self.sweeps}

    def to_json(self):
        doc = dict(self.metrics_dict())
        doc.update(timings=self.timings, source=self.config.source, analytic=self.config.analytic,
                   eps_cross=self.config.eps_cross, eps_solve=self.config.eps_solve, eps_round=self.config.eps_round)
        return json.dumps(doc, indent=2)


def solution_basis(geom_basis: Basis1D, degree: int, elements: int) -> Basis1D:
    """Bisection refinement of the geometry breakpoints (reference driver.py:259-288)."""
    kv = geom_basis.knot_vector
    uniq, counts = np.unique(kv.knots, return_counts=True)
    levels = 0
    while (uniq.size - 1) * 2 ** levels < elements:
        levels += 1
    breaks = list(uniq)
    for _ in range(levels):
        breaks = sorted(breaks + [0.5 * (a + b) for a, b in zip(breaks[:-1], breaks[1:])])
    mult = {float(v): max(1, degree - (kv.degree - int(c))) for v, c in zip(uniq[1:-1], counts[1:-1])}
    knots = [0.0] * (degree + 1)
    for b in breaks[1:-1]:
        knots.extend([b] * mult.get(float(b), 1))
    knots.extend([1.0] * (degree + 1))
    return Basis1D(KnotVector(np.asarray(knots), degree))


def solution_basis_exact(geom_basis: Basis1D, degree: int, n_basis: int) -> Basis1D:
    """EXTENSION: open uniform knots with exactly n_basis functions."""
    kv = geom_basis.knot_vector
    _, counts = np.unique(kv.knots, return_counts=True)
    if any(max(1, degree - (kv.degree - int(c))) > 1 for c in counts[1:-1]):
        raise DriverError("exact-count solution space cannot keep a reduced-continuity geometry line")
    return Basis1D(KnotVector.open_uniform(degree, n_basis - degree))


def _spawn_rngs(seed, n):
    return [np.random.default_rng(s) for s in np.random.SeedSequence(seed).spawn(n)]


def compression_ratio(t) -> float:
    """Dense element count over TT parameters (reference driver.py:360-368)."""
    if isinstance(t, TtMatrix):
        full = int(np.prod(t.row_sizes, dtype=np.int64)) * int(np.prod(t.col_sizes, dtype=np.int64))
    else:
        full = int(np.prod(t.mode_sizes, dtype=np.int64))
    return full / t.n_params


def evaluate_field(disc: Discretization, u: TtTensor, xi) -> float:
    """Field value at one parametric point (reference driver.py:371-379)."""
    v = torch.ones(1, 1, dtype=torch.float64, device=device())
    for d in range(3):
        ev = eval_basis(disc.solution_bases[d], float(xi[d]))
        sl = slice(ev.first_index, ev.first_index + ev.values.size)
        w = torch.as_tensor(ev.values, device=device())
        M = torch.einsum("a,ras->rs", w, u.cores[d][:, sl, :])
        v = v @ M
    return float(v[0, 0].item())


def _field_tables(disc: Discretization, u: TtTensor):
    out = []
    for d in range(3):
        G = u.cores[d]
        r, n, s = G.shape
        tab = disc.tables[d]
        nq = tab.points.size
        T = L.empty(r, nq, s)
        call("ttb_field_table", r, n, s, ptr(G), nq, ptr(tab.starts), ptr(tab.vals), disc.solution_bases[d].degree,
             ptr(T))
        out.append(T)
    return out


def l2_error(u: TtTensor, analytic, patch: GeometryPatch, disc: Discretization) -> float:
    """Reference l2_error (driver.py:388-422) as one device pass over the quadrature grid.

    ``analytic``: the PointFn an ANALYTIC factory returns (evaluated inside l1err_kernel by id) or any
    reference-style numpy callable of physical points (tabulated once at the quadrature points through
    the host bridge, pointfn.on_device)."""
    from .geometry import GridEvaluator
    ev = GridEvaluator(patch, disc.quad_axes())
    U0, U1, U2 = _field_tables(disc, u)
    nq = disc.quad_shape
    (f0, V0, D0), (f1, V1, D1), (f2, V2, D2) = ev.win
    p = patch.degrees
    n = ev.cw.shape[:3]
    if isinstance(analytic, PointFn) and analytic.analytic_id is not None:
        exact_id = analytic.analytic_id
        prm_t = torch.as_tensor(np.asarray(analytic.params, dtype=np.float64), device=device())
    elif callable(analytic):
        exact_id = -1                                   # table of exact values at every quadrature point
        idx = torch.stack(torch.meshgrid(*[torch.arange(k, device=device()) for k in nq], indexing="ij"),
                          -1).reshape(-1, 3)
        prm_t = on_device(analytic)(ev.points(idx)).to(torch.float64).contiguous()
    else:
        raise DriverError("analytic must be a callable of physical points")
    part = L.empty(2 * nq[0] * nq[1])
    out = L.empty(2)
    w = [t.w_dev for t in disc.tables]
    call("ttb_l1_error", ptr(f0), ptr(f1), ptr(f2), ptr(V0), ptr(V1), ptr(V2), ptr(D0), ptr(D1), ptr(D2), p[0], p[1],
         p[2], n[0], n[1], n[2], ptr(ev.cw), nq[0], nq[1], nq[2], ptr(U0.contiguous()), U0.shape[2], ptr(U1),
         U1.shape[2], ptr(U2.contiguous()), ptr(w[0]), ptr(w[1]), ptr(w[2]), int(exact_id), ptr(prm_t), ptr(part),
         ptr(out))
    num, den = out.cpu().numpy()
    if den == 0.0:
        raise DriverError("analytic solution has zero norm on this domain")
    return float(num / den)


def fit_slope(points_per_edge, errors) -> float:
    x = np.log(np.asarray(points_per_edge, dtype=float))
    y = np.log(np.asarray(errors, dtype=float))
    return float(-np.polyfit(x, y, 1)[0])


def field_on_grid(disc: Discretization, u: TtTensor, axes):
    """Field values on a tensor grid of parameters (reference driver.py:432-440)."""
    from .splines import tabulate
    tabs = [torch.as_tensor(tabulate(disc.solution_bases[d], np.asarray(ax, float))[0], device=device())
            for d, ax in enumerate(axes)]
    V = [torch.einsum("rns,qn->rqs", u.cores[d], tabs[d]) for d in range(3)]
    T = torch.einsum("qb,bpc->qpc", V[0][0], V[1])
    return torch.einsum("qpc,cm->qpm", T, V[2][:, :, 0]).cpu().numpy()


def _extend_interior(u_int: TtTensor, slices, sizes) -> TtTensor:
    cores = []
    for G, s, n in zip(u_int.cores, slices, sizes):
        full = L.zeros(G.shape[0], n, G.shape[2])
        full[:, s, :] = G
        cores.append(full)
    return TtTensor(cores)


def discretize(cfg: SolveConfig, patch: GeometryPatch) -> Discretization:
    if cfg.n_basis is not None:
        bases = tuple(solution_basis_exact(patch.bases[d], cfg.degree[d], cfg.n_basis[d]) for d in range(3))
    else:
        bases = tuple(solution_basis(patch.bases[d], cfg.degree[d], cfg.elements[d]) for d in range(3))
    return build_quadrature(bases, cfg.n_gauss)


def _sync():
    torch.cuda.synchronize()


def geometry_params(cfg: SolveConfig) -> dict:
    """cfg.geometry_params, plus -- for the seeded random cube on an exact-count (n_basis) open uniform
    solution space -- the solve's Gauss grid as its det J > 0 admissibility grid (BASELINE configs[3]:
    "rejected until det J > 0 at all Gauss points"; oracle/iga.py geometry_params)."""
    prm = dict(cfg.geometry_params)
    if cfg.geometry == "random_cube" and cfg.n_basis is not None and "check_gauss" not in prm:
        ng = cfg.n_gauss
        q = [d + 1 for d in cfg.degree] if ng is None else ([int(ng)] * 3 if np.isscalar(ng) else [int(g) for g in ng])
        prm["check_gauss"] = [[n - d, g] for n, d, g in zip(cfg.n_basis, cfg.degree, q)]
    return prm


def solve_poisson(cfg: SolveConfig, want_error: bool = True) -> SolutionReport:
    """Full TT pipeline for one configuration (reference driver.py:455-532; no operator cache)."""
    timings = {}
    _sync()
    t0 = time.perf_counter()
    patch = make_geometry(cfg.geometry, geometry_params(cfg))
    cfg.resolve_bc(patch)
    disc = discretize(cfg, patch)
    _sync()
    timings["t_setup_s"] = time.perf_counter() - t0
    rng_K, rng_f = _spawn_rngs(cfg.seed, 2)
    t0 = time.perf_counter()
    K, k_info = assemble_stiffness(patch, disc, cfg.eps_round, rank_cap=cfg.rank_cap, rng=rng_K)
    _sync()
    timings["t_assemble_K_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    f, f_info = assemble_load(patch, disc, cfg.source, cfg.eps_cross, rank_cap=cfg.rank_cap, rng=rng_f)
    _sync()
    timings["t_assemble_f_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    system = apply_dirichlet(K, f, cfg.bc, disc, patch, eps=cfg.eps_round)
    _sync()
    timings["t_bc_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    opts = AmenOptions(**cfg.solver) if cfg.solver else AmenOptions()
    result = amen_solve(system.K, system.f, cfg.eps_solve, opts)
    _sync()
    timings["t_solve_s"] = time.perf_counter() - t0
    u_full = tt_round(tt_add(_extend_interior(result.solution, system.interior, disc.mode_sizes), system.lift), 1e-14)
    err = None
    t0 = time.perf_counter()
    if cfg.analytic is not None and want_error:
        err = l2_error(u_full, ANALYTIC[cfg.analytic](cfg, patch), patch, disc)
    _sync()
    timings["t_error_s"] = time.perf_counter() - t0
    cross_ok = all(k_info["cross_converged"].values()) and f_info["cross_converged"]
    rep = SolutionReport(config=cfg, u=u_full, dofs=disc.n_dofs, mode_sizes=disc.mode_sizes, l2_error=err,
                         residual=result.residual, solver_converged=result.converged, cross_converged=bool(cross_ok),
                         ranks_K=K.ranks, ranks_f=f.ranks, ranks_u=u_full.ranks,
                         compression_K=compression_ratio(K), compression_f=compression_ratio(f),
                         compression_u=compression_ratio(u_full), timings=timings, sweeps=result.sweeps)
    rep.K, rep.f, rep.system, rep.disc, rep.patch = K, f, system, disc, patch
    rep.solution_interior = result.solution     # the AMEn solution of the eliminated system (tests)
    return rep


# ---------------------------------------------------------------------------
# classical full-grid anchor (reference driver.py:535-703)

@dataclass
class FullGridResult:
    """Reference FullGridResult (driver.py:535-544): K as a scipy CSR matrix and f, u as numpy arrays over
    the full coefficient space (boundary coefficients included), like the reference's."""

    K: object
    f: np.ndarray
    u: np.ndarray
    mode_sizes: tuple
    l2_error: float | None = None


def _stencil_to_csr(Kst, sizes, p):
    """Stencil storage (n_dofs, prod(2p_d+1)) -> scipy CSR (host; only for the API's return value)."""
    import scipy.sparse as sp
    K = Kst.cpu().numpy()
    n0, n1, n2 = sizes
    I = np.arange(n0 * n1 * n2).reshape(n0, n1, n2)
    rows, cols, vals = [], [], []
    w1, w2 = 2 * p[1] + 1, 2 * p[2] + 1
    for o0 in range(-p[0], p[0] + 1):
        for o1 in range(-p[1], p[1] + 1):
            for o2 in range(-p[2], p[2] + 1):
                sl_i = tuple(slice(max(0, -o), n - max(0, o)) for o, n in zip((o0, o1, o2), sizes))
                sl_j = tuple(slice(max(0, o), n - max(0, -o)) for o, n in zip((o0, o1, o2), sizes))
                ri, cj = I[sl_i].ravel(), I[sl_j].ravel()
                v = K[ri, ((o0 + p[0]) * w1 + (o1 + p[1])) * w2 + (o2 + p[2])]
                keep = v != 0.0
                rows.append(ri[keep])
                cols.append(cj[keep])
                vals.append(v[keep])
    nd = n0 * n1 * n2
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(nd, nd)).tocsr()


def full_grid_reference(cfg: SolveConfig) -> FullGridResult:
    """Classical IGA assembly and solve with the same quadrature (reference driver.py:561-703), on the device:
    Gauss-point metric and load from the geometry kernel, element-by-element stiffness/load into a stencil
    array (ttb_fullgrid_assemble), Dirichlet lift from the same Greville face interpolation as the TT path,
    and a Jacobi-preconditioned CG on the interior (ttb_stencil_spmv) to a relative residual of 1e-14 (the
    reference: scipy spsolve up to 50k interior dofs, CG at rtol 1e-12 above). Refuses above the dof guard,
    as the reference does: this path is the one the TT pipeline exists to avoid."""
    from .assembly import _face_coefficients
    from .geometry import GridEvaluator
    from .tensor_train import tt_from_full
    patch = make_geometry(cfg.geometry, cfg.geometry_params)
    cfg.resolve_bc(patch)
    bases = tuple(solution_basis(patch.bases[d], cfg.degree[d], cfg.elements[d]) for d in range(3))
    disc = build_quadrature(bases, cfg.n_gauss)
    sizes = disc.mode_sizes
    n_dofs = disc.n_dofs
    if n_dofs > FULL_GRID_DOF_GUARD:
        raise OracleRefusedError(f"full-grid oracle refused: {n_dofs} dofs exceed the {FULL_GRID_DOF_GUARD} guard")
    dev = device()
    nq = disc.quad_shape
    g = disc.n_gauss
    ne = tuple(nq[d] // g[d] for d in range(3))
    p = tuple(b.degree for b in bases)
    ev = GridEvaluator(patch, disc.quad_axes())
    idx = torch.stack(torch.meshgrid(*[torch.arange(k, device=dev) for k in nq], indexing="ij"), -1).reshape(-1, 3)
    rec = ev.records(idx)                                        # raises on a singular map, as the reference
    w = [t.w_dev for t in disc.tables]
    wq = (w[0][:, None, None] * w[1][None, :, None] * w[2][None, None, :]).reshape(-1)
    Rw = (rec[:, 13:] * wq[:, None]).contiguous()
    Fw = (ev.source_times_det(idx, cfg.source) * wq).contiguous()
    S = (2 * p[0] + 1) * (2 * p[1] + 1) * (2 * p[2] + 1)
    Kst = L.zeros(n_dofs, S)
    fvec = L.zeros(n_dofs)
    i3 = lambda v: (C.c_int * 3)(*[int(x) for x in v])          # noqa: E731
    tb = disc.tables
    call("ttb_fullgrid_assemble", i3(ne), i3(g), i3(p), i3(sizes), ptr(tb[0].starts), ptr(tb[1].starts),
         ptr(tb[2].starts), ptr(tb[0].vals), ptr(tb[1].vals), ptr(tb[2].vals), ptr(tb[0].ders), ptr(tb[1].ders),
         ptr(tb[2].ders), ptr(Rw), ptr(Fw), ptr(Kst), ptr(fvec))
    # Dirichlet elimination mirroring the TT path (reference _dense_lift, driver.py:547-558)
    lift = L.zeros(*sizes)
    for axis, side in cfg.bc.dirichlet_faces():
        fc = cfg.bc.condition(axis, side)
        if fc.is_zero():
            continue
        sl = [slice(None)] * 3
        sl[axis] = 0 if side == 0 else sizes[axis] - 1
        lift[tuple(sl)] = _face_coefficients(patch, disc, cfg.bc, axis, side)
    lift = lift.reshape(-1)
    mask_b = torch.zeros(sizes, dtype=torch.bool, device=dev)
    mask_b[tuple(cfg.bc.interior_slices(sizes))] = True
    mask = mask_b.reshape(-1).to(torch.uint8).contiguous()

    def spmv(x, m=None):
        y = L.empty(n_dofs)
        call("ttb_stencil_spmv", sizes[0], sizes[1], sizes[2], p[0], p[1], p[2], ptr(Kst), ptr(x), ptr(m), ptr(y))
        return y

    mf = mask.to(torch.float64)
    b = (fvec - spmv(lift)) * mf
    diag = Kst[:, S // 2]
    dinv = torch.where(mask.bool(), 1.0 / torch.where(diag != 0, diag, torch.ones_like(diag)), torch.zeros_like(diag))
    x = L.zeros(n_dofs)
    r = b.clone()
    z = dinv * r
    pv = z.clone()
    rz = torch.dot(r, z)
    bnorm = float(torch.linalg.vector_norm(b).item())
    converged = bnorm == 0.0
    it = 0
    while not converged and it < 20_000:
        Ap = spmv(pv, mask)
        alpha = rz / torch.dot(pv, Ap)
        x += alpha * pv
        r -= alpha * Ap
        it += 1
        if it % 10 == 0 and float(torch.linalg.vector_norm(r).item()) <= 1e-14 * bnorm:
            converged = True
            break
        z = dinv * r
        rz_new = torch.dot(r, z)
        pv = z + (rz_new / rz) * pv
        rz = rz_new
    if not converged:
        raise RuntimeError("full-grid CG failed to converge")
    u = lift + x
    err = None
    if cfg.analytic is not None:
        err = l2_error(tt_from_full(u.reshape(sizes), 1e-14), ANALYTIC[cfg.analytic](cfg, patch), patch, disc)
    return FullGridResult(_stencil_to_csr(Kst, sizes, p), fvec.cpu().numpy(), u.cpu().numpy(), sizes, err)
