"""End-to-end TT-IGA solves on one B200 (reference ``pkg/src/ttiga/driver.py``).

``solve_poisson`` runs geometry -> discretization -> TT assembly -> Dirichlet
elimination -> AMEn -> metrics with every numerical step on the device. The
error integral (reference l2_error: int|u-u*| / int|u*| with det J) is one
fused kernel over the whole tensor quadrature grid.
"""

from __future__ import annotations

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
from .splines import Basis1D, KnotVector, basis_windows, eval_basis
from .tensor_train import AmenOptions, TtMatrix, TtTensor, amen_solve, tt_add, tt_round

__all__ = ["DriverError", "SolveConfig", "SolutionReport", "SOURCES", "ANALYTIC", "solve_poisson", "l2_error",
           "compression_ratio", "evaluate_field", "solution_basis", "fit_slope", "field_on_grid"]


class DriverError(ValueError):
    """Invalid solve configuration (reference driver.py:69)."""


SOURCES = tuple(SOURCE_IDS)


def _t_sines(x):
    return torch.sin(math.pi * x[:, 0]) * torch.sin(math.pi * x[:, 1]) * torch.sin(math.pi * x[:, 2])


def _an_lshape(cfg, patch):
    return (0, (0.0, 0.0, 1.0, 1.0),
            lambda x: torch.sin(math.pi * x[:, 0]) * torch.sin(math.pi * x[:, 1]) / (2.0 * math.pi ** 2))


def _an_cube(cfg, patch):
    return 1, (0.0, 0.0, 1.0, 1.0), _t_sines


def _an_exp(cfg, patch):
    return 3, (0.0, 0.0, 1.0, 1.0), lambda x: torch.exp(x.sum(1)) * _t_sines(x)


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

    return 2, (ui, uo, ri, ro), u


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
                fn = ANALYTIC[self.analytic](self, patch)[2]
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

    ``analytic`` is the (id, params, fn) triple returned by an ANALYTIC factory.
    """
    exact_id, prm, _ = analytic
    from .geometry import GridEvaluator
    ev = GridEvaluator(patch, disc.quad_axes())
    U0, U1, U2 = _field_tables(disc, u)
    nq = disc.quad_shape
    (f0, V0, D0), (f1, V1, D1), (f2, V2, D2) = ev.win
    p = patch.degrees
    n = ev.cw.shape[:3]
    prm_t = torch.as_tensor(np.asarray(prm, dtype=np.float64), device=device())
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
    return rep
