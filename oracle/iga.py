"""Oracle: TT Galerkin assembly, Dirichlet elimination and the solve driver (TEST INFRASTRUCTURE ONLY).

Restates reference ``pkg/src/ttiga/assembly.py`` and ``pkg/src/ttiga/driver.py``
(quadrature, metric/load cross oracles, core contractions, TT summation with
rounding, boundary lift, elimination, AMEn solve, error metrics).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import tt as T
from .amen import AmenOpts, amen
from .bspline import Spline1D, basis_window, dense_tables, solution_space, solution_space_exact
from .cross import cross
from .patch import TensorGridEval, build_patch


class IgaFault(ValueError):
    """Mirror of reference AssemblyError / DriverError."""


@dataclass
class Quad:
    """Per-direction Gauss rule + active basis windows (reference _DirTables, assembly.py:56-64)."""

    x: np.ndarray
    w: np.ndarray
    first: np.ndarray
    V: np.ndarray
    D: np.ndarray


@dataclass
class Disc:
    """Reference Discretization (assembly.py:67-88)."""

    bases: tuple
    quads: tuple
    n_gauss: tuple

    @property
    def sizes(self):
        return tuple(b.n for b in self.bases)

    @property
    def qshape(self):
        return tuple(q.x.size for q in self.quads)

    def axes(self):
        return [q.x for q in self.quads]


def gauss_tables(bases, n_gauss=None) -> Disc:
    """Reference build_quadrature (assembly.py:91-135)."""
    bases = tuple(bases)
    if len(bases) != 3:
        raise IgaFault("need three bases")
    if n_gauss is None:
        g = [b.p + 1 for b in bases]
    elif np.isscalar(n_gauss):
        g = [int(n_gauss)] * 3
    else:
        g = [int(v) for v in n_gauss]
    quads = []
    for b, ng in zip(bases, g):
        if b.w is not None:
            raise IgaFault("solution bases must be polynomial")
        if ng < b.p + 1:
            raise IgaFault("too few Gauss points")
        xr, wr = np.polynomial.legendre.leggauss(ng)
        xs, ws = [], []
        for i in b.nonempty_spans():
            a, c = b.t[i], b.t[i + 1]
            xs.append(0.5 * (a + c) + 0.5 * (c - a) * xr)
            ws.append(0.5 * (c - a) * wr)
        x = np.concatenate(xs)
        first = np.empty(x.size, dtype=np.intp)
        V = np.empty((x.size, b.p + 1))
        D = np.empty((x.size, b.p + 1))
        for q, xv in enumerate(x):
            first[q], V[q], D[q] = basis_window(b, float(xv))
        quads.append(Quad(x, np.concatenate(ws), first, V, D))
    return Disc(bases, tuple(quads), tuple(g))


_CHUNK = 1 << 15


def _chunked(fn, idx):
    idx = np.asarray(idx, dtype=np.intp)
    if idx.shape[0] <= _CHUNK:
        return fn(idx)
    return np.concatenate([fn(idx[s: s + _CHUNK]) for s in range(0, idx.shape[0], _CHUNK)])


def metric_fn(ev: TensorGridEval, i, j):
    """Reference metric_oracle (assembly.py:153-160)."""
    return lambda idx: _chunked(lambda q: ev.det_metric(q)[1][:, i, j], idx)


def load_fn(ev: TensorGridEval, src):
    """Reference load_oracle (assembly.py:163-170): f(x(xi)) det J."""

    def one(q):
        J, x = ev.jac_points(q)
        return src(x) * np.linalg.det(J)

    return lambda idx: _chunked(one, idx)


def metric_rms(ev: TensorGridEval, rng, n_probe=512):
    """Reference metric_scale (assembly.py:173-182)."""
    idx = np.stack([rng.integers(0, n, size=n_probe) for n in ev.shape], 1)
    _, R = ev.det_metric(idx)
    return float(np.sqrt(np.mean(R ** 2)))


def op_core(G, q: Quad, dtest, dtrial):
    """(r, n, n, s) operator core from a quadrature-grid core (reference assembly.py:208-222)."""
    r, nq, s = G.shape
    n = int(q.first.max()) + q.V.shape[1]
    X = q.D if dtest else q.V
    Y = q.D if dtrial else q.V
    E = np.einsum("rqs,q,qa,qb->qabrs", G, q.w, X, Y, optimize=True)
    o = np.arange(X.shape[1])
    ia = (q.first[:, None] + o)[:, :, None]
    ib = (q.first[:, None] + o)[:, None, :]
    ia, ib = np.broadcast_arrays(ia, ib)
    M = np.zeros((n, n, r, s))
    np.add.at(M, (ia, ib), E)
    return M.transpose(2, 0, 1, 3)


def vec_core(G, q: Quad):
    """(r, n, s) load core (reference assembly.py:225-233)."""
    r, nq, s = G.shape
    n = int(q.first.max()) + q.V.shape[1]
    E = np.einsum("rqs,q,qa->qars", G, q.w, q.V, optimize=True)
    ia = q.first[:, None] + np.arange(q.V.shape[1])[None, :]
    out = np.zeros((n, r, s))
    np.add.at(out, (ia,), E)
    return out.transpose(1, 0, 2)


def stiffness(patch, disc: Disc, eps, rank_cap=64, rng=None):
    """Reference assemble_stiffness (assembly.py:236-275)."""
    rng = rng or np.random.default_rng()
    ev = TensorGridEval(patch, disc.axes())
    sc = metric_rms(ev, rng)
    info = {"eps": eps, "cross_errors": {}, "cross_converged": {}, "n_evals": 0, "cross_ranks": {}}
    K = None
    for i in range(3):
        for j in range(3):
            t, err, ok, nev, _ = cross(metric_fn(ev, i, j), ev.shape, eps, rank_cap=rank_cap, rng=rng, scale=sc)
            key = f"R{i + 1}{j + 1}"
            info["cross_errors"][key] = err
            info["cross_converged"][key] = ok
            info["cross_ranks"][key] = t.ranks
            info["n_evals"] += nev
            Kij = T.TTOp([op_core(t.cores[d], disc.quads[d], d == i, d == j) for d in range(3)])
            K = Kij if K is None else T.round_tt(T.add(K, Kij), eps)
    return K, info


def load(patch, disc: Disc, src, eps, rank_cap=64, rng=None):
    """Reference assemble_load (assembly.py:278-304)."""
    rng = rng or np.random.default_rng()
    ev = TensorGridEval(patch, disc.axes())
    t, err, ok, nev, _ = cross(load_fn(ev, src), ev.shape, eps, rank_cap=rank_cap, rng=rng)
    f = T.TT([vec_core(t.cores[d], disc.quads[d]) for d in range(3)])
    return f, {"eps": eps, "cross_error": err, "cross_converged": ok, "n_evals": nev, "cross_ranks": t.ranks}


# ---------------------------------------------------------------------------
# boundary conditions (reference assembly.py:307-504)

FACES = tuple((a, s) for a in range(3) for s in range(2))


@dataclass(frozen=True)
class Face:
    """Reference FaceCondition (assembly.py:310-331)."""

    kind: str
    value: object = None

    def __post_init__(self):
        if self.kind not in ("dirichlet", "natural"):
            raise IgaFault(f"face kind {self.kind!r}")

    def fn(self):
        if callable(self.value):
            return self.value
        c = 0.0 if self.value is None else float(self.value)
        return lambda x: np.full(np.asarray(x).shape[0], c)

    def zero(self):
        return not callable(self.value) and (self.value is None or float(self.value) == 0.0)


@dataclass(frozen=True)
class Bc:
    """Reference BoundarySpec (assembly.py:334-371); allow_adjacent: EXTENSION switch."""

    faces: dict = field(default_factory=dict)
    allow_adjacent: bool = False

    def __post_init__(self):
        for k, v in self.faces.items():
            if k not in FACES or not isinstance(v, Face):
                raise IgaFault(f"bad face {k!r}")

    def at(self, a, s):
        return self.faces.get((a, s), Face("natural"))

    def dirichlet(self):
        return [f for f in FACES if self.at(*f).kind == "dirichlet"]

    @staticmethod
    def all(value=0.0):
        return Bc({f: Face("dirichlet", value) for f in FACES})

    def interior(self, sizes):
        out = []
        for a, n in enumerate(sizes):
            lo = 1 if self.at(a, 0).kind == "dirichlet" else 0
            hi = n - (1 if self.at(a, 1).kind == "dirichlet" else 0)
            if hi - lo < 1:
                raise IgaFault(f"no interior along axis {a}")
            out.append(slice(lo, hi))
        return tuple(out)


def face_coeffs(patch, disc: Disc, bc: Bc, a, s):
    """Greville interpolation of face data (reference _face_coefficients, assembly.py:393-414)."""
    oth = [d for d in range(3) if d != a]
    gr = [disc.bases[d].greville() for d in oth]
    axes = [None] * 3
    axes[a] = np.array([float(s)])
    axes[oth[0]], axes[oth[1]] = gr
    ev = TensorGridEval(patch, axes)
    A, B = np.meshgrid(np.arange(gr[0].size), np.arange(gr[1].size), indexing="ij")
    idx = np.zeros((A.size, 3), dtype=np.intp)
    idx[:, oth[0]] = A.ravel()
    idx[:, oth[1]] = B.ravel()
    G = bc.at(a, s).fn()(ev.points(idx)).reshape(gr[0].size, gr[1].size)
    C0 = dense_tables(disc.bases[oth[0]], gr[0])[0]
    C1 = dense_tables(disc.bases[oth[1]], gr[1])[0]
    c = np.linalg.solve(C0, G)
    return np.linalg.solve(C1, c.T).T


def _face_tt(coeff, sizes, a, s):
    U, sv, Vt = np.linalg.svd(coeff, full_matrices=False)
    keep = max(1, int(np.sum(sv > 1e-14 * max(sv[0], 1e-300))))
    Us, V = U[:, :keep] * sv[:keep], Vt[:keep]
    e = np.zeros(sizes[a])
    e[0 if s == 0 else -1] = 1.0
    if a == 0:
        cores = [e[None, :, None], Us[None], V[:, :, None]]
    elif a == 1:
        cores = [Us[None], np.einsum("xy,i->xiy", np.eye(keep), e), V[:, :, None]]
    else:
        cores = [Us[None], V[:, :, None], e[None, :, None]]
    return T.TT(cores)


def lift_tt(patch, disc: Disc, bc: Bc):
    """Reference _lift_tensor (assembly.py:417-463).

    EXTENSION: nonzero data on adjacent faces (rejected by the reference) is
    accepted; an edge/corner coefficient is then owned by the nonzero face of
    lowest axis and masked out of the others, so no entry is counted twice
    (for consistent data both faces interpolate the same edge values).
    """
    sizes = disc.sizes
    nz = [f for f in bc.dirichlet() if not bc.at(*f).zero()]
    adjacent = any(fa[0] != fb[0] for i, fa in enumerate(nz) for fb in nz[i + 1:])
    if adjacent and not bc.allow_adjacent:
        raise IgaFault("nonzero Dirichlet data on adjacent faces is not supported")
    lift = T.TT.zeros(sizes)
    for a, s in nz:
        c = face_coeffs(patch, disc, bc, a, s)
        if adjacent:
            oth = [d for d in range(3) if d != a]
            for pos, d in enumerate(oth):
                if d > a:
                    continue
                for side in (0, 1):
                    if (d, side) in nz:
                        sl = [slice(None), slice(None)]
                        sl[pos] = 0 if side == 0 else sizes[d] - 1
                        c[tuple(sl)] = 0.0
        lift = T.round_tt(T.add(lift, _face_tt(c, sizes, a, s)), 1e-14)
    return lift


@dataclass
class System:
    """Reference AssembledSystem (assembly.py:374-382)."""

    K: object
    f: object
    lift: object
    interior: tuple
    meta: dict = field(default_factory=dict)


def eliminate(K, f, bc: Bc, disc: Disc, patch, eps=1e-12) -> System:
    """Reference apply_dirichlet (assembly.py:466-504)."""
    if not bc.dirichlet():
        raise IgaFault("no Dirichlet face")
    sizes = disc.sizes
    if K.row_sizes != sizes or f.mode_sizes != sizes:
        raise IgaFault("size mismatch")
    sl = bc.interior(sizes)
    lift = lift_tt(patch, disc, bc)
    fi = T.TT([G[:, s, :] for G, s in zip(f.cores, sl)])
    if float(np.max(np.abs(lift.cores[0]))) != 0.0:
        corr = T.matvec(K, lift)
        corr = T.TT([G[:, s, :] for G, s in zip(corr.cores, sl)])
        fi = T.round_tt(T.sub(fi, corr), eps)
    Ki = T.TTOp([G[:, s, s, :] for G, s in zip(K.cores, sl)])
    return System(Ki, fi, lift, sl, {"ranks_K": Ki.ranks, "ranks_f": fi.ranks, "ranks_lift": lift.ranks})


# ---------------------------------------------------------------------------
# sources / analytic solutions (reference driver.py:80-147)

def _s3(x):
    return np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1]) * np.sin(np.pi * x[:, 2])


def _exp_sines_source(x):
    """EXTENSION: -Laplace of exp(x+y+z) sin(pi x) sin(pi y) sin(pi z)."""
    e = np.exp(x.sum(1))
    s = [np.sin(np.pi * x[:, k]) for k in range(3)]
    c = [np.cos(np.pi * x[:, k]) for k in range(3)]
    S = s[0] * s[1] * s[2]
    mix = c[0] * s[1] * s[2] + s[0] * c[1] * s[2] + s[0] * s[1] * c[2]
    return -e * ((3.0 - 3.0 * np.pi ** 2) * S + 2.0 * np.pi * mix)


SOURCES = {
    "zero": lambda x: np.zeros(x.shape[0]),
    "one": lambda x: np.ones(x.shape[0]),
    "sin_pi_xy": lambda x: np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1]),
    "sin_pi_xyz": _s3,
    "manufactured_sines": lambda x: 3.0 * np.pi ** 2 * _s3(x),
    "exp_sines": _exp_sines_source,
}


def _an_lshape(cfg, patch):
    return lambda x: np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1]) / (2.0 * np.pi ** 2)


def _an_cube(cfg, patch):
    return _s3


def _an_exp(cfg, patch):
    return lambda x: np.exp(x.sum(1)) * _s3(x)


def _an_ring(cfg, patch):
    prm = patch.meta.get("params", {})
    ri, ro = prm.get("r_in", 0.5), prm.get("r_out", 1.0)
    ci, co = cfg.bc.at(1, 0), cfg.bc.at(1, 1)
    if ci.kind != "dirichlet" or co.kind != "dirichlet" or callable(ci.value) or callable(co.value):
        raise IgaFault("ring_radial needs constant Dirichlet radial faces")
    ui, uo = float(ci.value or 0.0), float(co.value or 0.0)
    lr = np.log(ro / ri)
    return lambda x: (ui * np.log(ro / np.hypot(x[:, 0], x[:, 1])) + uo * np.log(np.hypot(x[:, 0], x[:, 1]) / ri)) / lr


ANALYTIC = {"lshape_exact": _an_lshape, "cube_sines": _an_cube, "ring_radial": _an_ring, "exp_sines": _an_exp}


@dataclass
class Config:
    """Reference SolveConfig (driver.py:153-201) + EXTENSION fields.

    ``n_basis``: exact basis count per direction (open uniform knots) instead of
    the reference's bisection ladder. ``bc_from_analytic``: every default
    Dirichlet face takes the analytic solution as data.
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
    bc: object = None
    source: str = "zero"
    analytic: str | None = None
    seed: int = 0
    solver: dict = field(default_factory=dict)
    n_basis: object = None
    bc_from_analytic: bool = False

    def __post_init__(self):
        for nm in ("eps_cross", "eps_solve", "eps_round"):
            if not 0.0 < getattr(self, nm) < 1.0:
                raise IgaFault(f"{nm} outside (0,1)")
        tri = lambda v: tuple(int(x) for x in (v if not np.isscalar(v) else (v,) * 3))
        self.degree = tri(self.degree)
        self.elements = tri(self.elements)
        if self.n_basis is not None:
            self.n_basis = tri(self.n_basis)
        if min(self.degree) < 1 or min(self.elements) < 1:
            raise IgaFault("degree/elements")
        if self.source not in SOURCES:
            raise IgaFault("unknown source")
        if self.analytic is not None and self.analytic not in ANALYTIC:
            raise IgaFault("unknown analytic")

    def resolve(self, patch):
        if self.bc is None:
            if self.bc_from_analytic:
                fn = ANALYTIC[self.analytic](self, patch)
                self.bc = Bc({(int(a), int(s)): Face("dirichlet", fn) for a, s in patch.meta["default_dirichlet"]},
                             allow_adjacent=True)
            else:
                self.bc = Bc({(int(a), int(s)): Face("dirichlet", 0.0) for a, s in patch.meta["default_dirichlet"]})
        return self


def compression(t):
    """Reference compression_ratio (driver.py:360-368)."""
    if t.is_op:
        full = int(np.prod(t.row_sizes, dtype=np.int64)) * int(np.prod(t.col_sizes, dtype=np.int64))
    else:
        full = int(np.prod(t.mode_sizes, dtype=np.int64))
    return full / t.n_params


def field_at(disc: Disc, u, xi):
    """Reference evaluate_field (driver.py:371-379)."""
    v = np.ones((1, 1))
    for d in range(3):
        i0, val, _ = basis_window(disc.bases[d], float(xi[d]))
        v = v @ np.einsum("a,ras->rs", val, u.cores[d][:, i0: i0 + val.size, :])
    return float(v[0, 0])


def l1_rel_error(u, exact, patch, disc: Disc):
    """Reference l2_error (driver.py:388-422): int|u-u*| / int|u*| with det J."""
    Bq = [dense_tables(disc.bases[d], disc.quads[d].x)[0] for d in range(3)]
    V = [np.einsum("rns,qn->rqs", u.cores[d], Bq[d], optimize=True) for d in range(3)]
    T12 = np.einsum("qb,bpc->qpc", V[0][0], V[1], optimize=True)
    ev = TensorGridEval(patch, disc.axes())
    nq = disc.qshape
    w12 = np.outer(disc.quads[0].w, disc.quads[1].w)
    w3 = disc.quads[2].w
    i12 = np.stack([np.repeat(np.arange(nq[0]), nq[1]), np.tile(np.arange(nq[1]), nq[0]),
                    np.zeros(nq[0] * nq[1], dtype=np.intp)], 1)
    num = den = 0.0
    for k in range(nq[2]):
        idx = i12.copy()
        idx[:, 2] = k
        J, x = ev.jac_points(idx)
        wd = w12 * w3[k] * np.linalg.det(J).reshape(nq[0], nq[1])
        ue = exact(x).reshape(nq[0], nq[1])
        un = np.einsum("qpc,c->qp", T12, V[2][:, k, 0], optimize=True)
        num += float(np.sum(wd * np.abs(un - ue)))
        den += float(np.sum(wd * np.abs(ue)))
    if den == 0.0:
        raise IgaFault("analytic solution vanishes")
    return num / den


def _seeds(seed, n):
    return [np.random.default_rng(s) for s in np.random.SeedSequence(seed).spawn(n)]


def discretize(cfg: Config, patch):
    if cfg.n_basis is not None:
        bases = tuple(solution_space_exact(patch.sp[d], cfg.degree[d], cfg.n_basis[d]) for d in range(3))
    else:
        bases = tuple(solution_space(patch.sp[d], cfg.degree[d], cfg.elements[d]) for d in range(3))
    return gauss_tables(bases, cfg.n_gauss)


def extend(u_int, sl, sizes):
    """Reference _extend_interior (driver.py:446-452)."""
    out = []
    for G, s, n in zip(u_int.cores, sl, sizes):
        Z = np.zeros((G.shape[0], n, G.shape[2]))
        Z[:, s, :] = G
        out.append(Z)
    return T.TT(out)


def geometry_params(cfg: Config):
    """cfg.geometry_params, plus -- for the seeded random cube solved on an exact-count (n_basis) open
    uniform space -- the solve's Gauss grid as the det J > 0 admissibility grid (BASELINE configs[3]:
    "rejected until det J > 0 at all Gauss points")."""
    prm = dict(cfg.geometry_params)
    if cfg.geometry == "random_cube" and cfg.n_basis is not None and "check_gauss" not in prm:
        ng = cfg.n_gauss
        q = [d + 1 for d in cfg.degree] if ng is None else ([int(ng)] * 3 if np.isscalar(ng) else [int(g) for g in ng])
        prm["check_gauss"] = [[n - d, g] for n, d, g in zip(cfg.n_basis, cfg.degree, q)]
    return prm


def solve(cfg: Config, want_error=True):
    """Reference solve_poisson (driver.py:455-532) without the operator cache."""
    tm = {}
    t0 = time.perf_counter()
    patch = build_patch(cfg.geometry, geometry_params(cfg))
    cfg.resolve(patch)
    disc = discretize(cfg, patch)
    tm["t_setup_s"] = time.perf_counter() - t0
    rK, rf = _seeds(cfg.seed, 2)
    t0 = time.perf_counter()
    K, kinfo = stiffness(patch, disc, cfg.eps_round, cfg.rank_cap, rK)
    tm["t_assemble_K_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    f, finfo = load(patch, disc, SOURCES[cfg.source], cfg.eps_cross, cfg.rank_cap, rf)
    tm["t_assemble_f_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    sysm = eliminate(K, f, cfg.bc, disc, patch, eps=cfg.eps_round)
    tm["t_bc_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    u, res, conv, sweeps = amen(sysm.K, sysm.f, cfg.eps_solve, AmenOpts(**cfg.solver) if cfg.solver else None)
    tm["t_solve_s"] = time.perf_counter() - t0
    uf = T.round_tt(T.add(extend(u, sysm.interior, disc.sizes), sysm.lift), 1e-14)
    err = None
    t0 = time.perf_counter()
    if cfg.analytic is not None and want_error:
        err = l1_rel_error(uf, ANALYTIC[cfg.analytic](cfg, patch), patch, disc)
    tm["t_error_s"] = time.perf_counter() - t0
    return {
        "u": uf, "K": K, "f": f, "system": sysm, "disc": disc, "patch": patch,
        "dofs": int(np.prod(disc.sizes)), "mode_sizes": disc.sizes, "l2_error": err,
        "residual": res, "solver_converged": conv,
        "cross_converged": bool(all(kinfo["cross_converged"].values()) and finfo["cross_converged"]),
        "ranks_K": K.ranks, "ranks_f": f.ranks, "ranks_u": uf.ranks,
        "compression_K": compression(K), "compression_f": compression(f), "compression_u": compression(uf),
        "timings": tm, "sweeps": sweeps, "k_info": kinfo, "f_info": finfo,
    }
