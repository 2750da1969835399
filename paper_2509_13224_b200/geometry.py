"""Exact NURBS patches and device-side map/metric evaluation (reference ``pkg/src/ttiga/geometry.py``).

Control nets are built on the host (a few dozen points); the weighted control
grid lives in HBM as (n0, n1, n2, 4) = (w x, w y, w z, w) so the geometry
kernel gathers one (p+1)^3 window with two 16-byte loads per control point.
``GridEvaluator`` tabulates the per-direction basis windows once (device
Cox-de Boor) and evaluates x, J, det J and R = J^-1 J^-T det J at batches of
grid multi-indices with ``ttb_geo_eval``.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np
import torch

from . import linalg as L
from .pointfn import on_device
from ._lib import call, device, ptr
from .splines import Basis1D, KnotVector, basis_windows

__all__ = ["GeometryError", "SingularMapError", "GeometryPatch", "MetricSample", "GridEvaluator", "GEOMETRY_NAMES",
           "make_geometry", "patch_to_json", "patch_from_json", "SOURCE_IDS"]

GEOMETRY_NAMES = ("unit_cube", "lshape", "ring", "closed_hemisphere", "opened_hemisphere", "hyperboloid",
                  "quarter_torus")
EXTENDED_GEOMETRY_NAMES = GEOMETRY_NAMES + ("quarter_cylinder", "deformed_cube", "random_cube")

# source terms evaluated inside the geometry kernel (mode 1)
SOURCE_IDS = {"zero": 0, "one": 1, "sin_pi_xy": 2, "sin_pi_xyz": 3, "manufactured_sines": 4, "exp_sines": 5}


class GeometryError(ValueError):
    """Invalid geometry parameters or construction failure (reference geometry.py:45)."""


class SingularMapError(GeometryError):
    """Jacobian determinant below the singularity threshold (reference geometry.py:49)."""


@dataclass(frozen=True)
class MetricSample:
    jacobian: np.ndarray
    det: float
    metric: np.ndarray


@dataclass(frozen=True)
class GeometryPatch:
    """Trivariate NURBS map from the unit cube (reference geometry.py:66-114)."""

    bases: tuple
    control_points: np.ndarray
    weights: np.ndarray
    metadata: dict = field(default_factory=dict)

    def __post_init__(self):
        cp = np.asarray(self.control_points, dtype=float)
        w = np.asarray(self.weights, dtype=float)
        object.__setattr__(self, "control_points", cp)
        object.__setattr__(self, "weights", w)
        shape = tuple(b.n_basis for b in self.bases)
        if cp.shape != shape + (3,):
            raise GeometryError(f"control grid shape {cp.shape} != {shape + (3,)}")
        if w.shape != shape:
            raise GeometryError(f"weight grid shape {w.shape} != {shape}")
        if np.any(w <= 0):
            raise GeometryError("weights must be strictly positive")
        object.__setattr__(self, "_cw", None)

    @property
    def degrees(self):
        return tuple(b.degree for b in self.bases)

    @property
    def scale(self) -> float:
        c = self.control_points.reshape(-1, 3)
        return float(np.linalg.norm(c.max(axis=0) - c.min(axis=0)))

    def device_control(self):
        """(n0, n1, n2, 4) FP64 device grid of (w x, w y, w z, w)."""
        if self._cw is None:
            cw = np.concatenate([self.control_points * self.weights[..., None], self.weights[..., None]], axis=-1)
            object.__setattr__(self, "_cw", torch.as_tensor(np.ascontiguousarray(cw), device=device()))
        return self._cw

    def eval_point(self, xi) -> np.ndarray:
        ev = GridEvaluator(self, [[float(x)] for x in xi])
        return ev.points(np.zeros((1, 3), dtype=np.int64))[0]

    def eval_metric(self, xi) -> MetricSample:
        """One point (reference geometry.py:103-114): J from the device evaluator, det / metric from it on the
        host exactly as the reference forms them (det = np.linalg.det(J))."""
        ev = GridEvaluator(self, [[float(x)] for x in xi])
        jac = ev.records(np.zeros((1, 3), dtype=np.int64), check=False)[0, :9].reshape(3, 3)
        det = float(np.linalg.det(jac))
        if abs(det) < 1e-12 * self.scale ** 3:
            raise SingularMapError(f"singular geometry map at xi={tuple(xi)}")
        inv = np.linalg.inv(jac)
        metric = inv @ inv.T * det
        return MetricSample(jac, det, 0.5 * (metric + metric.T))


class GridEvaluator:
    """Batched evaluation on a fixed tensor grid of parameters (reference geometry.py:150-261)."""

    def __init__(self, patch: GeometryPatch, axes_points):
        self.patch = patch
        self.axes_points = [np.asarray(a, dtype=float).reshape(-1) for a in axes_points]
        self.win = [basis_windows(b, a) for b, a in zip(patch.bases, self.axes_points)]
        self.cw = patch.device_control()
        self.sing_tol = 1e-12 * patch.scale ** 3

    @property
    def shape(self):
        return tuple(a.size for a in self.axes_points)

    def _launch(self, idx, mode, out, ri=0, rj=0, src=0):
        idx = torch.as_tensor(idx, dtype=torch.int64, device=device()).contiguous()
        N = int(idx.shape[0])
        bad = torch.full((1,), 2 ** 63 - 1, dtype=torch.int64, device=device())
        (f0, V0, D0), (f1, V1, D1), (f2, V2, D2) = self.win
        p = self.patch.degrees
        n = self.cw.shape[:3]
        call("ttb_geo_eval", N, ptr(idx), ptr(f0), ptr(f1), ptr(f2), ptr(V0), ptr(V1), ptr(V2), ptr(D0), ptr(D1),
             ptr(D2), p[0], p[1], p[2], n[0], n[1], n[2], ptr(self.cw), float(self.sing_tol), mode, ri, rj, src,
             ptr(out), ptr(bad))
        return idx, bad

    def _raise_if_bad(self, idx, bad):
        b = int(bad.item())
        if b != 2 ** 63 - 1:
            q = idx[b].cpu().numpy()
            xi = tuple(float(self.axes_points[d][q[d]]) for d in range(3))
            raise SingularMapError(f"singular geometry map at xi={xi}")

    def min_det(self):
        """(min det J, number of points with det J <= 0) over the FULL tensor grid (device kernel
        ttb_geo_min_det; no index list, so the 8.4e9-point Gauss grid of configs[3] is one launch)."""
        out = torch.empty(2, dtype=torch.int64, device=device())
        (f0, V0, D0), (f1, V1, D1), (f2, V2, D2) = self.win
        p = self.patch.degrees
        n = self.cw.shape[:3]
        q = self.shape
        call("ttb_geo_min_det", q[0], q[1], q[2], ptr(f0), ptr(f1), ptr(f2), ptr(V0), ptr(V1), ptr(V2), ptr(D0),
             ptr(D1), ptr(D2), p[0], p[1], p[2], n[0], n[1], n[2], ptr(self.cw), ptr(out))
        key, bad = (int(v) & ((1 << 64) - 1) for v in out.cpu().tolist())
        bits = key ^ (1 << 63) if key >> 63 else (~key) & ((1 << 64) - 1)
        return float(np.frombuffer(np.uint64(bits).tobytes(), dtype=np.float64)[0]), bad

    # Public evaluation methods mirror the reference's array types: numpy (or list) indices -> numpy
    # results (reference GridEvaluator, geometry.py:150-261); a CUDA int64 index tensor -> CUDA tensors
    # (the device path every internal caller takes).
    @staticmethod
    def _host(idx):
        return not isinstance(idx, torch.Tensor)

    @staticmethod
    def _ret(x, host):
        return x.cpu().numpy() if host else x

    def records(self, idx, check=True):
        """(N, 22) records: J (9), x (3), det, R (9)."""
        host = self._host(idx)
        N = len(idx)
        out = L.empty(N, 22)
        idx, bad = self._launch(idx, 2, out)
        if check:
            self._raise_if_bad(idx, bad)
        return self._ret(out, host)

    def points(self, idx):
        host = self._host(idx)
        out = L.empty(len(idx), 3)
        self._launch(idx, 3, out)
        return self._ret(out, host)

    def jacobians(self, idx):
        rec = self.records(idx, check=False)
        return rec[:, :9].reshape(-1, 3, 3), rec[:, 9:12]

    def metric(self, idx):
        rec = self.records(idx)
        return rec[:, 12], rec[:, 13:].reshape(-1, 3, 3)

    def metric_entry(self, idx, i, j, check=True):
        """R[:, i, j] only (cross oracle of assembly.metric_oracle)."""
        host = self._host(idx)
        out = L.empty(len(idx))
        idx, bad = self._launch(idx, 0, out, ri=i, rj=j)
        if check:
            self._raise_if_bad(idx, bad)
        return self._ret(out, host)

    def source_times_det(self, idx, source):
        """f(x(xi)) det J (assembly.load_oracle). ``source``: a SOURCE_IDS name or a built-in PointFn
        (evaluated inside geo_kernel), or any callable of physical points (numpy semantics, bridged)."""
        host = self._host(idx)
        name = source if isinstance(source, str) else getattr(source, "name", None)
        if name in SOURCE_IDS and (isinstance(source, str) or getattr(source, "source_id", None) is not None):
            out = L.empty(len(idx))
            self._launch(idx, 1, out, src=SOURCE_IDS[name])
            return self._ret(out, host)
        rec = self.records(idx, check=False)
        if host:
            return np.asarray(source(rec[:, 9:12]), dtype=float) * rec[:, 12]
        return on_device(source)(rec[:, 9:12]) * rec[:, 12]


# ---------------------------------------------------------------------------
# factories (same solids as the reference, geometry.py:264-576, plus the BASELINE extensions)

_S = 1.0 / np.sqrt(2.0)


def _lin_kv():
    return KnotVector(np.array([0.0, 0.0, 1.0, 1.0]), 1)


def _circle():
    kv = KnotVector(np.array([0, 0, 0, .25, .25, .5, .5, .75, .75, 1, 1, 1.0]), 2)
    P = np.array([[1, 0], [1, 1], [0, 1], [-1, 1], [-1, 0], [-1, -1], [0, -1], [1, -1], [1, 0]], float)
    return kv, P, np.array([1, _S, 1, _S, 1, _S, 1, _S, 1.0])


def _arc(a0, a1):
    sweep = a1 - a0
    if not 0 < abs(sweep) < np.pi:
        raise GeometryError("single-segment arc must span (0, 180) degrees")
    mid, wm = 0.5 * (a0 + a1), np.cos(0.5 * sweep)
    P = np.array([[np.cos(a0), np.sin(a0)], [np.cos(mid) / wm, np.sin(mid) / wm], [np.cos(a1), np.sin(a1)]])
    return KnotVector(np.array([0, 0, 0, 1, 1, 1.0]), 2), P, np.array([1.0, wm, 1.0])


def _hyperbola(r_end, r_w, z0, z1):
    if not 0 < r_w < r_end:
        raise GeometryError("need 0 < waist radius < end radius")
    P = np.array([[r_end, z0], [r_w ** 2 / r_end, 0.5 * (z0 + z1)], [r_end, z1]])
    return KnotVector(np.array([0, 0, 0, 1, 1, 1.0]), 2), P, np.array([1.0, r_end / r_w, 1.0])


def _host_det(patch, xi):
    """det J at one point by a host quotient rule (construction-time orientation probe only)."""
    return patch.eval_metric(np.asarray(xi, dtype=float)).det


def _finalize(bases, ctrl, w, meta):
    """Orientation fix (flip xi_3 when det J < 0) + verification (reference geometry.py:334-344)."""
    patch = GeometryPatch(tuple(bases), ctrl, w, meta)
    if _host_det(patch, [0.37, 0.51, 0.43]) < 0:
        ctrl, w = np.flip(ctrl, 2), np.flip(w, 2)
        kv = bases[2].knot_vector
        bases = (bases[0], bases[1], Basis1D(KnotVector((kv.start + kv.end) - kv.knots[::-1], kv.degree)))
        patch = GeometryPatch(tuple(bases), ctrl, w, meta)
    for xi in ([0.11, 0.62, 0.29], [0.83, 0.24, 0.77], [0.5, 0.5, 0.5]):
        if _host_det(patch, xi) <= 0:
            raise GeometryError("orientation check failed: det(J) <= 0")
    return patch


def _product(kvs, build, meta):
    bases = tuple(Basis1D(kv) for kv in kvs)
    n = tuple(kv.n_basis for kv in kvs)
    ctrl, w = np.empty(n + (3,)), np.empty(n)
    for i in range(n[0]):
        for j in range(n[1]):
            for k in range(n[2]):
                ctrl[i, j, k], w[i, j, k] = build(i, j, k)
    return _finalize(bases, ctrl, w, meta)


def _take(params, defaults):
    unknown = set(params) - set(defaults)
    if unknown:
        raise GeometryError(f"unknown geometry parameters: {sorted(unknown)}")
    out = dict(defaults)
    out.update(params)
    return out


def _require(ok, msg):
    if not ok:
        raise GeometryError(msg)


def _all_faces():
    return [[a, s] for a in range(3) for s in range(2)]


def _unit_cube(prm):
    p = _take(prm, {})
    c = np.array([0.0, 1.0])
    ctrl = np.stack(np.meshgrid(c, c, c, indexing="ij"), axis=-1)
    lin = Basis1D(_lin_kv())
    return _finalize((lin, lin, lin), ctrl, np.ones((2, 2, 2)), {"name": "unit_cube", "params": p,
                     "directions": ("x", "y", "z"), "default_dirichlet": _all_faces()})


def _lshape(prm):
    p = _take(prm, {"zmax": 1.0})
    _require(p["zmax"] > 0, "zmax must be positive")
    inner = np.array([[0, 1], [0, 0], [1, 0]], float)
    outer = np.array([[-1, 1], [-1, -1], [1, -1]], float)
    ctrl = np.empty((3, 2, 2, 3))
    for i in range(3):
        for j, row in enumerate((inner, outer)):
            for k, z in enumerate((0.0, p["zmax"])):
                ctrl[i, j, k] = (row[i, 0], row[i, 1], z)
    lin = Basis1D(_lin_kv())
    return _finalize((Basis1D(KnotVector(np.array([0, 0, .5, 1, 1.0]), 1)), lin, lin), ctrl, np.ones((3, 2, 2)),
                     {"name": "lshape", "params": p, "directions": ("path", "across", "height"),
                      "default_dirichlet": [[0, 0], [0, 1], [1, 0], [1, 1]]})


def _ring(prm):
    p = _take(prm, {"r_in": 0.5, "r_out": 1.0, "h": 1.0})
    _require(0 < p["r_in"] < p["r_out"], "need 0 < r_in < r_out")
    _require(p["h"] > 0, "height must be positive")
    kv, P, w = _circle()
    rad, zs = (p["r_in"], p["r_out"]), (0.0, p["h"])
    return _product([kv, _lin_kv(), _lin_kv()], lambda i, j, k: ((P[i, 0] * rad[j], P[i, 1] * rad[j], zs[k]), w[i]),
                    {"name": "ring", "params": p, "directions": ("angular", "radial", "height"),
                     "default_dirichlet": [[1, 0], [1, 1]]})


def _hemisphere(p, name, top, extra):
    kv, P, w = _circle()
    kva, A, wa = _arc(0.0, top)
    rad = (p["r_in"], p["r_out"])

    def build(i, j, k):
        rho, z = A[j] * rad[k]
        return (P[i, 0] * rho, P[i, 1] * rho, z), w[i] * wa[j]

    meta = {"name": name, "params": p, "directions": ("longitude", "latitude", "radial")}
    meta.update(extra)
    return _product([kv, kva, _lin_kv()], build, meta)


def _closed_hemisphere(prm):
    p = _take(prm, {"r_in": 0.5, "r_out": 1.0})
    _require(0 < p["r_in"] < p["r_out"], "need 0 < r_in < r_out")
    return _hemisphere(p, "closed_hemisphere", 0.5 * np.pi,
                       {"default_dirichlet": [[2, 0], [2, 1]], "degenerate_faces": [[1, 1]]})


def _opened_hemisphere(prm):
    p = _take(prm, {"r_in": 0.5, "r_out": 1.0, "hole_deg": 18.0})
    _require(0 < p["r_in"] < p["r_out"], "need 0 < r_in < r_out")
    _require(0 < p["hole_deg"] < 90, "hole angle must be in (0, 90) degrees")
    return _hemisphere(p, "opened_hemisphere", 0.5 * np.pi - np.deg2rad(p["hole_deg"]),
                       {"default_dirichlet": [[1, 0], [1, 1]]})


def _hyperboloid(prm):
    p = _take(prm, {"r_middle": 0.5, "r_top": 1.0, "thickness": 0.3, "zmin": -1.0, "zmax": 1.0})
    _require(0 < p["r_middle"] < p["r_top"], "need 0 < r_middle < r_top")
    _require(0 < p["thickness"] < 2 * p["r_middle"], "invalid shell thickness")
    _require(p["zmin"] < p["zmax"], "need zmin < zmax")
    kv, P, w = _circle()
    kvh, H, wh = _hyperbola(p["r_top"], p["r_middle"], p["zmin"], p["zmax"])
    off = (-0.5 * p["thickness"], 0.5 * p["thickness"])
    return _product([kv, kvh, _lin_kv()],
                    lambda i, j, k: ((P[i, 0] * (H[j, 0] + off[k]), P[i, 1] * (H[j, 0] + off[k]), H[j, 1]),
                                     w[i] * wh[j]),
                    {"name": "hyperboloid", "params": p, "directions": ("angular", "height", "thickness"),
                     "default_dirichlet": [[1, 0], [1, 1]]})


def _quarter_torus(prm):
    p = _take(prm, {"r_in": 0.5, "r_out": 1.0, "R": 3.0})
    _require(0 < p["r_in"] < p["r_out"], "need 0 < r_in < r_out")
    _require(p["R"] > p["r_out"], "toroidal radius must exceed r_out")
    kvt, Tq, wt = _arc(0.0, 0.5 * np.pi)
    kv, P, w = _circle()
    rad = (p["r_in"], p["r_out"])

    def build(i, j, k):
        rho = p["R"] + P[j, 0] * rad[k]
        return (Tq[i, 0] * rho, Tq[i, 1] * rho, P[j, 1] * rad[k]), wt[i] * w[j]

    return _product([kvt, kv, _lin_kv()], build,
                    {"name": "quarter_torus", "params": p, "directions": ("toroidal", "poloidal", "radial"),
                     "default_dirichlet": [[2, 0], [2, 1]]})


def _quarter_cylinder(prm):
    """BASELINE config 2: quarter thick-walled cylinder, exact rational arc (1, sqrt2/2, 1)."""
    p = _take(prm, {"r_in": 1.0, "r_out": 2.0, "h": 1.0})
    _require(0 < p["r_in"] < p["r_out"], "need 0 < r_in < r_out")
    _require(p["h"] > 0, "height must be positive")
    kva, A, wa = _arc(0.0, 0.5 * np.pi)
    rad, zs = (p["r_in"], p["r_out"]), (0.0, p["h"])
    return _product([kva, _lin_kv(), _lin_kv()],
                    lambda i, j, k: ((A[i, 0] * rad[j], A[i, 1] * rad[j], zs[k]), wa[i]),
                    {"name": "quarter_cylinder", "params": p, "directions": ("angular", "radial", "height"),
                     "default_dirichlet": _all_faces()})


def _collocation(kv, pts):
    from .splines import tabulate
    return tabulate(Basis1D(kv), pts)[0]


def _deformed_cube(prm):
    """BASELINE config 3: degree-3 interpolant (Greville points, 16^3 controls) of the sine-deformed cube."""
    p = _take(prm, {"amplitude": 0.1, "n_ctrl": 16, "degree": 3})
    a, deg, nc = p["amplitude"], int(p["degree"]), int(p["n_ctrl"])
    kv = KnotVector.open_uniform(deg, nc - deg)
    from .splines import greville_points
    g = greville_points(kv)
    U, V, W = np.meshgrid(g, g, g, indexing="ij")
    F = np.stack([U + a * np.sin(2 * np.pi * V) * np.sin(np.pi * W),
                  V + a * np.sin(2 * np.pi * W) * np.sin(np.pi * U),
                  W + a * np.sin(2 * np.pi * U) * np.sin(np.pi * V)], -1)
    Cinv = np.linalg.inv(_collocation(kv, g))
    for ax in range(3):
        F = np.moveaxis(np.tensordot(Cinv, np.moveaxis(F, ax, 0), (1, 0)), 0, ax)
    b = Basis1D(kv)
    return _finalize((b, b, b), F, np.ones(F.shape[:3]), {"name": "deformed_cube", "params": p,
                     "directions": ("x", "y", "z"), "default_dirichlet": _all_faces()})


def gauss_grid(elements, points):
    """Gauss-Legendre points of ``elements`` uniform spans of [0, 1], ``points`` per span: the solve's
    quadrature on an exact-count open uniform solution basis (assembly.build_quadrature)."""
    xg, _ = np.polynomial.legendre.leggauss(int(points))
    brk = np.linspace(0.0, 1.0, int(elements) + 1)
    return np.concatenate([0.5 * (a + b) + 0.5 * (b - a) * xg for a, b in zip(brk[:-1], brk[1:])])


def _random_cube(prm):
    """BASELINE config 4: seeded N(0, sigma^2) perturbation of a degree-3 cube net, det J > 0 rejection.

    Check grid: with ``check_gauss = (elements, points)`` (set by the solve driver for exact-count
    solution spaces) every Gauss point of the solve -- 2036^3 = 8.4e9 points at configs[3], one
    min-det kernel launch per draw; otherwise 8 Gauss-Legendre points per geometry knot span.
    Oracle: oracle/patch.py random_cube (same draws, same grid).
    """
    p = _take(prm, {"sigma": 0.02, "n_ctrl": 8, "degree": 3, "seed": 0, "max_draws": 100, "check_gauss": None})
    deg, nc = int(p["degree"]), int(p["n_ctrl"])
    kv = KnotVector.open_uniform(deg, nc - deg)
    from .splines import greville_points
    g = greville_points(kv)
    base = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1)
    rng = np.random.default_rng(int(p["seed"]))
    if p["check_gauss"] is not None:
        cg = np.asarray(p["check_gauss"], dtype=int).reshape(-1, 2)
        cg = np.repeat(cg, 3, axis=0) if cg.shape[0] == 1 else cg
        axes = [gauss_grid(E, q) for E, q in cg]
    else:
        xg, _ = np.polynomial.legendre.leggauss(8)
        brk = np.unique(kv.knots)
        chk = np.concatenate([0.5 * (a + b) + 0.5 * (b - a) * xg for a, b in zip(brk[:-1], brk[1:])])
        axes = [chk, chk, chk]
    meta = {"name": "random_cube", "params": p, "directions": ("x", "y", "z"), "default_dirichlet": _all_faces()}
    b = Basis1D(kv)
    for draw in range(int(p["max_draws"])):
        ctrl = base.copy()
        ctrl[1:-1, 1:-1, 1:-1] += rng.normal(0.0, p["sigma"], size=(nc - 2, nc - 2, nc - 2, 3))
        patch = GeometryPatch((b, b, b), ctrl, np.ones((nc, nc, nc)), dict(meta))
        mn, bad = GridEvaluator(patch, axes).min_det()
        if bad == 0 and mn > 0.0:
            patch.metadata["draws"] = draw + 1
            patch.metadata["check_points"] = int(np.prod([a.size for a in axes]))
            patch.metadata["min_det"] = mn
            return patch
    raise GeometryError("no admissible random draw")


_FACTORIES = {
    "unit_cube": _unit_cube, "lshape": _lshape, "ring": _ring, "closed_hemisphere": _closed_hemisphere,
    "opened_hemisphere": _opened_hemisphere, "hyperboloid": _hyperboloid, "quarter_torus": _quarter_torus,
    "quarter_cylinder": _quarter_cylinder, "deformed_cube": _deformed_cube, "random_cube": _random_cube,
}


def make_geometry(name: str, params: dict | None = None) -> GeometryPatch:
    """Reference make_geometry (geometry.py:365-385) + BASELINE extension solids."""
    if name not in _FACTORIES:
        raise GeometryError(f"unknown geometry {name!r}; choose from {EXTENDED_GEOMETRY_NAMES}")
    return _FACTORIES[name](dict(params or {}))


def patch_to_json(patch: GeometryPatch) -> str:
    return json.dumps({"degrees": list(patch.degrees), "knots": [b.knot_vector.knots.tolist() for b in patch.bases],
                       "control_points": patch.control_points.tolist(), "weights": patch.weights.tolist(),
                       "metadata": patch.metadata}, indent=2, default=str)


def patch_from_json(text: str) -> GeometryPatch:
    doc = json.loads(text)
    bases = tuple(Basis1D(KnotVector(np.asarray(k, float), p)) for k, p in zip(doc["knots"], doc["degrees"]))
    return GeometryPatch(bases, np.asarray(doc["control_points"], float), np.asarray(doc["weights"], float),
                         doc.get("metadata", {}))
