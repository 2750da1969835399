"""Oracle: trivariate NURBS patches and batched metric evaluation (TEST INFRASTRUCTURE ONLY).

Restates reference ``pkg/src/ttiga/geometry.py``: exact rational patches for
the benchmark solids, pointwise and batched evaluation of the map x(xi), its
Jacobian J, det J and the metric factor R = J^-1 J^-T det J.
"""

from __future__ import annotations

import numpy as np

from .bspline import Spline1D, basis_window, dense_tables


class PatchFault(ValueError):
    """Mirror of reference GeometryError (geometry.py:45)."""


class SingularMap(PatchFault):
    """Mirror of reference SingularMapError (geometry.py:49)."""


class Patch:
    """Reference GeometryPatch (geometry.py:66-114)."""

    def __init__(self, splines, ctrl, w, meta=None):
        self.sp = tuple(splines)
        self.ctrl = np.asarray(ctrl, dtype=float)
        self.w = np.asarray(w, dtype=float)
        self.meta = dict(meta or {})
        shape = tuple(s.n for s in self.sp)
        if self.ctrl.shape != shape + (3,) or self.w.shape != shape:
            raise PatchFault("control grid shape")
        if np.any(self.w <= 0):
            raise PatchFault("weights must be positive")

    @property
    def degrees(self):
        return tuple(s.p for s in self.sp)

    @property
    def scale(self):
        c = self.ctrl.reshape(-1, 3)
        return float(np.linalg.norm(c.max(0) - c.min(0)))

    def _sums(self, xi):
        """num, den and their parametric derivatives (reference geometry.py:117-147)."""
        win = [basis_window(s, float(x)) for s, x in zip(self.sp, xi)]
        sl = tuple(slice(i0, i0 + v.size) for i0, v, _ in win)
        w = self.w[sl]
        wx = w[..., None] * self.ctrl[sl]
        v = [a[1] for a in win]
        d = [a[2] for a in win]

        def tri(a, b, c, T):
            return np.tensordot(np.tensordot(np.tensordot(a, T, (0, 0)), b, (0, 0)), c, (0, 0))

        den = tri(v[0], v[1], v[2], w)
        num = np.array([tri(v[0], v[1], v[2], wx[..., c]) for c in range(3)])
        dden = np.array([tri(d[0], v[1], v[2], w), tri(v[0], d[1], v[2], w), tri(v[0], v[1], d[2], w)])
        dnum = np.array([[tri(*(d[m] if m == e else v[m] for m in range(3)), wx[..., c]) for e in range(3)]
                         for c in range(3)])
        return num, den, dnum, dden

    def point(self, xi):
        num, den, _, _ = self._sums(xi)
        return num / den

    def metric(self, xi):
        """(J, det, R) at xi (reference eval_metric, geometry.py:103-114)."""
        num, den, dnum, dden = self._sums(xi)
        J = (dnum * den - np.outer(num, dden)) / den ** 2
        det = float(np.linalg.det(J))
        if abs(det) < 1e-12 * self.scale ** 3:
            raise SingularMap(f"singular map at {tuple(xi)}")
        Ji = np.linalg.inv(J)
        R = Ji @ Ji.T * det
        return J, det, 0.5 * (R + R.T)


class TensorGridEval:
    """Batched evaluation at multi-indices of a tensor grid of parameters.

    Restates reference GridEvaluator (geometry.py:150-261): per-direction
    active windows are tabulated once; each query gathers the (p+1)^3
    weighted control window and contracts direction by direction.
    """

    def __init__(self, patch: Patch, axes):
        self.patch = patch
        self.axes = [np.asarray(a, dtype=float) for a in axes]
        self.tabs = []
        for s, pts in zip(patch.sp, self.axes):
            st = np.empty(pts.size, dtype=np.intp)
            V = np.empty((pts.size, s.p + 1))
            D = np.empty((pts.size, s.p + 1))
            for q, x in enumerate(pts):
                st[q], V[q], D[q] = basis_window(s, float(x))
            self.tabs.append((st, V, D))
        self.wx = patch.w[..., None] * patch.ctrl
        self.sing = 1e-12 * patch.scale ** 3

    @property
    def shape(self):
        return tuple(a.size for a in self.axes)

    def _windows(self, idx):
        idx = np.asarray(idx, dtype=np.intp)
        v, d, ix = [], [], []
        for a in range(3):
            st, V, D = self.tabs[a]
            q = idx[:, a]
            v.append(V[q])
            d.append(D[q])
            ix.append(st[q][:, None] + np.arange(V.shape[1])[None, :])
        I0 = ix[0][:, :, None, None]
        I1 = ix[1][:, None, :, None]
        I2 = ix[2][:, None, None, :]
        return v, d, self.patch.w[I0, I1, I2], self.wx[I0, I1, I2]

    def jac_points(self, idx):
        """(J (N,3,3), x (N,3)) — reference GridEvaluator.jacobians (geometry.py:206-245)."""
        v, d, W, WX = self._windows(idx)
        # contract the third direction first, as the reference does
        Wc = np.einsum("nc,nabc->nab", v[2], W)
        Wc3 = np.einsum("nc,nabc->nab", d[2], W)
        Xc = np.einsum("nc,nabcx->nabx", v[2], WX)
        Xc3 = np.einsum("nc,nabcx->nabx", d[2], WX)
        Wb = np.einsum("nb,nab->na", v[1], Wc)
        Xb = np.einsum("nb,nabx->nax", v[1], Xc)
        den = np.einsum("na,na->n", v[0], Wb)
        num = np.einsum("na,nax->nx", v[0], Xb)
        dden = np.stack([
            np.einsum("na,na->n", d[0], Wb),
            np.einsum("na,na->n", v[0], np.einsum("nb,nab->na", d[1], Wc)),
            np.einsum("na,na->n", v[0], np.einsum("nb,nab->na", v[1], Wc3)),
        ], axis=1)
        dnum = np.stack([
            np.einsum("na,nax->nx", d[0], Xb),
            np.einsum("na,nax->nx", v[0], np.einsum("nb,nabx->nax", d[1], Xc)),
            np.einsum("na,nax->nx", v[0], np.einsum("nb,nabx->nax", v[1], Xc3)),
        ], axis=2)
        J = (dnum * den[:, None, None] - num[:, :, None] * dden[:, None, :]) / den[:, None, None] ** 2
        return J, num / den[:, None]

    def points(self, idx):
        return self.jac_points(idx)[1]

    def det_metric(self, idx):
        """(det (N,), R (N,3,3)) — reference GridEvaluator.metric (geometry.py:247-261)."""
        J, _ = self.jac_points(idx)
        det = np.linalg.det(J)
        bad = np.abs(det) < self.sing
        if np.any(bad):
            k = int(np.flatnonzero(bad)[0])
            raise SingularMap(f"singular map at grid index {tuple(np.asarray(idx)[k])}")
        Ji = np.linalg.inv(J)
        R = Ji @ Ji.transpose(0, 2, 1) * det[:, None, None]
        return det, 0.5 * (R + R.transpose(0, 2, 1))


# ---------------------------------------------------------------------------
# factories (reference geometry.py:264-576)

_H = 1.0 / np.sqrt(2.0)
_LIN = (0.0, 0.0, 1.0, 1.0)


def _circle9():
    """Nine-point exact circle (reference geometry.py:274-288)."""
    t = [0, 0, 0, .25, .25, .5, .5, .75, .75, 1, 1, 1]
    P = np.array([[1, 0], [1, 1], [0, 1], [-1, 1], [-1, 0], [-1, -1], [0, -1], [1, -1], [1, 0]], float)
    return t, P, np.array([1, _H, 1, _H, 1, _H, 1, _H, 1])


def _arc(a0, a1):
    """One rational quadratic arc of sweep < pi (reference geometry.py:291-306)."""
    sw = a1 - a0
    if not 0 < abs(sw) < np.pi:
        raise PatchFault("arc sweep")
    m = 0.5 * (a0 + a1)
    c = np.cos(0.5 * sw)
    P = np.array([[np.cos(a0), np.sin(a0)], [np.cos(m) / c, np.sin(m) / c], [np.cos(a1), np.sin(a1)]])
    return [0, 0, 0, 1, 1, 1], P, np.array([1.0, c, 1.0])


def _hyperbola(r_end, r_w, z0, z1):
    """Rational conic through the waist (reference geometry.py:309-320)."""
    if not 0 < r_w < r_end:
        raise PatchFault("waist radius")
    P = np.array([[r_end, z0], [r_w ** 2 / r_end, 0.5 * (z0 + z1)], [r_end, z1]])
    return [0, 0, 0, 1, 1, 1], P, np.array([1.0, r_end / r_w, 1.0])


def _orient(splines, ctrl, w, meta):
    """Flip xi_3 when det J < 0, then verify (reference _finalize, geometry.py:334-344)."""
    pt = Patch(splines, ctrl, w, meta)
    if pt.metric(np.array([0.37, 0.51, 0.43]))[1] < 0:
        ctrl = np.flip(ctrl, 2)
        w = np.flip(w, 2)
        s = splines[2]
        splines = (splines[0], splines[1], Spline1D((s.t[0] + s.t[-1]) - s.t[::-1], s.p))
        pt = Patch(splines, ctrl, w, meta)
    for xi in ([0.11, 0.62, 0.29], [0.83, 0.24, 0.77], [0.5, 0.5, 0.5]):
        if pt.metric(np.asarray(xi))[1] <= 0:
            raise PatchFault("orientation check failed")
    return pt


def _product(knots, degs, build, meta):
    sps = tuple(Spline1D(t, p) for t, p in zip(knots, degs))
    n = tuple(s.n for s in sps)
    ctrl = np.empty(n + (3,))
    w = np.empty(n)
    for i in range(n[0]):
        for j in range(n[1]):
            for k in range(n[2]):
                ctrl[i, j, k], w[i, j, k] = build(i, j, k)
    return _orient(sps, ctrl, w, meta)


def _params(given, defaults):
    bad = set(given) - set(defaults)
    if bad:
        raise PatchFault(f"unknown geometry parameters {sorted(bad)}")
    out = dict(defaults)
    out.update(given)
    return out


def _need(ok, msg):
    if not ok:
        raise PatchFault(msg)


def unit_cube(prm):
    p = _params(prm, {})
    c = np.array([0.0, 1.0])
    ctrl = np.stack(np.meshgrid(c, c, c, indexing="ij"), -1)
    lin = Spline1D(_LIN, 1)
    return _orient((lin, lin, lin), ctrl, np.ones((2, 2, 2)),
                   {"name": "unit_cube", "params": p, "directions": ("x", "y", "z"),
                    "default_dirichlet": [[a, s] for a in range(3) for s in range(2)]})


def lshape(prm):
    p = _params(prm, {"zmax": 1.0})
    _need(p["zmax"] > 0, "zmax")
    inner = np.array([[0, 1], [0, 0], [1, 0]], float)
    outer = np.array([[-1, 1], [-1, -1], [1, -1]], float)
    zs = (0.0, p["zmax"])
    ctrl = np.empty((3, 2, 2, 3))
    for i in range(3):
        for j, row in enumerate((inner, outer)):
            for k in range(2):
                ctrl[i, j, k] = (row[i, 0], row[i, 1], zs[k])
    lin = Spline1D(_LIN, 1)
    return _orient((Spline1D([0, 0, .5, 1, 1], 1), lin, lin), ctrl, np.ones((3, 2, 2)),
                   {"name": "lshape", "params": p, "directions": ("path", "across", "height"),
                    "default_dirichlet": [[0, 0], [0, 1], [1, 0], [1, 1]]})


def ring(prm):
    p = _params(prm, {"r_in": 0.5, "r_out": 1.0, "h": 1.0})
    _need(0 < p["r_in"] < p["r_out"], "radii")
    _need(p["h"] > 0, "height")
    t, P, w = _circle9()
    rad = (p["r_in"], p["r_out"])
    zs = (0.0, p["h"])
    return _product([t, _LIN, _LIN], (2, 1, 1),
                    lambda i, j, k: ((P[i, 0] * rad[j], P[i, 1] * rad[j], zs[k]), w[i]),
                    {"name": "ring", "params": p, "directions": ("angular", "radial", "height"),
                     "default_dirichlet": [[1, 0], [1, 1]]})


def _hemi(prm, name, top, meta_extra):
    t, P, w = _circle9()
    ta, A, wa = _arc(0.0, top)
    rad = (prm["r_in"], prm["r_out"])

    def build(i, j, k):
        rho, z = A[j] * rad[k]
        return (P[i, 0] * rho, P[i, 1] * rho, z), w[i] * wa[j]

    meta = {"name": name, "params": prm, "directions": ("longitude", "latitude", "radial")}
    meta.update(meta_extra)
    return _product([t, ta, _LIN], (2, 2, 1), build, meta)


def closed_hemisphere(prm):
    p = _params(prm, {"r_in": 0.5, "r_out": 1.0})
    _need(0 < p["r_in"] < p["r_out"], "radii")
    return _hemi(p, "closed_hemisphere", 0.5 * np.pi,
                 {"default_dirichlet": [[2, 0], [2, 1]], "degenerate_faces": [[1, 1]]})


def opened_hemisphere(prm):
    p = _params(prm, {"r_in": 0.5, "r_out": 1.0, "hole_deg": 18.0})
    _need(0 < p["r_in"] < p["r_out"], "radii")
    _need(0 < p["hole_deg"] < 90, "hole angle")
    return _hemi(p, "opened_hemisphere", 0.5 * np.pi - np.deg2rad(p["hole_deg"]),
                 {"default_dirichlet": [[1, 0], [1, 1]]})


def hyperboloid(prm):
    p = _params(prm, {"r_middle": 0.5, "r_top": 1.0, "thickness": 0.3, "zmin": -1.0, "zmax": 1.0})
    _need(0 < p["r_middle"] < p["r_top"], "radii")
    _need(0 < p["thickness"] < 2 * p["r_middle"], "thickness")
    _need(p["zmin"] < p["zmax"], "z range")
    t, P, w = _circle9()
    th, H, wh = _hyperbola(p["r_top"], p["r_middle"], p["zmin"], p["zmax"])
    off = (-0.5 * p["thickness"], 0.5 * p["thickness"])

    def build(i, j, k):
        rho = H[j, 0] + off[k]
        return (P[i, 0] * rho, P[i, 1] * rho, H[j, 1]), w[i] * wh[j]

    return _product([t, th, _LIN], (2, 2, 1), build,
                    {"name": "hyperboloid", "params": p, "directions": ("angular", "height", "thickness"),
                     "default_dirichlet": [[1, 0], [1, 1]]})


def quarter_torus(prm):
    p = _params(prm, {"r_in": 0.5, "r_out": 1.0, "R": 3.0})
    _need(0 < p["r_in"] < p["r_out"], "radii")
    _need(p["R"] > p["r_out"], "major radius")
    tt_, T, wt = _arc(0.0, 0.5 * np.pi)
    t, P, w = _circle9()
    rad = (p["r_in"], p["r_out"])

    def build(i, j, k):
        rho = p["R"] + P[j, 0] * rad[k]
        return (T[i, 0] * rho, T[i, 1] * rho, P[j, 1] * rad[k]), wt[i] * w[j]

    return _product([tt_, t, _LIN], (2, 2, 1), build,
                    {"name": "quarter_torus", "params": p, "directions": ("toroidal", "poloidal", "radial"),
                     "default_dirichlet": [[2, 0], [2, 1]]})


def quarter_cylinder(prm):
    """EXTENSION (BASELINE config 2): quarter thick-walled cylinder.

    Angle 0..pi/2 as one exact rational quadratic arc (weights 1, sqrt2/2, 1),
    linear radial r_in..r_out and linear height 0..h. Directions (angular,
    radial, height) as the reference ring.
    """
    p = _params(prm, {"r_in": 1.0, "r_out": 2.0, "h": 1.0})
    _need(0 < p["r_in"] < p["r_out"], "radii")
    _need(p["h"] > 0, "height")
    ta, A, wa = _arc(0.0, 0.5 * np.pi)
    rad = (p["r_in"], p["r_out"])
    zs = (0.0, p["h"])
    return _product([ta, _LIN, _LIN], (2, 1, 1),
                    lambda i, j, k: ((A[i, 0] * rad[j], A[i, 1] * rad[j], zs[k]), wa[i]),
                    {"name": "quarter_cylinder", "params": p, "directions": ("angular", "radial", "height"),
                     "default_dirichlet": [[a, s] for a in range(3) for s in range(2)]})


def _greville_interpolant(degree, n_ctrl, fn):
    """Tensor B-spline interpolant of a map at Greville points (EXTENSION helper)."""
    sp = Spline1D.uniform(degree, n_ctrl - degree)
    g = sp.greville()
    C = dense_tables(sp, g)[0]
    X = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1)
    F = fn(X[..., 0], X[..., 1], X[..., 2])
    for ax in range(3):
        F = np.moveaxis(np.tensordot(np.linalg.inv(C), np.moveaxis(F, ax, 0), (1, 0)), 0, ax)
    return sp, F


def deformed_cube(prm):
    """EXTENSION (BASELINE config 3): degree-3 interpolant of the sine-deformed cube.

    x = xi + a sin(2 pi eta) sin(pi zeta), y = eta + a sin(2 pi zeta) sin(pi xi),
    z = zeta + a sin(2 pi xi) sin(pi eta), interpolated at the Greville points
    of an open uniform degree-3 basis with ``n_ctrl`` (16) functions.
    """
    p = _params(prm, {"amplitude": 0.1, "n_ctrl": 16, "degree": 3})
    a = p["amplitude"]
    deg, nc = int(p["degree"]), int(p["n_ctrl"])

    def fmap(u, v, s):
        return np.stack([u + a * np.sin(2 * np.pi * v) * np.sin(np.pi * s),
                         v + a * np.sin(2 * np.pi * s) * np.sin(np.pi * u),
                         s + a * np.sin(2 * np.pi * u) * np.sin(np.pi * v)], -1)

    sp, ctrl = _greville_interpolant(deg, nc, fmap)
    return _orient((sp, sp, sp), ctrl, np.ones(ctrl.shape[:3]),
                   {"name": "deformed_cube", "params": p, "directions": ("x", "y", "z"),
                    "default_dirichlet": [[ax, s] for ax in range(3) for s in range(2)]})


def gauss_grid(elements, points):
    """Gauss-Legendre points of ``elements`` uniform spans of [0, 1], ``points`` per span (the solve's
    quadrature of an open uniform solution basis, reference assembly.py:91-135 / driver.py n_basis mode)."""
    xg, _ = np.polynomial.legendre.leggauss(int(points))
    brk = np.linspace(0.0, 1.0, int(elements) + 1)
    return np.concatenate([0.5 * (a + b) + 0.5 * (b - a) * xg for a, b in zip(brk[:-1], brk[1:])])


def min_det_polynomial_grid(pt, axes, chunk=4):
    """min det J (and the count of det J <= 0) over the full tensor grid ``axes`` of a NON-rational patch
    (weights 1), by sum factorization: the three Jacobian columns on a slab of ``chunk`` first-direction
    points are D0 B1 B2 P, B0 D1 B2 P and B0 B1 D2 P (dense per-direction basis tables), so the 8.4e9-point
    Gauss grid of configs[3] costs ~6e11 flops instead of a per-point window gather."""
    if not np.all(pt.w == 1.0):
        raise PatchFault("min_det_polynomial_grid needs a polynomial (weight-1) patch")
    tabs = []
    for s, pts in zip(pt.sp, axes):
        B = np.zeros((pts.size, s.n))
        Dm = np.zeros((pts.size, s.n))
        for q, x in enumerate(pts):
            st, V, D = basis_window(s, float(x))
            B[q, st:st + s.p + 1] = V
            Dm[q, st:st + s.p + 1] = D
        tabs.append((B, Dm))
    (B0, D0), (B1, D1), (B2, D2) = tabs
    P = pt.ctrl
    mn, bad = np.inf, 0
    for i0 in range(0, B0.shape[0], chunk):
        TB = np.einsum("ia,abcx->ibcx", B0[i0:i0 + chunk], P)
        TD = np.einsum("ia,abcx->ibcx", D0[i0:i0 + chunk], P)
        Xa = np.einsum("kc,ijcx->ijkx", B2, np.einsum("jb,ibcx->ijcx", B1, TD))
        Xb = np.einsum("kc,ijcx->ijkx", B2, np.einsum("jb,ibcx->ijcx", D1, TB))
        Xc = np.einsum("kc,ijcx->ijkx", D2, np.einsum("jb,ibcx->ijcx", B1, TB))
        det = (Xa[..., 0] * (Xb[..., 1] * Xc[..., 2] - Xb[..., 2] * Xc[..., 1])
               - Xb[..., 0] * (Xa[..., 1] * Xc[..., 2] - Xa[..., 2] * Xc[..., 1])
               + Xc[..., 0] * (Xa[..., 1] * Xb[..., 2] - Xa[..., 2] * Xb[..., 1]))
        mn = min(mn, float(det.min()))
        bad += int((det <= 0).sum())
    return mn, bad


def random_cube(prm):
    """EXTENSION (BASELINE config 4): seeded random perturbation of a degree-3 cube net.

    Control points at the Greville abscissae (identity map) of an open uniform
    degree-3 basis with ``n_ctrl`` (8) functions per direction; every interior
    point gets i.i.d. N(0, sigma^2) offsets per coordinate from
    ``np.random.default_rng(seed)``; draws are rejected (next draw from the same
    generator) until det J > 0 at every point of the check grid. With
    ``check_gauss = (elements, points)`` (set by the solve driver) the check grid is the solve's own
    quadrature -- every Gauss point, as BASELINE configs[3] asks; without it, 8 Gauss-Legendre points
    per geometry knot span per direction.
    """
    p = _params(prm, {"sigma": 0.02, "n_ctrl": 8, "degree": 3, "seed": 0, "max_draws": 100, "check_gauss": None})
    deg, nc = int(p["degree"]), int(p["n_ctrl"])
    sp = Spline1D.uniform(deg, nc - deg)
    g = sp.greville()
    base = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1)
    rng = np.random.default_rng(int(p["seed"]))
    if p["check_gauss"] is not None:
        cg = np.asarray(p["check_gauss"], dtype=int).reshape(-1, 2)
        cg = np.repeat(cg, 3, axis=0) if cg.shape[0] == 1 else cg
        axes = [gauss_grid(E, q) for E, q in cg]
    else:
        xg, _ = np.polynomial.legendre.leggauss(8)
        brk = np.unique(sp.t)
        chk = np.concatenate([0.5 * (a + b) + 0.5 * (b - a) * xg for a, b in zip(brk[:-1], brk[1:])])
        axes = [chk, chk, chk]
    meta = {"name": "random_cube", "params": p, "directions": ("x", "y", "z"),
            "default_dirichlet": [[ax, s] for ax in range(3) for s in range(2)]}
    for draw in range(int(p["max_draws"])):
        ctrl = base.copy()
        ctrl[1:-1, 1:-1, 1:-1] += rng.normal(0.0, p["sigma"], size=(nc - 2, nc - 2, nc - 2, 3))
        pt = Patch((sp, sp, sp), ctrl, np.ones((nc, nc, nc)), meta)
        mn, bad = min_det_polynomial_grid(pt, axes)
        if bad == 0 and mn > 0:
            pt.meta["draws"] = draw + 1
            pt.meta["check_points"] = int(np.prod([a.size for a in axes]))
            pt.meta["min_det"] = mn
            return pt
    raise PatchFault("no admissible random draw")


FACTORIES = {
    "unit_cube": unit_cube,
    "lshape": lshape,
    "ring": ring,
    "closed_hemisphere": closed_hemisphere,
    "opened_hemisphere": opened_hemisphere,
    "hyperboloid": hyperboloid,
    "quarter_torus": quarter_torus,
    "quarter_cylinder": quarter_cylinder,
    "deformed_cube": deformed_cube,
    "random_cube": random_cube,
}


def build_patch(name, params=None) -> Patch:
    """Reference make_geometry (geometry.py:365-385) plus the EXTENSION solids."""
    if name not in FACTORIES:
        raise PatchFault(f"unknown geometry {name!r}")
    return FACTORIES[name](dict(params or {}))
