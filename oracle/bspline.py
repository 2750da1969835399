"""Oracle: univariate B-spline / NURBS machinery (TEST INFRASTRUCTURE ONLY).

Restates reference ``pkg/src/ttiga/splines.py``. A basis is described by a
``Spline1D`` record (knots, degree, optional weights); evaluation follows
the Cox-de Boor triangle (NURBS Book A2.2) with first derivatives from the
degree p-1 row (A2.3), rational values by the quotient rule.
"""

from __future__ import annotations

import numpy as np


class SplineFault(ValueError):
    """Mirror of reference ``SplineError`` (splines.py:37)."""


class Spline1D:
    """Clamped knot vector + degree (+ weights for NURBS).

    Validation mirrors reference KnotVector.__post_init__ (splines.py:52-68)
    and Basis1D.__post_init__ (splines.py:108-115).
    """

    def __init__(self, knots, degree, weights=None):
        t = np.asarray(knots, dtype=float)
        p = int(degree)
        if p < 0:
            raise SplineFault("negative degree")
        if t.ndim != 1 or t.size < 2 * p + 2:
            raise SplineFault("too few knots")
        if np.any(t[1:] < t[:-1]):
            raise SplineFault("knots decrease")
        if np.any(t[: p + 1] != t[0]) or np.any(t[t.size - p - 1:] != t[-1]):
            raise SplineFault("ends not clamped")
        inner = t[p + 1: t.size - p - 1]
        if inner.size and np.max(np.unique(inner, return_counts=True)[1]) > p:
            raise SplineFault("interior multiplicity > degree")
        self.t = t
        self.p = p
        self.n = t.size - p - 1
        if weights is not None:
            w = np.asarray(weights, dtype=float)
            if w.shape != (self.n,):
                raise SplineFault("weight count")
            if np.any(w <= 0):
                raise SplineFault("weights must be positive")
            self.w = w
        else:
            self.w = None

    @staticmethod
    def uniform(p, spans):
        """Open uniform knots on [0,1] (reference splines.py:92-98)."""
        if spans < 1:
            raise SplineFault("need a span")
        mids = np.linspace(0.0, 1.0, spans + 1)[1:-1]
        return Spline1D(np.r_[np.zeros(p + 1), mids, np.ones(p + 1)], p)

    def nonempty_spans(self):
        """Reference KnotVector.spans (splines.py:86-89)."""
        return np.flatnonzero(self.t[1:] > self.t[:-1])

    def greville(self):
        """Knot averages (reference splines.py:284-291)."""
        if self.p == 0:
            return 0.5 * (self.t[:-1] + self.t[1:])
        return np.array([self.t[i + 1: i + self.p + 1].mean() for i in range(self.n)])


def span_index(sp: Spline1D, x: float) -> int:
    """Reference find_span (splines.py:146-161) incl. right-end clamp."""
    t = sp.t
    if x < t[0] or x > t[-1]:
        raise SplineFault(f"{x} outside [{t[0]}, {t[-1]}]")
    if x >= t[sp.n]:
        k = sp.n - 1
        while t[k] == t[k + 1]:
            k -= 1
        return k
    return int(np.searchsorted(t, x, side="right")) - 1


def _poly_window(t, p, k, x):
    """Nonzero degree-p values and derivatives on span k.

    Restates reference _bspline_values_derivs (splines.py:164-202): the
    triangular Cox-de Boor table with the 0/0 := 0 convention; derivatives
    from the saved degree-(p-1) row.
    """
    N = [1.0]
    low = [1.0]
    for j in range(1, p + 1):
        if j == p:
            low = list(N)
        nxt = [0.0] * (j + 1)
        carry = 0.0
        for r in range(j):
            a = x - t[k + 1 - j + r]          # left[j-r]
            b = t[k + 1 + r] - x              # right[r+1]
            den = a + b
            q = N[r] / den if den != 0.0 else 0.0
            nxt[r] = carry + b * q
            carry = a * q
        nxt[j] = carry
        N = nxt
    dN = np.zeros(p + 1)
    if p > 0:
        for j in range(p + 1):
            i = k - p + j
            acc = 0.0
            if j > 0:
                den = t[i + p] - t[i]
                if den != 0.0:
                    acc += p / den * low[j - 1]
            if j < p:
                den = t[i + p + 1] - t[i + 1]
                if den != 0.0:
                    acc -= p / den * low[j]
            dN[j] = acc
    return np.array(N), dN


def basis_window(sp: Spline1D, x: float):
    """(first_index, values, derivs) at x (reference eval_basis, splines.py:205-221)."""
    k = span_index(sp, x)
    v, d = _poly_window(sp.t, sp.p, k, x)
    if sp.w is not None:
        w = sp.w[k - sp.p: k + 1]
        W = float(v @ w)
        dW = float(d @ w)
        v, d = v * w / W, (d * w * W - v * w * dW) / (W * W)
    return k - sp.p, v, d


def dense_tables(sp: Spline1D, xs):
    """Dense (len(xs), n) value/derivative tables (reference tabulate, splines.py:294-310)."""
    xs = np.atleast_1d(np.asarray(xs, dtype=float))
    V = np.zeros((xs.size, sp.n))
    D = np.zeros((xs.size, sp.n))
    for r, x in enumerate(xs):
        i0, v, d = basis_window(sp, float(x))
        V[r, i0: i0 + sp.p + 1] = v
        D[r, i0: i0 + sp.p + 1] = d
    return V, D


def knot_insert(sp: Spline1D, ctrl, x):
    """Boehm insertion; rational bases in homogeneous coordinates.

    Restates reference insert_knot (splines.py:224-267).
    """
    t, p = sp.t, sp.p
    if not (t[0] < x < t[-1]):
        raise SplineFault("knot outside open range")
    if int(np.count_nonzero(t == x)) >= p:
        raise SplineFault("multiplicity would exceed degree")
    ctrl = np.asarray(ctrl, dtype=float)
    if ctrl.shape[0] != sp.n:
        raise SplineFault("control count")
    if sp.w is not None:
        flat = ctrl.reshape(sp.n, -1)
        hom = np.hstack([flat * sp.w[:, None], sp.w[:, None]])
        sp2, hom2 = knot_insert(Spline1D(t, p), hom, x)
        w2 = hom2[:, -1]
        return Spline1D(sp2.t, p, w2), (hom2[:, :-1] / w2[:, None]).reshape((w2.size,) + ctrl.shape[1:])
    k = span_index(sp, x)
    out = np.empty((sp.n + 1,) + ctrl.shape[1:])
    out[: k - p + 1] = ctrl[: k - p + 1]
    out[k + 1:] = ctrl[k:]
    for i in range(k - p + 1, k + 1):
        den = t[i + p] - t[i]
        a = (x - t[i]) / den if den != 0.0 else 0.0
        out[i] = a * ctrl[i] + (1.0 - a) * ctrl[i - 1]
    return Spline1D(np.insert(t, k + 1, x), p), out


def bisect_refine(sp: Spline1D, ctrl, levels: int):
    """Reference h_refine_uniform (splines.py:270-281)."""
    if levels < 0:
        raise SplineFault("levels < 0")
    for _ in range(levels):
        mids = [0.5 * (sp.t[i] + sp.t[i + 1]) for i in sp.nonempty_spans()]
        for m in mids:
            sp, ctrl = knot_insert(sp, ctrl, m)
    return sp, ctrl


def solution_space(geo: Spline1D, degree: int, elements: int) -> Spline1D:
    """Degree-p polynomial solution basis on a bisection of the geometry breaks.

    Restates reference driver.solution_basis (driver.py:259-288): span count
    snaps to base*2^k >= elements; geometry breakpoints keep multiplicity
    max(1, p - (p_geo - mult)).
    """
    vals, mult = np.unique(geo.t, return_counts=True)
    base = vals.size - 1
    lev = 0
    while base * 2 ** lev < elements:
        lev += 1
    brk = list(vals)
    for _ in range(lev):
        brk = sorted(brk + [0.5 * (a + b) for a, b in zip(brk[:-1], brk[1:])])
    keep = {float(v): max(1, degree - (geo.p - int(c))) for v, c in zip(vals[1:-1], mult[1:-1])}
    kn = [0.0] * (degree + 1)
    for b in brk[1:-1]:
        kn += [b] * keep.get(float(b), 1)
    kn += [1.0] * (degree + 1)
    return Spline1D(np.array(kn), degree)


def solution_space_exact(geo: Spline1D, degree: int, n_basis: int) -> Spline1D:
    """EXTENSION (BASELINE configs name an exact basis count per direction).

    Open uniform knots with ``n_basis`` functions. Geometry breakpoints of
    reduced continuity (multiplicity rule of :func:`solution_space` > 1)
    cannot be honoured by a uniform grid and are rejected; none of the
    BASELINE geometries has any.
    """
    spans = n_basis - degree
    if spans < 1:
        raise SplineFault("n_basis must exceed degree")
    vals, mult = np.unique(geo.t, return_counts=True)
    for c in mult[1:-1]:
        if max(1, degree - (geo.p - int(c))) > 1:
            raise SplineFault("exact-count solution space cannot keep a reduced-continuity geometry line")
    kn = np.linspace(0.0, 1.0, spans + 1)[1:-1]
    return Spline1D(np.r_[np.zeros(degree + 1), kn, np.ones(degree + 1)], degree)
