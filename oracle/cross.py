"""Oracle: maxvol pivoting and rank-adaptive TT-cross (TEST INFRASTRUCTURE ONLY).

Restates reference ``tensor_train/maxvol.py`` and ``tensor_train/cross.py``.
The random stream is consumed in exactly the reference order so a shared
seed reproduces the reference's holdout sample and column sets.
"""

from __future__ import annotations

import numpy as np

from . import tt as T


class MaxvolFault(np.linalg.LinAlgError):
    """Mirror of reference MaxvolError (maxvol.py:15)."""


def gepp_rows(M):
    """First r rows of the partial-pivoting row order (reference maxvol.py:19-34)."""
    A = np.array(M, dtype=float)
    n, r = A.shape
    order = np.arange(n)
    big = np.max(np.abs(A), initial=0.0)
    for k in range(r):
        j = k + int(np.argmax(np.abs(A[k:, k])))
        if abs(A[j, k]) <= 1e-14 * max(big, 1e-300):
            raise MaxvolFault("rank-deficient columns")
        if j != k:
            A[[k, j]] = A[[j, k]]
            order[[k, j]] = order[[j, k]]
        A[k + 1:, k] /= A[k, k]
        A[k + 1:, k + 1:] -= np.outer(A[k + 1:, k], A[k, k + 1:])
    return order[:r]


def maxvol(M, tol=1.01, max_iters=200):
    """Reference maxvol (maxvol.py:37-62): greedy Sherman-Morrison row swaps."""
    M = np.asarray(M, dtype=float)
    if M.ndim != 2:
        raise ValueError("maxvol expects a matrix")
    n, r = M.shape
    if tol < 1.0:
        raise ValueError("tol must be >= 1")
    if n <= r:
        return np.arange(n)
    rows = gepp_rows(M)
    C = np.linalg.solve(M[rows].T, M.T).T
    for _ in range(max_iters):
        i, j = np.unravel_index(int(np.argmax(np.abs(C))), C.shape)
        if abs(C[i, j]) <= tol:
            break
        u = C[i].copy()
        u[j] -= 1.0
        C -= np.outer(C[:, j], u) / C[i, j]
        rows[j] = i
    return np.sort(rows)


class Counted:
    """Evaluation counter around an index->value oracle (reference cross.py:58-69)."""

    def __init__(self, fn):
        self.fn, self.n = fn, 0

    def __call__(self, idx):
        idx = np.asarray(idx, dtype=np.intp)
        self.n += idx.shape[0]
        v = np.asarray(self.fn(idx), dtype=float)
        if v.shape != (idx.shape[0],):
            raise ValueError("oracle must return one value per index")
        return v


def fresh_tuples(rng, sizes, count, have=()):
    """Reference _random_tuples (cross.py:72-85), same rng call order."""
    out = list(have)
    seen = set(out)
    tries = 0
    while len(out) < count:
        c = tuple(int(rng.integers(0, n)) for n in sizes)
        if c not in seen:
            out.append(c)
            seen.add(c)
        tries += 1
        if tries > 100 * count + 1000:
            break
    return out


def fiber_index(left, nk, right, k, d):
    """Multi-indices of the unfolding C[(l, i_k), r] (reference cross.py:88-100)."""
    nl, nr = len(left), len(right)
    L = np.asarray(left, dtype=np.intp).reshape(nl, k)
    Rr = np.asarray(right, dtype=np.intp).reshape(nr, d - k - 1)
    idx = np.empty((nl * nk * nr, d), dtype=np.intp)
    if k > 0:
        idx[:, :k] = np.repeat(L, nk * nr, 0)
    idx[:, k] = np.tile(np.repeat(np.arange(nk), nr), nl)
    if k + 1 < d:
        idx[:, k + 1:] = np.tile(Rr, (nl * nk, 1))
    return idx


def cross(fn, sizes, eps, rank_cap=64, max_sweeps=20, holdout_size=1000, rng=None, scale=None):
    """Reference tt_cross (cross.py:103-222).

    Returns (TT, holdout_error, converged, n_evals, sweeps).
    """
    if eps <= 0 or rank_cap < 1 or max_sweeps < 1:
        raise ValueError("bad cross parameters")
    rng = rng or np.random.default_rng()
    sizes = tuple(int(n) for n in sizes)
    d = len(sizes)
    f = Counted(fn)
    hidx = np.stack([rng.integers(0, n, size=holdout_size) for n in sizes], 1)
    hval = f(hidx)
    hrms = float(np.sqrt(np.mean(hval ** 2)))
    if scale is None or scale <= 0.0:
        scale = hrms
    if hrms <= eps * scale:
        return T.TT.zeros(sizes), (hrms / scale if scale > 0 else 0.0), True, f.n, 0
    cap = [min(int(np.prod(sizes[: k + 1])), int(np.prod(sizes[k + 1:])), rank_cap) for k in range(d - 1)]
    ranks = [1] * (d - 1)
    rsets = [fresh_tuples(rng, sizes[k + 1:], ranks[k]) for k in range(d - 1)]

    def herr(t):
        return float(np.sqrt(np.mean((t.gather(hidx) - hval) ** 2))) / scale

    err, cores, done = np.inf, None, 0
    for sweep in range(max_sweeps):
        lsets = [[()]]
        for k in range(d - 1):
            C = f(fiber_index(lsets[k], sizes[k], rsets[k], k, d)).reshape(len(lsets[k]) * sizes[k], -1)
            Q, _ = np.linalg.qr(C)
            sel = maxvol(Q)
            cand = [l + (i,) for l in lsets[k] for i in range(sizes[k])]
            lsets.append([cand[s] for s in sel])
            ranks[k] = len(sel)
        cores = [None] * d
        rsets = [None] * (d - 1)
        cur = [()]
        for k in range(d - 1, 0, -1):
            nl, nr = len(lsets[k]), len(cur)
            C = f(fiber_index(lsets[k], sizes[k], cur, k, d)).reshape(nl * sizes[k], nr)
            Q, _ = np.linalg.qr(C.reshape(nl, sizes[k] * nr).T)
            sel = maxvol(Q)
            cores[k] = np.linalg.solve(Q[sel].T, Q.T).reshape(len(sel), sizes[k], nr)
            cand = [(i,) + r for i in range(sizes[k]) for r in cur]
            cur = [cand[s] for s in sel]
            rsets[k - 1] = cur
            ranks[k - 1] = len(sel)
        cores[0] = f(fiber_index([()], sizes[0], cur, 0, d)).reshape(1, sizes[0], len(cur))
        done = sweep + 1
        err = herr(T.TT(cores))
        if err <= eps:
            break
        if all(r >= c for r, c in zip(ranks, cap)):
            break
        for k in range(d - 1):
            rsets[k] = fresh_tuples(rng, sizes[k + 1:], min(2 * ranks[k], cap[k]), have=rsets[k])
    tens = T.TT(cores)
    trimmed = T.round_tt(tens, 0.5 * eps)
    et = herr(trimmed)
    if et <= max(eps, err):
        tens, err = trimmed, et
    return tens, err, err <= 10 * eps, f.n, done
