"""Synthetic BASELINE workloads and their algorithmic FLOP counts.

* ``matvec_round_instance``: the configs[4] kernel microbenchmark -- a 3-core
  TT-matrix with 1024 x 1024 modes and operator ranks 16 (cores i.i.d.
  N(0,1)/sqrt(rank), seeded), applied to a TT-vector with ranks 64 (same
  distribution), then rounded to 1e-8.
* ``solve_config``: the TT-IGA Poisson configs[0..4] as SolveConfig kwargs.

FLOP model: the nominal count of the reference algorithm's LAPACK path
(np.linalg.qr = dgeqrf + dorgqr; np.linalg.svd of a tall unfolding = dgesdd's m >> n path:
dgeqrf + dorgqr + SVD of R + Q U_R), independent of how the device executes it.
dense TT-matvec core k: 2 Ra Rb rc rd n m. Rounding: right-to-left per bond a
Householder QR of the (n r_k) x r_{k-1} unfolding (geqrf 2mn^2 - 2n^3/3, orgqr
the same) plus the R-carry GEMM 2 (r_{k-2} n_{k-1}) r_{k-1} k; left-to-right
per bond QR of the (r_{k-1} n) x r_k unfolding (both halves), the SVD
of the r x r factor (counted as 2 * 6 r^3 for ~6 Jacobi sweeps), U = Q U_R (2 m r
keep) and the carry GEMM 2 keep r_k (n r_{k+1}). The device path executes fewer flops on
very tall unfoldings (U = X V S^-1 without forming Q: the orgqr term is skipped), so the
GFLOP/s is nominal-flops / time; ms_per_step is the direct measure.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from .tensor_train import TtMatrix, TtTensor


def matvec_round_shapes(n=1024, R=16, r=64, d=3):
    Rs = [1] + [R] * (d - 1) + [1]
    rs = [1] + [r] * (d - 1) + [1]
    return Rs, rs


def matvec_round_instance(n=1024, R=16, r=64, d=3, seed=0, device="cuda"):
    """Seeded device instance (torch Philox on the GPU; the CPU sample re-draws with numpy)."""
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    Rs, rs = matvec_round_shapes(n, R, r, d)
    A = [torch.randn(Rs[k], n, n, Rs[k + 1], generator=g, device=device, dtype=torch.float64)
         / math.sqrt(R) for k in range(d)]
    X = [torch.randn(rs[k], n, rs[k + 1], generator=g, device=device, dtype=torch.float64) / math.sqrt(r)
         for k in range(d)]
    return TtMatrix(A), TtTensor(X)


def matvec_round_instance_np(n, R=16, r=64, d=3, seed=0):
    """Host (numpy) instance of the same shapes, for the CPU oracle sample."""
    rng = np.random.default_rng(seed)
    Rs, rs = matvec_round_shapes(n, R, r, d)
    A = [rng.standard_normal((Rs[k], n, n, Rs[k + 1])) / math.sqrt(R) for k in range(d)]
    X = [rng.standard_normal((rs[k], n, rs[k + 1])) / math.sqrt(r) for k in range(d)]
    return A, X


def _qr_flops(m, n):
    k = min(m, n)
    geqrf = 2.0 * m * n * k - (2.0 / 3.0) * k ** 3 if m >= n else 2.0 * n * m * k - (2.0 / 3.0) * k ** 3
    orgqr = 2.0 * m * k * k - (2.0 / 3.0) * k ** 3
    return geqrf + orgqr


def matvec_round_flops(n_rows, n_cols, Rs, rs, out_ranks):
    """Algorithmic FP64 flops of matvec + round for d cores (out_ranks: ranks after rounding)."""
    d = len(n_rows)
    f = 0.0
    Y = [Rs[k] * rs[k] for k in range(d + 1)]
    for k in range(d):
        f += 2.0 * Rs[k] * Rs[k + 1] * rs[k] * rs[k + 1] * n_rows[k] * n_cols[k]
    # right-to-left orthogonalization (ranks unchanged when full rank: k = min(n r, r_prev))
    ranks = list(Y)
    for k in range(d - 1, 0, -1):
        m, c = n_rows[k] * ranks[k + 1], ranks[k]
        kk = min(m, c)
        f += _qr_flops(m, c)
        f += 2.0 * (ranks[k - 1] * n_rows[k - 1]) * ranks[k] * kk
        ranks[k] = kk
    # left-to-right truncation
    for k in range(d - 1):
        m, c = ranks[k] * n_rows[k], ranks[k + 1]
        kk = min(m, c)
        keep = out_ranks[k + 1]
        f += _qr_flops(max(m, c), min(m, c)) + 12.0 * kk ** 3 + 2.0 * max(m, c) * kk * keep
        f += 2.0 * keep * ranks[k + 1] * n_rows[k + 1] * ranks[k + 2]
        ranks[k + 1] = keep
    return f


SOLVE_CONFIGS = {
    0: dict(geometry="unit_cube", degree=2, n_basis=32, source="manufactured_sines", analytic="cube_sines",
            eps_cross=1e-10, eps_round=1e-10, eps_solve=1e-10),
    1: dict(geometry="quarter_cylinder", degree=3, n_basis=128, source="manufactured_sines", analytic="cube_sines",
            bc_from_analytic=True, eps_cross=1e-8, eps_round=1e-8, eps_solve=1e-8),
    2: dict(geometry="deformed_cube", degree=3, n_basis=256, source="exp_sines", analytic="exp_sines",
            bc_from_analytic=True, eps_cross=1e-8, eps_round=1e-8, eps_solve=1e-8),
    3: dict(geometry="random_cube", degree=3, n_basis=512, source="one", eps_cross=1e-8, eps_round=1e-8,
            eps_solve=1e-8),
    4: dict(geometry="quarter_cylinder", degree=3, n_basis=1024, source="manufactured_sines", analytic="cube_sines",
            bc_from_analytic=True, eps_cross=1e-8, eps_round=1e-8, eps_solve=1e-8),
}
