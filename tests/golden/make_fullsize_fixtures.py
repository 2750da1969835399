"""Oracle fixtures at the FULL BASELINE sizes of configs[2] and configs[4] (plus configs[3]'s assembly).

    python tests/golden/make_fullsize_fixtures.py [c4] [c2] [c3]      (default: c4 c2)

* ``c4``: configs[4] (quarter cylinder, p=3, n=1024 per direction, 1.07e9 dofs) solved by the
  oracle restatement of reference driver.py:455-532 with the parity setting eps_solve = 1e-12
  (both sides then stop far below the 1e-9 parity bar instead of at the 1e-8 residual target, so
  their solutions can be compared at 1e-9). The operator ranks are 2, so the reference algorithm
  (explicit residual, amen.py:262-264) runs on the host. Stored: the stiffness cores in the banded
  layout (the dense ones are zero outside |i - j| <= p; checked here), load and solution cores,
  ranks, residual, sweeps.
* ``c2``: configs[2] (interpolated deformed cube, p=3, n=256, operator ranks ~109) ASSEMBLY
  (reference assembly.py:236-304): the load cores in full, and for the 190 MB stiffness TT its
  gauge-invariant summaries -- ranks, the singular values of both unfoldings, the Frobenius norm
  and 4096 seeded entries K[(i0,i1,i2),(j0,j1,j2)] with |i_d - j_d| <= p.
* ``c3``: the same assembly summaries for configs[3] (seeded random cube, n=512) -- beyond this
  container's memory (the oracle's dense operator cores are 30 GB each); ``c3n128`` is the same
  configuration at n=128 (geometry, det J check on the solve's Gauss grid, cross, rounding).

The AMEn solve of configs[2]/[3] is out of the oracle's reach (its explicit residual core is
~100 GB / ~0.5 TB), see DESIGN.md §5b.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import iga as OI  # noqa: E402
from oracle import tt as OT  # noqa: E402
from paper_2509_13224_b200.workloads import SOLVE_CONFIGS  # noqa: E402

PATH = os.path.join(HERE, "configs_fullsize_oracle.npz")
N_SAMPLE = 4096
PARITY_EPS_SOLVE = 1e-12


def banded(G, h):
    """(r0, n, n, r1) dense operator core -> (r0, n, 2h+1, r1) band [a, i, t, b] = G[a, i, i+t-h, b]."""
    r0, n, m, r1 = G.shape
    B = np.zeros((r0, n, 2 * h + 1, r1))
    ii = np.arange(n)
    for t in range(2 * h + 1):
        o = t - h
        ok = (ii + o >= 0) & (ii + o < m)
        B[:, ii[ok], t, :] = G[:, ii[ok], ii[ok] + o, :]
    mask = np.abs(ii[:, None] - np.arange(m)[None, :]) > h
    assert float(np.abs(G[:, mask, :]).max(initial=0.0)) == 0.0, "operator core not banded"
    return B


def op_bond_singular_values(K):
    """Singular values of both unfoldings of a 3-core operator TT (fused (i, j) modes)."""
    C = [G.reshape(G.shape[0], -1, G.shape[3]) for G in K.cores]
    C, _ = OT._rl_orth(C, False)               # cores 1, 2 right-orthonormal
    s1 = np.linalg.svd(C[0].reshape(-1, C[0].shape[2]), compute_uv=False)
    U, s, Vt = np.linalg.svd(C[0].reshape(-1, C[0].shape[2]), full_matrices=False)
    C1 = np.tensordot(s[:, None] * Vt, C[1], (1, 0))
    s2 = np.linalg.svd(C1.reshape(-1, C1.shape[2]), compute_uv=False)
    return s1, s2


def op_samples(K, p, seed=11):
    rng = np.random.default_rng(seed)
    n = K.row_sizes
    I = np.stack([rng.integers(0, n[d], N_SAMPLE) for d in range(3)], 1)
    J = np.stack([np.clip(I[:, d] + rng.integers(-p, p + 1, N_SAMPLE), 0, n[d] - 1) for d in range(3)], 1)
    v = np.ones((N_SAMPLE, 1))
    for d in range(3):
        G = K.cores[d][:, I[:, d], J[:, d], :]                   # (r0, N, r1)
        v = np.einsum("nr,rns->ns", v, G)
    return I.astype(np.int32), J.astype(np.int32), v[:, 0]


def c4():
    kw = dict(SOLVE_CONFIGS[4], eps_solve=PARITY_EPS_SOLVE)
    t = time.perf_counter()
    r = OI.solve(OI.Config(seed=0, **kw), want_error=False)
    dt = time.perf_counter() - t
    p = max(kw["degree"]) if not np.isscalar(kw["degree"]) else kw["degree"]
    out = {"c4_eps_solve": np.asarray(PARITY_EPS_SOLVE), "c4_oracle_s": np.asarray(dt)}
    for k, G in enumerate(r["K"].cores):
        out[f"c4_K{k}"] = banded(G, p)
    for k, G in enumerate(r["f"].cores):
        out[f"c4_f{k}"] = G
    for k, G in enumerate(r["u"].cores):
        out[f"c4_u{k}"] = G
    for key in ("ranks_K", "ranks_f", "ranks_u"):
        out[f"c4_{key}"] = np.asarray(r[key])
    out["c4_residual"] = np.asarray(r["residual"])
    out["c4_sweeps"] = np.asarray(r["sweeps"])
    out["c4_converged"] = np.asarray(bool(r["solver_converged"]))
    print(f"c4: oracle {dt:.1f}s timings {r['timings']} ranks K {r['ranks_K']} f {r['ranks_f']} u {r['ranks_u']} "
          f"residual {r['residual']:.3e} sweeps {r['sweeps']}", flush=True)
    return out


def assembly_summary(tag, c, n_basis=None):
    kw = dict(SOLVE_CONFIGS[c])
    if n_basis is not None:
        kw["n_basis"] = n_basis
    cfg = OI.Config(seed=0, **kw)
    t = time.perf_counter()
    patch = OI.build_patch(cfg.geometry, OI.geometry_params(cfg))
    cfg.resolve(patch)
    disc = OI.discretize(cfg, patch)
    rK, rf = OI._seeds(cfg.seed, 2)
    K, _ = OI.stiffness(patch, disc, cfg.eps_round, cfg.rank_cap, rK)
    tK = time.perf_counter() - t
    f, _ = OI.load(patch, disc, OI.SOURCES[cfg.source], cfg.eps_cross, cfg.rank_cap, rf)
    dt = time.perf_counter() - t
    p = cfg.degree[0]
    s1, s2 = op_bond_singular_values(K)
    I, J, v = op_samples(K, p)
    out = {f"{tag}_ranks_K": np.asarray(K.ranks), f"{tag}_ranks_f": np.asarray(f.ranks), f"{tag}_K_s1": s1,
           f"{tag}_K_s2": s2, f"{tag}_K_norm": np.asarray(OT.norm(K)), f"{tag}_K_I": I, f"{tag}_K_J": J,
           f"{tag}_K_vals": v, f"{tag}_oracle_s": np.asarray(dt)}
    for k, G in enumerate(f.cores):
        out[f"{tag}_f{k}"] = G
    print(f"{tag}: oracle assembly {dt:.1f}s (K {tK:.1f}s) ranks K {K.ranks} f {f.ranks}", flush=True)
    return out


def main():
    which = sys.argv[1:] or ["c4", "c2"]
    out = dict(np.load(PATH)) if os.path.exists(PATH) else {}
    for w in which:
        out = {k: v for k, v in out.items() if not k.startswith(w + "_")}
        if w == "c4":
            out.update(c4())
        elif w == "c3n128":
            out.update(assembly_summary(w, 3, 128))
        else:
            out.update(assembly_summary(w, int(w[1])))
        np.savez_compressed(PATH, **out)
    print("wrote", PATH)


if __name__ == "__main__":
    main()
