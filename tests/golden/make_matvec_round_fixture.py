"""Oracle fixture for the benchmarked workload itself: round(A x, 1e-8) of the configs[4] kernel
microbenchmark (3-core TT-matrix, 1024 x 1024 modes, operator ranks 16, TT-vector ranks 64).

    python tests/golden/make_matvec_round_fixture.py [n ...]     (default: 1024)

The rounded tensor at n = 1024 has ranks (1, 1024, 1024, 1) and an 8.6 GB middle core, so the
fixture stores gauge-invariant summaries of the oracle's result instead of its cores:

* ``ranks``: the TT ranks after rounding;
* ``s1``, ``s2``: the singular values of the two unfoldings of the rounded tensor (the values the
  reference's ``_chop`` sees, reference tensor_train/core.py:341-389);
* ``idx``, ``vals``: the rounded tensor at 4096 seeded multi-indices (``TtTensor.gather``);
* ``norm``: its Frobenius norm;
* ``in_sums``: checksums of the seeded inputs (sum and sum of squares of every core), so a change
  of the input generator is caught before the comparison.

The inputs are ``workloads.matvec_round_instance_np(n, 16, 64, 3, seed=0)`` (numpy Generator),
uploaded unchanged by the GPU test. The oracle is the numpy restatement of reference
tensor_train/core.py:327-389 (oracle/tt.py), itself pinned to the reference's golden vectors.
Takes ~10 min and ~45 GB of host memory at n = 1024 (8 host threads).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import tt as OT  # noqa: E402
from paper_2509_13224_b200.workloads import matvec_round_instance_np  # noqa: E402

N_SAMPLE = 4096


def bond_singular_values(cores):
    """Singular values of every unfolding of a 3-core TT whose first two cores are left-orthonormal
    (the rounding's output gauge): bond 2 from the last core, bond 1 after moving the last core's
    R factor left."""
    G0, G1, G2 = cores
    r2, n2, _ = G2.shape
    s2 = np.linalg.svd(G2.reshape(r2, n2), compute_uv=False)
    Q, R = np.linalg.qr(G2.reshape(r2, n2).T)                       # G2 = R^T Q^T
    r1, n1, _ = G1.shape
    G1r = np.tensordot(G1, R.T, (2, 0))                             # (r1, n1, k)
    Q1, R1 = np.linalg.qr(G1r.reshape(r1, -1).T)
    G0r = np.tensordot(G0, R1.T, (2, 0))
    s1 = np.linalg.svd(G0r.reshape(-1, G0r.shape[2]), compute_uv=False)
    return s1, s2


def input_sums(A, X):
    return np.array([[float(G.sum()), float((G * G).sum())] for G in list(A) + list(X)])


def make(n, seed=0):
    A, X = matvec_round_instance_np(n, 16, 64, 3, seed)
    sums = input_sums(A, X)
    t = time.perf_counter()
    Y = OT.round_tt(OT.matvec(OT.TTOp(A), OT.TT(X)), 1e-8)
    dt = time.perf_counter() - t
    del A, X
    s1, s2 = bond_singular_values(Y.cores)
    rng = np.random.default_rng(7)
    idx = np.stack([rng.integers(0, n, N_SAMPLE) for _ in range(3)], axis=1)
    vals = Y.gather(idx)
    out = {f"n{n}_ranks": np.asarray(Y.ranks), f"n{n}_s1": s1, f"n{n}_s2": s2, f"n{n}_idx": idx.astype(np.int32),
           f"n{n}_vals": vals, f"n{n}_norm": np.asarray(OT.norm(Y)), f"n{n}_in_sums": sums,
           f"n{n}_oracle_s": np.asarray(dt)}
    print(f"n={n}: oracle {dt:.1f}s ranks {Y.ranks} norm {float(out[f'n{n}_norm']):.6e} "
          f"s1 [{s1[0]:.4e}..{s1[-1]:.4e}] s2 [{s2[0]:.4e}..{s2[-1]:.4e}]", flush=True)
    return out


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [1024]
    path = os.path.join(HERE, "matvec_round_oracle.npz")
    out = dict(np.load(path)) if os.path.exists(path) else {}
    for n in sizes:
        out.update(make(n))
        np.savez_compressed(path, **out)
    print("wrote", path)


if __name__ == "__main__":
    main()
