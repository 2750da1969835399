"""Oracle fixtures for the non-separable BASELINE configs at sizes the CPU oracle needs minutes for.

configs[2] (interpolated deformed cube) and configs[3] (seeded random cube) are
EXTENSIONS (the reference ships neither geometry), so their fixtures
come from the oracle restatement -- itself pinned bit-for-bit to the reference's
golden vectors (tests/test_oracle_golden.py) -- run here once:

    python tests/golden/make_config_fixtures.py

Writes ``tests/golden/configs_oracle.npz``: solution cores, load cores, ranks,
residual, sweeps and L2 error for each case. At these sizes the device solve takes
the GEMM-staged banded operator and the compressed residual (operator ranks 55-75),
so tests/test_gpu_configs.py checks those paths against the oracle without running
the oracle on the GPU box.
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
from paper_2509_13224_b200.workloads import SOLVE_CONFIGS  # noqa: E402

CASES = {"c2_n16": (2, 16, None), "c3_n10": (3, 10, None)}


def main():
    out = {}
    for tag, (c, n, solver) in CASES.items():
        kw = dict(SOLVE_CONFIGS[c], n_basis=n)
        if solver:
            kw["solver"] = solver
        t = time.perf_counter()
        r = OI.solve(OI.Config(seed=0, **kw))
        print(tag, f"{time.perf_counter() - t:.1f}s", r["ranks_K"], r["ranks_u"], r["residual"], r["l2_error"])
        for k, G in enumerate(r["u"].cores):
            out[f"{tag}_u{k}"] = G
        for k, G in enumerate(r["f"].cores):
            out[f"{tag}_f{k}"] = G
        out[f"{tag}_ranks_K"] = np.asarray(r["ranks_K"])
        out[f"{tag}_ranks_f"] = np.asarray(r["ranks_f"])
        out[f"{tag}_ranks_u"] = np.asarray(r["ranks_u"])
        out[f"{tag}_residual"] = np.asarray(r["residual"])
        out[f"{tag}_converged"] = np.asarray(bool(r["solver_converged"]))
        out[f"{tag}_sweeps"] = np.asarray(r["sweeps"])
        out[f"{tag}_l2_error"] = np.asarray(np.nan if r["l2_error"] is None else float(r["l2_error"]))
    np.savez_compressed(os.path.join(HERE, "configs_oracle.npz"), **out)
    print("wrote configs_oracle.npz")


if __name__ == "__main__":
    main()
