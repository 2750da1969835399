"""The reference's own experiment set on the GPU, with the CPU oracle beside it.

SPEC acceptance criteria 1-5 (L-shape p=1 ladder, ring p=2 ladder, six-geometry
bench, ring compression ladder, ring_large 4.2e6 dofs): per run the GPU solve time
(assembly + BC + AMEn, device-synchronized) and, unless --gpu-only, the oracle's.
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import driver as D  # noqa: E402

RING_BC = {"faces": {(1, 0): 1.0, (1, 1): 2.0}}

RUNS = [
    ("lshape p1 e8", dict(geometry="lshape", degree=1, elements=8, source="sin_pi_xy", analytic="lshape_exact")),
    ("lshape p1 e32", dict(geometry="lshape", degree=1, elements=32, source="sin_pi_xy", analytic="lshape_exact")),
    ("ring p2 e16", dict(geometry="ring", degree=2, elements=16, source="zero", analytic="ring_radial", ring=True)),
    ("ring p2 e64", dict(geometry="ring", degree=2, elements=64, source="zero", ring=True)),
    ("ring p2 e160 (>=4e6 dofs)", dict(geometry="ring", degree=2, elements=160, source="zero", ring=True)),
    ("closed_hemisphere p2 e8", dict(geometry="closed_hemisphere", degree=2, elements=8, source="sin_pi_xyz")),
    ("opened_hemisphere p2 e8", dict(geometry="opened_hemisphere", degree=2, elements=8, source="sin_pi_xyz")),
    ("hyperboloid p2 e8", dict(geometry="hyperboloid", degree=2, elements=8, source="sin_pi_xyz")),
    ("quarter_torus p2 e8", dict(geometry="quarter_torus", degree=2, elements=8, source="sin_pi_xyz")),
    ("quarter_torus p2 e32", dict(geometry="quarter_torus", degree=2, elements=32, source="sin_pi_xyz")),
]


def solve_gpu(kw):
    kw = dict(kw)
    ring = kw.pop("ring", False)
    if ring:
        kw["bc"] = D.BoundarySpec({(1, 0): D.FaceCondition("dirichlet", 1.0), (1, 1): D.FaceCondition("dirichlet", 2.0)})
    D.solve_poisson(D.SolveConfig(seed=0, **kw), want_error=False)  # warm
    if ring:
        kw["bc"] = D.BoundarySpec({(1, 0): D.FaceCondition("dirichlet", 1.0), (1, 1): D.FaceCondition("dirichlet", 2.0)})
    torch.cuda.synchronize()
    r = D.solve_poisson(D.SolveConfig(seed=0, **kw), want_error=kw.get("analytic") is not None)
    t = sum(v for k, v in r.timings.items() if k != "t_error_s")
    return t, r


def solve_cpu(kw):
    from oracle import iga as OI
    kw = dict(kw)
    if kw.pop("ring", False):
        kw["bc"] = OI.Bc({(1, 0): OI.Face("dirichlet", 1.0), (1, 1): OI.Face("dirichlet", 2.0)})
    r = OI.solve(OI.Config(seed=0, **kw), want_error=False)
    return sum(v for k, v in r["timings"].items() if k != "t_error_s"), r


if __name__ == "__main__":
    gpu_only = "--gpu-only" in sys.argv
    for name, kw in RUNS:
        tg, r = solve_gpu(kw)
        rec = {"run": name, "dofs": r.dofs, "gpu_s": round(tg, 4), "ranks_K": r.ranks_K, "ranks_u": r.ranks_u,
               "residual": r.residual, "l2_error": r.l2_error, "sweeps": r.sweeps}
        if not gpu_only:
            tc, rc = solve_cpu(kw)
            rec.update(cpu_s=round(tc, 3), speedup=round(tc / tg, 1), cpu_ranks_u=rc["ranks_u"])
        print(json.dumps(rec), flush=True)
