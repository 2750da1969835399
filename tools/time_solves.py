"""Time GPU solves of the BASELINE configs (device time per phase) -- development probe."""
import json, sys, time
import torch
from paper_2509_13224_b200 import driver as D

CFG = {
    0: dict(geometry="unit_cube", degree=2, n_basis=32, source="manufactured_sines", analytic="cube_sines",
            eps_cross=1e-10, eps_round=1e-10, eps_solve=1e-10),
    1: dict(geometry="quarter_cylinder", degree=3, n_basis=128, source="manufactured_sines", analytic="cube_sines",
            bc_from_analytic=True, eps_cross=1e-8, eps_round=1e-8, eps_solve=1e-8),
}
which = [int(a) for a in sys.argv[1:]] or [0, 1]
for c in which:
    for rep in range(2):
        t = time.perf_counter()
        r = D.solve_poisson(D.SolveConfig(seed=0, **CFG[c]), want_error=True)
        torch.cuda.synchronize()
        print(json.dumps({"config": c, "rep": rep, "wall_s": time.perf_counter() - t, "ranks_K": r.ranks_K,
                          "ranks_f": r.ranks_f, "ranks_u": r.ranks_u, "l2": r.l2_error, "res": r.residual,
                          "sweeps": r.sweeps, "timings": {k: round(v, 4) for k, v in r.timings.items()}}), flush=True)
