"""Run one BASELINE solve config on the GPU and print its report (development / evidence tool)."""
import json, sys, time
import torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import driver as D
from paper_2509_13224_b200.workloads import SOLVE_CONFIGS

c = int(sys.argv[1])
kw = dict(SOLVE_CONFIGS[c])
for a in sys.argv[2:]:
    k, v = a.split("=")
    kw[k] = json.loads(v)
want_err = kw.pop("want_error", True)
t = time.perf_counter()
r = D.solve_poisson(D.SolveConfig(seed=0, **kw), want_error=want_err)
torch.cuda.synchronize()
print(json.dumps({"config": c, "overrides": sys.argv[2:], "wall_s": time.perf_counter() - t, "dofs": r.dofs,
                  "ranks_K": r.ranks_K, "ranks_f": r.ranks_f, "ranks_u": r.ranks_u, "l2_error": r.l2_error,
                  "residual": r.residual, "converged": r.solver_converged, "sweeps": r.sweeps,
                  "cross_converged": r.cross_converged, "compression_K": r.compression_K,
                  "compression_u": r.compression_u, "timings": {k: round(v, 4) for k, v in r.timings.items()},
                  "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
