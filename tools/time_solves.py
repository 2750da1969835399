"""Time GPU solves of the BASELINE configs at full size, several reps in one process (device-
synchronized phase times). Usage: python tools/time_solves.py [configs...] [--reps R]"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import driver as D  # noqa: E402
from paper_2509_13224_b200.workloads import SOLVE_CONFIGS  # noqa: E402

args = sys.argv[1:]
reps = 2
if "--reps" in args:
    i = args.index("--reps")
    reps = int(args[i + 1])
    del args[i:i + 2]
pool = 0
if "--pool-gb" in args:
    i = args.index("--pool-gb")
    pool = float(args[i + 1])
    del args[i:i + 2]
which = [int(a) for a in args] or [0, 1]
if pool:
    # reserve the caching allocator's pool up front (one cudaMalloc, kept by the allocator)
    t = time.perf_counter()
    blk = torch.empty(int(pool * 1e9) // 8, dtype=torch.float64, device="cuda")
    del blk
    torch.cuda.synchronize()
    print(json.dumps({"pool_gb": pool, "reserve_s": round(time.perf_counter() - t, 3)}), flush=True)
for c in which:
    for rep in range(reps):
        t = time.perf_counter()
        r = D.solve_poisson(D.SolveConfig(seed=0, **SOLVE_CONFIGS[c]), want_error=c in (0, 2))
        torch.cuda.synchronize()
        print(json.dumps({"config": c, "rep": rep, "wall_s": round(time.perf_counter() - t, 4), "ranks_K": r.ranks_K,
                          "ranks_u": r.ranks_u, "l2": r.l2_error, "res": r.residual, "sweeps": r.sweeps,
                          "timings": {k: round(v, 4) for k, v in r.timings.items()}}), flush=True)
