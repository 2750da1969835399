import sys, time, torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import driver as D, linalg as L
from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
for pad in (1.6, 0.0, 1.6, 0.0):
    L._OZAKI_MAX_PAD = pad
    torch.cuda.synchronize(); t = time.perf_counter()
    rep = D.solve_poisson(D.SolveConfig(seed=0, **SOLVE_CONFIGS[2]), want_error=False)
    torch.cuda.synchronize()
    print(f"pad {pad}: {time.perf_counter() - t:.3f} s solve {rep.timings['t_solve_s']:.3f} bc {rep.timings['t_bc_s']:.3f} res {rep.residual:.3e}", flush=True)
