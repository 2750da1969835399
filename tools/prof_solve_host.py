import cProfile, pstats, sys, io
sys.path.insert(0, ".")
import torch
from paper_2509_13224_b200 import driver as D
from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
kw = dict(SOLVE_CONFIGS[1]); kw.pop("want_error", None)
D.solve_poisson(D.SolveConfig(seed=0, **kw), want_error=False)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
r = D.solve_poisson(D.SolveConfig(seed=0, **kw), want_error=False)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue()[:6000])
print(r.timings)
