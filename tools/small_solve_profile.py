"""Where a small reference solve (L-shape p=1, 8 elements) spends its time on the GPU path: phase times,
kernel launches, device busy time, host syncs (cProfile)."""
import cProfile
import io
import pstats
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2509_13224_b200 import _lib, driver as D  # noqa: E402

kw = dict(geometry=sys.argv[1] if len(sys.argv) > 1 else "lshape", degree=1, elements=8, source="sin_pi_xy", seed=0)
if kw["geometry"] != "lshape":
    kw.update(degree=2, elements=16, source="zero")
D.solve_poisson(D.SolveConfig(**kw), want_error=False)
torch.cuda.synchronize()
lib = _lib.lib()
lib.ttb_launch_count(1)
t = time.perf_counter()
rep = D.solve_poisson(D.SolveConfig(**kw), want_error=False)
torch.cuda.synchronize()
print(f"wall {1e3 * (time.perf_counter() - t):.1f} ms, phases {rep.timings}, our launches {lib.ttb_launch_count(1)}")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    D.solve_poisson(D.SolveConfig(**kw), want_error=False)
    torch.cuda.synchronize()
tot = sum(e.device_time_total for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA)
n = sum(1 for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA)
print(f"device busy {tot / 1e3:.1f} ms over {n} device ops")
pr = cProfile.Profile()
pr.enable()
D.solve_poisson(D.SolveConfig(**kw), want_error=False)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(18)
print(s.getvalue()[:4000])
