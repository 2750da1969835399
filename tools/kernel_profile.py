"""Kernel-level time split of one BASELINE solve (CUPTI through torch.profiler; our ctypes-launched
kernels are traced like any other). Usage: python tools/kernel_profile.py <config> [key=json ...]
Runs the config once untraced (warm-up), then traced; prints the top kernels by device time."""
import json
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2509_13224_b200 import driver as D  # noqa: E402
from paper_2509_13224_b200.workloads import SOLVE_CONFIGS  # noqa: E402

if sys.argv[1] == "mr":
    # the configs[4] matvec+round microbenchmark step (bench.py)
    from paper_2509_13224_b200.tensor_train import tt_matvec, tt_round
    from paper_2509_13224_b200.workloads import matvec_round_instance
    A, X = matvec_round_instance(1024, 16, 64, 3, seed=0)
    tt_round(tt_matvec(A, X), 1e-8)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        Y = tt_round(tt_matvec(A, X), 1e-8)
        torch.cuda.synchronize()
    tot, cnt = {}, {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            tot[e.name[:110]] = tot.get(e.name[:110], 0.0) + e.device_time_total
            cnt[e.name[:110]] = cnt.get(e.name[:110], 0) + 1
    all_us = sum(tot.values())
    print(json.dumps({"workload": "matvec+round", "ranks": Y.ranks, "device_ms": all_us / 1e3}))
    for name, us in sorted(tot.items(), key=lambda x: -x[1])[:40]:
        print(f"{us / 1e3:10.2f} ms {100 * us / all_us:6.2f}% n={cnt[name]:6d}  {name}")
    sys.exit(0)
c = int(sys.argv[1])
kw = dict(SOLVE_CONFIGS[c])
for a in sys.argv[2:]:
    k, v = a.split("=", 1)
    kw[k] = json.loads(v)
cfg = D.SolveConfig(seed=0, **kw)
D.solve_poisson(cfg, want_error=False)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rep = D.solve_poisson(D.SolveConfig(seed=0, **kw), want_error=False)
    torch.cuda.synchronize()
tot = {}
cnt = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name[:110]
        tot[name] = tot.get(name, 0.0) + e.device_time_total
        cnt[name] = cnt.get(name, 0) + 1
all_us = sum(tot.values())
print(json.dumps({"config": c, "timings": rep.timings, "ranks_u": rep.ranks_u, "device_ms": all_us / 1e3}))
for name, us in sorted(tot.items(), key=lambda x: -x[1])[:30]:
    print(f"{us / 1e3:10.2f} ms {100 * us / all_us:6.2f}% n={cnt[name]:6d}  {name}")
