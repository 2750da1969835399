"""Where the TT assembly (stiffness + load) of one BASELINE config spends its time.

    python tools/profile_assembly.py <config> [n_basis]

Runs setup + assemble_stiffness + assemble_load once (warm-up), then again under (1) synchronized
wall-clock timers, (2) the CUPTI kernel trace (torch.profiler) and (3) cProfile of the host side,
and prints the device busy time, the top kernels and the top host functions."""
import cProfile
import io
import json
import pstats
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2509_13224_b200 import driver as D  # noqa: E402
from paper_2509_13224_b200.assembly import assemble_load, assemble_stiffness  # noqa: E402
from paper_2509_13224_b200.geometry import make_geometry  # noqa: E402
from paper_2509_13224_b200.workloads import SOLVE_CONFIGS  # noqa: E402

c = int(sys.argv[1])
kw = dict(SOLVE_CONFIGS[c])
if len(sys.argv) > 2:
    kw["n_basis"] = int(sys.argv[2])


def run():
    cfg = D.SolveConfig(seed=0, **kw)
    patch = make_geometry(cfg.geometry, cfg.geometry_params)
    cfg.resolve_bc(patch)
    disc = D.discretize(cfg, patch)
    rK, rf = D._spawn_rngs(cfg.seed, 2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    K, ki = assemble_stiffness(patch, disc, cfg.eps_round, rank_cap=cfg.rank_cap, rng=rK)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    f, fi = assemble_load(patch, disc, cfg.source, cfg.eps_cross, rank_cap=cfg.rank_cap, rng=rf)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return K, f, t1 - t0, t2 - t1


run()
K, f, tK, tf = run()
print(json.dumps({"config": c, "n": kw.get("n_basis"), "t_K_s": tK, "t_f_s": tf, "ranks_K": K.ranks,
                  "ranks_f": f.ranks}))
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
tot, cnt = {}, {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name[:100]] = tot.get(e.name[:100], 0.0) + e.device_time_total
        cnt[e.name[:100]] = cnt.get(e.name[:100], 0) + 1
all_us = sum(tot.values())
print(f"device busy {all_us / 1e3:.1f} ms of {1e3 * (tK + tf):.1f} ms wall")
for name, us in sorted(tot.items(), key=lambda x: -x[1])[:25]:
    print(f"{us / 1e3:10.2f} ms {100 * us / all_us:6.2f}% n={cnt[name]:6d}  {name}")
pr = cProfile.Profile()
pr.enable()
run()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue())
