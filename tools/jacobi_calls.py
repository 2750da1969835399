"""Sizes, sweep counts and times of every Jacobi SVD call in one assembly (or a whole solve).

    python tools/jacobi_calls.py <config> [solve]"""
import collections
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import driver as D  # noqa: E402
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200.assembly import assemble_stiffness  # noqa: E402
from paper_2509_13224_b200.geometry import make_geometry  # noqa: E402
from paper_2509_13224_b200.workloads import SOLVE_CONFIGS  # noqa: E402

rec = []
_orig = L._jacobi


def timed(Rcm, n, want_v=False, info=None):
    own = info is None
    if own:
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = _orig(Rcm, n, want_v, info)
    torch.cuda.synchronize()
    rec.append((n, bool(want_v), int(info.item()), time.perf_counter() - t))
    return out


c = int(sys.argv[1])
kw = dict(SOLVE_CONFIGS[c])


def run():
    cfg = D.SolveConfig(seed=0, **kw)
    if len(sys.argv) > 2:
        return D.solve_poisson(cfg, want_error=False)
    patch = make_geometry(cfg.geometry, cfg.geometry_params)
    cfg.resolve_bc(patch)
    disc = D.discretize(cfg, patch)
    rK, _ = D._spawn_rngs(cfg.seed, 2)
    return assemble_stiffness(patch, disc, cfg.eps_round, rank_cap=cfg.rank_cap, rng=rK)


run()
L._jacobi = timed
rec.clear()
run()
by = collections.defaultdict(list)
for n, v, sw, dt in rec:
    by[(n // 32 * 32, v)].append((sw, dt))
tot = sum(r[3] for r in rec)
print(f"{len(rec)} Jacobi calls, {tot * 1e3:.1f} ms synchronized")
for (nb, v), xs in sorted(by.items()):
    print(f"n in [{nb},{nb + 32}) want_v={v}: {len(xs)} calls, sweeps {min(x[0] for x in xs)}-{max(x[0] for x in xs)}, "
          f"{sum(x[1] for x in xs) * 1e3:.1f} ms ({sum(x[1] for x in xs) / len(xs) * 1e3:.2f} ms each)")
