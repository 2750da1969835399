"""How the leading-triplet route (linalg.topk_svd) behaves inside a BASELINE solve: calls, fallbacks, time."""
import collections
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import driver, linalg  # noqa: E402
from paper_2509_13224_b200.workloads import SOLVE_CONFIGS  # noqa: E402

T = collections.defaultdict(float)
N = collections.Counter()
_orig = linalg.topk_svd


def probe(X, kmax, delta):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = _orig(X, kmax, delta)
    torch.cuda.synchronize()
    key = (tuple(X.shape), kmax, "ok" if r is not None else "none", None if r is None else int(r[0].shape[1]))
    T[key] += time.perf_counter() - t
    N[key] += 1
    return r


linalg.topk_svd = probe
c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rep = driver.solve_poisson(driver.SolveConfig(seed=0, **SOLVE_CONFIGS[c]), want_error=False)
print(rep.timings, rep.ranks_u, rep.residual)
for k, v in sorted(T.items(), key=lambda x: -x[1]):
    print(f"{v:8.3f}s n={N[k]:4d} {1e3 * v / N[k]:8.2f} ms/call  {k}")
