"""Time spent in linalg.qr_colmajor / linalg._jacobi per shape during one BASELINE solve (synchronized timers)."""
import collections
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import driver, linalg  # noqa: E402
from paper_2509_13224_b200.workloads import SOLVE_CONFIGS  # noqa: E402

T = collections.defaultdict(float)
N = collections.Counter()
_qr, _jac = linalg.qr_colmajor, linalg._jacobi


def qr(Acm, m, n, *a, **k):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = _qr(Acm, m, n, *a, **k)
    torch.cuda.synchronize()
    key = ("qr", m, n, k.get("want_q", True))
    T[key] += time.perf_counter() - t
    N[key] += 1
    return r


def jac(Rcm, n, *a, **k):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = _jac(Rcm, n, *a, **k)
    torch.cuda.synchronize()
    key = ("jacobi", n, n, bool(a[0]) if a else k.get("want_v", False))
    T[key] += time.perf_counter() - t
    N[key] += 1
    return r


linalg.qr_colmajor = qr
linalg._jacobi = jac
c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
driver.solve_poisson(driver.SolveConfig(seed=0, **SOLVE_CONFIGS[c]), want_error=False)
tot = collections.defaultdict(float)
for k, v in T.items():
    tot[k[0]] += v
print({k: round(v, 3) for k, v in tot.items()})
for k, v in sorted(T.items(), key=lambda x: -x[1])[:40]:
    print(f"{v:8.3f}s n={N[k]:4d} {1e3 * v / N[k]:8.2f} ms/call  {k}")
