"""Host-side phase profile of a TT-IGA solve: wraps hot functions with synchronized timers."""
import collections
import functools
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import assembly, driver, linalg, splines, geometry  # noqa: E402
from paper_2509_13224_b200.tensor_train import amen, banded, core, cross  # noqa: E402
from paper_2509_13224_b200.workloads import SOLVE_CONFIGS  # noqa: E402

T = collections.defaultdict(float)
N = collections.Counter()
DEPTH = [0]


def wrap(mod, name):
    fn = getattr(mod, name)

    @functools.wraps(fn)
    def w(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        DEPTH[0] += 1
        try:
            return fn(*a, **k)
        finally:
            DEPTH[0] -= 1
            torch.cuda.synchronize()
            T[f"{mod.__name__.split('.')[-1]}.{name}"] += time.perf_counter() - t
            N[f"{mod.__name__.split('.')[-1]}.{name}"] += 1

    setattr(mod, name, w)


for mod, names in [
    (core, ["tt_round", "tt_norm", "tt_matvec", "tt_add"]),
    (cross, ["tt_cross"]),
    (amen, ["amen_solve", "_truncate_by_residual", "env_left_A", "env_right_A", "env_left_vec", "env_right_vec"]),
    (banded, ["compressed_residual", "env_left_A", "env_right_A"]),
    (assembly, ["_lift_tensor", "_face_coefficients", "_face_tt", "build_quadrature", "metric_scale"]),
    (linalg, ["qr_colmajor", "maxvol_colmajor", "solve", "cho_solve_or_lu", "_jacobi"]),
]:
    for nm in names:
        wrap(mod, nm)
# names imported into other modules' namespaces
for mod in (amen, cross, assembly, driver):
    for nm in ("tt_round", "tt_norm", "tt_matvec", "tt_cross", "amen_solve"):
        if hasattr(mod, nm):
            setattr(mod, nm, getattr(core, nm, None) or getattr(cross, nm, None) or getattr(amen, nm, None))
_orig_solve = amen.LocalSystem.solve


def _timed_solve(self, *a, **k):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = _orig_solve(self, *a, **k)
    torch.cuda.synchronize()
    key = f"LocalSystem.solve({'direct' if self.size <= a[3] else 'pcg'})"
    T[key] += time.perf_counter() - t
    N[key] += 1
    return r


amen.LocalSystem.solve = _timed_solve

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for rep in range(1 if cfg_id in (2, 3) else 2):
    T.clear(); N.clear()
    t0 = time.perf_counter()
    r = driver.solve_poisson(driver.SolveConfig(seed=0, **SOLVE_CONFIGS[cfg_id]), want_error=False)
    torch.cuda.synchronize()
    print(f"rep {rep} total {time.perf_counter() - t0:.4f}s timings", {k: round(v, 4) for k, v in r.timings.items()})
for k, v in sorted(T.items(), key=lambda x: -x[1]):
    print(f"{v:9.4f}s n={N[k]:5d} {k}")
