"""Host-side profile of the small reference experiments (L-shape 8 el., ring 16 el.): per-phase
timings and the top Python functions by own time under cProfile (second, warm call)."""
import cProfile
import io
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import driver as D  # noqa: E402
from paper_2509_13224_b200 import _lib  # noqa: E402


def cfg(name):
    if name == "lshape":
        return D.SolveConfig(seed=0, geometry="lshape", degree=1, elements=8, source="sin_pi_xy", analytic="lshape_exact")
    bc = D.BoundarySpec({(1, 0): D.FaceCondition("dirichlet", 1.0), (1, 1): D.FaceCondition("dirichlet", 2.0)})
    return D.SolveConfig(seed=0, geometry="ring", degree=2, elements=16, source="zero", bc=bc)


for name in sys.argv[1:] or ["lshape", "ring"]:
    for _ in range(3):
        D.solve_poisson(cfg(name), want_error=False)
    torch.cuda.synchronize()
    n0 = _lib.call_raw("ttb_launch_count", 0)
    t = time.perf_counter()
    r = D.solve_poisson(cfg(name), want_error=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    n1 = _lib.call_raw("ttb_launch_count", 0)
    print(name, f"{dt*1e3:.1f} ms", {k: round(v * 1e3, 2) for k, v in r.timings.items()}, "sweeps", r.sweeps,
          "launches", n1 - n0, flush=True)
    pr = cProfile.Profile()
    pr.enable()
    D.solve_poisson(cfg(name), want_error=False)
    torch.cuda.synchronize()
    pr.disable()
    s = io.StringIO()
    st = pstats.Stats(pr, stream=s)
    st.sort_stats("tottime").print_stats(35)
    st.sort_stats("cumulative").print_stats(45)
    print(s.getvalue())
