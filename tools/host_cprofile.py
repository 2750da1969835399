"""cProfile of one (warm) solve: where the host time of small, latency-bound solves goes.
Usage: python tools/host_cprofile.py <config|torus32|lshape32>"""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import driver as D  # noqa: E402
from paper_2509_13224_b200.workloads import SOLVE_CONFIGS  # noqa: E402

EXTRA = {
    "torus32": dict(geometry="quarter_torus", degree=2, elements=32, source="sin_pi_xyz"),
    "lshape32": dict(geometry="lshape", degree=1, elements=32, source="sin_pi_xy", analytic="lshape_exact"),
    "lshape8": dict(geometry="lshape", degree=1, elements=8, source="sin_pi_xy", analytic="lshape_exact"),
    "hemi8": dict(geometry="closed_hemisphere", degree=2, elements=8, source="sin_pi_xyz"),
}
name = sys.argv[1]
kw = dict(EXTRA[name]) if name in EXTRA else dict(SOLVE_CONFIGS[int(name)])
D.solve_poisson(D.SolveConfig(seed=0, **kw), want_error=False)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
r = D.solve_poisson(D.SolveConfig(seed=0, **kw), want_error=False)
torch.cuda.synchronize()
pr.disable()
print(name, {k: round(v, 4) for k, v in r.timings.items()}, r.ranks_u, r.sweeps)
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(40)
