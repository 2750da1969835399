"""Host-side cost structure of the small-solve assembly (L-shape p=1, 8 elements): cProfile by cumulative time."""
import cProfile
import io
import pstats
import sys
import torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import driver as D  # noqa: E402
from paper_2509_13224_b200.assembly import assemble_stiffness  # noqa: E402
from paper_2509_13224_b200.geometry import make_geometry  # noqa: E402

cfg = D.SolveConfig(geometry="lshape", degree=1, elements=8, source="sin_pi_xy", seed=0)
patch = make_geometry(cfg.geometry, cfg.geometry_params)
cfg.resolve_bc(patch)
disc = D.discretize(cfg, patch)
for _ in range(2):
    rK, rf = D._spawn_rngs(0, 2)
    assemble_stiffness(patch, disc, cfg.eps_round, rank_cap=cfg.rank_cap, rng=rK)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
rK, rf = D._spawn_rngs(0, 2)
assemble_stiffness(patch, disc, cfg.eps_round, rank_cap=cfg.rank_cap, rng=rK)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(30)
print(s.getvalue()[:6000])
