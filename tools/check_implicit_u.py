"""matvec+round on the configs[4] microbenchmark: implicit-U tall SVD vs explicit Q (same inputs);
prints ranks, the relative difference of the rounded tensors (via TT norms) and U orthogonality."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200.tensor_train import tt_matvec, tt_norm, tt_round, tt_sub  # noqa: E402
from paper_2509_13224_b200.workloads import matvec_round_instance  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
A, X = matvec_round_instance(n, 16, 64, 3, seed=0)
Y1 = tt_round(tt_matvec(A, X), 1e-8)
L._IMPLICIT_U = False
Y2 = tt_round(tt_matvec(A, X), 1e-8)
d = tt_norm(tt_sub(Y1, Y2)) / tt_norm(Y2)
G = Y1.cores[1].reshape(-1, Y1.cores[1].shape[2])
orth = float((G.t() @ G - torch.eye(G.shape[1], dtype=G.dtype, device=G.device)).abs().max())
print(f"n={n} ranks implicit {Y1.ranks} explicit {Y2.ranks} rel.diff {d:.3e} core1 orthogonality {orth:.3e}")
