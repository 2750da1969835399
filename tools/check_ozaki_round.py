"""matvec+round with/without Ozaki GEMMs and implicit-U: pairwise relative differences of the results."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200.tensor_train import tt_matvec, tt_norm, tt_round, tt_sub  # noqa: E402
from paper_2509_13224_b200.workloads import matvec_round_instance  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
A, X = matvec_round_instance(n, 16, 64, 3, seed=0)
res = {}
for oz in (True, False):
    for imp in (True, False):
        L._OZAKI, L._IMPLICIT_U = oz, imp
        res[(oz, imp)] = tt_round(tt_matvec(A, X), 1e-8)
        torch.cuda.synchronize()
ref = res[(False, False)]
for k, Y in res.items():
    print(f"ozaki={k[0]} implicit_u={k[1]} ranks {Y.ranks} rel.diff vs (dmma, explicit) "
          f"{tt_norm(tt_sub(Y, ref)) / tt_norm(ref):.3e}", flush=True)
# the matvec alone
L._OZAKI = True
Y1 = tt_matvec(A, X)
L._OZAKI = False
Y2 = tt_matvec(A, X)
print("matvec core1 rel.diff", float((Y1.cores[1] - Y2.cores[1]).norm() / Y2.cores[1].norm()))
