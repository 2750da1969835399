"""Which permutes (and their bytes) one matvec+round step issues (bench workload)."""
import sys
import traceback
import torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200.tensor_train import tt_matvec, tt_round  # noqa: E402
from paper_2509_13224_b200.workloads import matvec_round_instance  # noqa: E402

A, X = matvec_round_instance(1024, 16, 64, 3, seed=0)
tt_round(tt_matvec(A, X), 1e-8)
orig = L.permute
log = []


def spy(Xt, perm, out=None):
    st = traceback.extract_stack()[-2]
    log.append((Xt.numel() * 8, tuple(Xt.shape), perm, f"{st.filename.split('/')[-1]}:{st.lineno}"))
    return orig(Xt, perm, out=out)


L.permute = spy
import paper_2509_13224_b200.tensor_train.core as C  # noqa: E402
C.L.permute = spy
torch.cuda.synchronize()
tt_round(tt_matvec(A, X), 1e-8)
torch.cuda.synchronize()
tot = 0
for b, sh, p, where in log:
    if b > 1e8:
        print(f"{b / 1e9:6.2f} GB {sh} {p} {where}")
    tot += b
print(f"total {tot / 1e9:.2f} GB in {len(log)} permutes")
