"""Does a column-norm ordering of R reduce the Jacobi sweep count? (probe)"""
import sys, torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L
from paper_2509_13224_b200.workloads import matvec_round_instance
from paper_2509_13224_b200.tensor_train import tt_matvec
from paper_2509_13224_b200.tensor_train.core import _rl_orthogonalize


def run(M, label):
    n = M.shape[0]
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); L._jacobi(M.clone(), n, False, info); b.record(); torch.cuda.synchronize()
    print(f"{label:28s} {a.elapsed_time(b):7.2f} ms sweeps={int(info.item())}", flush=True)


for src in ("random", "bench"):
    if src == "random":
        n = 1024
        X = torch.randn(n, n, dtype=torch.float64, device="cuda")
        Qt, Rt = L.qr_colmajor(L.permute(X, (1, 0)), n, n)
    else:
        A, X = matvec_round_instance(1024, 16, 64, 3, seed=0)
        Y = tt_matvec(A, X)
        cores, _ = _rl_orthogonalize(list(Y.cores))
        G = cores[1]
        r0, nn, r1 = G.shape
        Z = L.gemm(L.SVDFactors(cores[0].reshape(-1, r0)).SVt(r0), G.reshape(r0, -1)).reshape(-1, r1)
        Qt, Rt = L.qr_colmajor(L.permute(Z, (1, 0)), Z.shape[0], r1)
        n = r1
    Rt = Rt.contiguous()
    run(Rt, f"{src}: R")
    norms = (Rt * Rt).sum(dim=1)
    order = torch.argsort(norms, descending=True)
    run(Rt[order].contiguous(), f"{src}: R, norm-sorted")
    order = torch.argsort(norms, descending=False)
    run(Rt[order].contiguous(), f"{src}: R, norm-ascending")
