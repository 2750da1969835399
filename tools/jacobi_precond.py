"""Does a static column ordering before the Cholesky (diag(G) descending) shorten the one-sided
Jacobi on R^T? 1024^2 square cases and a tall carried core (1M x 1024 = M . Q, M ill-conditioned)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200._lib import call, ptr  # noqa: E402

n = 1024
g = torch.Generator(device="cuda").manual_seed(0)


def run(G, label):
    for order in ("none", "diag_desc", "diag_asc"):
        Gp = G.clone()
        if order != "none":
            perm = torch.argsort(torch.diagonal(G), descending=(order == "diag_desc"))
            Gp = G[perm][:, perm].contiguous()
        info2 = torch.zeros(1, dtype=torch.int32, device="cuda")
        call("ttb_potrf", n, ptr(Gp), n, ptr(info2))
        R = torch.triu(Gp).contiguous()
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        U, S, V = L._jacobi(R, n, False, info)
        e1.record()
        torch.cuda.synchronize()
        print(f"{label:10s} {order:9s}: {e0.elapsed_time(e1):7.2f} ms, sweeps {int(info.item())}", flush=True)


X = torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64)
run(L.gemm(X, X, tA=True), "gaussian")
X = X @ torch.tril(torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64) / n ** 0.5
                   + torch.eye(n, device="cuda", dtype=torch.float64))
run(L.gemm(X, X, tA=True), "product")
# graded columns (the kind of spectrum truncation acts on)
Xg = torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64) * torch.logspace(0, -6, n, device="cuda",
                                                                                       dtype=torch.float64)
run(L.gemm(Xg, Xg, tA=True), "graded")
