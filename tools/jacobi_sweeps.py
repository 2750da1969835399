"""One-sided Jacobi SVD of a 1024^2 matrix: on X directly vs on R^T with R the Cholesky factor of
X^T X (the shape of the rounding's first LR SVD); time and sweep count."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200._lib import call, ptr  # noqa: E402

n = 1024
g = torch.Generator(device="cuda").manual_seed(0)
for kind in ("gaussian", "product"):
    X = torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64)
    if kind == "product":   # like c0 = core0 . R^T
        X = X @ torch.tril(torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64) / n ** 0.5
                           + torch.eye(n, device="cuda", dtype=torch.float64))
    for mode in ("direct", "chol_rt", "chol_r"):
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        if mode == "direct":
            A = L.permute(X, (1, 0))
        else:
            G = L.gemm(X, X, tA=True)
            inf2 = torch.zeros(1, dtype=torch.int32, device="cuda")
            call("ttb_potrf", n, ptr(G), n, ptr(inf2))
            R = torch.triu(G).contiguous()          # row-major R = col-major R^T
            A = R if mode == "chol_rt" else R.t().contiguous()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        U, S, V = L._jacobi(A, n, False, info)
        e1.record()
        torch.cuda.synchronize()
        S_ref = torch.linalg.svdvals(X)
        err = float(((S.sort(descending=True).values - S_ref).abs() / S_ref[0]).max())
        print(f"{kind:9s} {mode:8s}: {e0.elapsed_time(e1):7.2f} ms, sweeps {int(info.item())}, s err {err:.1e}",
              flush=True)
