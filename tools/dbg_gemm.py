import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L
for (M, N, K, lda, ldb) in ((96, 16, 131057, 131073, 131057), (112, 16, 131073, 131073, 131073), (96, 16, 131056, 131072, 131056)):
    Abig = torch.randn(M, lda, dtype=torch.float64, device="cuda")
    A = Abig[:, :K]
    Bbig = torch.randn(N, ldb, dtype=torch.float64, device="cuda")
    B = Bbig[:, :K]
    try:
        W = L.gemm(A, B, tB=True)
        torch.cuda.synchronize()
        ref = (A.cpu().numpy() @ B.cpu().numpy().T)
        print(M, N, K, lda, ldb, "ok", np.abs(W.cpu().numpy() - ref).max(), flush=True)
    except Exception as e:
        print(M, N, K, lda, ldb, "ERR", str(e)[:100], flush=True)
        break
