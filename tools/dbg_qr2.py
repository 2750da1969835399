import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L
from paper_2509_13224_b200._lib import call
for rep in range(3):
    for m, n in ((131073, 150), (131073, 16), (200000, 40), (5000, 33)):
        X = torch.randn(n, m, dtype=torch.float64, device="cuda")
        Qt, Rt = L.qr_colmajor(X.clone(), m, n)
        torch.cuda.synchronize()
        print(rep, m, n, "ok", flush=True)
