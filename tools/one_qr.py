import sys, torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L
m, n = 1 << 20, 1024
X = torch.randn(n, m, dtype=torch.float64, device="cuda")
L.qr_colmajor(X, m, n, want_q=False)
torch.cuda.synchronize()
print("ok")
