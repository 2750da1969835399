"""One geqrf+orgqr of the rounding's 1M x 1024 unfolding (for ncu launch lists)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L
m, n = 1 << 20, 1024
X = torch.randn(n, m, dtype=torch.float64, device="cuda")
L.qr_colmajor(X, m, n, want_q=True)
torch.cuda.synchronize()
print("ok")
