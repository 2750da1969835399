"""One Jacobi SVD of a 1024 x 1024 triangular factor (for ncu captures)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L
n = 1024
g = torch.Generator(device="cuda").manual_seed(n)
X = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
Qt, Rt = L.qr_colmajor(L.permute(X, (1, 0)), n, n)
L._jacobi(Rt.contiguous(), n, False, None)
torch.cuda.synchronize()
print("ok")
