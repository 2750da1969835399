"""One WY trailing-update GEMM (C -= A B, 896 x 1M, K = 128) for ncu."""
import sys, torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L
m, nq, K = 1 << 20, 896, 128
A = torch.randn(nq, K, dtype=torch.float64, device="cuda")
B = torch.randn(K, m, dtype=torch.float64, device="cuda")
C = torch.randn(nq, m, dtype=torch.float64, device="cuda")
L.gemm(A, B, alpha=-1.0, beta=1.0, out=C)
torch.cuda.synchronize()
print("ok")
