import sys, time, torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L
g = torch.Generator(device="cuda").manual_seed(0)
for n in (256, 1024):
    A = torch.randn(n, n, generator=g, dtype=torch.float64, device="cuda").tril() + n * torch.eye(n, dtype=torch.float64, device="cuda")
    e = L._norm2_est(A); torch.cuda.synchronize()
    t = time.perf_counter(); e = L._norm2_est(A); torch.cuda.synchronize(); dt = time.perf_counter() - t
    true = torch.linalg.matrix_norm(A, 2).item()
    print(f"n={n}: est {e:.6e} true {true:.6e} rel {(true - e) / true:.2e} time {1e3 * dt:.2f} ms")
