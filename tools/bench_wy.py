"""WY trailing-update GEMM shapes (C -= A B, beta = 1) as the blocked QR issues them."""
import sys, torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L

def timeit(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best

m = 1 << 20
for nq, K in ((896, 128), (512, 128), (128, 128), (768, 256), (256, 256), (1024, 64)):
    A = torch.randn(nq, K, dtype=torch.float64, device="cuda")
    B = torch.randn(K, m, dtype=torch.float64, device="cuda")
    C = torch.randn(nq, m, dtype=torch.float64, device="cuda")
    ms = timeit(lambda: L.gemm(A, B, alpha=-1.0, beta=1.0, out=C))
    print(f"C({nq} x {m}) -= A({nq} x {K}) B: {ms:7.2f} ms  {2.0 * nq * m * K / ms / 1e9:6.2f} TF/s", flush=True)
    del A, B, C

# cuBLAS on the same update (torch.addmm, beta = 1, alpha = -1) as the ceiling reference
for nq, K in ((896, 128), (512, 128)):
    A = torch.randn(nq, K, dtype=torch.float64, device="cuda")
    B = torch.randn(K, m, dtype=torch.float64, device="cuda")
    C = torch.randn(nq, m, dtype=torch.float64, device="cuda")
    ms = timeit(lambda: C.addmm_(A, B, beta=1.0, alpha=-1.0))
    print(f"cuBLAS C({nq} x {m}) -= A B (K={K}): {ms:7.2f} ms  {2.0 * nq * m * K / ms / 1e9:6.2f} TF/s", flush=True)
    del A, B, C
