"""Device GEMM throughput: libttiga_b200 DMMA kernel vs cuBLAS (torch) on the shapes the TT path uses."""
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

shapes = [(8192, 8192, 8192, 0, 0), (8192, 8192, 8192, 1, 0), (8192, 8192, 8192, 0, 1),
          (262144, 4096, 1024, 0, 0), (1048576, 1024, 1024, 0, 0), (1024, 1048576, 128, 0, 0),
          (1024, 128, 1048576, 0, 1), (1024, 1024, 1048576, 1, 1),
          (1048576, 1024, 1024, 1, 1), (1024, 1048576, 1024, 0, 0)]
for M, N, K, tA, tB in shapes:
    A = torch.randn((K, M) if tA else (M, K), dtype=torch.float64, device="cuda")
    B = torch.randn((N, K) if tB else (K, N), dtype=torch.float64, device="cuda")
    C = torch.empty(M, N, dtype=torch.float64, device="cuda")
    ms = timeit(lambda: L.gemm(A, B, tA=bool(tA), tB=bool(tB), out=C))
    At = A.t() if tA else A
    Bt = B.t() if tB else B
    ms_ref = timeit(lambda: torch.matmul(At, Bt, out=C))
    fl = 2.0 * M * N * K
    print(f"M={M} N={N} K={K} tA={tA} tB={tB}: ours {fl/ms/1e9:7.2f} TF/s  cuBLAS {fl/ms_ref/1e9:7.2f} TF/s", flush=True)
    del A, B, C
