"""QR timing on the rounding's big unfoldings (development probe)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L


def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


for m, n in ((1 << 20, 1024), (1 << 18, 1024), (1 << 20, 256), (4096, 1024), (1024, 1024)):
    X = torch.randn(n, m, dtype=torch.float64, device="cuda")  # col-major m x n
    k = min(m, n)
    fl = 2.0 * m * n * k - 2.0 / 3.0 * k ** 3
    ms_r = timed(lambda: L.qr_colmajor(X.clone(), m, n, want_q=False))
    ms_qr = timed(lambda: L.qr_colmajor(X.clone(), m, n))
    ms_c = timed(lambda: X.clone())
    print(f"m={m} n={n}: geqrf {ms_r - ms_c:8.2f} ms ({fl / (ms_r - ms_c) / 1e9:6.2f} TF/s)  "
          f"geqrf+orgqr {ms_qr - ms_c:8.2f} ms ({2 * fl / (ms_qr - ms_c) / 1e9:6.2f} TF/s)", flush=True)
    del X
