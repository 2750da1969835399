"""Ozaki-scheme FP64 GEMM on the INT8 tensor cores vs the DMMA DGEMM: accuracy and time."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for (M, N, K, tB, graded) in ((256, 256, 128, 0, 0), (1024, 512, 1024, 1, 0), (4096, 1024, 1024, 0, 1),
                              (262144, 4096, 1024, 0, 0), (1 << 20, 1024, 1024, 0, 0)):
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, generator=g, device="cuda", dtype=torch.float64)
    B = torch.randn((N, K) if tB else (K, N), generator=g, device="cuda", dtype=torch.float64)
    if graded:
        A *= torch.logspace(0, -12, K, device="cuda", dtype=torch.float64)[None, :]
        B *= torch.logspace(0, -6, N, device="cuda", dtype=torch.float64)[None, :]
    C = torch.empty(M, N, device="cuda", dtype=torch.float64)
    ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, K)), dtype=torch.uint8, device="cuda")
    oz = lambda: call("ttb_dgemm_ozaki", tB, M, N, K, ptr(A), K, ptr(B), K if tB else N, ptr(C), N, ptr(ws))  # noqa
    ms_oz = timeit(oz)
    Cd = L.gemm(A, B, tB=bool(tB))
    ms_d = timeit(lambda: L.gemm(A, B, tB=bool(tB), out=Cd))
    # exact-ish reference on a row subset in long double? use FP64 DGEMM and its own error scale
    scale = (A.abs() @ (B.abs().t() if tB else B.abs()))
    err_oz = float(((C - Cd).abs() / scale.clamp_min(1e-300)).max())
    fl = 2.0 * M * N * K
    print(f"M={M} N={N} K={K} tB={tB} graded={graded}: ozaki {ms_oz:.2f} ms ({fl / ms_oz / 1e9:.1f} TF/s)  "
          f"dmma {ms_d:.2f} ms ({fl / ms_d / 1e9:.1f} TF/s)  max|C_oz - C_dmma| / (|A||B|) = {err_oz:.2e}",
          flush=True)
    del A, B, C, ws, Cd, scale
