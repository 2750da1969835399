"""Whole ttb_dgemm_ozaki calls on the step's two slicing-heavy shapes (A row-sliced 1M x 1024; B
column-sliced 1024 x 1M), CUDA-event timed, plus the error against DMMA on a small shape."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402


def run(M, N, K, reps=10):
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(M, K, generator=g, device="cuda", dtype=torch.float64)
    B = torch.randn(K, N, generator=g, device="cuda", dtype=torch.float64)
    C = torch.empty(M, N, device="cuda", dtype=torch.float64)
    ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, K)), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        call("ttb_dgemm_ozaki", 0, M, N, K, ptr(A), K, ptr(B), N, ptr(C), N, ptr(ws))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        call("ttb_dgemm_ozaki", 0, M, N, K, ptr(A), K, ptr(B), N, ptr(C), N, ptr(ws))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    i = torch.randint(0, M, (64,), device="cuda")
    ref = A[i] @ B
    err = float((C[i] - ref).abs().max() / ref.abs().max())
    print(f"M={M} N={N} K={K}: {ms:.3f} ms  err {err:.2e}", flush=True)
    del A, B, C, ws
    torch.cuda.empty_cache()


run(1 << 20, 1024, 1024)
run(1024, 1 << 20, 1024)
run(4096, 2048, 512)
