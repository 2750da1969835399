"""Jacobi SVD timing / sweep counts on the shapes the rounding meets (development probe)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L


def timed(fn):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); r = fn(); b.record(); torch.cuda.synchronize()
    return r, a.elapsed_time(b)


for n in (64, 128, 256, 512, 1024):
    g = torch.Generator(device="cuda").manual_seed(n)
    X = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    Qt, Rt = L.qr_colmajor(L.permute(X, (1, 0)), n, n)
    for label, M, wv in (("R", Rt.contiguous(), False), ("R^T", L.permute(Rt, (1, 0)), False),
                         ("R^T+V", L.permute(Rt, (1, 0)), True)):
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        (U, S, V), ms = timed(lambda: L._jacobi(M.clone(), n, wv, info))
        print(f"n={n:5d} jacobi on {label:3s}: {ms:8.2f} ms, sweeps={int(info.item())}", flush=True)
