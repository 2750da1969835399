"""Band contraction at the configs[3] local shape (n=512, X=8184, Ra=Rb=121, h=3): DMMA batch vs Ozaki."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402

n, h, Rin, Rout, X = (int(v) for v in sys.argv[1:6]) if len(sys.argv) > 5 else (512, 3, 121, 121, 8184)
B = 2 * h + 1
g = torch.Generator(device="cuda").manual_seed(1)
Tp = torch.randn(n + 2 * h, Rin, X, generator=g, dtype=torch.float64, device="cuda")
Mt = torch.randn(n, B, Rin, Rout, generator=g, dtype=torch.float64, device="cuda")
out = L.empty(n, X, Rout)
flop = 2.0 * n * X * Rout * B * Rin


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


ms = timed(lambda: L.gemm_strided(1, 0, X, Rout, B * Rin, Tp, X, Rin * X, Mt, Rout, B * Rin * Rout, out, Rout,
                                  X * Rout, n))
ref = out.clone()
print(f"DMMA batch: {ms:.2f} ms = {flop / ms / 1e9:.1f} TF/s")
for G in ((32,) if len(sys.argv) > 5 else (1, 8, 32, 64)):
    ws = torch.empty(int(call_raw("ttb_band_gemm_ozaki_workspace", n, h, Rin, Rout, X, G)), dtype=torch.uint8,
                     device="cuda")
    ms = timed(lambda: call("ttb_band_gemm_ozaki", n, h, Rin, Rout, X, ptr(Tp), ptr(Mt), ptr(out), ptr(ws), G))
    err = ((out - ref).norm() / ref.norm()).item()
    print(f"Ozaki G={G}: {ms:.2f} ms = {flop / ms / 1e9:.1f} TF/s FP64-eq, ws {ws.numel() / 1e9:.2f} GB, err {err:.1e}")
