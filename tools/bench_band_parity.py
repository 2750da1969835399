import sys, torch
sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L
from paper_2509_13224_b200._lib import call, ptr
def run(n, h, Ra, Rb, X):
    g = torch.Generator(device="cuda").manual_seed(0)
    Mt = torch.randn(n, 2*h+1, Ra, Rb, generator=g, device="cuda", dtype=torch.float64)
    Tp = torch.randn((n+2*h)*Ra*X, generator=g, device="cuda", dtype=torch.float64)
    out = L.empty(n, X, Rb)
    for _ in range(2): call("ttb_band_gemm", n, h, Ra, Rb, X, ptr(Tp), ptr(Mt), ptr(out))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): call("ttb_band_gemm", n, h, Ra, Rb, X, ptr(Tp), ptr(Mt), ptr(out))
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)/3
    print(f"Ra={Ra} Rb={Rb} X={X}: {ms:.2f} ms {2.0*n*X*(2*h+1)*Ra*Rb/ms/1e9:.1f} TF/s", flush=True)
for Rb in (121, 122, 128):
    for X in (7998, 8000):
        run(510, 3, 121, Rb, X)
