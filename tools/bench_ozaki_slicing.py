"""Time the Ozaki operand preparation on a W-GEMM-shaped operand (1024 x 1M rows, the geqrf trailing
matrix): row maxima + slicing vs the GEMM itself (ttb_dgemm_ozaki_ex, M=1024 N=128 K=1M)."""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402

M, N, K = 1024, 128, 1 << 20
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(M, K, generator=g, device="cuda", dtype=torch.float64)
B = torch.randn(N, K, generator=g, device="cuda", dtype=torch.float64)
C = torch.empty(M, N, device="cuda", dtype=torch.float64)
ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, K)), dtype=torch.uint8, device="cuda")
f = lambda: call("ttb_dgemm_ozaki_ex", 1, M, N, K, 1.0, ptr(A), K, ptr(B), K, 0.0, ptr(C), N, ptr(ws))  # noqa
f()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    for _ in range(3):
        f()
    torch.cuda.synchronize()
tot = {}
for e in p.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name.split("(")[1] if e.name.startswith("(") else e.name
        tot[e.name[:60]] = tot.get(e.name[:60], 0.0) + e.device_time_total / 3 / 1e3
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:8.3f} ms  {k}")
print("bytes A:", A.numel() * 8 / 1e9, "GB")
