"""CUPTI kernel split of one Ozaki FP64 GEMM (1M x 1024 x 1024)."""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402

M, N, K = 1 << 20, 1024, 1024
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(M, K, generator=g, device="cuda", dtype=torch.float64)
B = torch.randn(K, N, generator=g, device="cuda", dtype=torch.float64)
C = torch.empty(M, N, device="cuda", dtype=torch.float64)
ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, K)), dtype=torch.uint8, device="cuda")
call("ttb_dgemm_ozaki", 0, M, N, K, ptr(A), K, ptr(B), N, ptr(C), N, ptr(ws))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    call("ttb_dgemm_ozaki", 0, M, N, K, ptr(A), K, ptr(B), N, ptr(C), N, ptr(ws))
    torch.cuda.synchronize()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        print(f"{e.device_time_total / 1e3:8.2f} ms  {e.name[:90]}")
