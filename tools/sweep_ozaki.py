"""Ozaki FP64 GEMM time vs K at fixed M x N (separates the per-tile fixed cost -- prologue, epilogue,
C write -- from the per-k main loop), plus the slicing kernels' share (torch.profiler)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402

M, N = 1 << 17, 4096
for K in (256, 512, 1024, 2048, 4096):
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(M, K, generator=g, device="cuda", dtype=torch.float64)
    B = torch.randn(K, N, generator=g, device="cuda", dtype=torch.float64)
    C = torch.empty(M, N, device="cuda", dtype=torch.float64)
    ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, K)), dtype=torch.uint8, device="cuda")
    f = lambda: call("ttb_dgemm_ozaki", 0, M, N, K, ptr(A), K, ptr(B), N, ptr(C), N, ptr(ws))  # noqa
    f()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as p:
        for _ in range(3):
            f()
        torch.cuda.synchronize()
    tot = {}
    for e in p.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            tot[e.name] = tot.get(e.name, 0.0) + e.device_time_total / 3 / 1e3
    main = sum(v for k, v in tot.items() if "oz_gemm" in k)
    rest = sum(v for k, v in tot.items() if "oz_gemm" not in k)
    print(f"K={K}: oz_gemm {main:.2f} ms ({2.0 * M * N * K / main / 1e9:.1f} TF/s fp64-eq), slicing etc {rest:.2f} ms",
          flush=True)
    del A, B, C, ws
