"""ttb_i8gemm (tcgen05 kind::i8) vs an exact FP64 reference; throughput in int8 TOPS."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200._lib import call, ptr  # noqa: E402

for (M, N, K) in ((128, 128, 128), (256, 384, 512), (1024, 1024, 4096), (8192, 8192, 8192)):
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randint(-127, 128, (M, K), generator=g, device="cuda", dtype=torch.int8)
    B = torch.randint(-127, 128, (N, K), generator=g, device="cuda", dtype=torch.int8)
    C = torch.empty(M, N, dtype=torch.int32, device="cuda")
    call("ttb_i8gemm", M, N, K, ptr(A), ptr(B), ptr(C))
    torch.cuda.synchronize()
    ref = (A.double() @ B.double().t())
    err = float((C.double() - ref).abs().max())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        call("ttb_i8gemm", M, N, K, ptr(A), ptr(B), ptr(C))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"M={M} N={N} K={K}: max|err| {err:.0f}  {ms:.3f} ms  {2.0 * M * N * K / ms / 1e9:.1f} TOPS", flush=True)
