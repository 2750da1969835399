"""DMMA GEMM throughput on the rank-wide shapes of the large AMEn solves (N = TT rank ~ 70-96)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


g = torch.Generator(device="cuda").manual_seed(0)
# stage 3 of the local operator (configs[3]): y (n r0 x r1) = t2 (n r0 x r1p Rb') phiRp^T
for (M, N, K) in ((510 * 93, 89, 90 * 122), (254 * 71, 67, 68 * 110), (510 * 93, 93, 94 * 122)):
    A = torch.randn(M, K, generator=g, device="cuda", dtype=torch.float64)
    B = torch.randn(N, K, generator=g, device="cuda", dtype=torch.float64)
    C = torch.empty(M, N, device="cuda", dtype=torch.float64)
    ms = timeit(lambda: L.gemm(A, B, tB=True, out=C))
    print(f"stage3 M={M} N={N} K={K}: {ms:.3f} ms {2.0 * M * N * K / ms / 1e9:.1f} TF/s", flush=True)
# stage 1 (batched over n): Tp_j (Ra r0 x r1) = phiLp (Ra r0 x r0) v_j (r0 x r1)
for (n, Ra, r0, r1) in ((510, 121, 93, 89), (254, 109, 71, 67)):
    A = torch.randn(Ra * r0, r0, generator=g, device="cuda", dtype=torch.float64)
    V = torch.randn(n, r0, r1, generator=g, device="cuda", dtype=torch.float64)
    T = torch.empty(n, Ra * r0, r1, device="cuda", dtype=torch.float64)
    ms = timeit(lambda: L.gemm_strided(0, 0, Ra * r0, r1, r0, A, r0, 0, V, r1, r0 * r1, T, r1, Ra * r0 * r1, n))
    print(f"stage1 n={n} M={Ra * r0} N={r1} K={r0}: {ms:.3f} ms {2.0 * n * Ra * r0 * r0 * r1 / ms / 1e9:.1f} TF/s",
          flush=True)
