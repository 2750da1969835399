"""One banded-operator GEMM (ttb_band_gemm) at the configs[3] local-system shape, for an ncu capture:
n=510 mode indices, h=3, operator ranks 121, X = r0 r1 = 93 * 86. Launch 0 is a warm-up, launch 1 is
the one to profile (ncu -k regex:dgemm_kernel --launch-skip 1 --launch-count 1)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200._lib import call, ptr  # noqa: E402

n, h, R, X = 510, 3, 121, 93 * 86
g = torch.Generator(device="cuda").manual_seed(0)
Mt = torch.randn(n, 2 * h + 1, R, R, generator=g, device="cuda", dtype=torch.float64)
Tp = torch.randn((n + 2 * h) * R * X, generator=g, device="cuda", dtype=torch.float64)
out = L.empty(n, X, R)
for _ in range(2):
    call("ttb_band_gemm", n, h, R, R, X, ptr(Tp), ptr(Mt), ptr(out))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
call("ttb_band_gemm", n, h, R, R, X, ptr(Tp), ptr(Mt), ptr(out))
e1.record()
torch.cuda.synchronize()
fl = 2.0 * n * X * (2 * h + 1) * R * R
ms = e0.elapsed_time(e1)
print(f"band_gemm n={n} h={h} R={R} X={X}: {ms:.3f} ms, {fl / ms / 1e9:.1f} TFLOP/s, "
      f"algorithmic bytes {8.0 * ((n + 2 * h) * R * X + n * (2 * h + 1) * R * R + n * X * R) / 1e9:.3f} GB")
