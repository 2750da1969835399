"""One 1024^2 Cholesky factorization (ttb_potrf) for ncu."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2509_13224_b200._lib import call, ptr  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(4 * n, n, generator=g, device="cuda", dtype=torch.float64)
G = X.t() @ X
info = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(2):
    A = G.clone()
    call("ttb_potrf", n, ptr(A), n, ptr(info))
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
A = G.clone()
a.record()
call("ttb_potrf", n, ptr(A), n, ptr(info))
b.record()
torch.cuda.synchronize()
L = torch.tril(A.t())     # col-major lower
print(f"potrf n={n}: {a.elapsed_time(b):.3f} ms, info {int(info)}, rel err {float((L @ L.t() - G).norm() / G.norm()):.2e}")
