"""Wall time of one 1M x 1024 ttb_geqrf (CUDA events), 3 reps, best."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402

m, n = (1 << 20), 1024
X = torch.randn(n, m, dtype=torch.float64, device="cuda")
ws = L.empty(int(call_raw("ttb_qr_workspace", m, n)))
tau = L.empty(n)
best = 1e9
for _ in range(4):
    A = X.clone()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    call("ttb_geqrf", m, n, ptr(A), m, ptr(tau), ptr(ws))
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(f"geqrf 1M x 1024: {best:.2f} ms", flush=True)
