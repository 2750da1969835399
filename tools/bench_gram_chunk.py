"""Ozaki Gram of rows (1024 x 1M) timing; run with TTB_OZAKI_LONGK_CHUNK=<k> to compare K-range lengths."""
import os
import sys
import torch
sys.path.insert(0, ".")
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402

n, m = 1024, 1 << 20
T = torch.randn(n, m, device="cuda", dtype=torch.float64)
G = torch.empty(n, n, device="cuda", dtype=torch.float64)
ws = torch.empty(int(call_raw("ttb_ozaki_gram_rows_workspace", n, m)), dtype=torch.uint8, device="cuda")
for _ in range(2):
    call("ttb_ozaki_gram_rows", n, m, ptr(T), m, ptr(G), n, ptr(ws))
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    call("ttb_ozaki_gram_rows", n, m, ptr(T), m, ptr(G), n, ptr(ws))
b.record()
torch.cuda.synchronize()
ref = (T @ T.t())
err = ((G - ref).norm() / ref.norm()).item()
print(f"chunk {os.environ.get('TTB_OZAKI_LONGK_CHUNK', 'default')}: {a.elapsed_time(b) / 5:.2f} ms, err {err:.1e}")
