"""Time the Ozaki Gram of rows (1024 x 1M, the CholeskyQR2 Gram) for several long-K range policies."""
import os
import subprocess
import sys

if len(sys.argv) == 1:
    for kc in ("0", "4096", "8192", "16384"):
        env = dict(os.environ, TTB_OZAKI_LONGK_CHUNK=kc)
        out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
        print(f"chunk {kc}: {out.stdout.strip()} {out.stderr.strip()[-300:] if out.returncode else ''}", flush=True)
    sys.exit(0)

import torch  # noqa: E402

sys.path.insert(0, ".")
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402

n, m = 1024, 1 << 20
T = torch.randn(n, m, device="cuda", dtype=torch.float64)
G = torch.empty(n, n, device="cuda", dtype=torch.float64)
ws = torch.empty(int(call_raw("ttb_ozaki_gram_rows_workspace", n, m)), dtype=torch.uint8, device="cuda")
f = lambda: call("ttb_ozaki_gram_rows", n, m, ptr(T), m, ptr(G), n, ptr(ws))  # noqa
f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    f()
e1.record()
torch.cuda.synchronize()
Gd = T @ T.t()
print(f"{e0.elapsed_time(e1) / 3:.2f} ms per Gram (incl. slicing), rel err {float((G - Gd).norm() / Gd.norm()):.2e}")
