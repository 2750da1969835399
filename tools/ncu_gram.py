"""One Ozaki Gram of rows (1024 x 1M, the CholeskyQR Gram) inside the NVTX range "prof", for ncu."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402

n, m = 1024, 1 << 20
T = torch.randn(n, m, device="cuda", dtype=torch.float64)
G = torch.empty(n, n, device="cuda", dtype=torch.float64)
ws = torch.empty(int(call_raw("ttb_ozaki_gram_rows_workspace", n, m)), dtype=torch.uint8, device="cuda")
call("ttb_ozaki_gram_rows", n, m, ptr(T), m, ptr(G), n, ptr(ws))
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prof")
call("ttb_ozaki_gram_rows", n, m, ptr(T), m, ptr(G), n, ptr(ws))
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("done")
