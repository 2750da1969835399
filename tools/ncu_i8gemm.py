"""One TMA-fed tcgen05 INT8 GEMM launch (8192^3) inside the NVTX range "prof", for ncu."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200._lib import call, ptr  # noqa: E402

M = N = K = 8192
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randint(-127, 128, (M, K), generator=g, device="cuda", dtype=torch.int8)
B = torch.randint(-127, 128, (N, K), generator=g, device="cuda", dtype=torch.int8)
C = torch.empty(M, N, dtype=torch.int32, device="cuda")
call("ttb_i8gemm", M, N, K, ptr(A), ptr(B), ptr(C))
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prof")
call("ttb_i8gemm", M, N, K, ptr(A), ptr(B), ptr(C))
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("done")
