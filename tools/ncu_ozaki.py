"""One Ozaki FP64 GEMM inside the NVTX range "prof", for ncu. Default shape = the bench's middle-core
TT-matvec product (262144 x 4096 x 1024); override with M N K."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402

M, N, K = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (1 << 18, 4096, 1024)
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(M, K, generator=g, device="cuda", dtype=torch.float64)
B = torch.randn(K, N, generator=g, device="cuda", dtype=torch.float64)
C = torch.empty(M, N, device="cuda", dtype=torch.float64)
ws = torch.empty(int(call_raw("ttb_ozaki_workspace", M, N, K)), dtype=torch.uint8, device="cuda")
call("ttb_dgemm_ozaki", 0, M, N, K, ptr(A), K, ptr(B), N, ptr(C), N, ptr(ws))
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prof")
call("ttb_dgemm_ozaki", 0, M, N, K, ptr(A), K, ptr(B), N, ptr(C), N, ptr(ws))
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("done")
