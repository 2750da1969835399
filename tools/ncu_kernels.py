"""Representative single launches of the non-GEMM kernel families, for `ncu --set full`: a warm-up
call, then the profiled call inside the NVTX range "prof" (ncu --nvtx --nvtx-include "prof/").
Usage: python tools/ncu_kernels.py geo|maxvol|tsqr|l1err

geo    -- geo_kernel mode 0 (one metric entry R_01) at 8M points of the configs[2] deformed cube
maxvol -- maxvol_kernel on a 122400 x 60 fiber matrix (configs[3] cross shape)
tsqr   -- one 1M x 1024 geqrf (tsqr_factor_kernel<16> leaf launches of the tall panels)
l1err  -- the configs[1] error integral (l1err_kernel over all quadrature points)
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402

what = sys.argv[1]
if what == "geo":
    from paper_2509_13224_b200 import driver as D
    from paper_2509_13224_b200.geometry import GridEvaluator
    from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
    cfg = D.SolveConfig(seed=0, **SOLVE_CONFIGS[2])
    patch = D.make_geometry(cfg.geometry, cfg.geometry_params)
    nq = 1016
    ax = [np.linspace(0.001, 0.999, nq)] * 3
    ev = GridEvaluator(patch, ax)
    g = torch.Generator(device="cuda").manual_seed(0)
    idx = torch.randint(0, nq, (1 << 23, 3), generator=g, device="cuda", dtype=torch.int64)
    ev.metric_entry(idx, 0, 1, check=False)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("prof")
    ev.metric_entry(idx, 0, 1, check=False)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
elif what == "maxvol":
    g = torch.Generator(device="cuda").manual_seed(0)
    n, r = 122400, 60
    Q = torch.randn(r, n, generator=g, device="cuda", dtype=torch.float64)
    L.maxvol_colmajor(Q, n, r)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("prof")
    L.maxvol_colmajor(Q, n, r)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
elif what == "tsqr":
    m, n = (1 << 20), 1024
    X = torch.randn(n, m, dtype=torch.float64, device="cuda")
    ws = L.empty(int(call_raw("ttb_qr_workspace", m, n)))
    tau = L.empty(n)
    for rep in range(2):
        A = X.clone()
        if rep:
            torch.cuda.nvtx.range_push("prof")
        call("ttb_geqrf", m, n, ptr(A), m, ptr(tau), ptr(ws))
        if rep:
            torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
elif what == "l1err":
    from paper_2509_13224_b200 import driver as D
    from paper_2509_13224_b200.workloads import SOLVE_CONFIGS
    for rep in range(2):
        if rep:
            torch.cuda.nvtx.range_push("prof")
        D.solve_poisson(D.SolveConfig(seed=0, **SOLVE_CONFIGS[1]), want_error=True)
        if rep:
            torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
print(what, "done")
