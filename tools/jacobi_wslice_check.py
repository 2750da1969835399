"""Jacobi SVD of n x n matrices: time, sweeps and accuracy against LAPACK (numpy, host) for the
kernel selected by TTB_JACOBI (unset = warp-sliced default, g = previous Gram-block kernel)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402

alg = os.environ.get("TTB_JACOBI", "default")
rng = np.random.default_rng(0)
CASES = ((130, "gauss"), (256, "gauss"), (512, "gauss"), (1000, "gauss"), (1024, "gauss"), (1024, "graded"),
         (1024, "R^T gram"))
if os.environ.get("ODD"):
    CASES = ((130, "gauss"), (134, "graded"), (258, "gauss"), (510, "gauss"), (766, "R^T gram"), (1022, "gauss"))
if os.environ.get("SMALL"):
    CASES = ((32, "gauss"), (64, "gauss"), (72, "gauss"), (100, "gauss"), (110, "graded"), (128, "gauss"))
for n, kind in CASES:
    X = rng.standard_normal((n, n))
    if kind == "graded":
        X = X * np.logspace(0, -8, n)[None, :]
    if kind == "R^T gram":
        Y = rng.standard_normal((4 * n, n))
        X = np.linalg.qr(Y, mode="r").T.copy()
    s_ref = np.linalg.svd(X, compute_uv=False)
    for want_v in (False, True):
        M = torch.as_tensor(X.T.copy(), device="cuda")   # col-major X
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        L._jacobi(M.clone(), n, want_v, info)            # warm
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        U, S, V = L._jacobi(M.clone(), n, want_v, info)
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        Uh = U.cpu().numpy().T   # column-major storage -> columns are singular vectors
        Sh = S.cpu().numpy()
        es = np.abs(Sh - s_ref).max() / s_ref[0]
        esr = np.max(np.abs(Sh - s_ref) / s_ref)
        orth = np.abs(Uh.T @ Uh - np.eye(n)).max()
        rec = ""
        if want_v:
            Vh = V.cpu().numpy().T
            rec = f" recon {np.abs(Uh @ np.diag(Sh) @ Vh.T - X).max() / s_ref[0]:.1e} Vorth {np.abs(Vh.T @ Vh - np.eye(n)).max():.1e}"
        print(f"[{alg}] n={n:5d} {kind:9s} V={int(want_v)}: {ms:7.2f} ms sweeps {int(info.item()):2d}  "
              f"S err {es:.1e} (of s_max) {esr:.1e} (rel) U orth {orth:.1e}{rec}", flush=True)
