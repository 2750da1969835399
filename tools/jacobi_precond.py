"""Sweep counts and times of the two 1024^2 Jacobi SVDs of the matvec+round step on the step's own
matrices (captured from linalg._jacobi), direct vs QR-preconditioned (Jacobi on R2^T, X^T = Q2 R2,
optionally with the columns pre-sorted by norm)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200 import workloads as W  # noqa: E402
from paper_2509_13224_b200.tensor_train import core as C  # noqa: E402

caps = []
orig = L._jacobi


def spy(Rcm, n, want_v=False, info=None):
    if n == 1024:
        caps.append(Rcm.clone())
    return orig(Rcm, n, want_v, info)


L._jacobi = spy
A, x = W.matvec_round_instance(1024)
C.tt_round(C.tt_matvec(A, x), 1e-8)
torch.cuda.synchronize()
L._jacobi = orig
print("captured", len(caps), flush=True)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), out


n = 1024
for ci, Acm in enumerate(caps):
    X = Acm.t()                                   # row-major view of the col-major matrix
    S_ref = torch.linalg.svdvals(X)
    norms = torch.linalg.vector_norm(Acm, dim=1)  # column norms of the col-major matrix
    print(f"matrix {ci}: cond {float(S_ref[0] / S_ref[-1]):.2e}, col norms {float(norms.min()):.2e}..{float(norms.max()):.2e}")
    for mode in ("direct", "qr", "sorted_qr"):
        info = torch.zeros(1, dtype=torch.int32, device="cuda")

        def run():
            if mode == "direct":
                return L._jacobi(Acm.clone(), n, False, info)
            src = Acm
            if mode == "sorted_qr":
                src = Acm[torch.argsort(norms, descending=True)]
            _, Rt2 = L.qr_colmajor(src.clone(), n, n, want_q=False)
            return L._jacobi(Rt2.t().contiguous(), n, False, info)

        for _ in range(2):
            ms, (U, S, V) = timed(run)
        err = float(((S.sort(descending=True).values - S_ref).abs() / S_ref[0]).max())
        print(f"  {mode:10s}: {ms:7.2f} ms, sweeps {int(info.item())}, s err {err:.1e}", flush=True)
