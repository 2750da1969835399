"""e2e (host path) timing variants at the bench workload: pinned vs pageable inputs, preallocated vs
allocated outputs."""
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_2509_13224_b200.tensor_train import tt_matvec_round_host
from paper_2509_13224_b200.workloads import matvec_round_instance

A, X = matvec_round_instance(1024, 16, 64, 3, seed=0)
npA = [G.cpu().numpy() for G in A.cores]
npX = [G.cpu().numpy() for G in X.cores]
pA = [torch.from_numpy(a).pin_memory() for a in npA]
pX = [torch.from_numpy(a).pin_memory() for a in npX]
out = tt_matvec_round_host(pA, pX, 1e-8)


def t(label, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
        del r
    torch.cuda.synchronize()
    print(f"{label}: {1e3 * (time.perf_counter() - t0) / reps:.1f} ms", flush=True)


t("pinned in, out=", lambda: tt_matvec_round_host(pA, pX, 1e-8, out=out))
t("pinned in, alloc out", lambda: tt_matvec_round_host(pA, pX, 1e-8))
t("numpy in, out=", lambda: tt_matvec_round_host(npA, npX, 1e-8, out=out))
t("numpy in, alloc out", lambda: tt_matvec_round_host(npA, npX, 1e-8))
