"""Time the banded operator contraction: GEMM-staged (ttb_band_gemm / ttb_local_matvec_gemm) vs the
elementwise kernels, at configs[2]/[3]-like ranks. Prints one JSON line per case."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def case(n, h, R, r0, r1, naive=True):
    B = 2 * h + 1
    g = torch.Generator(device="cuda").manual_seed(0)
    M = torch.randn(R, n, B, R, generator=g, device="cuda", dtype=torch.float64)
    Mf = L.permute(M, (1, 2, 0, 3))
    phiL = torch.randn(r0, R, r0, generator=g, device="cuda", dtype=torch.float64)
    phiR = torch.randn(r1, R, r1, generator=g, device="cuda", dtype=torch.float64)
    v = torch.randn(n, r0, r1, generator=g, device="cuda", dtype=torch.float64)
    y = torch.empty_like(v)
    phiLp = L.permute(phiL, (1, 0, 2))
    r1p = r1 + (r0 & r1 & 1)
    phiRp = torch.zeros(r1, r1p, R, device="cuda", dtype=torch.float64)
    phiRp[:, :r1] = L.permute(phiR, (0, 2, 1))
    ws = L.empty(int(call_raw("ttb_local_gemm_workspace", r0, n, r1, R, R, h)))
    call("ttb_local_gemm_ws_init", r0, n, r1, R, h, ptr(ws))
    flops = 2.0 * n * r0 * r1 * B * R * R + 2 * 2.0 * n * r0 * r0 * r1 * R
    t_g = timeit(lambda: call("ttb_local_matvec_gemm", r0, n, r1, R, R, h, ptr(phiLp), ptr(Mf), ptr(phiRp), ptr(v),
                              ptr(y), ptr(ws)))
    Tp = ws[: (n + 2 * h) * R * r0 * r1p]
    out = L.empty(n, r0 * r1p, R)
    t_b = timeit(lambda: call("ttb_band_gemm", n, h, R, R, r0 * r1p, ptr(Tp), ptr(Mf), ptr(out)))
    res = {"n": n, "h": h, "R": R, "r0": r0, "r1": r1, "matvec_gemm_ms": t_g * 1e3,
           "matvec_gemm_tflops": flops / t_g / 1e12, "band_gemm_ms": t_b * 1e3,
           "band_gemm_tflops": 2.0 * n * r0 * r1 * B * R * R / t_b / 1e12}
    if naive:
        wsn = L.empty(r0 * R * n * r1 + r0 * n * R * r1)
        vn = L.permute(v, (1, 0, 2))
        yn = L.empty(r0, n, r1)
        t_n = timeit(lambda: call("ttb_local_matvec", r0, n, r1, R, R, h, ptr(phiL), ptr(M), ptr(phiR), ptr(vn),
                                  ptr(yn), ptr(wsn)), reps=2)
        res.update(matvec_naive_ms=t_n * 1e3, matvec_naive_tflops=flops / t_n / 1e12,
                   rel_diff=float((L.permute(y, (1, 0, 2)) - yn).norm() / yn.norm()))
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    case(64, 3, 40, 20, 20)
    case(256, 3, 109, 20, 20)
    case(256, 3, 109, 63, 63)
    case(512, 3, 121, 40, 40, naive=False)
    case(512, 3, 121, 64, 64, naive=False)
    case(510, 3, 122, 93, 89, naive=False)
