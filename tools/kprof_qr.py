"""CUPTI kernel split of one 1M x 1024 geqrf (+ orgqr) -- the rounding's dominant factorization."""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402

m, n = 1 << 20, 1024
X = torch.randn(n, m, dtype=torch.float64, device="cuda")
ws = L.empty(int(call_raw("ttb_qr_workspace", m, n)))
tau = L.empty(n)
for want_q in (False, True):
    A = X.clone()
    call("ttb_geqrf", m, n, ptr(A), m, ptr(tau), ptr(ws))
    torch.cuda.synchronize()
    A = X.clone()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        e0.record()
        call("ttb_geqrf", m, n, ptr(A), m, ptr(tau), ptr(ws))
        if want_q:
            Q = L.empty(n, m)
            call("ttb_orgqr", m, n, n, ptr(A), m, ptr(Q), m, ptr(ws), n)
        e1.record()
        torch.cuda.synchronize()
    tot, cnt = {}, {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            tot[e.name[:100]] = tot.get(e.name[:100], 0.0) + e.device_time_total
            cnt[e.name[:100]] = cnt.get(e.name[:100], 0) + 1
    print(f"{'geqrf+orgqr' if want_q else 'geqrf'}: wall {e0.elapsed_time(e1):.2f} ms, kernel sum {sum(tot.values()) / 1e3:.2f} ms")
    for name, us in sorted(tot.items(), key=lambda x: -x[1])[:16]:
        print(f"  {us / 1e3:8.2f} ms n={cnt[name]:4d} {name}")
