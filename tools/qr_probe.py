"""geqrf + orgqr time and launch count for a few (m, n) (development probe): python tools/qr_probe.py m n [m n ...]"""
import sys
import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, ".")
from paper_2509_13224_b200 import _lib, linalg as L  # noqa: E402

lib = _lib.lib()
args = [int(a) for a in sys.argv[1:]] or [2040, 510, 1016, 254, 260100, 510, 8160, 510, 510, 510]
for m, n in zip(args[::2], args[1::2]):
    X = torch.randn(n, m, dtype=torch.float64, device="cuda")
    for want_q in (False, True):
        L.qr_colmajor(X.clone(), m, n, want_q=want_q)
        torch.cuda.synchronize()
        lib.ttb_launch_count(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        Xc = X.clone()
        a.record()
        L.qr_colmajor(Xc, m, n, want_q=want_q)
        b.record()
        torch.cuda.synchronize()
        print(f"m={m} n={n} want_q={want_q}: {a.elapsed_time(b):8.2f} ms, {lib.ttb_launch_count(1)} launches", flush=True)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        L.qr_colmajor(X.clone(), m, n)
        torch.cuda.synchronize()
    tot, cnt = {}, {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            tot[e.name[:70]] = tot.get(e.name[:70], 0.0) + e.device_time_total
            cnt[e.name[:70]] = cnt.get(e.name[:70], 0) + 1
    for name, us in sorted(tot.items(), key=lambda x: -x[1])[:6]:
        print(f"    {us / 1e3:8.2f} ms n={cnt[name]:5d} {name}")
