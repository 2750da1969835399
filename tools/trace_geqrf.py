"""Kernel timeline (CUPTI, torch.profiler) of one 1M x 1024 geqrf: per-stream busy time and overlap."""
import json
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2509_13224_b200 import linalg as L  # noqa: E402
from paper_2509_13224_b200._lib import call, call_raw, ptr  # noqa: E402

m, n = (1 << 20), 1024
X = torch.randn(n, m, dtype=torch.float64, device="cuda")
ws = L.empty(int(call_raw("ttb_qr_workspace", m, n)))
tau = L.empty(n)
A = X.clone()
call("ttb_geqrf", m, n, ptr(A), m, ptr(tau), ptr(ws))
A = X.clone()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    call("ttb_geqrf", m, n, ptr(A), m, ptr(tau), ptr(ws))
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/geqrf_trace.json")
ev = [e for e in json.load(open("gpurun_out/geqrf_trace.json"))["traceEvents"] if e.get("cat") == "kernel"]
t0 = min(e["ts"] for e in ev)
t1 = max(e["ts"] + e["dur"] for e in ev)
print(f"span {(t1 - t0) / 1e3:.2f} ms, kernels {len(ev)}")
by = {}
for e in ev:
    s = e["args"].get("stream")
    by.setdefault(s, []).append(e)
for s, es in by.items():
    busy = sum(e["dur"] for e in es)
    print(f"stream {s}: {len(es)} kernels busy {busy / 1e3:.2f} ms")
# coarse timeline: 2 ms bins, which streams are active
bins = int((t1 - t0) / 2000) + 1
act = [[0.0] * bins for _ in by]
keys = list(by)
for si, s in enumerate(keys):
    for e in by[s]:
        a, b = e["ts"] - t0, e["ts"] - t0 + e["dur"]
        for k in range(int(a // 2000), min(bins, int(b // 2000) + 1)):
            lo, hi = max(a, k * 2000), min(b, (k + 1) * 2000)
            if hi > lo:
                act[si][k] += (hi - lo) / 2000
for k in range(bins):
    print(f"{k * 2:4d} ms " + " ".join(f"{keys[si]}:{min(act[si][k], 9.99):4.2f}" for si in range(len(keys))))
for e in sorted(ev, key=lambda e: e["ts"])[:400]:
    print(f"{(e['ts'] - t0) / 1e3:8.3f} {e['dur'] / 1e3:7.3f} s{e['args'].get('stream')} {e['name'][:70]}")
