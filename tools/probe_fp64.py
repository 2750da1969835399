"""Probe: measured FP64 GEMM throughput (cuBLAS DGEMM via torch) and copy bandwidth.

Used only to fix the FP64 roofline denominator (MEASURED_PEAKS.json has no FP64 entry).
"""
import json, torch, subprocess
dev = torch.device("cuda:0")
out = {"gpu": torch.cuda.get_device_name(0)}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); c = a @ b; e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    out[f"dgemm_{n}_tflops"] = 2 * n**3 / best / 1e12
x = torch.empty(1 << 30, dtype=torch.uint8, device=dev); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); y.copy_(x); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e) / 1e3)
out["copy_gbs"] = 2 * (1 << 30) / best / 1e9
p = torch.cuda.get_device_properties(0)
out["sms"] = p.multi_processor_count
out["smem_optin"] = getattr(p, "shared_memory_per_block_optin", None)
print(json.dumps(out))
print(subprocess.run(["nvidia-smi", "-q", "-d", "CLOCK"], capture_output=True, text=True).stdout[:1500])
