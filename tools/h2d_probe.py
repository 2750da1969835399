"""Host->device staging options for pageable numpy inputs (2.1 GB, the configs[4] operator core)."""
import time
import numpy as np
import torch

n = 2 * 1024 ** 3 // 8
a = np.random.default_rng(0).standard_normal(n)
d = torch.empty(n, dtype=torch.float64, device="cuda")
p = torch.empty(n, dtype=torch.float64, pin_memory=True)
print("torch threads", torch.get_num_threads())
for rep in range(2):
    t = time.perf_counter(); p.copy_(torch.from_numpy(a)); dt = time.perf_counter() - t
    print(f"pageable->pinned torch copy_: {n * 8 / dt / 1e9:.1f} GB/s")
    t = time.perf_counter(); np.copyto(p.numpy(), a); dt = time.perf_counter() - t
    print(f"pageable->pinned np.copyto: {n * 8 / dt / 1e9:.1f} GB/s")
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(p, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"pinned H2D: {n * 8 / dt / 1e9:.1f} GB/s")
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(torch.from_numpy(a)); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"pageable H2D (driver staging): {n * 8 / dt / 1e9:.1f} GB/s")
    cr = torch.cuda.cudart()
    t = time.perf_counter()
    rc = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    d.copy_(torch.from_numpy(a), non_blocking=True); torch.cuda.synchronize()
    t2 = time.perf_counter()
    cr.cudaHostUnregister(a.ctypes.data)
    t3 = time.perf_counter()
    print(f"cudaHostRegister rc={rc}: register {1e3 * (t1 - t):.1f} ms, H2D {n * 8 / (t2 - t1) / 1e9:.1f} GB/s, unregister {1e3 * (t3 - t2):.1f} ms")
    # D2H into pinned, and pinned->pageable
    torch.cuda.synchronize(); t = time.perf_counter(); p.copy_(d, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"D2H pinned: {n * 8 / dt / 1e9:.1f} GB/s")
