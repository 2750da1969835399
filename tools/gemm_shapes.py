"""Histogram of the large DMMA GEMM shapes of one BASELINE solve (TTB_GEMM_LOG stderr lines)."""
import collections
import sys
c = collections.Counter()
for line in open(sys.argv[1]):
    if line.startswith("ttb_gemm"):
        c[line.split(" ", 1)[1].strip()] += 1
tot = []
for k, n in c.items():
    d = dict(kv.split("=") for kv in k.split())
    fl = 2.0 * int(d["M"]) * int(d["N"]) * int(d["K"]) * int(d["batch"])
    tot.append((fl * n, n, k))
for fl, n, k in sorted(tot, reverse=True)[:20]:
    print(f"{fl / 1e12:9.2f} TFLOP  n={n:5d}  {k}")
