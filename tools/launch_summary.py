"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name:
python tools/launch_summary.py launches.csv [top]"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ms": 1.0, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "nsecond": 1e-6, "s": 1e3, "second": 1e3}
tot, cnt = {}, {}
for r in rows[1:]:
    name = r[ik].split("(")[0] if not r[ik].startswith("(") else r[ik].split(")")[1].split("(")[0]
    name = name.replace("void ", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    t = float(r[iv].replace(",", "")) * scale.get(r[iu], 1e-6)
    tot[name] = tot.get(name, 0.0) + t
    cnt[name] = cnt.get(name, 0) + 1
T = sum(tot.values())
print(f"launches {sum(cnt.values())}  total {T:.2f} ms")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v:10.3f} ms {100 * v / T:6.2f}%  n={cnt[k]:5d}  {k[:90]}")
