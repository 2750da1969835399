"""Summarize an ncu --metrics gpu__time_duration.sum CSV: per-kernel totals and shares."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
tot = collections.defaultdict(float); cnt = collections.Counter(); allt = 0.0
scale = {'nsecond': 1.0, 'usecond': 1e3, 'msecond': 1e6, 'second': 1e9}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
    name = r[ki].split('(')[0].replace('void ', '').replace('<unnamed>::', '')[:70]
    tot[name] += v; cnt[name] += 1; allt += v
print(f"launches {sum(cnt.values())}  total {allt/1e6:.2f} ms")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v/1e6:10.3f} ms {100*v/allt:6.2f}%  n={cnt[k]:5d}  {k}")
