"""Summarise an ncu launch list (gpu__time_duration.sum CSV): per-kernel count, total, share."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[h], rows[h + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
for r in data:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(r[ui], 1e-9)
    name = r[ki].split("(")[0]
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:70]:70s} {cnt[k]:8d} {tot[k]*1e3:10.3f} {tot[k]/T*100:6.2f}%")
print(f"{'TOTAL':70s} {sum(cnt.values()):8d} {T*1e3:10.3f}")
