"""Summarise an ncu source-page CSV of a warp-specialised tcgen05 kernel: stall samples and
executions of the mbarrier try-wait loops (by smem offset), and the top stalled instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = 1 if "Address" in rows[1] else 0
hdr = rows[hi]
idx = {h: k for k, h in enumerate(hdr)}
data = rows[hi + 1:]
S = lambda r: float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
E = lambda r: int(r[idx["Instructions Executed"]] or 0)
tot = sum(S(r) for r in data)
keys = sys.argv[2:] or ["TRYWAIT", "UTCIMMA", "LDTM", "BAR.SYNC", "STL", "LDL", "SHFL", "MUFU", "F2F"]
for key in keys:
    rs = [r for r in data if key in r[1]]
    print(f"{key:10s} n={len(rs):4d} samples={sum(S(r) for r in rs) / tot * 100:5.1f}% executed={sum(E(r) for r in rs)}")
for r in [r for r in data if "TRYWAIT" in r[1]]:
    print(f"   {r[1][:70]:70s} exec={E(r):10d} samples={S(r) / tot * 100:.2f}%")
