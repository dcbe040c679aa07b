"""Summarise an `ncu --page source --csv --print-source sass` export: top
instructions by warp-stall samples with their dominant stall reasons, and the
sample totals per stall reason. python scripts/sass_hotspots.py file.csv [N]"""
import csv
import sys
from collections import Counter

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
tot = Counter()
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    st = {h: int(r[idx[h]] or 0) for h in stalls}
    tot.update(st)
    data.append((s, r[idx["Address"]], r[idx["Source"]], st, r[idx["Instructions Executed"]]))
allsamp = sum(d[0] for d in data)
print(f"total samples {allsamp}")
for k, v in tot.most_common(10):
    print(f"  {k:28s} {v:8d} {100 * v / max(allsamp, 1):5.1f}%")
print()
for s, a, src, st, ie in sorted(data, key=lambda d: -d[0])[:top]:
    top3 = ", ".join(f"{k[6:]}={v}" for k, v in Counter(st).most_common(3) if v)
    print(f"{s:7d} {100 * s / max(allsamp, 1):5.1f}%  {a:>6s}  {src[:60]:60s} exec={ie:>8s}  {top3}")
