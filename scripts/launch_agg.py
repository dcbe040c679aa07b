"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel:
python scripts/launch_agg.py gpurun_out/x.csv [top]"""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
rows = [r for r in csv.DictReader(io.StringIO(txt)) if r.get("Metric Name") == "gpu__time_duration.sum"]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    k = r["Kernel Name"][:70] + " " + r["Grid Size"] + r["Block Size"]
    agg[k][0] += 1
    agg[k][1] += float(r["Metric Value"].replace(",", ""))
print("total kernel us %.1f, launches %d" % (sum(v[1] for v in agg.values()) / 1e3, len(rows)))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v[1] / 1e3:9.1f} us {v[0]:5d} x {v[1] / v[0] / 1e3:7.2f} us  {k}")
