"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0].split("<")[0]
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    v = v / 1e3 if u in ("ns", "nsecond") else v * 1e3 if u in ("ms", "msecond") else v
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[-40:]:40s} {v[0]:8d} {v[1]:12.1f} {v[1] / v[0]:10.2f} {v[1] / tot:6.3f}")
