"""Mean per-kernel duration from an ncu --csv launch list (gpu__time_duration)."""
import csv
import collections
import sys

rows = collections.defaultdict(list)
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("fcpd::", "")
    v = float(r["Metric Value"].replace(",", ""))
    rows[name].append(v / 1e3 if r["Metric Unit"] == "ns" else v)
tot = sum(sum(v) for v in rows.values())
for k, v in sorted(rows.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:40s} n={len(v):3d} mean={sum(v)/len(v):9.1f} us  share={100*sum(v)/tot:5.1f}%")
