"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(list)
for d in data:
    name = d["Kernel Name"]
    name = name.split("(")[0][:70]
    agg[name].append(float(d["Metric Value"]))
tot = sum(sum(v) for v in agg.values())
print(f"launches {len(data)}  total {tot/1e6:.2f} ms (serialised, cold-cache)")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{100*sum(v)/tot:5.1f}%  {sum(v)/1e6:8.2f} ms  n={len(v):5d}  avg={sum(v)/len(v)/1e3:8.1f} us  {k}")
