"""Development aid: per-kernel time table of an ncu launch list (gpu__time_duration.sum CSV)."""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))]
agg = collections.OrderedDict()
tot = 0.0
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0]
    if "<" in r["Kernel Name"].split("(")[0] or True:
        name = r["Kernel Name"]
        name = name[:name.index("(")] if "(" in name and "<" not in name[:name.index("(")] else name.split(">(")[0] + ">" if ">(" in name else name
    us = float(r["Metric Value"].replace(",", "")) / (1000.0 if r["Metric Unit"] == "ns" else 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
    tot += us
print(f"{len(rows)} launches, {tot/1000:.3f} ms total")
for name, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{us/1000:9.3f} ms {100*us/tot:5.1f}% {c:4d}x {us/c:9.1f} us  {name[:90]}")
