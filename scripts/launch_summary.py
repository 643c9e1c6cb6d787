"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import re
import sys

path = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
lines = [l for l in open(path) if not l.startswith("==")]
agg = collections.defaultdict(lambda: [0, 0.0])
for x in csv.DictReader(lines):
    if x.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(x["Metric Value"]) * (1e-3 if x["Metric Unit"] == "ns" else 1.0 if x["Metric Unit"] == "us" else 1e3)
    k = re.sub(r"\(.*", "", x["Kernel Name"]).replace("void ", "").replace("<unnamed>::", "").replace("nat::", "")
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':58s} {'launches':>8s} {'us/step':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:58]:58s} {v[0] / div:8.1f} {v[1] / div:10.1f} {100 * v[1] / tot:5.1f}%")
print(f"{'total':58s} {'':8s} {tot / div:10.1f}")
