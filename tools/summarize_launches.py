"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel
name: launches, total / mean device time and share of the total.  Usage:
    python tools/summarize_launches.py launches.csv [out.json]"""
import csv, json, re, sys
from collections import defaultdict

rows = []
with open(sys.argv[1]) as fh:
    lines = [l for l in fh if l.startswith('"')]
rd = csv.DictReader(lines)
tot = defaultdict(float); cnt = defaultdict(int)
for r in rd:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    short = re.sub(r"\(.*", "", name)
    short = re.sub(r"^void ", "", short)
    unit = r.get("Metric Unit", "nsecond")
    v = float(r["Metric Value"].replace(",", ""))
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
    tot[short] += v * scale; cnt[short] += 1
T = sum(tot.values())
out = {"total_ms": T, "launches": sum(cnt.values()),
       "kernels": sorted([{"kernel": k, "launches": cnt[k], "total_ms": tot[k], "mean_us": tot[k] / cnt[k] * 1e3,
                           "share": tot[k] / T} for k in tot], key=lambda e: -e["total_ms"])}
js = json.dumps(out, indent=1)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(js)
print(js[:4000])
