"""Summarise round-2 ncu --set full captures (gpurun_out/ncu_r2_<tag>_raw.csv.gz):
per capture the kernel, duration, DRAM bytes read / written, DRAM throughput, achieved
occupancy, registers, IPC.  Writes profiles/ncu_r2_summary.json and the per-launch DRAM
traffic that bench.py puts into roofline.traffic (profiles/ncu_traffic_r2.json).

    python tools/ncu_extract.py [gpurun_out]
"""
import csv, glob, gzip, json, os, sys

SRC = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3, "second": 1e6,
         "us": 1.0, "ns": 1e-3, "ms": 1e3, "s": 1e6}
WANT = {"duration_us": "gpu__time_duration.sum", "dram_read_B": "dram__bytes_read.sum",
        "dram_write_B": "dram__bytes_write.sum", "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "registers": "launch__registers_per_thread", "ipc": "sm__inst_executed.avg.per_cycle_active"}

out = {}
for path in sorted(glob.glob(os.path.join(SRC, "ncu_r2_*_raw.csv.gz"))):
    tag = os.path.basename(path)[len("ncu_r2_"):-len("_raw.csv.gz")]
    rows = [r for r in csv.reader(gzip.open(path, "rt")) if r]
    rows = [r for r in rows if len(r) > 10]
    if len(rows) < 3:
        continue
    h, u = rows[0], rows[1]
    v = rows[2]
    if len(rows) > 3 and "gpu__time_duration.sum" in h:      # several launches captured: the longest one
        di = h.index("gpu__time_duration.sum")
        def dur(r):
            try:
                return float(r[di].replace(",", ""))
            except ValueError:
                return 0.0
        v = max(rows[2:], key=dur)
    e = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "?"}
    for k, name in WANT.items():
        if name in h:
            i = h.index(name)
            try:
                x = float(v[i].replace(",", ""))
            except ValueError:
                continue
            e[k] = x * SCALE.get(u[i], 1.0)
    if "dram_read_B" in e:
        e["dram_bytes_per_launch"] = e["dram_read_B"] + e.get("dram_write_B", 0.0)
    out[tag] = e
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_r2_summary.json"), "w"), indent=1)
# bench classes: the dominant kernel of each class in the c3 bench step
cls = {"sweep_row": "sweep", "eval": "eval", "cg": "treecl", "ksweep": "ksweep"}
traffic = {c: {"dram_bytes_per_launch": out[t]["dram_bytes_per_launch"], "kernel": out[t]["kernel"],
               "source": f"profiles/ncu_r2_{t}_details.txt (ncu --set full, one launch)"}
           for c, t in cls.items() if t in out and "dram_bytes_per_launch" in out[t]}
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic_r2.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
