#!/bin/bash
# K-sweep with unit records: tests, per-class times, A/B, ncu launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "kernel_matrix or sinkhorn_phase" > gpurun_out/pytest_ks.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_ks.log
tail -3 gpurun_out/pytest_ks.log
PINS_LIST_STATS=1 timeout 300 python tools/probe_trace.py c3_gmm10k sort '{"K": 200000, "outer_rule": 3, "outer_tol": 1e-7, "newton_tol": 1e-8}' > gpurun_out/probe_c3_sort.log 2> gpurun_out/probe_c3_sort.err
python - <<PY
import json
d=json.loads(open("gpurun_out/probe_c3_sort.log").read().strip().splitlines()[-1])
print({k:(v["launches"], round(v["ms"],1)) for k,v in d["prof"].items() if v["launches"]})
PY
grep "lists:" gpurun_out/probe_c3_sort.err | head -3
python tools/ab_env.py c3_gmm10k 2 - PINS_KSWEEP_NOCOOL=1 PINS_LIST_MARGIN=12 > gpurun_out/ab_ks.log 2>&1
cut -c1-330 gpurun_out/ab_ks.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_ks.csv python tools/probe_trace.py c3_gmm10k x '{"K": 1}' > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches_ks.csv gpurun_out/launches_ks.json > /dev/null; python -c "import json; d=json.load(open(\"gpurun_out/launches_ks.json\")); [print(k[\"kernel\"][:60], k[\"launches\"], round(k[\"mean_us\"],1), round(k[\"share\"],3)) for k in d[\"kernels\"][:7]]"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lse_ksweep -s 300 -c 1 -o /tmp/prof_ks -f python tools/probe_trace.py c3_gmm10k x '{"K": 1}' > gpurun_out/ncu_ks.log 2>&1
ncu -i /tmp/prof_ks.ncu-rep --page details > gpurun_out/ncu_r2_ksweep_details.txt 2>&1
ncu -i /tmp/prof_ks.ncu-rep --page raw --csv 2>&1 | gzip > gpurun_out/ncu_r2_ksweep_raw.csv.gz
ncu -i /tmp/prof_ks.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu_r2_ksweep_src_sass.csv.gz
grep -E "Duration|Registers Per|Achieved Occupancy|Issued Ipc|DRAM Throughput|Mem Busy|L1/TEX Hit|Theoretical Occ|Memory Throughput" gpurun_out/ncu_r2_ksweep_details.txt
