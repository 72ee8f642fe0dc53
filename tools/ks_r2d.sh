#!/bin/bash
# K-sweep with the TMA bulk pipeline: tests, per-class times (sorted vs row order), stats, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "kernel_matrix or sinkhorn_phase" > gpurun_out/pytest_ks.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_ks.log
tail -3 gpurun_out/pytest_ks.log
for v in sort nosort; do
if [ $v = nosort ]; then export PINS_KNOSORT=1; else unset PINS_KNOSORT; fi
PINS_LIST_STATS=1 timeout 300 python tools/probe_trace.py c3_gmm10k $v '{"K": 200000, "outer_rule": 3, "outer_tol": 1e-7, "newton_tol": 1e-8}' > gpurun_out/probe_c3_$v.log 2> gpurun_out/probe_c3_$v.err
grep "lists:" gpurun_out/probe_c3_$v.err | head -2
python - <<PY
import json
d=json.loads(open("gpurun_out/probe_c3_$v.log").read().strip().splitlines()[-1])
print("$v", {k:(v["launches"], round(v["ms"],1)) for k,v in d["prof"].items() if v["launches"]})
PY
done
unset PINS_KNOSORT
python tools/ab_env.py c3_gmm10k 2 - PINS_KNOSORT=1 PINS_LIST_MARGIN=12 > gpurun_out/ab_ks.log 2>&1
cut -c1-330 gpurun_out/ab_ks.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lse_ksweep -s 300 -c 1 -o /tmp/prof_ks -f python tools/probe_trace.py c3_gmm10k x '{"K": 1}' > gpurun_out/ncu_ks.log 2>&1
ncu -i /tmp/prof_ks.ncu-rep --page details > gpurun_out/ncu_r2_ksweep_details.txt 2>&1
ncu -i /tmp/prof_ks.ncu-rep --page raw --csv 2>&1 | gzip > gpurun_out/ncu_r2_ksweep_raw.csv.gz
ncu -i /tmp/prof_ks.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu_r2_ksweep_src_sass.csv.gz
grep -E "Duration|Registers Per|Achieved Occupancy|Issued Ipc|DRAM Throughput|Mem Busy|L1/TEX Hit|Theoretical Occ|Memory Throughput" gpurun_out/ncu_r2_ksweep_details.txt
