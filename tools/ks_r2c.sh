#!/bin/bash
# K-sweep: tests, per-class device times of a c3 solve, ncu --set full of the ELL walk and the merge
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "kernel_matrix" > gpurun_out/pytest_ks.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_ks.log
tail -3 gpurun_out/pytest_ks.log
timeout 300 python tools/probe_trace.py c3_gmm10k y '{"K": 200000, "outer_rule": 3, "outer_tol": 1e-7, "newton_tol": 1e-8}' > gpurun_out/probe_c3_prof.log 2>&1
python - <<'PY'
import json
d=json.loads(open("gpurun_out/probe_c3_prof.log").read().strip().splitlines()[-1])
for k,v in d["prof"].items(): print(k, v)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lse_ksweep -s 300 -c 1 -o /tmp/prof_ks -f python tools/probe_trace.py c3_gmm10k x '{"K": 1}' > gpurun_out/ncu_ks.log 2>&1
ncu -i /tmp/prof_ks.ncu-rep --page details > gpurun_out/ncu_r2_ksweep_details.txt 2>&1
ncu -i /tmp/prof_ks.ncu-rep --page raw --csv 2>&1 | gzip > gpurun_out/ncu_r2_ksweep_raw.csv.gz
ncu -i /tmp/prof_ks.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu_r2_ksweep_src_sass.csv.gz
timeout 600 ncu --set full --clock-control none -k regex:lse_merge -s 300 -c 1 -o /tmp/prof_mg -f python tools/probe_trace.py c3_gmm10k x '{"K": 1}' > gpurun_out/ncu_mg.log 2>&1
ncu -i /tmp/prof_mg.ncu-rep --page details > gpurun_out/ncu_r2_lsemerge_details.txt 2>&1
grep -E "Duration|Registers Per|Achieved Occupancy|Issued Ipc|DRAM Throughput|Mem Busy|L1/TEX Hit|Theoretical Occ|Memory Throughput" gpurun_out/ncu_r2_ksweep_details.txt gpurun_out/ncu_r2_lsemerge_details.txt
