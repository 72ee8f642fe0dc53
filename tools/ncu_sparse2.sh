#!/bin/bash
mkdir -p gpurun_out
PINS_LIST_STATS=1 python tools/probe_trace.py c3_gmm10k x '{"K": 1}' 2>&1 | grep lists
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lse_sparse -s 2000 -c 1 -o /tmp/prof_sp -f python tools/probe_trace.py c3_gmm10k x '{"K": 1}' > gpurun_out/ncu_sp.log 2>&1
ncu -i /tmp/prof_sp.ncu-rep --page details > gpurun_out/ncu_r2_sparse_details.txt 2>&1
ncu -i /tmp/prof_sp.ncu-rep --page raw --csv 2>&1 | gzip > gpurun_out/ncu_r2_sparse_raw.csv.gz
ncu -i /tmp/prof_sp.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu_r2_sparse_src_sass.csv.gz
PINS_NO_SPARSE_SWEEP=1 timeout 600 ncu --set full --clock-control none -k regex:lse_pass -s 4000 -c 1 -o /tmp/prof_dn -f python tools/probe_trace.py c3_gmm10k x '{"K": 1}' > gpurun_out/ncu_dn.log 2>&1
ncu -i /tmp/prof_dn.ncu-rep --page details > gpurun_out/ncu_r2_sweepk0_details.txt 2>&1
ncu -i /tmp/prof_dn.ncu-rep --page raw --csv 2>&1 | gzip > gpurun_out/ncu_r2_sweepk0_raw.csv.gz
grep -E "Duration|Registers Per|Achieved Occupancy|Issued Ipc|Avg. Active Threads|Issued Instructions  |Mem Busy|L1/TEX Hit" gpurun_out/ncu_r2_sparse_details.txt gpurun_out/ncu_r2_sweepk0_details.txt
