#!/bin/bash
mkdir -p gpurun_out
python tools/ncu_target.py sweep > gpurun_out/ncu_sp_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lse_sparse -s 20 -c 1 -o /tmp/prof_sp -f python tools/ncu_target.py sweep > gpurun_out/ncu_sp.log 2>&1
ncu -i /tmp/prof_sp.ncu-rep --page details > gpurun_out/ncu_r2_sparse_details.txt 2>&1
ncu -i /tmp/prof_sp.ncu-rep --page raw --csv 2>&1 | gzip > gpurun_out/ncu_r2_sparse_raw.csv.gz
ncu -i /tmp/prof_sp.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu_r2_sparse_src_sass.csv.gz
ncu -i /tmp/prof_sp.ncu-rep --page source --csv --print-source cuda 2>&1 | gzip > gpurun_out/ncu_r2_sparse_src_cuda.csv.gz
grep -E "Duration|Registers|Achieved Occupancy|Issued Ipc|No Eligible" gpurun_out/ncu_r2_sparse_details.txt
