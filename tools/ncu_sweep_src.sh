#!/bin/bash
# ncu --set full with source counters of one k = 0 half-sweep (after the plain run exits 0)
mkdir -p gpurun_out
TAG=${TAG:-r2}
python tools/ncu_target.py sweep ${CFG:-c3_gmm10k} > gpurun_out/ncu_plain_$TAG.log 2>&1 && {
ncu --set full --clock-control none --import-source on -k regex:lse_pass -s ${SKIP:-40} -c 1 -o /tmp/prof_sweep -f python tools/ncu_target.py sweep ${CFG:-c3_gmm10k} > gpurun_out/ncu_sweep_$TAG.log 2>&1
ncu -i /tmp/prof_sweep.ncu-rep --page details > gpurun_out/ncu_${TAG}_sweep_details.txt 2>&1
ncu -i /tmp/prof_sweep.ncu-rep --page raw --csv 2>&1 | gzip > gpurun_out/ncu_${TAG}_sweep_raw.csv.gz
ncu -i /tmp/prof_sweep.ncu-rep --page source --csv --print-source cuda 2>&1 | gzip > gpurun_out/ncu_${TAG}_sweep_src_cuda.csv.gz
ncu -i /tmp/prof_sweep.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu_${TAG}_sweep_src_sass.csv.gz
}
