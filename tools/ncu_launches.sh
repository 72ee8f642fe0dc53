#!/bin/bash
# ncu launch list (device time per launch) of a short target; summary by kernel
mkdir -p gpurun_out
TAG=${TAG:-r2}
python tools/ncu_target.py ${MODE:-late} ${CFG:-c3_gmm10k} > gpurun_out/ncu_launch_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c ${NL:-20000} --csv --log-file gpurun_out/launches_$TAG.csv \
    python tools/ncu_target.py ${MODE:-late} ${CFG:-c3_gmm10k} > gpurun_out/ncu_launch_$TAG.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1
cat gpurun_out/launches_$TAG.txt | head -30
