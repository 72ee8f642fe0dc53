#!/bin/bash
# ncu --set full of one k = 0 half-sweep (after the plain run exits 0)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/ncu_target.py sweep > gpurun_out/ncu_plain.log 2>&1 && {
ncu --set full --clock-control none --import-source on -k regex:lse_pass -s 40 -c 1 -o /tmp/prof_sweep -f python tools/ncu_target.py sweep > gpurun_out/ncu_sweep.log 2>&1
ncu -i /tmp/prof_sweep.ncu-rep --page details > gpurun_out/prof8_sweep_details.txt 2>&1
ncu -i /tmp/prof_sweep.ncu-rep --page raw --csv 2>&1 | gzip > gpurun_out/prof8_sweep_raw.csv.gz
}
