#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "sparse_sweeps" > gpurun_out/pytest_r2g.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_r2g.log
tail -3 gpurun_out/pytest_r2g.log
PINS_LIST_STATS=1 timeout 300 python tools/probe_trace.py c3_gmm10k ls '{"K": 200000, "outer_rule": 3, "outer_tol": 1e-7, "newton_tol": 1e-8}' > gpurun_out/pt_c3_ls.log 2>&1
grep lists gpurun_out/pt_c3_ls.log | head -3; tail -1 gpurun_out/pt_c3_ls.log | cut -c 300-900
head -2 gpurun_out/trace_c3_gmm10k_ls.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_ls.csv python tools/ncu_target.py sweep > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches_ls.csv | head -40
