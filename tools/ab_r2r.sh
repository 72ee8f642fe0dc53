#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "sparse_sweeps or uninitialised or sinkhorn_phase or reproducible" > gpurun_out/pytest_r2r.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_r2r.log
tail -4 gpurun_out/pytest_r2r.log
python tools/ab_env.py c3_gmm10k 2 - PINS_SPARSE_SWEEP=1 PINS_SPARSE_SWEEP=1,PINS_LIST_MARGIN=8 > gpurun_out/ab_r2r.log 2>&1
cut -c1-330 gpurun_out/ab_r2r.log
PINS_SPARSE_SWEEP=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_ls.csv python tools/probe_trace.py c3_gmm10k x '{"K": 1}' > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches_ls.csv gpurun_out/launches_ls.json > /dev/null; python -c "import json; d=json.load(open(\"gpurun_out/launches_ls.json\")); [print(k[\"kernel\"][:50], k[\"launches\"], round(k[\"mean_us\"],1), round(k[\"share\"],3)) for k in d[\"kernels\"][:12]]"
