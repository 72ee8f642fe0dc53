#!/bin/bash
# K-sweep bring-up: tests, A/B on c3 (dense vs absorbed kernel-matrix sweeps), list stats, launch list
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "kernel_matrix or sparse_sweeps or sinkhorn_phase or sinkhorn_sweep" > gpurun_out/pytest_ks.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_ks.log
tail -15 gpurun_out/pytest_ks.log
PINS_LIST_STATS=1 python tools/ab_env.py c3_gmm10k 2 PINS_KSWEEP=0 - > gpurun_out/ab_ks.log 2>&1
cut -c1-400 gpurun_out/ab_ks.log
PINS_LIST_STATS=1 timeout 300 python tools/probe_trace.py c3_gmm10k x '{"K": 1}' 2>&1 | grep -i "lists:" | head -5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_ks.csv python tools/probe_trace.py c3_gmm10k x '{"K": 1}' > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches_ks.csv gpurun_out/launches_ks.json > /dev/null; python -c "import json; d=json.load(open(\"gpurun_out/launches_ks.json\")); [print(k[\"kernel\"][:60], k[\"launches\"], round(k[\"mean_us\"],1), round(k[\"share\"],3)) for k in d[\"kernels\"][:14]]"
