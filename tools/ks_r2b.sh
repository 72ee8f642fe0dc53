#!/bin/bash
# K-sweep tuning: tests, margin A/B on c3 and c3_r / c4, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "kernel_matrix or sinkhorn_phase" > gpurun_out/pytest_ks.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_ks.log
tail -5 gpurun_out/pytest_ks.log
PINS_LIST_STATS=1 python tools/ab_env.py c3_gmm10k 2 - PINS_LIST_MARGIN=8 PINS_LIST_MARGIN=12 PINS_LIST_MARGIN=20 > gpurun_out/ab_ks.log 2>&1
cut -c1-330 gpurun_out/ab_ks.log
python tools/ab_env.py c3_gmm10k_r 1 PINS_KSWEEP=0 - PINS_LIST_MARGIN=12 > gpurun_out/ab_ks_r.log 2>&1
cut -c1-330 gpurun_out/ab_ks_r.log
python tools/ab_env.py c4_l1rect 1 PINS_KSWEEP=0 - PINS_LIST_MARGIN=12 > gpurun_out/ab_ks_c4.log 2>&1
cut -c1-330 gpurun_out/ab_ks_c4.log
for mg in 4 12; do
PINS_LIST_MARGIN=$mg PINS_LIST_STATS=1 timeout 300 python tools/probe_trace.py c3_gmm10k x '{"K": 1}' 2>&1 | grep -i "lists:" | head -3
PINS_LIST_MARGIN=$mg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_ks$mg.csv python tools/probe_trace.py c3_gmm10k x '{"K": 1}' > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches_ks$mg.csv gpurun_out/launches_ks$mg.json > /dev/null; python -c "import json; d=json.load(open(\"gpurun_out/launches_ks$mg.json\")); [print(k[\"kernel\"][:60], k[\"launches\"], round(k[\"mean_us\"],1), round(k[\"share\"],3)) for k in d[\"kernels\"][:7]]"
done
