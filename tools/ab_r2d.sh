#!/bin/bash
mkdir -p gpurun_out
python tools/ab_env.py c3_gmm10k 2 - PINS_SPLIT_F=14.4 PINS_SPLIT_F=19.2 PINS_SPLIT_F=24 > gpurun_out/ab_r2d.log 2>&1
PINS_SKIP_STATS=1 PINS_SPLIT_F=14.4 timeout 300 python tools/probe_trace.py c3_gmm10k sk2 '{"K": 200000, "outer_rule": 3, "outer_tol": 1e-7, "newton_tol": 1e-8}' > gpurun_out/pt_c3_sk2.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "skip or bit or sinkhorn or reuse or fixed" > gpurun_out/pytest_r2d.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_r2d.log
cat gpurun_out/ab_r2d.log | cut -c1-300; grep "chunk skip" gpurun_out/pt_c3_sk2.log; tail -3 gpurun_out/pytest_r2d.log
