#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "sparse_sweeps or sinkhorn or tile_skip or fixed_iterations or reproducible" > gpurun_out/pytest_r2e.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_r2e.log
tail -15 gpurun_out/pytest_r2e.log
PINS_LIST_STATS=1 timeout 300 python tools/probe_trace.py c3_gmm10k ls '{"K": 200000, "outer_rule": 3, "outer_tol": 1e-7, "newton_tol": 1e-8}' > gpurun_out/pt_c3_ls.log 2>&1
grep lists gpurun_out/pt_c3_ls.log | head -20
python tools/ab_env.py c3_gmm10k 2 - PINS_NO_SPARSE_SWEEP=1 PINS_LIST_MARGIN=2 PINS_LIST_MARGIN=8 > gpurun_out/ab_r2e.log 2>&1
python tools/ab_env.py c3_gmm10k_r 1 - PINS_NO_SPARSE_SWEEP=1 >> gpurun_out/ab_r2e.log 2>&1
python tools/ab_env.py c4_l1rect 1 - PINS_NO_SPARSE_SWEEP=1 >> gpurun_out/ab_r2e.log 2>&1
cut -c1-330 gpurun_out/ab_r2e.log
