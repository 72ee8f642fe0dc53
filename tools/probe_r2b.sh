#!/bin/bash
# per-outer trace of the bench solve (c3, certified stop) + tree-PCG cycle stats; dense ncu captures
mkdir -p gpurun_out
P='{"K": 200000, "outer_rule": 3, "outer_tol": 1e-7, "newton_tol": 1e-8}'
timeout 300 python tools/probe_trace.py c3_gmm10k b "$P" > gpurun_out/pt_c3.log 2>&1
PINS_TREE_STATS=2 timeout 300 python tools/probe_trace.py c3_gmm10k ts "$P" > gpurun_out/pt_c3_ts.log 2>&1
timeout 300 python tools/probe_trace.py c3_gmm10k_r b "$P" > gpurun_out/pt_c3r.log 2>&1
PINS_SKIP_STATS=1 timeout 300 python tools/probe_trace.py c3_gmm10k sk "$P" > gpurun_out/pt_c3_sk.log 2>&1
if [ -n "$NCU" ]; then
source <(sed -n '/^cap()/,/^}/p' tools/ncu_r2.sh)
cap denserow dense 'lse_pass_kernel<\(int\)7' 6
cap densecol dense 'lse_pass_kernel<\(int\)8' 6
fi
