#!/bin/bash
# late-phase structure of the bench solve: per-outer trace + tree-PCG cycle split (dev probe)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
P='{"K": 200000, "outer_rule": 3, "outer_tol": 1e-7, "newton_tol": 1e-8}'
timeout 300 python tools/probe_trace.py c3_gmm10k r2h "$P" > gpurun_out/r2h_c3.log 2>&1
PINS_TREE_STATS=1 timeout 300 python tools/probe_trace.py c3_gmm10k r2hs "$P" > gpurun_out/r2hs_c3.log 2>&1
timeout 300 python tools/probe_trace.py c1_rand1k r2h "$P" > gpurun_out/r2h_c1.log 2>&1
