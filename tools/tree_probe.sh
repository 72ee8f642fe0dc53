#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PINS_TREE_STATS=2 timeout 300 python tools/probe_trace.py c3_gmm10k tp '{"newton_tol": 1e-8, "K": 400, "outer_rule": 0, "outer_tol": 0.0}' > gpurun_out/tp_c3.log 2>&1
