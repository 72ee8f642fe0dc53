#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/probe_trace.py c1_rand1k base > gpurun_out/p2_c1_base.log 2>&1
timeout 300 python tools/probe_trace.py c3_gmm10k base > gpurun_out/p2_c3_base.log 2>&1
timeout 300 python tools/probe_trace.py c3_gmm10k nt8 '{"newton_tol": 1e-8}' > gpurun_out/p2_c3_nt8.log 2>&1
