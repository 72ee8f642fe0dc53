#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in c3_gmm10k c4_l1rect c2_img4k; do
timeout 300 python tools/probe_trace.py $c ws2 '{"newton_tol": 1e-8, "warm_start": 2}' > gpurun_out/ws2_${c}.log 2>&1
done
timeout 600 python tools/probe_trace.py c1_rand1k ws2 '{"newton_tol": 1e-8, "warm_start": 2, "outer_tol": 2e-8, "K": 200000}' > gpurun_out/ws2_c1_rand1k.log 2>&1
