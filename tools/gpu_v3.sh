#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/v3_pytest.log 2>&1; echo "rc $?" >> gpurun_out/v3_pytest.log
for c in c3_gmm10k c2_img4k c4_l1rect c1_rand1k; do
timeout 300 python tools/probe_trace.py $c v3nt8 '{"newton_tol": 1e-8}' > gpurun_out/v3_${c}_nt8.log 2>&1
done
