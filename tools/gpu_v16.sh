#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/probe_passes.py c2_img4k c3_gmm10k c4_l1rect c1_rand1k > gpurun_out/v17_passes.log 2>&1
for c in c3_gmm10k c4_l1rect c2_img4k; do
PINS_TREE_STATS=1 timeout 300 python tools/probe_trace.py $c v17 '{"newton_tol": 1e-8}' > gpurun_out/v17_${c}.log 2>&1
done
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/v17_pytest.log 2>&1; echo "rc $?" >> gpurun_out/v17_pytest.log
