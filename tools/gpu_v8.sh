#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/probe_passes.py c1_rand1k c2_img4k c3_gmm10k c4_l1rect > gpurun_out/v8_passes.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/v8_pytest.log 2>&1; echo "rc $?" >> gpurun_out/v8_pytest.log
for c in c3_gmm10k c2_img4k c4_l1rect c1_rand1k; do
timeout 300 python tools/probe_trace.py $c v8 '{"newton_tol": 1e-8}' > gpurun_out/v8_${c}.log 2>&1
done
