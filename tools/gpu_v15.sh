#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/probe_passes.py c2_img4k c3_gmm10k c4_l1rect > gpurun_out/v15_passes.log 2>&1
for c in c3_gmm10k c4_l1rect; do
timeout 300 python tools/probe_trace.py $c v15 '{"newton_tol": 1e-8}' > gpurun_out/v15_${c}.log 2>&1
done
timeout 600 python tools/probe_trace.py c1_rand1k v15tol '{"newton_tol": 1e-8, "outer_tol": 3e-8, "K": 200000}' > gpurun_out/v15_c1tol.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/v15_pytest.log 2>&1; echo "rc $?" >> gpurun_out/v15_pytest.log
