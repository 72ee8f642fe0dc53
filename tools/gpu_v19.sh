#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/probe_passes.py c2_img4k c3_gmm10k c4_l1rect > gpurun_out/v19_passes.log 2>&1
PINS_TREE_STATS=1 timeout 300 python tools/probe_trace.py c3_gmm10k v19 '{"newton_tol": 1e-8}' > gpurun_out/v19_c3.log 2>&1
timeout 300 python tools/probe_trace.py c4_l1rect v19 '{"newton_tol": 1e-8}' > gpurun_out/v19_c4.log 2>&1
timeout 300 python tools/probe_trace.py c2_img4k v19 '{"newton_tol": 1e-8}' > gpurun_out/v19_c2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/v19_pytest.log 2>&1; echo "rc $?" >> gpurun_out/v19_pytest.log
