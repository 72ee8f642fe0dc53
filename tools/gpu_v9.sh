#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PINS_TREE_STATS=1 timeout 300 python tools/probe_trace.py c3_gmm10k v11 '{"newton_tol": 1e-8}' > gpurun_out/v11_c3.log 2>&1
PINS_TREE_STATS=1 timeout 300 python tools/probe_trace.py c2_img4k v11 '{"newton_tol": 1e-8}' > gpurun_out/v11_c2.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "newton or solve or cg" > gpurun_out/v11_pytest.log 2>&1; echo "rc $?" >> gpurun_out/v11_pytest.log
