#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/probe_passes.py c1_rand1k c2_img4k c3_gmm10k c4_l1rect > gpurun_out/v2_passes.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/v2_pytest.log 2>&1; echo "rc $?" >> gpurun_out/v2_pytest.log
timeout 400 python tools/probe_trace.py c3_gmm10k v2nt8 '{"newton_tol": 1e-8}' > gpurun_out/v2_c3_nt8.log 2>&1
