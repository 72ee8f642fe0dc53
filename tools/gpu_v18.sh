#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PINS_TREE_STATS=1 timeout 300 python tools/probe_trace.py c3_gmm10k v18 '{"newton_tol": 1e-8}' > gpurun_out/v18_c3.log 2>&1
PINS_CLUSTER_NNZ_MAX=100000 timeout 300 python tools/probe_trace.py c3_gmm10k v18b '{"newton_tol": 1e-8}' > gpurun_out/v18b_c3.log 2>&1
PINS_CLUSTER_NNZ_MAX=1000000 timeout 300 python tools/probe_trace.py c3_gmm10k v18c '{"newton_tol": 1e-8}' > gpurun_out/v18c_c3.log 2>&1
timeout 300 python tools/probe_trace.py c4_l1rect v18 '{"newton_tol": 1e-8}' > gpurun_out/v18_c4.log 2>&1
timeout 600 python tools/probe_trace.py c1_rand1k v18 '{"newton_tol": 1e-8, "outer_tol": 2e-8, "K": 200000}' > gpurun_out/v18_c1.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/v18_pytest.log 2>&1; echo "rc $?" >> gpurun_out/v18_pytest.log
