#!/bin/bash
# Development check on a B200 (via gpurun): build, per-pass timings, full solves with the
# per-outer trace and launch profile for the large configs, then the GPU test suite.
#   bash tools/gpu_check.sh TAG
T=${1:-chk}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/probe_passes.py c2_img4k c3_gmm10k c4_l1rect > gpurun_out/${T}_passes.log 2>&1
for c in c3_gmm10k c4_l1rect c2_img4k; do
  PINS_TREE_STATS=1 timeout 300 python tools/probe_trace.py $c $T '{"newton_tol": 1e-8}' > gpurun_out/${T}_${c}.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc $?" >> gpurun_out/${T}_pytest.log
