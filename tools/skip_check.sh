#!/bin/bash
# tile-skip A/B: pass timings and c3/c4 traces with and without PINS_NO_TILESKIP, then GPU tests
T=${1:-skip}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/probe_passes.py c2_img4k c3_gmm10k c4_l1rect > gpurun_out/${T}_passes.log 2>&1
PINS_NO_TILESKIP=1 timeout 300 python tools/probe_passes.py c2_img4k c3_gmm10k c4_l1rect > gpurun_out/${T}_passes_noskip.log 2>&1
for c in c3_gmm10k c4_l1rect c2_img4k; do
  timeout 300 python tools/probe_trace.py $c $T '{"newton_tol": 1e-8}' > gpurun_out/${T}_${c}.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tile_skip or tensor_core" > gpurun_out/${T}_pytest_skip.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc $?" >> gpurun_out/${T}_pytest.log
