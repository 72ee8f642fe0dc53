#!/bin/bash
# same-box A/B (chunk skip on / off) of c3 / c4 / c2 solves, then the GPU test suite
T=${1:-ab}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in c3_gmm10k c4_l1rect c2_img4k; do
  PINS_SKIP_STATS=1 timeout 300 python tools/probe_trace.py $c $T '{"newton_tol": 1e-8}' > gpurun_out/${T}_${c}.log 2>&1
  PINS_NO_X0=1 timeout 300 python tools/probe_trace.py $c ${T}n '{"newton_tol": 1e-8}' > gpurun_out/${T}n_${c}.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc $?" >> gpurun_out/${T}_pytest.log
