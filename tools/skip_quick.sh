#!/bin/bash
# quick A/B of the chunk skip: pass timings (skip / no skip) and c3 / c4 traces
T=${1:-q}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/probe_passes.py c3_gmm10k c4_l1rect > gpurun_out/${T}_passes.log 2>&1
PINS_NO_TILESKIP=1 timeout 300 python tools/probe_passes.py c3_gmm10k c4_l1rect >> gpurun_out/${T}_passes.log 2>&1
for c in c3_gmm10k c4_l1rect; do
  timeout 300 python tools/probe_trace.py $c $T '{"newton_tol": 1e-8}' > gpurun_out/${T}_${c}.log 2>&1
done
for c in c3_gmm10k c4_l1rect; do
  PINS_NO_TILESKIP=1 timeout 300 python tools/probe_trace.py $c ${T}n '{"newton_tol": 1e-8}' > gpurun_out/${T}n_${c}.log 2>&1
done
for c in c3_gmm10k; do
  timeout 300 python tools/probe_trace.py $c ${T}r '{"newton_tol": 1e-8}' > gpurun_out/${T}r_${c}.log 2>&1
done
