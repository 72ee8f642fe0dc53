#!/bin/bash
# A/B of the tree-PCG nnz cap on c3 / c2 (same box)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for lim in 400000 200000 100000 50000; do
  for c in c3_gmm10k c2_img4k; do
    PINS_TREE_NNZ_MAX=$lim timeout 300 python tools/probe_trace.py $c cap$lim '{"newton_tol": 1e-8}' > gpurun_out/cap${lim}_${c}.log 2>&1
  done
done
