#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "newton" > gpurun_out/tcl_pytest.log 2>&1; echo "rc $?" >> gpurun_out/tcl_pytest.log
for c in c3_gmm10k c4_l1rect; do
PINS_CG=treecl timeout 300 python tools/probe_trace.py $c tcl '{"newton_tol": 1e-8}' > gpurun_out/tcl_${c}.log 2>&1
done
