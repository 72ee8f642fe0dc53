#!/bin/bash
# same-box A/B of the sum kernel's launch bounds: (kPT, 5) as built, then (kPT)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/probe_passes.py c3_gmm10k c4_l1rect > gpurun_out/lb5_passes.log 2>&1
timeout 300 python tools/probe_trace.py c3_gmm10k lb5 '{"newton_tol": 1e-8}' > gpurun_out/lb5_c3.log 2>&1
timeout 300 python tools/probe_trace.py c3_gmm10k lb5b '{"newton_tol": 1e-8}' > gpurun_out/lb5b_c3.log 2>&1
sed -i 's/__launch_bounds__(kPT, 5) sum_pass_kernel/__launch_bounds__(kPT) sum_pass_kernel/' paper_2502_03749_b200/csrc/pins_pass.cuh
python -c "import __graft_entry__ as g; g.build()" >> gpurun_out/build.log 2>&1
timeout 300 python tools/probe_passes.py c3_gmm10k c4_l1rect > gpurun_out/lb0_passes.log 2>&1
timeout 300 python tools/probe_trace.py c3_gmm10k lb0 '{"newton_tol": 1e-8}' > gpurun_out/lb0_c3.log 2>&1
timeout 300 python tools/probe_trace.py c3_gmm10k lb0b '{"newton_tol": 1e-8}' > gpurun_out/lb0b_c3.log 2>&1
