#!/bin/bash
# first GPU call of the session: state of the GPU tests + full-size solve probes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
for c in c1_rand1k c2_img4k c3_gmm10k c4_l1rect; do
  timeout 420 python tools/probe_solve.py $c > gpurun_out/probe_$c.log 2>&1; echo "rc $?" >> gpurun_out/probe_$c.log
done
