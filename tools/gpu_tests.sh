#!/bin/bash
# GPU test pass: build, then pytest -m gpu (all failures, durations)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -30 gpurun_out/build.log; exit 1; }
timeout ${PT_TIMEOUT:-1500} python -m pytest tests -m gpu -q -rf --durations=25 ${PT_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -40 gpurun_out/pytest_gpu.log
