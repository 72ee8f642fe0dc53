#!/bin/bash
# build, optional probe script(s), then the GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -30 gpurun_out/build.log; exit 1; }
for p in $PROBES; do
  timeout 600 python $p > gpurun_out/$(basename $p .py).log 2>&1; echo "rc $?" >> gpurun_out/$(basename $p .py).log
done
timeout ${PT_TIMEOUT:-1800} python -m pytest tests -m gpu -q -rf --durations=30 ${PT_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -45 gpurun_out/pytest_gpu.log
