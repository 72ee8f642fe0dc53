#!/bin/bash
# full GPU pass: build, tests, bench (full), ncu sweep capture with source counters
mkdir -p gpurun_out
TAG=${TAG:-r2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -30 gpurun_out/build.log; exit 1; }
if [ -z "$NO_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=30 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc $?" >> gpurun_out/bench_$TAG.log
tail -c 400 gpurun_out/bench_$TAG.log
if [ -n "$NCU" ]; then bash tools/ncu_sweep_src.sh; fi
