#!/bin/bash
# round-2 full GPU pass: tests, bench (full), launch list of the bench command, ncu captures
mkdir -p gpurun_out
TAG=${TAG:-r2a}
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_$TAG.log
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=30 -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 1500 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc $?" >> gpurun_out/bench_$TAG.log
tail -c 600 gpurun_out/bench_$TAG.log
if [ -z "$NO_NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400000 --csv --log-file gpurun_out/launches_$TAG.csv \
      python bench.py --steps 1 --warmup 3 --quick --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
  python tools/summarize_launches.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1
  timeout 2400 bash tools/ncu_r2.sh
fi
