#!/bin/bash
# bench line + launch list of the same command + smoke
T=${1:-b}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python bench.py > gpurun_out/bench_$T.log 2>&1; echo "rc $?" >> gpurun_out/bench_$T.log
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file /tmp/launches.csv python bench.py > gpurun_out/ncu_bench_$T.log 2>&1
python tools/summarize_launches.py /tmp/launches.csv gpurun_out/launches_$T.json > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "rc $?" >> gpurun_out/smoke_$T.log
