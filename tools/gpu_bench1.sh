#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/clocks_pre.csv
python bench.py --steps 2 --warmup 3 > gpurun_out/bench_r1.log 2>&1; echo "rc $?" >> gpurun_out/bench_r1.log
python tools/ncu_target.py sweep > gpurun_out/ncu_plain.log 2>&1 && python tools/ncu_target.py eval >> gpurun_out/ncu_plain.log 2>&1 && python tools/ncu_target.py cg >> gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lse_pass -s 40 -c 1 -o gpurun_out/prof_sweep -f python tools/ncu_target.py sweep > gpurun_out/ncu_sweep.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:sum_pass -s 22 -c 1 -o gpurun_out/prof_eval -f python tools/ncu_target.py eval > gpurun_out/ncu_eval.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:cg_schur -s 3 -c 1 -o gpurun_out/prof_cg -f python tools/ncu_target.py cg > gpurun_out/ncu_cg.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
