#!/bin/bash
# bench + ncu evidence; large artefacts stay in /tmp on the box, summaries go to gpurun_out/
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python bench.py --steps 2 --warmup 3 > gpurun_out/bench_r1.log 2>&1; echo "rc $?" >> gpurun_out/bench_r1.log
python tools/ncu_target.py sweep > gpurun_out/ncu_plain.log 2>&1 && python tools/ncu_target.py eval >> gpurun_out/ncu_plain.log 2>&1 && python tools/ncu_target.py cg >> gpurun_out/ncu_plain.log 2>&1 && {
ncu --set full --clock-control none --import-source on -k regex:lse_pass -s 40 -c 1 -o /tmp/prof_sweep -f python tools/ncu_target.py sweep > gpurun_out/ncu_sweep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sum_pass -s 22 -c 1 -o /tmp/prof_eval -f python tools/ncu_target.py eval > gpurun_out/ncu_eval.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cg_schur -s 3 -c 1 -o /tmp/prof_cg -f python tools/ncu_target.py cg > gpurun_out/ncu_cg.log 2>&1
for p in sweep eval cg; do
  ncu -i /tmp/prof_$p.ncu-rep --page raw --csv > gpurun_out/prof_${p}_raw.csv 2>&1
  ncu -i /tmp/prof_$p.ncu-rep --page details > gpurun_out/prof_${p}_details.txt 2>&1
  ncu -i /tmp/prof_$p.ncu-rep --page source --csv 2>&1 | gzip > gpurun_out/prof_${p}_source.csv.gz
done
ls -la /tmp/prof_*.ncu-rep > gpurun_out/prof_sizes.txt
}
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 25000 --csv --log-file /tmp/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
python tools/summarize_launches.py /tmp/launches.csv gpurun_out/launches_summary.json > /dev/null 2>&1
gzip -c /tmp/launches.csv > gpurun_out/launches.csv.gz
du -sh gpurun_out >> gpurun_out/prof_sizes.txt
