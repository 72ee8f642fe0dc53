#!/bin/bash
# round evidence: bench, ncu launch list of the same command, ncu --set full per hot kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python bench.py > gpurun_out/bench_r1d.log 2>&1; echo "rc $?" >> gpurun_out/bench_r1d.log
python tools/ncu_target.py sweep > gpurun_out/ncu_plain.log 2>&1 && python tools/ncu_target.py eval >> gpurun_out/ncu_plain.log 2>&1 && python tools/ncu_target.py late >> gpurun_out/ncu_plain.log 2>&1 && {
ncu --set full --clock-control none --import-source on -k regex:lse_pass -s 40 -c 1 -o /tmp/prof_sweep -f python tools/ncu_target.py sweep > gpurun_out/ncu_sweep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sum_pass -s 4 -c 1 -o /tmp/prof_eval -f python tools/ncu_target.py eval > gpurun_out/ncu_eval.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tree_pcg -s 150 -c 1 -o /tmp/prof_tree -f python tools/ncu_target.py late > gpurun_out/ncu_tree.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sum_pass -s 400 -c 1 -o /tmp/prof_evallate -f python tools/ncu_target.py late > gpurun_out/ncu_evallate.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cg_tree_cluster -s 150 -c 1 -o /tmp/prof_treecl -f python tools/ncu_target.py late > gpurun_out/ncu_treecl.log 2>&1
for p in sweep eval tree evallate treecl; do
  ncu -i /tmp/prof_$p.ncu-rep --page details > gpurun_out/prof5_${p}_details.txt 2>&1
  ncu -i /tmp/prof_$p.ncu-rep --page raw --csv 2>&1 | gzip > gpurun_out/prof5_${p}_raw.csv.gz
  ncu -i /tmp/prof_$p.ncu-rep --page source --csv 2>&1 | gzip > gpurun_out/prof5_${p}_source.csv.gz
done
}
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file /tmp/launches.csv python bench.py > gpurun_out/ncu_bench.log 2>&1
python tools/summarize_launches.py /tmp/launches.csv gpurun_out/launches_r1d.json > /dev/null 2>&1
gzip -c /tmp/launches.csv > gpurun_out/launches_r1d.csv.gz
du -sh gpurun_out > gpurun_out/sizes.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc $?" >> gpurun_out/smoke.log
