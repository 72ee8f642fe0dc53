#!/bin/bash
# fresh per-kernel evidence: plain runs first, then one ncu --set full per hot kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in c3_gmm10k c2_img4k c4_l1rect c1_rand1k; do
timeout 300 python tools/probe_trace.py $c v14 '{"newton_tol": 1e-8}' > gpurun_out/v14_${c}.log 2>&1
done
python tools/ncu_target.py sweep > gpurun_out/ncu_plain.log 2>&1 && python tools/ncu_target.py eval >> gpurun_out/ncu_plain.log 2>&1 && PINS_CG=tree python tools/ncu_target.py cg >> gpurun_out/ncu_plain.log 2>&1 && {
ncu --set full --clock-control none --import-source on -k regex:lse_pass -s 40 -c 1 -o /tmp/prof_sweep -f python tools/ncu_target.py sweep > gpurun_out/ncu_sweep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sum_pass -s 4 -c 1 -o /tmp/prof_eval -f python tools/ncu_target.py eval > gpurun_out/ncu_eval.log 2>&1
PINS_CG=tree ncu --set full --clock-control none --import-source on -k regex:tree_pcg -s 8 -c 1 -o /tmp/prof_tree -f python tools/ncu_target.py cg > gpurun_out/ncu_tree.log 2>&1
for p in sweep eval tree; do
  ncu -i /tmp/prof_$p.ncu-rep --page details > gpurun_out/prof2_${p}_details.txt 2>&1
  ncu -i /tmp/prof_$p.ncu-rep --page raw --csv 2>&1 | gzip > gpurun_out/prof2_${p}_raw.csv.gz
  ncu -i /tmp/prof_$p.ncu-rep --page source --csv 2>&1 | gzip > gpurun_out/prof2_${p}_source.csv.gz
done
}
du -sh gpurun_out > gpurun_out/sizes.txt
