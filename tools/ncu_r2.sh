#!/bin/bash
# round-2 ncu evidence: one --set full capture per kernel family (each after its plain
# run exits 0), details + raw csv; source counters for the TC half-sweep.
mkdir -p gpurun_out
cap() {   # tag mode regex skip
  local tag=$1 mode=$2 re=$3 skip=$4
  python tools/ncu_target.py $mode > gpurun_out/ncu_${tag}_plain.log 2>&1 || { echo "$tag plain failed"; return; }
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$re" -s $skip -c 1 -o /tmp/prof_$tag -f \
      python tools/ncu_target.py $mode > gpurun_out/ncu_${tag}.log 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page details > gpurun_out/ncu_r2_${tag}_details.txt 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv 2>&1 | gzip > gpurun_out/ncu_r2_${tag}_raw.csv.gz
  if [ -n "$5" ]; then ncu -i /tmp/prof_$tag.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/ncu_r2_${tag}_src_sass.csv.gz; fi
}
cap sweep sweep 'lse_pass' 40 src
# kernel-matrix mode: three consecutive launches each (a launch of a record half-sweep exits at once)
capn() {   # tag mode regex skip count
  local tag=$1 mode=$2 re=$3 skip=$4 cnt=$5
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$re" -s $skip -c $cnt -o /tmp/prof_$tag -f \
      python tools/ncu_target.py $mode > gpurun_out/ncu_${tag}.log 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page details > gpurun_out/ncu_r2_${tag}_details.txt 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv 2>&1 | gzip > gpurun_out/ncu_r2_${tag}_raw.csv.gz
}
python tools/ncu_target.py ksweep > gpurun_out/ncu_ksweep_plain.log 2>&1
capn ksweep ksweep 'lse_ksweep' 1001 3
capn ksmerge ksweep 'lse_merge' 1001 3
capn ksfallback ksweep 'lse_fallback_k' 1001 3
cap eval eval 'sum_pass' 5
cap denserow dense 'lse_pass_kernel<\(int\)7' 6
cap densecol dense 'lse_pass_kernel<\(int\)8' 6
cap densesum dense 'sum_pass' 0
cap treecl late 'cg_tree_cluster' 150
cap treefac late 'tree_pcg' 150
cap spmv spmv 'cg_kernel' 0
ls -la gpurun_out | grep ncu_r2_
