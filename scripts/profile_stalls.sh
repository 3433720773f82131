#!/bin/bash
# ncu --set full of chosen step kernels with stall reasons; exports the raw
# page and the per-SASS source page on the box (the .ncu-rep stays there).
# usage (repo root, under gpurun): bash scripts/profile_stalls.sh TAG NX NY NZ KIND:REGEX [KIND:REGEX ...]
TAG=$1; NX=$2; NY=$3; NZ=$4; shift 4
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for spec in "$@"; do
  kind=${spec%%:*}; rx=${spec#*:}
  out=gpurun_out/st_${TAG}_${kind}
  timeout 300 python scripts/profile_passes.py $NX $NY $NZ $kind > $out.plain.log 2>&1 || { echo "plain run failed" >> $out.plain.log; continue; }
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"$rx" -s 1 -c 1 -o $out -f \
     python scripts/profile_passes.py $NX $NY $NZ $kind > $out.ncu.log 2>&1
  $NCU -i $out.ncu-rep --page raw --csv > $out.raw.csv 2>&1
  $NCU -i $out.ncu-rep --page source --csv --print-source sass > $out.sass.csv 2>&1
  $NCU -i $out.ncu-rep --page details --csv > $out.details.csv 2>&1
  rm -f $out.ncu-rep
done
