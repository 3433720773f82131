#!/bin/bash
# Round-end evidence on one B200: reference arm line, ncu launch list of bench.py, ncu --set full of the four step kernels.
# usage (from the repo root, under gpurun): bash scripts/profile_round.sh
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 400 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/p_ref.log 2>&1; echo rc=$? >> gpurun_out/p_ref.log
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p_launches.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p_ncu1.log 2>&1; echo rc=$? >> gpurun_out/p_ncu1.log
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:'ring_kernel|zline_kernel|tile_kernel' -c 8 -o gpurun_out/p_full -f python scripts/profile_passes.py 512 512 512 Z_MID,Y_FWD,X_KIN,Y_INV > gpurun_out/p_ncu2.log 2>&1; echo rc=$? >> gpurun_out/p_ncu2.log
# the report itself (~100 MB with sources) stays on the box; keep text summaries
python scripts/ncu_summary.py full gpurun_out/p_full.ncu-rep 134217728 > gpurun_out/p_full_summary.txt 2>&1
$NCU -i gpurun_out/p_full.ncu-rep --page details --csv --section WarpStateStats --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis > gpurun_out/p_full_details.csv 2>&1
rm -f gpurun_out/p_full.ncu-rep
