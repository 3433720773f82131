#!/bin/bash
# Round-end evidence on one B200 (usage, from the repo root under gpurun:
#   bash scripts/profile_round.sh TAG):
#   bench line and reference arm, ncu launch list of the bench command,
#   ncu --set full of the four step kernels at 512^3, long parity runs.
TAG=${1:-r02}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
BENCH="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_bench.log
timeout 400 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/${TAG}_ref.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_ref.log
# launch list in plane order (CTAP_PBLOCK=0): the slab schedule runs the same kernels on 4-plane
# slabs, hundreds per step, which ncu serialises cold-cache; per-pass shares read from plane order
export CTAP_PBLOCK=0
timeout 600 $BENCH > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $BENCH > gpurun_out/${TAG}_ncu1.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_ncu1.log
unset CTAP_PBLOCK
timeout 300 python scripts/profile_passes.py 512 512 512 Z_MID,Y_FWD,X_KIN,Y_INV > gpurun_out/${TAG}_pp.log 2>&1 && \
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:'ring_kernel|zline_kernel|tile_kernel' -c 8 -o gpurun_out/${TAG}_full -f python scripts/profile_passes.py 512 512 512 Z_MID,Y_FWD,X_KIN,Y_INV > gpurun_out/${TAG}_ncu2.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_ncu2.log
python scripts/ncu_summary.py full gpurun_out/${TAG}_full.ncu-rep 134217728 > gpurun_out/${TAG}_full_summary.txt 2>&1
$NCU -i gpurun_out/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_raw.csv 2>&1
rm -f gpurun_out/${TAG}_full.ncu-rep
if [ "${PARITY:-1}" = 1 ]; then
  timeout 2400 python scripts/parity_run.py cfg1 cfg2b cfg3 cfg4 cfg3c64 cfg2 --out gpurun_out/${TAG}_parity.json > gpurun_out/${TAG}_parity.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_parity.log
fi
