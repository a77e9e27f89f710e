#!/bin/bash
# One ncu --set full capture per named kernel (first launch of the warm solve's
# kind in tools/prof_solve.py), raw pages summarised into gpurun_out/ncu_<k>.txt.
#   bash tools/ncu_full.sh quad3d_indoor k_regions_once k_round_tail ...
sc=$1; shift
for k in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -c 1 \
    -o gpurun_out/ncu_${k} -f python tools/prof_solve.py $sc 1 > gpurun_out/ncu_${k}.log 2>&1
  python tools/ncu_summary.py gpurun_out/ncu_${k}.ncu-rep > gpurun_out/ncu_${k}.txt 2>&1
done
