#!/bin/bash
# One ncu --set full capture per named kernel of a quad3d solve (tools/prof_solve.py,
# one solve), raw pages summarised into gpurun_out/ncu_<k>.txt.  "name:skip" skips
# the first `skip` matching launches (e.g. k_expand:6 for a mid-explore round).
#   bash tools/ncu_full.sh quad3d_indoor k_regions_once k_round_tail:6 ...
sc=$1; shift
for spec in "$@"; do
  k=${spec%%:*}; skip=0
  [[ "$spec" == *:* ]] && skip=${spec##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${k}" --launch-skip $skip -c 1 \
    -o gpurun_out/ncu_${k} -f python tools/prof_solve.py $sc 1 > gpurun_out/ncu_${k}.log 2>&1
  python tools/ncu_summary.py gpurun_out/ncu_${k}.ncu-rep > gpurun_out/ncu_${k}.txt 2>&1
done
