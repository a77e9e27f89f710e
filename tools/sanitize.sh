#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over small
# full solves (graph, bank, cooperative explore rounds, MC, smoothing).
# Summaries -> gpurun_out/sanitizer_<tool>_<case>.txt
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool case path samples mc
  timeout 1500 $CS --tool $1 --print-limit 20 --error-exitcode 9 python tools/sanitize_solve.py $3 $4 $5 \
    > gpurun_out/sanitizer_$1_$2.txt 2>&1
  echo "$1 $2 rc=$?" | tee -a gpurun_out/sanitizer_summary.txt
  tail -3 gpurun_out/sanitizer_$1_$2.txt | tee -a gpurun_out/sanitizer_summary.txt
}
: > gpurun_out/sanitizer_summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  run $tool minimal tests/golden/scenarios/minimal.json 0 2000
  run $tool three_obstacle tests/golden/scenarios/three_obstacle.json 200 2000
  run $tool quad3d_forest scenarios/quad3d_forest.json 400 2000
done
