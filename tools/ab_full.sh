#!/bin/bash
# Same-box A/B of libpump_gpu.so (A) against libpump_gpu_b.so (B): GPU parity
# tests on B, indoor A/B (tools/ab_lib.sh), forest A/B, round stamps of B.
#   bash tools/ab_full.sh [rounds]
L=paper_1607_06886_b200/libpump_gpu.so
B=paper_1607_06886_b200/libpump_gpu_b.so
cp $L /tmp/A0.so
cp $B $L
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
PUMP_DEBUG_COOP=1 python tools/coop_stamps.py quad3d_indoor > gpurun_out/coop_b.txt 2>&1
cp /tmp/A0.so $L
bash tools/ab_lib.sh ${1:-3} > gpurun_out/ablib.txt 2>&1
cut -c1-12 gpurun_out/ablib.txt | paste -sd' '
grep -o "round_tail.: [0-9.]*" gpurun_out/ablib.txt | paste -sd' '
for i in 1 2; do
  for v in A B; do
    if [ $v = A ]; then cp /tmp/A0.so $L; else cp $B $L; fi
    python bench.py --config quad3d_forest --no-cpu-baseline --no-mc-sweep --no-rrt --steps 5 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('forest $v', d['ms_per_step'], d['kernels']['round_tail']['ms_per_step'])"
  done
done
cp /tmp/A0.so $L
python - <<'PY'
import numpy as np
rows = [[float(x) for x in l.split()[2:13]] for l in open("gpurun_out/coop_b.txt").read().split("---- second solve")[-1].splitlines() if l.startswith("[coop]")]
a = np.array(rows); print("B stamps", a.mean(0).round(1), a.sum(1).mean().round(1))
PY
