#!/bin/bash
# Same-box A/B of per-phase times: A = libpump_gpu_a.so, B = libpump_gpu.so, alternating.
L=paper_1607_06886_b200/libpump_gpu.so
cp $L /tmp/B.so
for i in 1 2 3; do
  cp paper_1607_06886_b200/libpump_gpu_a.so $L; echo -n "A "; python tools/phase_ab.py ${1:-quad3d_forest} 2>/dev/null
  cp /tmp/B.so $L; echo -n "B "; python tools/phase_ab.py ${1:-quad3d_forest} 2>/dev/null
done
cp /tmp/B.so $L
