#!/bin/bash
# Same-box A/B of two builds: A = paper_1607_06886_b200/libpump_gpu.so, B = libpump_gpu_b.so
# (swapped in place for B), alternating A B A B; prints ms/step and per-family ms.
#   bash tools/ab_lib.sh [rounds]
L=paper_1607_06886_b200/libpump_gpu.so
cp $L /tmp/libA.so
for i in $(seq ${1:-2}); do
  cp /tmp/libA.so $L; bash tools/ab_bench.sh "" | sed 's/^default/A/'
  cp paper_1607_06886_b200/libpump_gpu_b.so $L; bash tools/ab_bench.sh "" | sed 's/^default/B/'
done
cp /tmp/libA.so $L
