#!/bin/bash
# Same-box A/B of two builds on the named configs: A = libpump_gpu.so, B = libpump_gpu_b.so
#   bash tools/ab_lib_cfg.sh ROUNDS CONFIG...
R=${1:-2}; shift
L=paper_1607_06886_b200/libpump_gpu.so
cp $L /tmp/libA.so
for i in $(seq $R); do
  for cfg in "$@"; do
    cp /tmp/libA.so $L; bash tools/ab_env.sh $cfg "" 2>&1 | head -1 | sed 's/ default / A /'
    cp paper_1607_06886_b200/libpump_gpu_b.so $L; bash tools/ab_env.sh $cfg "" 2>&1 | head -1 | sed 's/ default / B /'
  done
done
cp /tmp/libA.so $L
