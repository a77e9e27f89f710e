#!/bin/bash
# Same-box comparison of several library builds with tools/e2e_dbg.py, round-robin:
#   bash tools/ab_multi.sh a b c   (paper_1607_06886_b200/libpump_gpu_{a,b,c}.so; "cur" = the in-tree build)
L=paper_1607_06886_b200/libpump_gpu.so
cp $L /tmp/cur.so
for i in 1 2 3; do
  for v in "$@"; do
    if [ "$v" = cur ]; then cp /tmp/cur.so $L; else cp paper_1607_06886_b200/libpump_gpu_$v.so $L; fi
    echo "$v"; python tools/e2e_dbg.py 2>/dev/null | cut -c1-60
  done
done
cp /tmp/cur.so $L
