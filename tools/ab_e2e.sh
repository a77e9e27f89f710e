#!/bin/bash
# Same-box A/B of libpump_gpu_a.so (A) vs libpump_gpu.so (B) with tools/e2e_dbg.py, alternating.
L=paper_1607_06886_b200/libpump_gpu.so
cp $L /tmp/B.so
for i in 1 2 3; do
  cp paper_1607_06886_b200/libpump_gpu_a.so $L; echo "A"; python tools/e2e_dbg.py 2>/dev/null | cut -c1-60
  cp /tmp/B.so $L; echo "B"; python tools/e2e_dbg.py 2>/dev/null | cut -c1-60
done
cp /tmp/B.so $L
