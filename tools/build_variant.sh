#!/bin/bash
# Build an A/B variant of the library: bash tools/build_variant.sh "-DFLAG ..." -> paper_1607_06886_b200/libpump_gpu_b.so
make -s -j16 -C paper_1607_06886_b200/csrc VARIANT=_b EXTRA="$1"
