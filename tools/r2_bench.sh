#!/bin/bash
# Round-2 measurement pass on the box: bench (both arms, driver flags), the
# ncu launch list of one warm forest solve, and ncu --set full captures of the
# top kernels.  usage: bash tools/r2_bench.sh TAG [ncu-kernel-specs...]
TAG=${1:-r2}; shift
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; tail -c 400 gpurun_out/${TAG}_bench.json
if [ -z "$NO_REF" ]; then
  python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
  echo "ref rc=$?"; tail -c 300 gpurun_out/${TAG}_bench_ref.json
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python tools/one_solve.py quad3d_forest 2 > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
[ $# -gt 0 ] && bash tools/ncu_full.sh quad3d_forest "$@"
ls gpurun_out | head -50
