#!/bin/bash
# GPU test pass on the box: the -m gpu suite (all failures listed), durations.
# usage: bash tools/gpu_tests.sh [pytest -k expr] [tag]
K=${1:-}
TAG=${2:-run}
if [ -n "$K" ]; then
  timeout 3000 python -m pytest tests -q -m gpu -k "$K" --durations=15 -p no:cacheprovider > gpurun_out/gputests_$TAG.log 2>&1
else
  timeout 3000 python -m pytest tests -q -m gpu --durations=25 -p no:cacheprovider > gpurun_out/gputests_$TAG.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/gputests_$TAG.log
tail -60 gpurun_out/gputests_$TAG.log
