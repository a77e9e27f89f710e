#!/bin/bash
# Perf check on the box: explore/solve parity tests, the bench (ours only) on
# forest and indoor, and ncu --set full captures of the top forest kernels.
TAG=${1:-r2p}; shift
bash tools/gpu_tests.sh "explore or run_pump or fullsize or golden or dropin" $TAG > /dev/null; tail -3 gpurun_out/gputests_$TAG.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_forest.json 2>gpurun_out/${TAG}_forest.err; echo "forest rc=$?"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config quad3d_indoor > gpurun_out/${TAG}_indoor.json 2>gpurun_out/${TAG}_indoor.err; echo "indoor rc=$?"
[ $# -gt 0 ] && bash tools/ncu_full.sh quad3d_forest "$@"
python - <<PY
import json
for c in ("forest", "indoor"):
    d = json.loads(open("gpurun_out/${TAG}_%s.json" % c).read().strip().splitlines()[-1])
    print(c, d["value"], d["e2e"]["value"], {k: v["ms_per_step"] for k, v in d["kernels"].items() if v["ms_per_step"] > 0.1}, d["solve"])
PY
