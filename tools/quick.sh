#!/bin/bash
# Quick loop on the box: a pytest -k selection, then the forest (and optionally indoor) bench, ours only.
#   bash tools/quick.sh TAG "pytest -k expr" [indoor]
TAG=$1; K=$2
if [ -n "$K" ]; then bash tools/gpu_tests.sh "$K" $TAG | tail -3; fi
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-mc-sweep --no-rrt > gpurun_out/${TAG}_forest.json 2>gpurun_out/${TAG}_forest.err; echo forest rc=$?
[ -n "$3" ] && { python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-mc-sweep --no-rrt --config quad3d_indoor > gpurun_out/${TAG}_indoor.json 2>gpurun_out/${TAG}_indoor.err; echo indoor rc=$?; }
python - <<PY
import json, os
for c in ("forest", "indoor"):
    p = "gpurun_out/${TAG}_%s.json" % c
    if not os.path.exists(p): continue
    d = json.loads(open(p).read().strip().splitlines()[-1])
    print(c, d["value"], d["e2e"]["value"], {k: v["ms_per_step"] for k, v in d["kernels"].items() if v["ms_per_step"] > 0.05}, d["solve"])
PY
