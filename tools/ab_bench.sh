#!/bin/bash
# A/B: bench.py (solve only) under each env setting given; prints ms/step and per-family ms.
for e in "$@"; do
  env $e python bench.py --no-cpu-baseline --no-mc-sweep --no-rrt --steps 10 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python - "$e" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
k = {n: v["ms_per_step"] for n, v in d["kernels"].items()}
print(sys.argv[1] or "default", d["ms_per_step"], k)
PY
done
