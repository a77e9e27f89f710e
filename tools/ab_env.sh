#!/bin/bash
# Same-box A/B of env settings on one config: bash tools/ab_env.sh CONFIG "ENV1" "ENV2" ...
cfg=$1; shift
for rep in 1 2; do
for e in "$@"; do
  env $e python bench.py --config $cfg --no-cpu-baseline --no-mc-sweep --no-rrt --steps 10 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python - "$e" "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
k = {n: v["ms_per_step"] for n, v in d["kernels"].items() if v["ms_per_step"] > 0.1}
print(sys.argv[2], sys.argv[1] or "default", d["ms_per_step"], k, flush=True)
PY
done
done
