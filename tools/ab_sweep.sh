#!/bin/bash
# A/B over env settings on a sweep workload set: prints ms per solve per workload.
#   bash tools/ab_sweep.sh scaling "" "PUMP_X=1"
kind=$1; shift
for e in "$@"; do
  env $e python tools/sweep.py $kind 3 > gpurun_out/abs.jsonl 2>gpurun_out/abs.err
  python - "$e" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("gpurun_out/abs.jsonl")]
print(sys.argv[1] or "default", " ".join(f"{r['workload']}={r.get('ms_per_solve')}" for r in rows))
PY
done
