#!/bin/bash
# Named-config and scaling sweeps (BASELINE configs[0..2], [4]) with oracle parity on sampled points.
TAG=${1:-r2}
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_forest.json 2>gpurun_out/${TAG}_forest.err; echo "forest rc=$?"
timeout 1800 python tools/sweep.py named 5 oracle > gpurun_out/${TAG}_sweep_named.jsonl 2> gpurun_out/${TAG}_sweep_named.err; echo "named rc=$?"
timeout 2400 python tools/sweep.py scaling 3 oracle > gpurun_out/${TAG}_sweep_scaling.jsonl 2> gpurun_out/${TAG}_sweep_scaling.err; echo "scaling rc=$?"
cut -c1-300 gpurun_out/${TAG}_sweep_named.jsonl; cut -c1-200 gpurun_out/${TAG}_sweep_scaling.jsonl
