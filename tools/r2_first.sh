set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --config quad3d_forest --steps 10 --warmup 3 --no-cpu-baseline --no-rrt > gpurun_out/r2_forest_bench0.json 2> gpurun_out/r2_forest_bench0.err
tail -c 600 gpurun_out/r2_forest_bench0.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_forest_launches0.csv python tools/one_solve.py quad3d_forest 2 > gpurun_out/r2_ncu_launch.log 2>&1
bash tools/ncu_full.sh quad3d_forest k_regions k_round_tail:6 k_expand:6
ls gpurun_out
