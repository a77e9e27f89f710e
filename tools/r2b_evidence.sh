#!/bin/bash
# Round-2 evidence refresh on the box: ncu --set full captures of the forest
# kernels (per-kernel table -> profiles/r2_ncu_kernels.json, which bench.py
# reads for roofline.traffic), the -m gpu suite, the bench (both arms) and the
# ncu launch list of one warm forest solve.   usage: bash tools/r2b_evidence.sh TAG
TAG=${1:-r2b}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
rm -f gpurun_out/ncu_k_*.ncu-rep
bash tools/ncu_full.sh quad3d_forest k_regions_once k_round_tail:15 k_expand:15 k_pair_filter_grid k_bank_rec_sep \
  k_mcnoise_sep k_connect k_collide k_mc_tab k_smooth_probe k_wp_prep k_task_map:15
python tools/ncu_kernels.py gpurun_out/ncu_k_*.ncu-rep > gpurun_out/${TAG}_ncu_kernels.json
python tools/ncu_summary.py gpurun_out/ncu_k_*.ncu-rep > gpurun_out/${TAG}_ncu_full.txt
cp gpurun_out/${TAG}_ncu_kernels.json profiles/r2_ncu_kernels.json
bash tools/gpu_tests.sh "" $TAG > /dev/null; tail -3 gpurun_out/gputests_$TAG.log
python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; tail -c 300 gpurun_out/${TAG}_bench.json
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
echo "ref rc=$?"; tail -c 300 gpurun_out/${TAG}_bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python tools/one_solve.py quad3d_forest 2 > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv 2 > gpurun_out/${TAG}_launches.txt
# keep gpurun_out under the 64 MiB copy-back limit: the summaries stay, the reports go
mkdir -p gpurun_out/keep && mv gpurun_out/ncu_k_regions_once.ncu-rep gpurun_out/keep/ 2>/dev/null
rm -f gpurun_out/ncu_k_*.ncu-rep
du -sh gpurun_out
