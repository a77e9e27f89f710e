#!/bin/bash
# Evidence pass on the box: the -m gpu suite, the glibc-vs-portable decision
# report and the reference acceptance suite output (for profiles/), then the
# bench (both arms, driver flags) and the launch list.  usage: bash tools/r2_evidence.sh TAG
TAG=${1:-r2}
bash tools/gpu_tests.sh "" $TAG > /dev/null
tail -5 gpurun_out/gputests_$TAG.log
timeout 900 python -m pytest tests/test_normals_vs_glibc.py -q -s -m gpu -p no:cacheprovider > gpurun_out/${TAG}_glibc_vs_portable.txt 2>&1
grep -E "differing|passed|failed" gpurun_out/${TAG}_glibc_vs_portable.txt | cut -c1-300
timeout 900 tools/acceptance_ref tests/golden/scenarios > gpurun_out/${TAG}_acceptance_ref.txt 2>&1; echo "acceptance rc=$?" >> gpurun_out/${TAG}_acceptance_ref.txt
cat gpurun_out/${TAG}_acceptance_ref.txt
NO_REF=${NO_REF:-} bash tools/r2_bench.sh $TAG
