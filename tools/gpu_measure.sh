#!/bin/bash
# One measurement pass on the GPU box (run from the repo root under gpurun): GPU tests, the C4 bench line,
# the ncu launch list + per-pass DRAM bytes, the issue counters (stamped with libpa's source hash) and
# ncu --set full captures of the two dominant kernels.  Everything lands in gpurun_out/<tag>_*.
#   usage: bash tools/gpu_measure.sh <tag> [tests|notests]
set -u
TAG=${1:-r2}
MODE=${2:-tests}
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${TAG}_build.txt 2>&1 || { echo "build failed"; tail $O/${TAG}_build.txt; exit 1; }
if [ "$MODE" = tests ]; then
  PARITY_OUT=$O/${TAG}_parity.json timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${TAG}_gpu_tests.txt 2>&1
  echo "pytest rc=$?"; tail -3 $O/${TAG}_gpu_tests.txt
fi
timeout 900 python tools/issue_capture.py run $TAG > $O/${TAG}_issue.log 2>&1 && \
  timeout 300 python tools/issue_capture.py parse $O/${TAG}_issue_c4.csv $TAG >> $O/${TAG}_issue.log 2>&1
echo "issue rc=$?"; tail -2 $O/${TAG}_issue.log
cp profiles/${TAG}_issue_c4.json $O/ 2>/dev/null
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $O/${TAG}_launch_bench.json 2>&1
echo "launches rc=$?"
STEP_MS=$(python -c "import json,sys; print(json.loads(open('$O/${TAG}_launch_bench.json').read().strip().splitlines()[-1])['ms_per_step'])" 2>/dev/null || echo 0)
python tools/launch_profile.py $O/${TAG}_launches_c4.csv $TAG $STEP_MS > $O/${TAG}_launch_profile.log 2>&1; echo "launch profile rc=$?"
cp profiles/${TAG}_traffic_c4.json profiles/${TAG}_launches_c4.md $O/ 2>/dev/null
timeout 900 python bench.py --steps 3 --warmup 3 > $O/${TAG}_bench_c4.json 2> $O/${TAG}_bench_c4.err
echo "bench rc=$?"; tail -c 300 $O/${TAG}_bench_c4.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_adjoint_tay2 -s 1 -c 1 \
  -o $O/${TAG}_k2c python tools/profile_step.py c4 16 1 > $O/${TAG}_ncu_k2c.log 2>&1
echo "ncu k2c rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fwd_dep -s 1 -c 1 \
  -o $O/${TAG}_k1d python tools/profile_step.py c4 16 1 > $O/${TAG}_ncu_k1d.log 2>&1
echo "ncu k1d rc=$?"
