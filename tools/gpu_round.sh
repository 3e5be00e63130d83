#!/bin/bash
# One GPU call: build, gpu tests, smoke, bench (default line + sweep), launch list, ncu --set full of K4.
# Usage (from the repo root on the box): tools/gpu_round.sh [tag]
TAG=${1:-r01}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_${TAG}.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_${TAG}.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest gpu exit $?"; tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench exit $?"; cat gpurun_out/bench_${TAG}.json
bash tools/sweep.sh "0 1 2" "2 3 4 5" 200
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "ncu launches exit $?"
$CMD > gpurun_out/plain2_${TAG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k4_bf16x3 -s 5 -c 1 -o gpurun_out/prof_k4_c3_${TAG} -f $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full c3 exit $?"
CMD5="python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3"
$CMD5 > gpurun_out/plain5_${TAG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k4_bf16x3 -s 4 -c 1 -o gpurun_out/prof_k4_c5_${TAG} -f $CMD5 > gpurun_out/ncu_full5_${TAG}.log 2>&1
echo "ncu full c5 exit $?"
