#!/bin/bash
# One GPU call: build, GPU tests, smoke, default bench line + reference arm, K4 sweep, ncu launch list and
# --set full captures of k4_bf16x3 on configs 3 and 5.   Usage: tools/evidence_round.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_${TAG}.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_${TAG}.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest gpu exit $?"; tail -2 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench exit $?"; cat gpurun_out/bench_${TAG}.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref exit $?"
bash tools/sweep.sh "0" "4 5 6" 200
bash tools/sweep.sh "1 2" "3" 300
bash tools/profile_round.sh ${TAG}
# statistics path (NEXT-3): bench lines for configs 3-5 and the config-4 launch list (K8 / K7c / K7b shares)
for c in 3 4 5; do timeout 300 python bench.py --stats --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/stats_c${c}_${TAG}.json 2> gpurun_out/stats_c${c}_${TAG}.err; echo "stats c$c exit $?"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_stats_c4_${TAG}.csv python bench.py --stats --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_stats_${TAG}.log 2>&1; echo "stats launch list rc $?"
# NEXT-row kernels: one --set full capture each (K8, K7c, K7a, K6 12W) + summary
bash tools/profile_next.sh ${TAG}
