#!/bin/bash
# Round-2 evidence in one GPU call: build, GPU tests, smoke, bench lines (driver-like and long), reference arm,
# 2-rank run, NEXT-row lines, ncu launch list + --set full captures of k4_bf16x3 (configs 3 and 5).
TAG=${1:-r02}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_${TAG}.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_${TAG}.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest gpu exit $?"; tail -2 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?"
# K4 pair mode (cta_group::2) forced on every K4 shape with >= 2 column tiles: the same parity / guard-band tests
CE_K4_PAIR=1 timeout 900 python -m pytest tests/test_gpu_tc_paths.py tests/test_gpu_parity.py tests/test_gpu_guard.py -q -m gpu \
  -k "not stats and not comb" > gpurun_out/pytest_gpu_pair_${TAG}.log 2>&1; echo "pytest gpu (pair forced) exit $?"; tail -2 gpurun_out/pytest_gpu_pair_${TAG}.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_driverlike.json 2> gpurun_out/bench_${TAG}_driverlike.err; echo "bench20 exit $?"
timeout 900 python bench.py --steps 2000 --warmup 50 --sweep-steps 40 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench2000 exit $?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref exit $?"
timeout 600 python bench.py --gpus 2 --backend gloo --steps 20 --warmup 5 --sweep "" --no-cpu-baseline > gpurun_out/bench_2rank_${TAG}.json 2> gpurun_out/bench_2rank_${TAG}.err; echo "2rank exit $?"
for k in 1 2; do timeout 300 python bench.py --kernel $k --steps 200 --warmup 10 --sweep "" --no-cpu-baseline > gpurun_out/bench_k${k}_${TAG}.json 2>/dev/null; done
timeout 300 python bench.py --config 6 --steps 100 --warmup 10 --sweep "" --no-cpu-baseline > gpurun_out/bench_c6_${TAG}.json 2>/dev/null
for c in massive_12w paper_12w paper_3w; do timeout 300 python bench.py --comb $c --steps 50 --warmup 5 > gpurun_out/comb_${c}_${TAG}.json 2>/dev/null; done
for c in 3 4 5; do timeout 300 python bench.py --stats --config $c --steps 20 --warmup 3 > gpurun_out/stats_c${c}_${TAG}.json 2>/dev/null; done
CMD="python bench.py --launch direct --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 3 --sweep ''"
eval $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
  eval ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list rc $?"
eval ncu --set full --clock-control none --import-source on -k regex:k4_bf16x3 -s 10 -c 1 -f -o gpurun_out/prof_c3_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full c3 rc $?"
CMD5="python bench.py --config 5 --launch direct --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 3 --sweep ''"
eval $CMD5 > gpurun_out/plain5_${TAG}.log 2>&1 && \
  eval ncu --set full --clock-control none --import-source on -k regex:k4_bf16x3 -s 3 -c 1 -f -o gpurun_out/prof_c5_${TAG} $CMD5 > gpurun_out/ncu_full5_${TAG}.log 2>&1
echo "full c5 rc $?"
# K10 (comb 12W on tcgen05): launch list and ncu --set full of the main kernel
CMDC="python bench.py --comb massive_12w --steps 10 --warmup 3 --e2e-steps 3"
eval $CMDC > gpurun_out/plainc_${TAG}.log 2>&1 && \
  eval ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -c 40 --csv --log-file gpurun_out/launches_comb_${TAG}.csv $CMDC > /dev/null 2>&1
echo "comb launch list rc $?"
eval ncu --set full --clock-control none --import-source on -k regex:k10_comb_tc -s 3 -c 1 -f -o gpurun_out/prof_k10_${TAG} $CMDC > gpurun_out/ncu_k10_${TAG}.log 2>&1
echo "full k10 rc $?"
for c in 4 5; do
CMDS="python bench.py --stats --config $c --steps 3 --warmup 3"
eval ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --cache-control none -c 30 --csv --log-file gpurun_out/launches_stats_c${c}_${TAG}.csv $CMDS > /dev/null 2>&1
echo "stats c$c launch list rc $?"
done
# the NCCL plumbing through the driver's launcher (one rank: torch.distributed.run, backend nccl)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 20 --warmup 5 --sweep "" --no-cpu-baseline > gpurun_out/bench_nccl1_${TAG}.json 2> gpurun_out/bench_nccl1_${TAG}.err
echo "nccl torchrun rc $?"
