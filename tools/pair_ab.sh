#!/bin/bash
# K4 pair mode: parity under CE_K4_PAIR=1 (subset), timing A/B, trace
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pair.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_pair.log; exit 1; }
CE_K4_PAIR=1 timeout 900 python -m pytest tests/test_gpu_tc_paths.py tests/test_gpu_parity.py tests/test_gpu_guard.py -x -q -m gpu \
  --timeout 240 --timeout-method=thread -k "not stats and not comb" > gpurun_out/pair_pytest.log 2>&1
echo "pair pytest rc $?"; tail -3 gpurun_out/pair_pytest.log
for pr in 0 1 0 1; do CE_K4_PAIR=$pr timeout 600 python tools/time_configs.py 3 ${PAIR_CFGS:-3,4,5,6}; done > gpurun_out/pair_time.log 2>&1
cat gpurun_out/pair_time.log
tools/k4_trace.sh pt > gpurun_out/trace_build.log 2>&1 || { echo TRACE BUILD FAILED; exit 0; }
for pr in 0 1; do
  echo "=== config 3 pair=$pr"; CE_K4_PAIR=$pr timeout 120 tools/k4_trace_pt 1200 100 100 128 12 1
  echo "=== config 5 T=2 pair=$pr"; CE_K4_PAIR=$pr timeout 120 tools/k4_trace_pt 3276 126 126 256 24 2
done > gpurun_out/pair_trace.log 2>&1
