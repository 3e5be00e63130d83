#!/bin/bash
# K4 pair mode (cta_group::2, CE_K4_PAIR=1): parity of every K4 test under it, then a same-box timing A/B.
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pair.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_pair.log; exit 1; }
CE_K4_PAIR=1 timeout 1200 python -m pytest tests/test_gpu_tc_paths.py tests/test_gpu_parity.py tests/test_gpu_guard.py -x -q -m gpu \
  --timeout 240 --timeout-method=thread -k "not stats and not comb" > gpurun_out/pair_pytest.log 2>&1
echo "pair pytest rc $?"; tail -8 gpurun_out/pair_pytest.log
for pr in 0 1 0 1; do CE_K4_PAIR=$pr timeout 600 python tools/time_configs.py 3 ${PAIR_CFGS:-3,4,5,6}; done > gpurun_out/pair_time.log 2>&1
cat gpurun_out/pair_time.log
if [ -n "$PAIR_FULL" ]; then
timeout 1800 python -m pytest tests -q -m gpu --timeout 400 --timeout-method=thread > gpurun_out/pytest_gpu_pair_base.log 2>&1; echo "full pytest rc $?"; tail -4 gpurun_out/pytest_gpu_pair_base.log
fi
