#!/bin/bash
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pair.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_pair.log; exit 1; }
for rep in 1 2; do
CE_K4_PAIR=0 timeout 600 python tools/time_configs.py 3 3,4,5
CE_K4_PAIR=1 timeout 600 python tools/time_configs.py 3 3,4,5
done 2>&1 | tee gpurun_out/pair_quick.log
CE_K4_PAIR=1 timeout 900 python -m pytest tests/test_gpu_tc_paths.py tests/test_gpu_parity.py tests/test_gpu_guard.py -x -q -m gpu \
  --timeout 240 --timeout-method=thread -k "not stats and not comb" > gpurun_out/pair_quick_pytest.log 2>&1
echo "pair pytest rc $?"; tail -2 gpurun_out/pair_quick_pytest.log
