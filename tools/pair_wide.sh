#!/bin/bash
# K4 pair mode: wide raw stages (CE_K4_WIDE=1) and A/B ring depth (CE_K4_SAB) -- parity, then same-box timing
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pair.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_pair.log; exit 1; }
CE_K4_PAIR=1 CE_K4_WIDE=1 timeout 900 python -m pytest tests/test_gpu_tc_paths.py tests/test_gpu_parity.py tests/test_gpu_guard.py -x -q -m gpu \
  --timeout 240 --timeout-method=thread -k "not stats and not comb" > gpurun_out/pair_wide_pytest.log 2>&1
echo "pair wide pytest rc $?"; tail -3 gpurun_out/pair_wide_pytest.log
{
for rep in 1 2; do
CE_K4_PAIR=0 timeout 600 python tools/time_configs.py 3 4,5
for sab in 3 4; do for w in 0 1; do
CE_K4_PAIR=1 CE_K4_SAB=$sab CE_K4_WIDE=$w timeout 600 python tools/time_configs.py 3 4,5
done; done
done
} > gpurun_out/pair_wide.log 2>&1
cat gpurun_out/pair_wide.log
