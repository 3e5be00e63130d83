#!/bin/bash
# K4 pair mode: separate, deeper filter-chunk ring (K4_S_B_P) -- parity with pairs forced, then same-box timing matrix
mkdir -p gpurun_out
: > gpurun_out/pair_bring.log
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pair.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_pair.log; exit 1; }
CE_K4_PAIR=1 timeout 900 python -m pytest tests/test_gpu_tc_paths.py tests/test_gpu_parity.py tests/test_gpu_guard.py -x -q -m gpu \
  --timeout 240 --timeout-method=thread -k "not stats and not comb" > gpurun_out/pair_bring_pytest.log 2>&1
echo "pair pytest rc $?"; tail -3 gpurun_out/pair_bring_pytest.log
IFS='|' read -ra FL <<< "${PAIR_FLAGS:-|-DK4_S_AB_P=3 -DK4_S_B_P=3|-DK4_S_AB_P=4 -DK4_S_B_P=4|-DK4_S_AB_P=3 -DK4_S_B_P=6|-DK4_S_AB_P=2 -DK4_S_B_P=5|-DK4_S_AB_P=4 -DK4_S_B_P=5}"
for rep in 1 2; do
for fl in "${FL[@]}"; do
  CE_NVCC_EXTRA="$fl" python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pair.log 2>&1 || { echo "BUILD FAILED $fl" >> gpurun_out/pair_bring.log; continue; }
  echo "== flags: $fl" >> gpurun_out/pair_bring.log
  CE_K4_PAIR=1 timeout 600 python tools/time_configs.py 3 4,5 >> gpurun_out/pair_bring.log 2>&1
done
CE_K4_PAIR=0 timeout 600 python tools/time_configs.py 3 4,5 >> gpurun_out/pair_bring.log 2>&1
done
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pair.log 2>&1
cat gpurun_out/pair_bring.log
