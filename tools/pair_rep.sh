#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/pair_rep.log
for rep in 1 2; do
for fl in "" "-DK4_S_AB_P=4"; do
  CE_NVCC_EXTRA="$fl" python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pair.log 2>&1 || { echo "BUILD FAILED $fl" >> gpurun_out/pair_rep.log; continue; }
  echo "== flags: $fl" >> gpurun_out/pair_rep.log
  for pr in 0 1; do CE_K4_PAIR=$pr timeout 600 python tools/time_configs.py 3 4,5 >> gpurun_out/pair_rep.log 2>&1; done
done
done
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pair.log 2>&1
cat gpurun_out/pair_rep.log
timeout 1800 python -m pytest tests -q -m gpu --timeout 400 --timeout-method=thread > gpurun_out/pytest_gpu_pairpolicy.log 2>&1; echo "full pytest rc $?"; tail -4 gpurun_out/pytest_gpu_pairpolicy.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_pairpolicy.json 2> gpurun_out/bench_pairpolicy.err; echo "bench rc $?"
