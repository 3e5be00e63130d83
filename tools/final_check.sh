#!/bin/bash
# HEAD check: build, whole GPU suite, pairs-forced K4 tests, smoke, same-box timing with and without pairs
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_final.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_final.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest gpu rc $?"; tail -2 gpurun_out/pytest_gpu_final.log
CE_K4_PAIR=1 timeout 900 python -m pytest tests/test_gpu_tc_paths.py tests/test_gpu_parity.py tests/test_gpu_guard.py -q -m gpu \
  -k "not stats and not comb" > gpurun_out/pytest_gpu_pair_final.log 2>&1; echo "pair pytest rc $?"; tail -2 gpurun_out/pytest_gpu_pair_final.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_final.log 2>&1; echo "smoke rc $?"
for rep in 1 2; do
CE_K4_PAIR=0 timeout 600 python tools/time_configs.py 3 3,4,5
timeout 600 python tools/time_configs.py 3 3,4,5
done 2>&1 | tee gpurun_out/final_time.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final20.json 2>/dev/null; echo "bench20 rc $?"
python -c 'import json; d=json.loads(open("gpurun_out/bench_final20.json").read().strip().splitlines()[-1]); print("bench20 %.2f us frac %.3f" % (d["ms_per_step"]*1e3, d["roofline"]["frac"]), [(s["workload"][:7], round(s["ms_per_step"]*1e3,1), round(s["roofline"]["frac"],3)) for s in d["sweep"]])'
