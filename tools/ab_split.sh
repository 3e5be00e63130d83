#!/bin/bash
# After splitting the pair kernel into its own translation unit: K4 (single CTAs) must be back at the old speed;
# parity of the whole suite; pair forced parity; bench driver-like + 2000.
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_split.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_split.log; exit 1; }
{
for rep in 1 2; do
CE_K4_PAIR=0 timeout 600 python tools/time_configs.py 3 3,4,5
timeout 600 python tools/time_configs.py 3 3,4,5
done
} > gpurun_out/ab_split.log 2>&1
cat gpurun_out/ab_split.log
CE_K4_PAIR=1 timeout 900 python -m pytest tests/test_gpu_tc_paths.py tests/test_gpu_parity.py tests/test_gpu_guard.py -x -q -m gpu \
  --timeout 240 --timeout-method=thread -k "not stats and not comb" > gpurun_out/pair_split_pytest.log 2>&1
echo "pair pytest rc $?"; tail -2 gpurun_out/pair_split_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_split20.json 2>/dev/null; echo "bench20 rc $?"
python -c 'import json; d=json.loads(open("gpurun_out/bench_split20.json").read().strip().splitlines()[-1]); print("bench20 %.2f us frac %.3f" % (d["ms_per_step"]*1e3, d["roofline"]["frac"]), [(s["workload"][:7], round(s["ms_per_step"]*1e3,1), round(s["roofline"]["frac"],3)) for s in d["sweep"]])'
