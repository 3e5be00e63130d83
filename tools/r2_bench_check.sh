#!/bin/bash
# round-2 GPU check: FFMA peak, bench tests, default bench line (+ a direct-launch line), traffic range capture
set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma_peak tools/ffma_peak.cu && /tmp/ffma_peak > gpurun_out/ffma_peak.json
python -m pytest tests/test_gpu_bench.py -q -x > gpurun_out/r2_bench_tests.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err
python bench.py --steps 2000 --warmup 50 --sweep "" --no-cpu-baseline > gpurun_out/r2_bench_2000.json 2> gpurun_out/r2_bench_2000.err
tail -3 gpurun_out/r2_bench_tests.log
