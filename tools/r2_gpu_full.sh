#!/bin/bash
# round-2 full GPU check: the whole -m gpu suite, the default bench line, the traffic range capture
mkdir -p gpurun_out
python -m pytest tests/test_gpu_comb.py -q -x > gpurun_out/r2_gpu_comb.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_comb.log
python bench.py --comb massive_12w --steps 50 --warmup 5 > gpurun_out/r2_comb12w.json 2>&1
CE_K6_POLY=0 python bench.py --comb massive_12w --steps 50 --warmup 5 > gpurun_out/r2_comb12w_old.json 2>&1
python -m pytest tests -m gpu -q > gpurun_out/r2_gpu_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_all.log
python tools/traffic_range.py --config 3 --kernel 3 --steps 50 > gpurun_out/traffic_plain.log 2>&1 && \
ncu --replay-mode range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
    --log-file gpurun_out/traffic_c3.csv python tools/traffic_range.py --config 3 --kernel 3 --steps 50 > gpurun_out/traffic_ncu.log 2>&1
tail -3 gpurun_out/r2_gpu_comb.log gpurun_out/r2_gpu_all.log
