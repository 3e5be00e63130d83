#!/bin/bash
mkdir -p gpurun_out
python bench.py --comb massive_12w --steps 5 --warmup 3 > gpurun_out/p_comb.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k6_estimate -s 3 -c 1 -o gpurun_out/prof_k6c \
    python bench.py --comb massive_12w --steps 5 --warmup 3 > gpurun_out/p_comb_ncu.log 2>&1
python tools/traffic_range.py --config 5 --kernel 3 --steps 6 > gpurun_out/traffic_plain5.log 2>&1 && \
ncu --replay-mode range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
    --log-file gpurun_out/traffic_c5.csv python tools/traffic_range.py --config 5 --kernel 3 --steps 6 > gpurun_out/traffic_ncu5.log 2>&1
ls -la gpurun_out/prof_k6c* gpurun_out/traffic_c5.csv
