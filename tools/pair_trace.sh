#!/bin/bash
mkdir -p gpurun_out
tools/k4_trace.sh pt > gpurun_out/trace_build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/trace_build.log; exit 1; }
for pr in 0 1; do
  echo "=== config 3 pair=$pr"; CE_K4_PAIR=$pr timeout 120 tools/k4_trace_pt 1200 100 100 128 12 1
  echo "=== config 5 T=2 pair=$pr"; CE_K4_PAIR=$pr timeout 120 tools/k4_trace_pt 3276 126 126 256 24 2
done > gpurun_out/pair_trace.log 2>&1
wc -l gpurun_out/pair_trace.log
