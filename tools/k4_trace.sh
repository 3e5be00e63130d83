#!/bin/bash
# Build the traced libce + K4 trace harness: tools/k4_trace[_SUFFIX] (binaries, not tracked).
# Usage: tools/k4_trace.sh [suffix] [extra nvcc -D flags...]
cd "$(dirname "$0")/.."
SUF=${1:+_$1}; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DCE_K4_TRACE "$@" -Iinclude \
  -o tools/k4_trace$SUF tools/k4_trace.cu paper_1802_05427_b200/csrc/*.cu -lcuda
