set -x
for c in 1 2 4; do
  CE_K4_CLUSTER=$c timeout 60 tools/k4_trace_v5 1200 100 100 128 12 1 > gpurun_out/trace_c3_v5_C$c.txt 2>&1; echo "rc $?"
  CE_K4_CLUSTER=$c timeout 60 tools/k4_trace_v5 3276 126 126 256 24 2 > gpurun_out/trace_c5_v5_C$c.txt 2>&1; echo "rc $?"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "not kernels_agree" 2>&1 | tail -3
