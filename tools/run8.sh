for k in 3 4; do
  timeout 60 tools/k4_trace_v8 1200 100 100 128 12 1 $k > gpurun_out/trace_c3_v8_k$k.txt 2>&1; echo "c3 k$k rc $?"
  timeout 60 tools/k4_trace_v8 3276 126 126 256 24 2 $k > gpurun_out/trace_c5_v8_k$k.txt 2>&1; echo "c5 k$k rc $?"
  timeout 60 tools/k4_trace_v8 1200 150 100 128 12 4 $k > gpurun_out/trace_c4_v8_k$k.txt 2>&1; echo "c4 k$k rc $?"
done
grep -h "per call" gpurun_out/trace_c*_v8_k*.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_v8.txt 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_v8.txt
