for v in v16 e3b; do
  timeout 60 tools/k4_trace_$v 1200 100 100 128 12 1 3 > gpurun_out/trace_c3_$v.txt 2>&1
  timeout 60 tools/k4_trace_$v 3276 126 126 256 24 2 3 > gpurun_out/trace_c5_$v.txt 2>&1
  timeout 60 tools/k4_trace_$v 1200 150 100 128 12 4 3 > gpurun_out/trace_c4_$v.txt 2>&1
  echo "== $v"; grep -h "per call" gpurun_out/trace_c3_$v.txt gpurun_out/trace_c5_$v.txt gpurun_out/trace_c4_$v.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "kernel3 or 3-" > gpurun_out/pytest_v16.txt 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_v16.txt
