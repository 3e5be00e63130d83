for v in e1 e2 e3; do
  timeout 60 tools/k4_trace_$v 1200 100 100 128 12 1 3 > gpurun_out/trace_c3_$v.txt 2>&1
  timeout 60 tools/k4_trace_$v 3276 126 126 256 24 2 3 > gpurun_out/trace_c5_$v.txt 2>&1
  echo "== $v"; grep -h "per call" gpurun_out/trace_c3_$v.txt gpurun_out/trace_c5_$v.txt
done
