for cg in 1 2; do
  CE_K4_CG=$cg timeout 60 tools/k4_trace_v7 1200 100 100 128 12 1 > gpurun_out/trace_c3_v7_cg$cg.txt 2>&1; echo "c3 cg$cg rc $?"
  CE_K4_CG=$cg timeout 60 tools/k4_trace_v7 3276 126 126 256 24 2 > gpurun_out/trace_c5_v7_cg$cg.txt 2>&1; echo "c5 cg$cg rc $?"
done
for cg in 1 2; do
CE_K4_CG=$cg timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_v7_cg$cg.txt 2>&1; echo "pytest cg$cg rc $?"; tail -3 gpurun_out/pytest_v7_cg$cg.txt
done
