v=v13
timeout 60 tools/k4_trace_$v 1200 100 100 128 12 1 3 > gpurun_out/trace_c3_$v.txt 2>&1
timeout 60 tools/k4_trace_$v 3276 126 126 256 24 2 3 > gpurun_out/trace_c5_$v.txt 2>&1
timeout 60 tools/k4_trace_$v 1200 150 100 128 12 4 3 > gpurun_out/trace_c4_$v.txt 2>&1
grep -h "per call" gpurun_out/trace_c3_$v.txt gpurun_out/trace_c5_$v.txt gpurun_out/trace_c4_$v.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_v13.txt 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_v13.txt
timeout 600 python bench.py --steps 1000 --warmup 20 > gpurun_out/bench_v13.json 2> gpurun_out/bench_v13.err; echo "bench rc $?"; cat gpurun_out/bench_v13.json
